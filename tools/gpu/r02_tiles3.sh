for T in 32 40 48 56 64 72 80 88 96; do
  PB_GEMM_T=$T python bench.py --config c3 --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/t3_$T.json 2>&1; echo T=$T rc=$?
done
