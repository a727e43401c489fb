python -m pytest tests -m gpu -x -q -k "gemm or syrk" > gpurun_out/pt_gemm.log 2>&1; echo pytest=$?; tail -1 gpurun_out/pt_gemm.log
for T in 72 64 56 48 40 32; do
  PB_GEMM_T=$T python bench.py --config c3 --no-e2e --no-cpu --steps 3 --warmup 3 > gpurun_out/c3_T$T.jsonl 2>gpurun_out/c3_T$T.err; echo T$T=$?
done
python bench.py --config c3 --no-e2e --no-cpu --steps 3 --warmup 3 > gpurun_out/c3_auto.jsonl 2>gpurun_out/c3_auto.err; echo auto=$?
