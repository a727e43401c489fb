ONLY="gemm_nt 68x68x68,gemm_nt 72x72x72,gemm_nt 76x76x76,gemm_nt 80x80x80,gemm_nt 84x84x84,gemm_nt 88x88x88,gemm_nt 92x92x92,gemm_nt 96x96x96,gemm_nt 100x100x100,gemm_nt 132x132x132,gemm_nt 136x136x136,gemm_nt 164x164x164,gemm_nt 196x196x196"
for T in 0 40 72 80 88 96; do
  if [ $T = 0 ]; then unset PB_GEMM_T; else export PB_GEMM_T=$T; fi
  python bench.py --config c3 --steps 3 --warmup 3 --no-cpu --no-e2e --only "$ONLY" > gpurun_out/t2_$T.json 2>&1; echo T=$T rc=$?
done
