CMD="python bench.py --config c3 --steps 2 --warmup 3 --no-cpu --no-e2e --only"
$CMD "gemm_nt 64x64x64,gemm_nt 68x68x68,gemm_nt 76x76x76,gemm_nt 84x84x84" > gpurun_out/c3_sub.json 2>&1 && \
ncu --set full --clock-control none -k regex:"gemm_tma" -s 12 -c 4 -o gpurun_out/prof_c3 \
  $CMD "gemm_nt 64x64x64,gemm_nt 68x68x68,gemm_nt 76x76x76,gemm_nt 84x84x84" > gpurun_out/ncu_c3.log 2>&1; echo ncu_rc=$?
