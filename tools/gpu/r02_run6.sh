CMD="python bench.py --steps 3 --warmup 3 --no-cpu --no-gemm --no-e2e --no-inplace --only"
$CMD "potrf_l n=32,potrf_l n=64" > gpurun_out/bench_sub2.json 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"potrf_reg" -s 2 -c 2 -o gpurun_out/prof_reg \
  $CMD "potrf_l n=32,potrf_l n=64" > gpurun_out/ncu.log 2>&1; echo ncu_rc=$?
