CMD="python bench.py --steps 1 --warmup 3 --no-cpu --no-gemm --no-e2e --no-inplace --only"
$CMD "potrf_l n=16" > gpurun_out/plain16.json 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"potrf_small" -s 3 -c 1 -o gpurun_out/prof_n16 \
  $CMD "potrf_l n=16" > gpurun_out/ncu16.log 2>&1; echo ncu_rc=$?
