CMD="python bench.py --steps 1 --warmup 3 --no-cpu --no-gemm --no-e2e --no-inplace"
$CMD > gpurun_out/plain_ll.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"potrf|trsm|gemm_tma|gemm_direct|gemm_item|commit" -s 156 -c 52 --csv \
  --log-file gpurun_out/launches_c2.csv $CMD > gpurun_out/ncu_ll.log 2>&1; echo ncu_rc=$?
