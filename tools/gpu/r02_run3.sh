timeout 900 python -m pytest tests -m gpu -x -q -k "potrf" > gpurun_out/pytest_potrf.log 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/pytest_potrf.log
CMD="python bench.py --steps 3 --warmup 3 --no-cpu --no-gemm --no-e2e --no-inplace --only potrf_l_n=64,potrf_l_n=128"
CMD="python bench.py --steps 3 --warmup 3 --no-cpu --no-gemm --no-e2e --no-inplace --only"
$CMD "potrf_l n=32,potrf_l n=64,potrf_l n=128,potrf_l n=256" > gpurun_out/bench_sub.json 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"potrf_cta|potrf_reg" -s 2 -c 4 -o gpurun_out/prof_cta \
  $CMD "potrf_l n=64,potrf_l n=128" > gpurun_out/ncu.log 2>&1; echo ncu_rc=$?
tail -3 gpurun_out/ncu.log
