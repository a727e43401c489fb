timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/pytest_gpu.log
CMD="python bench.py --steps 1 --warmup 3 --no-cpu --no-gemm --no-e2e --no-inplace --only"
$CMD "potrf_l n=4,potrf_l n=8,potrf_l n=16" > gpurun_out/plain_small.json 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"potrf_small" -s 3 -c 1 -o gpurun_out/prof_n4 \
  $CMD "potrf_l n=4" > gpurun_out/ncu_n4.log 2>&1; echo ncu4_rc=$?
ncu --set full --clock-control none --import-source on -k regex:"potrf_small" -s 3 -c 1 -o gpurun_out/prof_n8 \
  $CMD "potrf_l n=8" > gpurun_out/ncu_n8.log 2>&1; echo ncu8_rc=$?
ncu --set full --clock-control none --import-source on -k regex:"potrf_small" -s 3 -c 1 -o gpurun_out/prof_n16 \
  $CMD "potrf_l n=16" > gpurun_out/ncu_n16.log 2>&1; echo ncu16_rc=$?
python bench.py --steps 1 --warmup 3 --no-cpu --no-gemm --no-e2e --no-inplace > gpurun_out/plain_c2.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -s 180 -c 400 --csv --log-file gpurun_out/launches_c2_all.csv \
  python bench.py --steps 1 --warmup 3 --no-cpu --no-gemm --no-e2e --no-inplace > gpurun_out/ncu_launch.log 2>&1; echo launch_rc=$?
