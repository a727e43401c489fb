CMD="python bench.py --steps 1 --warmup 3 --no-cpu --no-gemm --no-e2e --no-inplace --only"
$CMD "potrf_l n=128,potrf_l n=256" > gpurun_out/plain_team.json 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"potrf_team" -s 3 -c 1 -o gpurun_out/prof_team \
  $CMD "potrf_l n=128" > gpurun_out/ncu_team.log 2>&1; echo ncu_rc=$?
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"pb::|potrf|gemm|trsm|commit" -s 20 -c 40 --csv --log-file gpurun_out/launches_256.csv \
  $CMD "potrf_l n=256" > gpurun_out/ncu_256.log 2>&1; echo launch_rc=$?
