# launch list of the C2 bench (per-launch durations, cold-cache, serialised) + one full capture of the n=4 kernel
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r01_c2_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:potrf_small1_kernel -s 3 -c 1 -o gpurun_out/ncu_small1_4 -f \
  python bench.py --no-e2e --no-cpu --steps 1 --warmup 3 --only "potrf_l n=4" > gpurun_out/ncu_small1_4.log 2>&1
echo done
