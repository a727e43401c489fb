ncu --set full --clock-control none --import-source on -k regex:potrf_team_kernel -s 1 -c 1 -o gpurun_out/ncu_team128 -f \
  python bench.py --no-e2e --no-cpu --steps 1 --warmup 3 --only "potrf_l n=128" > gpurun_out/ncu_team128.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"potrf|gemm|syrk|pb" --csv --log-file gpurun_out/r01_c2_launches_ours.csv \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_launch2.log 2>&1
echo done
