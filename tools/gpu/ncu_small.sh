ncu --set full --clock-control none -k regex:trsm_team_kernel -s 2 -c 1 -o /tmp/ncu_trsm -f \
  python bench.py --config c4 --no-e2e --no-cpu --steps 1 --warmup 3 --only "trsm_rltn 72x48" > /tmp/ncu_trsm.log 2>&1
ncu -i /tmp/ncu_trsm.ncu-rep --page raw --csv > gpurun_out/ncu_trsm_raw.csv 2>/dev/null
echo done
