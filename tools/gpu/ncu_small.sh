ncu --set full --clock-control none -k regex:getrf -s 2 -c 1 -o /tmp/ncu_lu -f \
  python bench.py --config c6 --no-e2e --no-cpu --steps 1 --warmup 3 --only "getrf_pivot 32x32" > /tmp/ncu_lu.log 2>&1
ncu -i /tmp/ncu_lu.ncu-rep --page raw --csv > gpurun_out/ncu_lu_raw.csv 2>/dev/null
echo done
