PB_SMALL_CFG=t1_128x1 ncu --set full --clock-control none --import-source on -k regex:potrf_small_kernel -s 1 -c 1 -o /tmp/ncu_t1s -f \
  python bench.py --no-e2e --no-cpu --steps 1 --warmup 1 --only "potrf_l n=16" > gpurun_out/ncu_t1s.log 2>&1; echo ncu=$?
ncu -i /tmp/ncu_t1s.ncu-rep --page raw --csv > gpurun_out/ncu_t1s_raw.csv 2>/dev/null
ncu -i /tmp/ncu_t1s.ncu-rep --page details > gpurun_out/ncu_t1s_details.txt 2>/dev/null
ncu -i /tmp/ncu_t1s.ncu-rep --page source --csv --print-source sass > gpurun_out/ncu_t1s_src.csv 2>/dev/null
ls -la gpurun_out/ncu_t1s*
