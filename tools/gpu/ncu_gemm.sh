ncu --set full --clock-control none --import-source on -k regex:gemm_tma -s 1 -c 1 -o /tmp/ncu_g -f \
  python tools/prof_gemm.py gemm 64x64x64 4096 2 > gpurun_out/ncu_g.log 2>&1; echo ncu=$?
ncu -i /tmp/ncu_g.ncu-rep --page raw --csv > gpurun_out/ncu_gemm_raw.csv 2>/dev/null
ncu -i /tmp/ncu_g.ncu-rep --page source --csv --print-source sass > gpurun_out/ncu_gemm_src.csv 2>/dev/null
ncu -i /tmp/ncu_g.ncu-rep --page details > gpurun_out/ncu_gemm_details.txt 2>/dev/null
ls -la gpurun_out/ncu_gemm*
