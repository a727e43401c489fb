ncu --set full --clock-control none --import-source on -k regex:potrf_reg_kernel -s 2 -c 1 -o gpurun_out/ncu_reg32 -f \
  python bench.py --no-e2e --no-cpu --steps 1 --warmup 3 --only "potrf_l n=32" > gpurun_out/ncu_reg32.log 2>&1
echo done
