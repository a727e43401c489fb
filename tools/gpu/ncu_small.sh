ncu --set full --clock-control none --import-source on -k regex:potrf_small1_kernel -s 2 -c 1 -o gpurun_out/ncu_small1_8 -f \
  python bench.py --no-e2e --no-cpu --steps 1 --warmup 3 --only "potrf_l n=8" > gpurun_out/ncu_small1_8.log 2>&1
echo done
