# ncu: product potrf_warp_kernel<4> (one launch of the C2 n=4 point) and the microbench V2
ncu --set full --clock-control none --import-source on -k regex:potrf_warp_kernel -s 2 -c 1 -o gpurun_out/ncu_warp4 -f \
  python bench.py --no-e2e --no-cpu --steps 1 --warmup 3 --only "potrf_l n=4" > gpurun_out/ncu_warp4.log 2>&1
ncu --set full --clock-control none -k regex:k4 -s 9 -c 1 -o gpurun_out/ncu_exp4 -f ./tools/potrf4_exp > gpurun_out/ncu_exp4.log 2>&1
echo done
