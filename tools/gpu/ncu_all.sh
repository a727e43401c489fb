# one full ncu capture per C2 point's kernel (current code), for profiles/r01_c2_kernels_ncu.txt
cap() { ncu --set full --clock-control none -k regex:"$2" -s 2 -c 1 -o /tmp/ncu_$1 -f \
  python bench.py --no-e2e --no-cpu --steps 1 --warmup 3 --only "potrf_l n=$1" > /tmp/ncu_$1.log 2>&1; }
cap 8 potrf_small1_kernel
cap 16 potrf_small_kernel
cap 32 potrf_reg_kernel
cap 64 potrf_reg_kernel
cap 128 potrf_team_kernel
python tools/ncu_summarize.py /tmp/ncu_ gpurun_out/r01_c2_kernels_ncu.txt
