# ncu --set full source-level captures of one launch per C2 potrf regime (n = 16, 32, 64, 128)
CMD="python bench.py --steps 1 --warmup 3 --no-cpu --no-gemm --no-e2e --no-inplace --only"
$CMD "potrf_l n=16,potrf_l n=32,potrf_l n=64,potrf_l n=128" > gpurun_out/plain_all.json 2>&1 || exit 1
for n in 16 32 64 128; do
  ncu --set full --clock-control none --import-source on -k regex:"potrf_" -s 3 -c 1 -o gpurun_out/prof_potrf$n \
    $CMD "potrf_l n=$n" > gpurun_out/ncu_potrf$n.log 2>&1; echo ncu${n}_rc=$?
done
