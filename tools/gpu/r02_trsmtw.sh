for tw in 0 8 6 4 3 2 1; do
  if [ $tw = 0 ]; then unset PB_TRSM_TW; else export PB_TRSM_TW=$tw; fi
  python bench.py --steps 5 --warmup 3 --no-cpu --no-gemm --no-e2e --no-inplace --only "potrf_l n=256" > gpurun_out/tw_$tw.json 2>&1
  python bench.py --config c4 --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/twc4_$tw.json 2>&1; echo tw=$tw rc=$?
done
