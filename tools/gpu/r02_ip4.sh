for c in 0 1 2 3 4 5; do
  PB_IP4=$c python bench.py --steps 3 --warmup 3 --no-cpu --no-gemm --no-e2e --only "potrf_l n=4" > gpurun_out/ip4_$c.json 2>&1; echo c=$c rc=$?
done
