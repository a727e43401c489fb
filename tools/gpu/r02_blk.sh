for d in 128 64; do
  PB_DIRECT_MAX=$d python bench.py --steps 5 --warmup 3 --no-cpu --no-gemm --no-e2e --no-inplace --only "potrf_l n=128,potrf_l n=256" > gpurun_out/blk_$d.json 2>&1; echo d=$d rc=$?
done
PB_DIRECT_MAX=64 timeout 600 python -m pytest tests -m gpu -x -q -k "potrf" > gpurun_out/pblk.log 2>&1; echo pytest_rc=$?; tail -2 gpurun_out/pblk.log
