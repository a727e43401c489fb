timeout 600 python -m pytest tests -m gpu -x -q -k "potrf_small or golden or potrf_l_random or failure_index or guard_bands_potrf" > gpurun_out/pytest_pair.log 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/pytest_pair.log
for c in 0 1 2 3; do
  PB_PAIR=$c timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu --no-gemm --no-e2e --no-inplace --only "potrf_l n=12,potrf_l n=16" > gpurun_out/pair_$c.json 2>&1; echo cfg=$c rc=$?
done
