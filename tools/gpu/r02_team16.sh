timeout 600 python -m pytest tests -m gpu -x -q -k "potrf" > gpurun_out/pytest_t16.log 2>&1; echo pytest_rc=$?
tail -2 gpurun_out/pytest_t16.log
python bench.py --steps 5 --warmup 3 --no-cpu --no-gemm --no-e2e --no-inplace --only "potrf_l n=128,potrf_l n=256" > gpurun_out/team16.json 2>&1; echo rc=$?
