timeout 900 python -m pytest tests -m gpu -x -q -k "potrf" > gpurun_out/pytest_potrf.log 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/pytest_potrf.log
python bench.py --steps 5 --warmup 3 --no-cpu --no-gemm --no-e2e --no-inplace > gpurun_out/bench_c2.json 2>&1; echo bench_rc=$?
