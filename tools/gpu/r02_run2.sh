set -x
timeout 900 python -m pytest tests -m gpu -x -q -k "potrf" > gpurun_out/pytest_potrf.log 2>&1; echo pytest_rc=$?
tail -15 gpurun_out/pytest_potrf.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --no-gemm --no-e2e > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo bench_rc=$?
tail -c 2000 gpurun_out/bench_c2.err
