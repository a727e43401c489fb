timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/pytest_gpu.log
python bench.py --config pack --steps 5 --warmup 3 --no-cpu > gpurun_out/bench_pack.json 2> gpurun_out/bench_pack.err; echo rc=$?
tail -3 gpurun_out/bench_pack.err
