timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?; tail -2 gpurun_out/pytest_gpu.log
python bench.py --config c3 --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/c3_new.json 2>&1; echo c3=$?
python bench.py --config c1 --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/c1_new.json 2>&1; echo c1=$?
