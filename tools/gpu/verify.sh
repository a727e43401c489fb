# Verification run (one gpurun call): full GPU suite, smoke, the default bench line.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_final.log 2>&1; echo pytest_rc=$?; tail -2 gpurun_out/pytest_gpu_final.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_final.log 2>&1; echo smoke_rc=$?
( time python bench.py ) > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo ours_rc=$?
