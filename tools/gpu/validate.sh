timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_final.log 2>&1; echo pytest_rc=$?; tail -2 gpurun_out/pytest_gpu_final.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_final.log 2>&1; echo smoke_rc=$?
( time python bench.py ) > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo ours_rc=$?
( time python bench.py --impl reference ) > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err; echo ref_rc=$?
tail -3 gpurun_out/bench_default.err gpurun_out/bench_reference.err
