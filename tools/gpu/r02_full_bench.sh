( time python bench.py ) > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo ours_rc=$?
tail -4 gpurun_out/bench_default.err
( time python bench.py --impl reference ) > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err; echo ref_rc=$?
tail -4 gpurun_out/bench_reference.err
