python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -1 gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?; cat gpurun_out/smoke.log
python bench.py > gpurun_out/bench_c2.jsonl 2> gpurun_out/bench_c2.err; echo c2=$?
for c in c3 c1; do python bench.py --config $c --no-e2e > gpurun_out/bench_$c.jsonl 2> gpurun_out/bench_$c.err; echo $c=$?; done
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r01_c2_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_launch.log 2>&1; echo ncu=$?
