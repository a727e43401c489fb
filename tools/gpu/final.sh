python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -1 gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?; cat gpurun_out/smoke.log
python bench.py > gpurun_out/bench_c2.jsonl 2> gpurun_out/bench_c2.err; echo c2=$?
for c in c1 c3 c4 c5 c6; do python bench.py --config $c --no-e2e > gpurun_out/bench_$c.jsonl 2> gpurun_out/bench_$c.err; echo $c=$?; done
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.jsonl 2>gpurun_out/bench_ref.err; echo ref=$?
