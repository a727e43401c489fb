python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?; tail -2 gpurun_out/smoke.log
for c in c4 c5 c6; do
  timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo $c rc=$?; tail -2 gpurun_out/bench_$c.err
done
