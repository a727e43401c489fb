for c in c1 c4 c6; do python bench.py --config $c --no-e2e > gpurun_out/bench_$c.jsonl 2> gpurun_out/bench_$c.err; echo $c=$?; done
