python bench.py --config c3 --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/s2_0.json 2>&1; echo a=$?
PB_S2=1 python bench.py --config c3 --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/s2_1.json 2>&1; echo b=$?
PB_S2=2 python bench.py --config c3 --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/s2_2.json 2>&1; echo c=$?
