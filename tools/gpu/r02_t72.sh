ONLY="gemm_nt 68x68x68,gemm_nt 72x72x72,gemm_nt 132x132x132,gemm_nt 136x136x136,gemm_nt 200x200x200,gemm_nt 204x204x204"
python bench.py --config c3 --steps 3 --warmup 3 --no-cpu --no-e2e --only "$ONLY" > gpurun_out/t72_a.json 2>&1; echo a=$?
PB_T72S2=1 python bench.py --config c3 --steps 3 --warmup 3 --no-cpu --no-e2e --only "$ONLY" > gpurun_out/t72_b.json 2>&1; echo b=$?
