python -m pytest tests -m gpu -x -q -k "gemm or syrk or trmm or golden or randomised or special or alias" > gpurun_out/pt_d.log 2>&1; echo pytest=$?; tail -1 gpurun_out/pt_d.log
timeout 200 python tools/stress.py 300 21 > gpurun_out/stress_d.log 2>&1; echo stress=$?; tail -1 gpurun_out/stress_d.log
python bench.py --no-e2e --no-cpu --steps 5 --warmup 3 --config c3 2>>gpurun_out/ab.err > gpurun_out/c3_d.jsonl; python -c "
import json; d=json.loads(open('gpurun_out/c3_d.jsonl').read()); print('c3', round(d['value'],1), round(d['ms_per_step'],3))
[print(' ', p['point'], round(p['gflops'],1), round(p['roofline_frac'],4), round(p['ms'],4)) for p in d['points'][:8]]"
