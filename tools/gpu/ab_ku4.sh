python -m pytest tests -m gpu -x -q -k "gemm or syrk" > gpurun_out/pt_ku4.log 2>&1; echo pytest=$?; tail -1 gpurun_out/pt_ku4.log
python bench.py --no-e2e --no-cpu --steps 5 --warmup 3 --config c3 2>>gpurun_out/ab.err | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('c3', round(d['value'],1), round(d['ms_per_step'],3), ' '.join('%s:%.4f' % (p['point'].split()[1], p['ms']) for p in d['points'][:7]))"
