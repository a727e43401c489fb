run() { python bench.py --no-e2e --no-cpu --steps 5 --warmup 3 --config $3 --only "$1" 2>>gpurun_out/ab.err | python -c "
import json,sys; d=json.loads(sys.stdin.read()); p=d['points'][0]; print('$2', p['point'], round(p['gflops'],1), round(p['roofline_frac'],4), round(p['ms'],3))"; }
for tw in 2 1 4; do PB_CHAIN_TW=$tw run "riccati nx=32 nu=8 N=50" tw$tw c5; done
