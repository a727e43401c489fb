run() { python bench.py --no-e2e --no-cpu --steps 5 --warmup 3 --config $3 --only "$1" 2>>gpurun_out/ab.err | python -c "
import json,sys; d=json.loads(sys.stdin.read()); p=d['points'][0]; print('$2', p['point'], round(p['gflops'],1), round(p['roofline_frac'],4), round(p['ms'],3))"; }
for pf in 1 3 1 3; do PB_REG_PF=$pf run "potrf_l n=32" pf$pf c2; PB_REG_PF=$pf run "potrf_l n=64" pf$pf c2; done
