PB_SMALL_CFG=t1_64x1 python -m pytest tests -m gpu -x -q -k "potrf_small and 16 or host_pinned" > gpurun_out/pt_t1.log 2>&1; echo pytest=$?; tail -1 gpurun_out/pt_t1.log
run() { python bench.py --no-e2e --no-cpu --steps 5 --warmup 3 --config $3 --only "$1" 2>>gpurun_out/ab.err | python -c "
import json,sys; d=json.loads(sys.stdin.read()); [print('$2', p['point'], round(p['gflops'],1), round(p['roofline_frac'],4), round(p['ms'],4)) for p in d['points']]"; }
run "potrf_l n=16" quad c2
for v in t1_32x1 t1_32x2 t1_64x1 t1_64x2 t1_96x1 t1_128x1; do PB_SMALL_CFG=$v run "potrf_l n=16" $v c2; done
