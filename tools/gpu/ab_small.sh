PB_SMALL_S1=1 python -m pytest tests -m gpu -x -q -k "potrf_small or potrf_l_random or failure" > gpurun_out/pt_potrf.log 2>&1; echo pytest=$?; tail -1 gpurun_out/pt_potrf.log
run() { python bench.py --no-e2e --no-cpu --steps 5 --warmup 3 --config $3 --only "$1" 2>>gpurun_out/ab.err | python -c "
import json,sys; d=json.loads(sys.stdin.read()); [print('$2', p['point'], round(p['gflops'],1), round(p['roofline_frac'],4), round(p['ms'],4)) for p in d['points']]"; }
for v in 0 1 2 3; do PB_SMALL_S1=$v run "potrf_l n=16" s1_$v c2; done
