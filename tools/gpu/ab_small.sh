python -m pytest tests -m gpu -x -q -k "potrf" > gpurun_out/pt_potrf.log 2>&1; echo pytest=$?; tail -1 gpurun_out/pt_potrf.log
run() { python bench.py --no-e2e --no-cpu --steps 5 --warmup 3 --config $3 --only "$1" 2>>gpurun_out/ab.err | python -c "
import json,sys; d=json.loads(sys.stdin.read()); p=d['points'][0]; print('$2', p['point'], round(p['gflops'],1), round(p['roofline_frac'],4), round(p['ms'],3))"; }
run "potrf_l n=32" reg c2
run "potrf_l n=64" reg c2
run "syrk_potrf_ln 40x40x32" reg c6
