python -m pytest tests -m gpu -x -q -k "trsm or golden or riccati or composite or randomised" > gpurun_out/pt_trsm.log 2>&1; echo pytest=$?; tail -1 gpurun_out/pt_trsm.log
run() { python bench.py --no-e2e --no-cpu --steps 10 --warmup 3 --config $3 --only "$1" 2>>gpurun_out/ab.err | python -c "
import json,sys; d=json.loads(sys.stdin.read()); [print('$2', p['point'], round(p['gflops'],1), round(p['roofline_frac'],4), round(p['ms'],4)) for p in d['points']]"; }
run "trsm_rltn 72x48" new c4
run "trsm_rltn 72x48" new c4
