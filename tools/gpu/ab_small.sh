python -m pytest tests -m gpu -x -q -k "trsm or chain or riccati or kkt or composite or golden" > gpurun_out/pt_trsm.log 2>&1; echo pytest=$?; tail -1 gpurun_out/pt_trsm.log
run() { python bench.py --no-e2e --no-cpu --steps 5 --warmup 3 --config $3 --only "$1" 2>>gpurun_out/ab.err | python -c "
import json,sys; d=json.loads(sys.stdin.read()); p=d['points'][0]; print('$2', p['point'], round(p['gflops'],1), round(p['roofline_frac'],4), round(p['ms'],3))"; }
run "trsm_rltn 72x48" tw c4
