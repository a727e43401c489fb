python -m pytest tests -m gpu -x -q -k "trsm or golden or riccati or composite or randomised or potrf" > gpurun_out/pt_tdb.log 2>&1; echo pytest=$?; tail -1 gpurun_out/pt_tdb.log
timeout 200 python tools/stress.py 300 61 > gpurun_out/stress_tdb.log 2>&1; echo stress=$?; tail -1 gpurun_out/stress_tdb.log
run() { python bench.py --no-e2e --no-cpu --steps 10 --warmup 3 --config $3 --only "$1" 2>>gpurun_out/ab.err | python -c "
import json,sys; d=json.loads(sys.stdin.read()); [print('$2', p['point'], round(p['gflops'],1), round(p['roofline_frac'],4), round(p['ms'],4)) for p in d['points']]"; }
for i in 1 2; do
PB_TRSM_DB=0 run "trsm_rltn 72x48" single c4
run "trsm_rltn 72x48" db c4
done
