python -m pytest tests -m gpu -x -q -k "potrf" > gpurun_out/pt_potrf.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pt_potrf.log
for only in "potrf_l n=4"; do
 for legacy in 0 1; do
  if [ $legacy = 1 ]; then export PB_SMALL_LEGACY=1; else unset PB_SMALL_LEGACY; fi
  python bench.py --no-e2e --no-cpu --steps 5 --warmup 3 --only "$only" 2>>gpurun_out/ab.err | python -c "
import json,sys; d=json.loads(sys.stdin.read()); p=d['points'][0]; print('legacy=$legacy', p['point'], round(p['gflops'],1), round(p['roofline_frac'],4), round(p['ms'],3))"
 done
done
