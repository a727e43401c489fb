python -m pytest tests -m gpu -x -q -k "potrf" > gpurun_out/pt_r8.log 2>&1; echo pytest=$?; tail -1 gpurun_out/pt_r8.log
timeout 200 python tools/stress.py 300 41 > gpurun_out/stress_r8.log 2>&1; echo stress=$?; tail -1 gpurun_out/stress_r8.log
run() { python bench.py --no-e2e --no-cpu --steps 5 --warmup 3 --config $3 --only "$1" 2>>gpurun_out/ab.err | python -c "
import json,sys; d=json.loads(sys.stdin.read()); [print('$2', p['point'], round(p['gflops'],1), round(p['roofline_frac'],4), round(p['ms'],4)) for p in d['points']]"; }
for i in 1 2; do
for v in 0 1 2; do PB_SMALL_R8=$v run "potrf_l n=8" r8_$v c2; done
done
