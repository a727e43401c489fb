python -m pytest tests -m gpu -x -q -k "gemm or syrk or golden or randomised or special or alias or potrf_l_random or composite" > gpurun_out/pt_pf.log 2>&1; echo pytest=$?; tail -1 gpurun_out/pt_pf.log
timeout 200 python tools/stress.py 300 51 > gpurun_out/stress_pf.log 2>&1; echo stress=$?; tail -1 gpurun_out/stress_pf.log
run() { python bench.py --no-e2e --no-cpu --steps 10 --warmup 3 --config $3 --only "$1" 2>>gpurun_out/ab.err | python -c "
import json,sys; d=json.loads(sys.stdin.read()); [print('$2', p['point'], round(p['gflops'],1), round(p['roofline_frac'],4), round(p['ms'],4)) for p in d['points']]"; }
for i in 1 2; do
PB_DIRECT_PF=0 run "gemm_nt 8x8x8" old c3
run "gemm_nt 8x8x8" pf c3
done
