python -m pytest tests -m gpu -x -q -k "gemm or syrk or trmm or riccati or chain" > gpurun_out/pt_gemm.log 2>&1; echo pytest=$?; tail -1 gpurun_out/pt_gemm.log
run() { python bench.py --no-e2e --no-cpu --steps 10 --warmup 3 --config $3 --only "$1" 2>>gpurun_out/ab.err | python -c "
import json,sys; d=json.loads(sys.stdin.read()); [print('$2', p['point'], round(p['gflops'],1), round(p['roofline_frac'],4), round(p['ms'],4)) for p in d['points']]"; }
for i in 1 2; do
run "gemm_nt 64x64x64" new c1
run "syrk_ln 96x40" new c4
run "gemm_nn 64x64x64,trmm_rlnn 40x0" new c6
done
python bench.py --no-e2e --no-cpu --steps 3 --warmup 3 --config c3 2>>gpurun_out/ab.err | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('c3', d['value'], d['ms_per_step'])"
