run() { python bench.py --no-e2e --no-cpu --steps 10 --warmup 3 --config $3 --only "$1" 2>>gpurun_out/ab.err | python -c "
import json,sys; d=json.loads(sys.stdin.read()); [print('$2', p['point'], round(p['gflops'],1), round(p['roofline_frac'],4), round(p['ms'],4)) for p in d['points']]"; }
for i in 1 2; do
run "gemm_nt 64x64x64" s2c1 c1
for v in k16s4 k16s3 k8s6; do PB_TMA_CS=$v run "gemm_nt 64x64x64" $v c1; done
done
PB_TMA_CS=k16s4 python -m pytest tests -m gpu -x -q -k "gemm_nt" > gpurun_out/pt_gemm.log 2>&1; echo pytest=$?; tail -1 gpurun_out/pt_gemm.log
