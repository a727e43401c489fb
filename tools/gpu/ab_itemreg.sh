run() { python bench.py --no-e2e --no-cpu --steps 10 --warmup 3 --config $3 --only "$1" 2>>gpurun_out/ab.err | python -c "
import json,sys; d=json.loads(sys.stdin.read()); [print('$2', p['point'], round(p['gflops'],1), round(p['roofline_frac'],4), round(p['ms'],4)) for p in d['points']]"; }
for i in 1 2; do
for v in 1 2 3 4; do PB_ITEM_REG=$v run "gemm_nt 4x4x4" reg$v c3; done
done
for v in 2 3 4; do PB_ITEM_REG=$v python -m pytest tests -m gpu -x -q -k "gemm_nt_random or syrk_ln_random" > gpurun_out/pt_ir$v.log 2>&1; echo v$v pytest=$?; done
