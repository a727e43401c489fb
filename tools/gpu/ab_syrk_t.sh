run() { python bench.py --no-e2e --no-cpu --steps 10 --warmup 3 --config $3 --only "$1" 2>>gpurun_out/ab.err | python -c "
import json,sys; d=json.loads(sys.stdin.read()); [print('$2', p['point'], round(p['gflops'],1), round(p['roofline_frac'],4), round(p['ms'],4)) for p in d['points']]"; }
run "syrk_ln 96x40" auto c4
for T in 32 40 48 56 64 72; do PB_GEMM_T=$T run "syrk_ln 96x40" T$T c4; done
