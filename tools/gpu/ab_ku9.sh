c3() { python bench.py --no-e2e --no-cpu --steps 5 --warmup 3 --config c3 2>>gpurun_out/ab.err | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$1', round(d['value'],1), round(d['ms_per_step'],3), ' '.join('%s:%.4f' % (p['point'].split()[1], p['ms']) for p in d['points'][:7]))"; }
c3 ku1_lb3
PB_DIRECT_LB=1 c3 ku1_lb1
sed -i 's/#define PB_KU9 1/#define PB_KU9 2/' paper_1704_02457_b200/csrc/pb_gemm.cu
python -c "import sys; sys.path.insert(0,'.'); from paper_1704_02457_b200 import _build; _build.build()" > gpurun_out/rebuild.log 2>&1; echo rebuild=$?
c3 ku2_lb3
PB_DIRECT_LB=1 c3 ku2_lb1
python -m pytest tests -m gpu -x -q -k "gemm or syrk" > gpurun_out/pt_ku.log 2>&1; echo pytest=$?; tail -1 gpurun_out/pt_ku.log
