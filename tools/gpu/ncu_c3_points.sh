# ncu --set full digests (text only) of C3 gemm points: usage ncu_c3_points.sh "12 20 36"
mkdir -p gpurun_out
for n in $1; do
ncu --set full --clock-control none --import-source on -k regex:"gemm" -s 3 -c 1 -o /tmp/prof_c3_n$n python bench.py --config c3 --steps 1 --warmup 3 --no-cpu --only "gemm_nt ${n}x${n}x${n}" > /tmp/ncu_c3_$n.log 2>&1; echo ncu_rc=$?
items=$(python -c "
import json
d=json.loads([l for l in open('/tmp/ncu_c3_$n.log') if l.startswith('{')][-1]); print(d['points'][0]['chunk'])")
python tools/ncu_sass.py /tmp/prof_c3_n$n.ncu-rep $items 30 > gpurun_out/c3_n${n}_digest.txt 2>&1
done
