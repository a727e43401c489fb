# usage: ncu_one.sh <n> <kernel-regex> <out-name>: ncu --set full source-level capture of one launch of a C2 potrf point
CMD="python bench.py --steps 1 --warmup 3 --no-cpu --no-gemm --no-e2e --no-inplace --only"
ncu --set full --clock-control none --import-source on -k regex:"$2" -s 3 -c 1 -o gpurun_out/$3 \
    $CMD "potrf_l n=$1" > gpurun_out/ncu_$3.log 2>&1; echo ncu_rc=$?
