# usage: ncu_cfg.sh <config> <kernel-regex> <out-name> [skip]: ncu --set full source-level capture of one launch of a bench config
ncu --set full --clock-control none --import-source on -k regex:"$2" -s ${4:-3} -c 1 -o gpurun_out/$3 \
    python bench.py --config $1 --steps 1 --warmup 3 --no-cpu > gpurun_out/ncu_$3.log 2>&1; echo ncu_rc=$?
