# End-of-round measurement run (one gpurun call): full GPU suite, smoke, every bench config, the reference arm,
# the C2 launch list and the ncu --set full captures of the two kernels new in this session.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_final.log 2>&1; echo pytest_rc=$?; tail -2 gpurun_out/pytest_gpu_final.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_final.log 2>&1; echo smoke_rc=$?
( time python bench.py ) > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo ours_rc=$?
for c in c4 c5 c6 pack; do python bench.py --config $c --steps 5 --warmup 3 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo ${c}_rc=$?; done
( time python bench.py --impl reference ) > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err; echo ref_rc=$?
CMD="python bench.py --steps 1 --warmup 3 --no-cpu --no-gemm --no-e2e --no-inplace"
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"potrf|trsm|gemm_tma|gemm_direct|gemm_item|commit" -s 156 -c 52 --csv \
  --log-file gpurun_out/launches_c2.csv $CMD > gpurun_out/ncu_ll.log 2>&1; echo launchlist_rc=$?
ncu --set full --clock-control none --import-source on -k regex:"potrf_chain" -s 3 -c 1 -o gpurun_out/prof_chain128_final \
  $CMD --only "potrf_l n=128" > gpurun_out/ncu_chain.log 2>&1; echo ncu_chain_rc=$?
ncu --set full --clock-control none --import-source on -k regex:"trsm_wide" -s 3 -c 1 -o gpurun_out/prof_trsm_wide_final \
  $CMD --only "potrf_l n=256" > gpurun_out/ncu_trsm.log 2>&1; echo ncu_trsm_rc=$?
for n in 32 64; do ncu --set full --clock-control none --import-source on -k regex:"potrf_reg" -s 3 -c 1 -o gpurun_out/prof_reg${n}_final \
  $CMD --only "potrf_l n=$n" > gpurun_out/ncu_reg$n.log 2>&1; echo ncu_reg${n}_rc=$?; done
