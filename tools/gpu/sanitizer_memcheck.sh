export PYTORCH_NO_CUDA_MEMORY_CACHING=1
timeout 600 python tools/sanitize_suite.py > gpurun_out/san_plain.log 2>&1; rc=$?; echo plain_rc=$rc; tail -2 gpurun_out/san_plain.log
if [ $rc -eq 0 ]; then
  timeout 1500 compute-sanitizer --tool memcheck --leak-check no --print-limit 50 python tools/sanitize_suite.py > gpurun_out/san_memcheck.log 2>&1; echo memcheck_rc=$?
  tail -5 gpurun_out/san_memcheck.log
fi
