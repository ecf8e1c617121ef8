mkdir -p gpurun_out/san
timeout 1200 compute-sanitizer --tool memcheck --leak-check full --error-exitcode 9 python tools/all_kernels_smoke.py > gpurun_out/san/memcheck.log 2>&1; echo "memcheck rc=$?"
tail -15 gpurun_out/san/memcheck.log
timeout 1500 python -m pytest tests/test_gpu_protocol.py -m gpu -q -p no:cacheprovider -rA -k "free_running" > gpurun_out/r2_gpu_tests15.log 2>&1; echo "tests rc=$?"
grep -E "free-running config|passed|failed" gpurun_out/r2_gpu_tests15.log | cut -c1-1500
