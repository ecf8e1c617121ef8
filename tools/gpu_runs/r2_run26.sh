timeout 1800 python -m pytest tests/test_gpu_protocol.py tests/test_gpu_adm.py -m gpu -q -p no:cacheprovider -rA -k "free_running or range" > gpurun_out/r2_gpu_tests26.log 2>&1; echo "tests rc=$?"
grep -E "free-running config|passed|failed|FAILED|RuntimeError|oracle failed" gpurun_out/r2_gpu_tests26.log | cut -c1-900
