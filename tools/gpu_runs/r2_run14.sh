timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -rA > gpurun_out/r2_gpu_tests14.log 2>&1; echo "tests rc=$?"
grep -v "^PASSED" gpurun_out/r2_gpu_tests14.log | grep -E "free-running|re-synced|gate decisions|passed|failed|FAILED|Error" | cut -c1-1200
