timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -rA > gpurun_out/r2_gpu_tests10.log 2>&1; echo "tests rc=$?"
grep -v "^PASSED" gpurun_out/r2_gpu_tests10.log | tail -30
