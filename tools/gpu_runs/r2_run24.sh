# full -m gpu suite + smoke at HEAD
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -rA > gpurun_out/r2_gpu_tests24.log 2>&1; echo "tests rc=$?"
grep -E "free-running|re-synced|gate decisions|passed|failed|FAILED" gpurun_out/r2_gpu_tests24.log | cut -c1-600
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke.log 2>&1; echo "smoke rc=$?"; tail -3 gpurun_out/r2_smoke.log
