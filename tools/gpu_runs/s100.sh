cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/r2s3_pytest_gpu_s100.log 2>&1; echo pytest_rc=$?
tail -1 gpurun_out/r2s3_pytest_gpu_s100.log
timeout 1500 python tools/configs_bench.py --configs 3 2>&1 | cut -c1-400
