cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/r2s3_pytest_gpu_head.log 2>&1; echo pytest_rc=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2s3_smoke_head.log 2>&1; echo smoke_rc=$?
timeout 900 python tools/configs_bench.py --configs 1,2,4 > gpurun_out/r2s3_configs124.log 2>&1; echo cfg_rc=$?
