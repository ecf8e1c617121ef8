cd $GRAFT_REPO_ROOT
timeout 1500 python tools/configs_bench.py --configs 3 > gpurun_out/r2s3_config3.log 2>&1; echo rc=$?
