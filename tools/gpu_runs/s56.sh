cd $GRAFT_REPO_ROOT
timeout 300 python tools/prof_solve.py --batch 2368 --inner 30 --ns 4 --cfg 2 --reps 3 2>&1 | tail -1
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/r2s3_pytest_gpu_s56.log 2>&1; echo pytest_rc=$?
tail -1 gpurun_out/r2s3_pytest_gpu_s56.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python tools/configs_bench.py --configs 1,2 2>&1 | cut -c1-260
