cd $GRAFT_REPO_ROOT
timeout 120 python tools/k1_run.py 65536
timeout 600 python -m pytest tests/test_gpu_steps.py -m gpu -q -k "warp" -x 2>&1 | tail -3
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
