cd $GRAFT_REPO_ROOT
timeout 120 python tools/write_bw.py
timeout 600 python tools/tail_probe.py --cps 4,3,2
