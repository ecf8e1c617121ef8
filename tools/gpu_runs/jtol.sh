cd $GRAFT_REPO_ROOT
timeout 900 python tools/jtol_probe.py --batch 4096 --tols 0,1e-5,3e-5,0
