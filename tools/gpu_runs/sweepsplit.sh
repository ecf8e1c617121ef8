cd $GRAFT_REPO_ROOT
for ms in 0 1 2 3; do timeout 300 python tools/prof_solve.py --batch 2368 --inner 30 --ns 4 --cfg 2 --reps 3 --max-sweeps $ms 2>&1 | tail -1; done
