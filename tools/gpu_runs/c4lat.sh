cd $GRAFT_REPO_ROOT
for b in 1 4 16 64 256; do timeout 300 python tools/c4_prof.py --batch $b --inner 30 2>&1 | tail -1; done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c4_b1_launches.csv python tools/c4_prof.py --batch 1 --inner 10 > /dev/null 2>&1
echo ncu_rc=$?
