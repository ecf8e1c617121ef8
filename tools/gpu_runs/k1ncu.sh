cd $GRAFT_REPO_ROOT
timeout 120 python tools/k1_run.py 65536
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_warp -s 2 -c 1 -o gpurun_out/k1_head python tools/k1_run.py 16384 > gpurun_out/k1_ncu.log 2>&1
echo ncu_rc=$?
