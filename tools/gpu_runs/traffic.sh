cd $GRAFT_REPO_ROOT
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_warp -s 1 -c 1 -o gpurun_out/k1_128x5 python tools/k1_run.py 65536 > gpurun_out/k1_128x5_ncu.log 2>&1
echo k1_ncu_rc=$?
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:k_solve -c 1 --csv --log-file gpurun_out/k_solve_slab_dram.csv python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu --no-k1 > gpurun_out/k_solve_slab_dram.log 2>&1
echo ksolve_ncu_rc=$?
