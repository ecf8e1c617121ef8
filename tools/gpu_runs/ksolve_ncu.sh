cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/ncu6
python tools/prof_solve.py --batch 592 --inner 30 --ns 4 > gpurun_out/ncu6/prof_plain.log 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_solve -c 1 -o gpurun_out/ncu6/k_solve_r2s3 -f python tools/prof_solve.py --batch 592 --inner 30 --ns 4 > gpurun_out/ncu6/ncu_full.log 2>&1; echo "ncu rc=$?"
ncu -i gpurun_out/ncu6/k_solve_r2s3.ncu-rep --page source --csv --print-source=cuda,sass > gpurun_out/ncu6/k_solve_src.csv 2>/dev/null; echo src_rc=$?
