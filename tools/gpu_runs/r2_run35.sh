# ncu of the hybrid-layout k_solve (jl 0) for comparison with the shared-column layout profile
mkdir -p gpurun_out/ncu_hyb
python tools/prof_solve.py --batch 592 --inner 30 --ns 4 --jl 0 > gpurun_out/ncu_hyb/plain.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_solve -c 1 -o gpurun_out/ncu_hyb/k_solve_hyb -f python tools/prof_solve.py --batch 592 --inner 30 --ns 4 --jl 0 > gpurun_out/ncu_hyb/ncu.log 2>&1; echo "ncu rc=$?"
