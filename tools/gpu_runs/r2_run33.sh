# crash isolation for the register-resident Jacobi: CTAs per SM and register budget
python tools/rr_diag.py 592,1,30,0,0 592,1,30,2,0 592,1,30,3,0 1024,0,0,0,0 2>&1 | tee gpurun_out/r2_rr_diag3.log
for jl in 0 1; do timeout 300 python tools/prof_solve.py --batch 592 --inner 30 --ns 4 --jl $jl 2>&1 | tail -1 | tee -a gpurun_out/r2_rr_diag3.log; done
cp paper_1205_5351_b200/libtilt_m3.so paper_1205_5351_b200/libtilt.so
echo "--- MINB 3 build" | tee -a gpurun_out/r2_rr_diag3.log
python tools/rr_diag.py 444,1,30,0,0 1024,0,0,0,0 2>&1 | tee -a gpurun_out/r2_rr_diag3.log
for jl in 0 1; do timeout 300 python tools/prof_solve.py --batch 444 --inner 30 --ns 4 --jl $jl 2>&1 | tail -1 | tee -a gpurun_out/r2_rr_diag3.log; done
