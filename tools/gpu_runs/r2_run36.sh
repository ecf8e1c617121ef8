# V-register Jacobi sidecar: parity vs the shared layout, crash check, timing (MINB 4 and MINB 3 builds)
python tools/rr_diag.py 592,1,30,0,0 1024,0,0,0,0 2>&1 | tee gpurun_out/r2_vreg_diag.log
timeout 600 python tools/rr_check.py --cfg 2 --batch 64 --free 1024 2>&1 | tee -a gpurun_out/r2_vreg_diag.log
for jl in 0 1 0 1; do timeout 300 python tools/prof_solve.py --batch 592 --inner 30 --ns 4 --jl $jl 2>&1 | tail -1 | tee -a gpurun_out/r2_vreg_diag.log; done
cp paper_1205_5351_b200/libtilt_m3.so paper_1205_5351_b200/libtilt.so
echo "--- MINB 3" | tee -a gpurun_out/r2_vreg_diag.log
for jl in 0 1 0 1; do timeout 300 python tools/prof_solve.py --batch 444 --inner 30 --ns 4 --jl $jl 2>&1 | tail -1 | tee -a gpurun_out/r2_vreg_diag.log; done
timeout 600 python tools/rr_check.py --cfg 2 --batch 8 --free 1024 2>&1 | tail -2 | tee -a gpurun_out/r2_vreg_diag.log
