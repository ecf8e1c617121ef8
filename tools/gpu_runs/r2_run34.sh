# hybrid Jacobi (B by columns in smem, V by rows in registers): parity vs the smem layout, crash check, timing
python tools/rr_diag.py 592,1,30,0,0 1024,0,0,0,0 2>&1 | tee gpurun_out/r2_hyb_diag.log
timeout 600 python tools/rr_check.py --cfg 2 --batch 64 --free 1024 2>&1 | tee -a gpurun_out/r2_hyb_diag.log
for jl in 0 1 0 1; do timeout 300 python tools/prof_solve.py --batch 592 --inner 30 --ns 4 --jl $jl 2>&1 | tail -1 | tee -a gpurun_out/r2_hyb_diag.log; done
