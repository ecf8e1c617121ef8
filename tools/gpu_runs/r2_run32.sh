# named barrier vs __syncthreads variant of the register-resident Jacobi
python tools/rr_diag.py 592,1,30,0,0 1024,0,0,0,0 592,1,30,0,1 2>&1 | tee gpurun_out/r2_rr_diag2.log
cp paper_1205_5351_b200/libtilt.so /tmp/libtilt_named.so
cp paper_1205_5351_b200/libtilt_nb.so paper_1205_5351_b200/libtilt.so
echo "--- __syncthreads variant" | tee -a gpurun_out/r2_rr_diag2.log
python tools/rr_diag.py 592,1,30,0,0 1024,0,0,0,0 2>&1 | tee -a gpurun_out/r2_rr_diag2.log
for jl in 0 1; do timeout 300 python tools/prof_solve.py --batch 592 --inner 30 --ns 4 --jl $jl 2>&1 | tail -1 | tee -a gpurun_out/r2_rr_diag2.log; done
