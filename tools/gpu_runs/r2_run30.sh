# register-resident Jacobi: layout A/B on the same patches, then kernel timing, then fixed-count parity tests
timeout 600 python tools/rr_check.py --cfg 2 --batch 64 --free 1024 2>&1 | tee gpurun_out/r2_rr_check.log
for jl in 0 1; do timeout 300 python tools/prof_solve.py --batch 592 --inner 30 --ns 4 --jl $jl 2>&1 | tail -1 | tee -a gpurun_out/r2_rr_prof.log; done
timeout 900 python -m pytest tests/test_gpu_steps.py tests/test_gpu_tilt.py -m gpu -x -q 2>&1 | tail -15 | tee gpurun_out/r2_rr_tests.log
