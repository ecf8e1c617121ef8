# idle-unit load skip + warp_tap perspective-division skip: kernel timing, 8192-patch bench (K1 roofline), step/tilt tests
for i in 1 2; do timeout 300 python tools/prof_solve.py --batch 592 --inner 30 --ns 4 2>&1 | tail -1 | tee -a gpurun_out/r2_run37.log; done
timeout 900 python bench.py --global-batch 8192 --steps 4 --warmup 3 --no-cpu --no-e2e 2>&1 | tail -1 > gpurun_out/r2_bench_8192j.log
timeout 1200 python -m pytest tests/test_gpu_steps.py tests/test_gpu_tilt.py -m gpu -x -q 2>&1 | tail -3 | tee -a gpurun_out/r2_run37.log
