# rank-compacted output product A = sum_{h_j > 0} h_j b_j v_j^T: probe timing, step/tilt tests, 8192 bench, config 2
for i in 1 2; do timeout 300 python tools/prof_solve.py --batch 592 --inner 30 --ns 4 2>&1 | tail -1 | tee -a gpurun_out/r2_run46.log; done
timeout 1200 python -m pytest tests/test_gpu_steps.py tests/test_gpu_tilt.py -m gpu -x -q 2>&1 | tail -2 | tee -a gpurun_out/r2_run46.log
timeout 900 python bench.py --global-batch 8192 --steps 4 --warmup 3 --no-cpu --no-e2e 2>&1 | tail -1 > gpurun_out/r2_bench_8192l.log
timeout 900 python tools/configs_bench.py --configs 2 2>&1 | tail -1 | tee -a gpurun_out/r2_run46.log
