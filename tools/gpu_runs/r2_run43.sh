# K1 v2 (geometry once per CTA, 16-byte plane stores, fp32-rcp + Newton 1/w): roofline, warp/step/tilt tests, 8192 bench
for N in 8192 65536; do echo "$N $(timeout 300 python tools/k1_run.py $N 2>&1 | tail -1)" | tee -a gpurun_out/r2_k1_v2.log; done
timeout 1200 python -m pytest tests/test_gpu_steps.py tests/test_gpu_tilt.py -m gpu -x -q 2>&1 | tail -3 | tee -a gpurun_out/r2_k1_v2.log
timeout 900 python bench.py --global-batch 8192 --steps 4 --warmup 3 --no-cpu --no-e2e 2>&1 | tail -1 > gpurun_out/r2_bench_8192k.log
