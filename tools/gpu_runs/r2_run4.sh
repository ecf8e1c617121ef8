# round 2, run 4: column-reuse Jacobi schedule (parity + speed), K1 back on smem, free-running trace
timeout 1500 python -m pytest tests/test_gpu_steps.py tests/test_gpu_tilt.py tests/test_gpu_adm.py -m gpu -q -x -p no:cacheprovider > gpurun_out/r2_gpu_tests4.log 2>&1; echo "tests rc=$?"
tail -5 gpurun_out/r2_gpu_tests4.log
timeout 900 python bench.py --global-batch 8192 --steps 4 --warmup 3 --no-cpu --no-e2e > gpurun_out/r2_bench_8192c.log 2>&1; echo "bench8192 rc=$?"
tail -c 1800 gpurun_out/r2_bench_8192c.log
timeout 1200 python tools/free_running_trace.py --out gpurun_out/r2_free_trace.jsonl > gpurun_out/r2_free_trace.log 2>&1; echo "trace rc=$?"
cat gpurun_out/r2_free_trace.log | cut -c1-600
