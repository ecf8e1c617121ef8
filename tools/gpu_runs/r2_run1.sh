set -x
nproc; nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -q -x --deselect tests/test_gpu_large.py -p no:cacheprovider > gpurun_out/r2_gpu_tests.log 2>&1; echo "tests rc=$?"
tail -5 gpurun_out/r2_gpu_tests.log
timeout 600 python bench.py --global-batch 8192 --steps 4 --warmup 3 --no-cpu > gpurun_out/r2_bench_8192.log 2>&1; echo "bench8192 rc=$?"
tail -c 3000 gpurun_out/r2_bench_8192.log
timeout 1700 python bench.py --steps 20 --warmup 5 > gpurun_out/r2_bench_full.log 2>&1; echo "benchfull rc=$?"
tail -c 4000 gpurun_out/r2_bench_full.log
