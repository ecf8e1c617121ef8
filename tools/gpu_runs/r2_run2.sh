# round 2, run 2: full -m gpu suite (new GEMM / LU / protocol tests), quick and full bench
nproc
timeout 2400 python -m pytest tests -m gpu -q -rA -p no:cacheprovider -k "not free_running_convergence_config2_64" > gpurun_out/r2_gpu_tests2.log 2>&1; echo "tests rc=$?"
tail -30 gpurun_out/r2_gpu_tests2.log | grep -v "^PASSED"
timeout 900 python bench.py --global-batch 8192 --steps 4 --warmup 3 > gpurun_out/r2_bench_8192.log 2>&1; echo "bench8192 rc=$?"
tail -c 2500 gpurun_out/r2_bench_8192.log
timeout 1700 python bench.py --steps 20 --warmup 5 > gpurun_out/r2_bench_full.log 2>&1; echo "benchfull rc=$?"
tail -c 4500 gpurun_out/r2_bench_full.log
