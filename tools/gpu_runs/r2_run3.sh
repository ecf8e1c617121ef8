# round 2, run 3: tau in fp32 (Z28), new K1, large SVDWS steps, 64-patch free-running, launch list
timeout 1800 python -m pytest tests -m gpu -q -rA -p no:cacheprovider -k "resync or svdws or warp or free_running or pyramid or two_rank or bad_box or large_configs or full_batch" > gpurun_out/r2_gpu_tests3.log 2>&1; echo "tests rc=$?"
grep -v "^PASSED" gpurun_out/r2_gpu_tests3.log | tail -40
timeout 900 python bench.py --global-batch 8192 --steps 4 --warmup 3 --no-cpu --no-e2e > gpurun_out/r2_bench_8192b.log 2>&1; echo "bench8192 rc=$?"
tail -c 1500 gpurun_out/r2_bench_8192b.log
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_warp -c 5 --csv python bench.py --global-batch 8192 --steps 2 --warmup 1 --no-cpu --no-e2e > gpurun_out/r2_ncu_k1.csv 2> gpurun_out/r2_ncu_k1.err; echo "ncu k1 rc=$?"
tail -8 gpurun_out/r2_ncu_k1.csv
