# full GPU suite + smoke at HEAD, then the configs table (c1-c4) at HEAD
timeout 3000 python -m pytest tests -m gpu -q 2>&1 | tail -15 > gpurun_out/r2_gpu_tests45.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke45.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r2_smoke45.log
timeout 1500 python tools/configs_bench.py --configs 1,2,4 2>&1 | tail -8 > gpurun_out/r2_configs45.log
