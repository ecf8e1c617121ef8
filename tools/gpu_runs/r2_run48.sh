# multi-CTA Jacobi loop with the lagged active-count read (no host wait between sweeps): config 4 probe + full, large tests; ragged K1 tests
python tools/c4_prof.py --batch 256 --outer 1 --inner 30 2>&1 | tail -1 | tee gpurun_out/r2_run48.log
python tools/c4_prof.py --batch 256 --outer 1 --inner 30 2>&1 | tail -1 | tee -a gpurun_out/r2_run48.log
timeout 1500 python -m pytest tests/test_gpu_large.py tests/test_gpu_steps.py -m gpu -x -q 2>&1 | tail -2 | tee -a gpurun_out/r2_run48.log
timeout 900 python tools/configs_bench.py --configs 4 2>&1 | tail -1 | tee -a gpurun_out/r2_run48.log
