python tools/c4_prof.py --batch 256 --outer 1 --inner 30 > gpurun_out/c4_plain2.log 2>&1; echo "plain rc=$?"; cat gpurun_out/c4_plain2.log
timeout 1500 python -m pytest tests/test_gpu_large.py tests/test_gpu_tilt.py -m gpu -q -x -p no:cacheprovider -k "large or multi_cta or svdws or pyramid" > gpurun_out/r2_gpu_tests20.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r2_gpu_tests20.log
timeout 1200 python tools/configs_bench.py --configs 4 > gpurun_out/r2_configs_4b.log 2>&1; echo "configs rc=$?"; cat gpurun_out/r2_configs_4b.log
