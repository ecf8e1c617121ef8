timeout 900 python bench.py --global-batch 8192 --steps 4 --warmup 3 --no-cpu --no-e2e --no-k1 > gpurun_out/r2_bench_8192i.log 2>&1; echo "bench rc=$?"
python -c "
import json; l=[x for x in open('gpurun_out/r2_bench_8192i.log') if x.startswith('{')][-1]; d=json.loads(l)
print(d['value'], d['inner_iters_per_s'], d['mean_inner_iters_per_patch'], d['converged_fraction'], d['roofline']['frac'], d['stop_rules'])"
timeout 600 python -m pytest tests/test_gpu_tilt.py tests/test_gpu_steps.py -m gpu -q -x -p no:cacheprovider > gpurun_out/r2_gpu_tests17.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/r2_gpu_tests17.log
timeout 1200 python tools/configs_bench.py --configs 2,4 > gpurun_out/r2_configs_24.log 2>&1; echo "configs rc=$?"
cat gpurun_out/r2_configs_24.log | tail -3
