timeout 900 python tools/inner_drift.py --patch 21 --ks 20,200,400,800 > gpurun_out/r2_inner_drift21c.log 2>&1; echo "drift rc=$?"
cat gpurun_out/r2_inner_drift21c.log
timeout 900 python bench.py --global-batch 8192 --steps 4 --warmup 3 --no-cpu --no-e2e --no-k1 > gpurun_out/r2_bench_8192h.log 2>&1; echo "bench rc=$?"
python -c "
import json; l=[x for x in open('gpurun_out/r2_bench_8192h.log') if x.startswith('{')][-1]; d=json.loads(l)
print(d['value'], d['inner_iters_per_s'], d['mean_inner_iters_per_patch'], d['converged_fraction'], d['roofline']['frac'], d['stop_rules'], d['recovery']['fraction'])"
timeout 1800 python -m pytest tests/test_gpu_protocol.py -m gpu -q -p no:cacheprovider -rA -k "free_running or resync" > gpurun_out/r2_gpu_tests13.log 2>&1; echo "tests rc=$?"
grep -E "free-running|re-synced|passed|failed" gpurun_out/r2_gpu_tests13.log | cut -c1-1500
