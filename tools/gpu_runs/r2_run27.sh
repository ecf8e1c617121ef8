timeout 900 python bench.py --global-batch 8192 --steps 4 --warmup 3 --no-cpu --no-e2e --no-k1 > gpurun_out/r2_bench_8192l.log 2>&1; echo "bench rc=$?"
python -c "
import json; l=[x for x in open('gpurun_out/r2_bench_8192l.log') if x.startswith('{')][-1]; d=json.loads(l)
print('bench8192', d['value'], d['inner_iters_per_s'], d['mean_inner_iters_per_patch'], d['roofline']['frac'])"
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -rA > gpurun_out/r2_gpu_tests27.log 2>&1; echo "tests rc=$?"
grep -E "free-running|re-synced|passed|failed|FAILED" gpurun_out/r2_gpu_tests27.log | cut -c1-500
python tools/c4_prof.py --batch 256 --outer 1 --inner 30 2>&1 | tail -1
