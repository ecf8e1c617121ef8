timeout 900 python tools/inner_drift.py --patch 21 --ks 20,100,200,400,800 > gpurun_out/r2_inner_drift21b.log 2>&1; echo "drift rc=$?"
cat gpurun_out/r2_inner_drift21b.log
timeout 900 python tools/inner_trace.py --patch 21 --outer 1 --variants "default" > gpurun_out/r2_inner_trace21e.log 2>&1; echo "trace21 rc=$?"
cut -c1-400 gpurun_out/r2_inner_trace21e.log
timeout 900 python bench.py --global-batch 8192 --steps 4 --warmup 3 --no-cpu --no-e2e --no-k1 > gpurun_out/r2_bench_8192g.log 2>&1; echo "bench rc=$?"
python -c "
import json; l=[x for x in open('gpurun_out/r2_bench_8192g.log') if x.startswith('{')][-1]; d=json.loads(l)
print(d['value'], d['inner_iters_per_s'], d['mean_inner_iters_per_patch'], d['converged_fraction'], d['roofline']['frac'], d['stop_rules'], d['recovery']['fraction'])"
