# round 2, run 7: Moreau-form SVT (CTA + multi-CTA): traces, full -m gpu suite, bench 8192
timeout 900 python tools/inner_trace.py --patch 0 --outer 1 --variants "default" > gpurun_out/r2_inner_trace0c.log 2>&1; echo "trace0 rc=$?"
timeout 900 python tools/inner_trace.py --patch 21 --outer 1 --variants "default" > gpurun_out/r2_inner_trace21c.log 2>&1; echo "trace21 rc=$?"
cut -c1-600 gpurun_out/r2_inner_trace0c.log gpurun_out/r2_inner_trace21c.log
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -rA -k "not free_running_convergence_config2_64" > gpurun_out/r2_gpu_tests7.log 2>&1; echo "tests rc=$?"
grep -v "^PASSED" gpurun_out/r2_gpu_tests7.log | tail -30
timeout 900 python bench.py --global-batch 8192 --steps 4 --warmup 3 --no-cpu --no-e2e > gpurun_out/r2_bench_8192f.log 2>&1; echo "bench rc=$?"
python -c "
import json; l=[x for x in open('gpurun_out/r2_bench_8192f.log') if x.startswith('{')][-1]; d=json.loads(l)
print(d['value'], d['inner_iters_per_s'], d['mean_inner_iters_per_patch'], d['converged_fraction'], d['roofline']['frac'], d['stop_rules'], d['recovery']['fraction'])"
timeout 1200 python tools/free_running_trace.py --patches 25,62,22,21,0,1 --out gpurun_out/r2_free_trace2.jsonl > gpurun_out/r2_free_trace2.log 2>&1; echo "trace rc=$?"
python -c "
import json
for l in open('gpurun_out/r2_free_trace2.jsonl'):
    d=json.loads(l); print(d['patch'], d['outer'], 'final dtau %.2e' % d['dtau'][-1], 'max %.2e' % max(d['dtau']), 'gpu caps', sum(x>=1000 for x in d['inner_gpu']), 'inner gpu/oracle', sum(d['inner_gpu']), sum(d['inner_oracle']))"
