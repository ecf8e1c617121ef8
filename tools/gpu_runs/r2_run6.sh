# round 2, run 6: exact-residual (res3) + Moreau-form SVT: inner traces, parity, bench
timeout 900 python tools/inner_trace.py --patch 0 --outer 1 --variants "default" > gpurun_out/r2_inner_trace0b.log 2>&1; echo "trace0 rc=$?"
timeout 900 python tools/inner_trace.py --patch 21 --outer 1 --variants "default" > gpurun_out/r2_inner_trace21b.log 2>&1; echo "trace21 rc=$?"
cut -c1-700 gpurun_out/r2_inner_trace0b.log gpurun_out/r2_inner_trace21b.log
timeout 1500 python -m pytest tests/test_gpu_steps.py tests/test_gpu_tilt.py tests/test_gpu_adm.py tests/test_gpu_protocol.py -m gpu -q -p no:cacheprovider -rA -k "not free_running_convergence_config2_64" > gpurun_out/r2_gpu_tests6.log 2>&1; echo "tests rc=$?"
grep -v "^PASSED" gpurun_out/r2_gpu_tests6.log | tail -25
timeout 900 python bench.py --global-batch 8192 --steps 4 --warmup 3 --no-cpu --no-e2e > gpurun_out/r2_bench_8192e.log 2>&1; echo "bench rc=$?"
python -c "
import json; l=[x for x in open('gpurun_out/r2_bench_8192e.log') if x.startswith('{')][-1]; d=json.loads(l)
print(d['value'], d['inner_iters_per_s'], d['mean_inner_iters_per_patch'], d['converged_fraction'], d['roofline']['frac'], d['stop_rules'], d['recovery']['fraction'])"
