# round 2, run 5: inner-loop traces (why fp32 loops run to max_inner), K1 with one fp64 division
timeout 900 python tools/inner_trace.py --patch 0 --outer 1 > gpurun_out/r2_inner_trace0.log 2>&1; echo "trace0 rc=$?"
timeout 900 python tools/inner_trace.py --patch 21 --outer 1 > gpurun_out/r2_inner_trace21.log 2>&1; echo "trace21 rc=$?"
cut -c1-900 gpurun_out/r2_inner_trace0.log gpurun_out/r2_inner_trace21.log
timeout 600 python bench.py --global-batch 8192 --steps 4 --warmup 3 --no-cpu --no-e2e > gpurun_out/r2_bench_8192d.log 2>&1; echo "bench rc=$?"
python -c "
import json; l=[x for x in open('gpurun_out/r2_bench_8192d.log') if x.startswith('{')][-1]; d=json.loads(l)
print(d['value'], d['inner_iters_per_s'], d['roofline']['frac'], d['roofline_k1'])"
