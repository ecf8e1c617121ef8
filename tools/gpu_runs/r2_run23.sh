for v in 1 0 0 1; do TILT_L2_PERSIST=$v python tools/prof_solve.py --batch 2368 --inner 30 --ns 4 --reps 3 2>&1 | tail -1 | sed "s/^/persist=$v /"; done
for v in 0 1; do TILT_L2_PERSIST=$v timeout 900 python bench.py --global-batch 8192 --steps 4 --warmup 3 --no-cpu --no-e2e --no-k1 > gpurun_out/r2_bench_p$v.log 2>&1; python -c "
import json; l=[x for x in open('gpurun_out/r2_bench_p$v.log') if x.startswith('{')][-1]; d=json.loads(l)
print('persist=$v bench8192', d['value'], d['inner_iters_per_s'], d['mean_inner_iters_per_patch'], d['roofline']['frac'])"; done
