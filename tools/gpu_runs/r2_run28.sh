# A/B: ladmap_inner inlined (default) vs __noinline__ (separate register allocation)
for v in inline noinline inline noinline; do cp build/libtilt_$v.so paper_1205_5351_b200/libtilt.so; python tools/prof_solve.py --batch 2368 --inner 30 --ns 4 --reps 3 2>&1 | tail -1 | sed "s/^/$v /"; done
cp build/libtilt_noinline.so paper_1205_5351_b200/libtilt.so
timeout 900 python bench.py --global-batch 8192 --steps 4 --warmup 3 --no-cpu --no-e2e --no-k1 > gpurun_out/r2_bench_noinl.log 2>&1; python -c "
import json; l=[x for x in open('gpurun_out/r2_bench_noinl.log') if x.startswith('{')][-1]; d=json.loads(l)
print('noinline bench8192', d['value'], d['inner_iters_per_s'], d['mean_inner_iters_per_patch'], d['roofline']['frac'])"
