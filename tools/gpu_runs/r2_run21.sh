python tools/prof_solve.py --batch 592 --inner 30 --ns 4 --reps 3 > gpurun_out/prof_l2.log 2>&1; echo "plain rc=$?"; cat gpurun_out/prof_l2.log
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:k_solve --csv python tools/prof_solve.py --batch 592 --inner 30 --ns 4 --reps 1 > gpurun_out/prof_l2_ncu.csv 2>gpurun_out/prof_l2_ncu.err; echo "ncu rc=$?"
grep -E "dram__|lts__t_sector_hit|gpu__time" gpurun_out/prof_l2_ncu.csv | cut -d, -f12- 
timeout 900 python -m pytest tests/test_gpu_tilt.py -m gpu -q -x -p no:cacheprovider > gpurun_out/r2_gpu_tests21.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/r2_gpu_tests21.log
timeout 900 python bench.py --global-batch 8192 --steps 4 --warmup 3 --no-cpu --no-e2e --no-k1 > gpurun_out/r2_bench_8192j.log 2>&1; echo "bench rc=$?"
python -c "
import json; l=[x for x in open('gpurun_out/r2_bench_8192j.log') if x.startswith('{')][-1]; d=json.loads(l)
print(d['value'], d['inner_iters_per_s'], d['mean_inner_iters_per_patch'], d['roofline']['frac'])"
