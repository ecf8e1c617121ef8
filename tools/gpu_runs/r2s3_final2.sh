# final measurement at HEAD (S56 / S100 classes): driver bench command, launch list, ncu of k_solve<S56>
cd $GRAFT_REPO_ROOT
timeout 1700 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2s3_bench_final2.log 2>&1; echo "bench rc=$?"
mkdir -p gpurun_out/ncu7
python bench.py --global-batch 4096 --steps 2 --warmup 1 --no-cpu --no-e2e > gpurun_out/ncu7/bench_plain.log 2>&1 && \
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/ncu7/bench_launches.csv python bench.py --global-batch 4096 --steps 2 --warmup 1 --no-cpu --no-e2e > gpurun_out/ncu7/ncu_launches.log 2>&1; echo "ncu launches rc=$?"
python tools/prof_solve.py --batch 592 --inner 30 --ns 4 > gpurun_out/ncu7/prof_plain.log 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_solve -c 1 -o gpurun_out/ncu7/k_solve_s56 -f python tools/prof_solve.py --batch 592 --inner 30 --ns 4 > gpurun_out/ncu7/ncu_full.log 2>&1; echo "ncu full rc=$?"
ncu -i gpurun_out/ncu7/k_solve_s56.ncu-rep --page source --csv --print-source=cuda,sass > gpurun_out/ncu7/k_solve_src.csv 2>/dev/null
ncu -i gpurun_out/ncu7/k_solve_s56.ncu-rep --page raw --csv > gpurun_out/ncu7/k_solve_raw.csv 2>/dev/null
rm -f gpurun_out/ncu7/k_solve_s56.ncu-rep
