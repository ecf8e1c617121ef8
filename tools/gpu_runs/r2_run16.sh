# ncu: --set full of the CTA k_solve (S64, 592 patches x 30 inner iterations, NS period 4) and the
# launch list of a bench command (one ncu tool per call; each command first exits 0 without ncu)
mkdir -p gpurun_out/ncu
python tools/prof_solve.py --batch 592 --inner 30 --ns 4 > gpurun_out/ncu/prof_plain.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_solve -c 1 -o gpurun_out/ncu/k_solve_r2 -f python tools/prof_solve.py --batch 592 --inner 30 --ns 4 > gpurun_out/ncu/ncu_full.log 2>&1; echo "ncu full rc=$?"
tail -3 gpurun_out/ncu/ncu_full.log
python bench.py --global-batch 4096 --steps 2 --warmup 1 --no-cpu --no-e2e > gpurun_out/ncu/bench_plain.log 2>&1 && \
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/ncu/bench_launches.csv python bench.py --global-batch 4096 --steps 2 --warmup 1 --no-cpu --no-e2e > gpurun_out/ncu/ncu_launches.log 2>&1; echo "ncu launches rc=$?"
wc -l gpurun_out/ncu/bench_launches.csv
