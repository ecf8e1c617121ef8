# final measurement set at HEAD: the driver's bench command, the reference arm, ncu of k_solve and the launch list
timeout 1700 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2_bench_final4.log 2>&1; echo "bench rc=$?"
grep "^\[bench\]" gpurun_out/r2_bench_final4.log
timeout 900 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2_ref_final4.log 2>&1; echo "ref rc=$?"
mkdir -p gpurun_out/ncu4
python tools/prof_solve.py --batch 592 --inner 30 --ns 4 > gpurun_out/ncu4/prof_plain.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_solve -c 1 -o gpurun_out/ncu4/k_solve_r2_final4 -f python tools/prof_solve.py --batch 592 --inner 30 --ns 4 > gpurun_out/ncu4/ncu_full.log 2>&1; echo "ncu full rc=$?"
python bench.py --global-batch 4096 --steps 2 --warmup 1 --no-cpu --no-e2e > gpurun_out/ncu4/bench_plain.log 2>&1 && \
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/ncu4/bench_launches.csv python bench.py --global-batch 4096 --steps 2 --warmup 1 --no-cpu --no-e2e > gpurun_out/ncu4/ncu_launches.log 2>&1; echo "ncu launches rc=$?"
