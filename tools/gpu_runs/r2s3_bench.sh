# measurement at HEAD (session 3): the driver's bench command and the launch list of the same program
cd $GRAFT_REPO_ROOT
timeout 1700 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2s3_bench.log 2>&1; echo "bench rc=$?"
mkdir -p gpurun_out/ncu5
python bench.py --global-batch 4096 --steps 2 --warmup 1 --no-cpu --no-e2e > gpurun_out/ncu5/bench_plain.log 2>&1 && \
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/ncu5/bench_launches.csv python bench.py --global-batch 4096 --steps 2 --warmup 1 --no-cpu --no-e2e > gpurun_out/ncu5/ncu_launches.log 2>&1; echo "ncu launches rc=$?"
