# the driver's bench command (N=1, K=20, W=5) and the reference arm, then a 2-rank gloo smoke of the N>1 path
timeout 1700 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2_bench_final1.log 2>&1; echo "bench rc=$?"
grep "^\[bench\]" gpurun_out/r2_bench_final1.log; tail -c 4000 gpurun_out/r2_bench_final1.log
timeout 900 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2_ref_final1.log 2>&1; echo "ref rc=$?"
tail -c 1500 gpurun_out/r2_ref_final1.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 2 --steps 4 --warmup 3 --global-batch 2048 --backend gloo --no-cpu --no-k1 > gpurun_out/r2_bench_gloo2.log 2>&1; echo "gloo2 rc=$?"
tail -c 2500 gpurun_out/r2_bench_gloo2.log
