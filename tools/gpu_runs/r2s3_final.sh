# final measurement at HEAD: the driver's bench command and the reference arm
cd $GRAFT_REPO_ROOT
timeout 1700 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2s3_bench_final.log 2>&1; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2s3_ref_final.log 2>&1; echo "ref rc=$?"
