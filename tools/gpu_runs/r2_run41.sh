# K1 with the footprint staged in shared memory: roofline at 8192 / 65536 patches, warp parity tests
for N in 8192 65536; do echo "$N $(timeout 300 python tools/k1_run.py $N 2>&1 | tail -1)" | tee -a gpurun_out/r2_k1_foot.log; done
timeout 900 python -m pytest tests/test_gpu_steps.py -m gpu -x -q 2>&1 | tail -3 | tee -a gpurun_out/r2_k1_foot.log
