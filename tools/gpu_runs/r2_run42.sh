# two-pass K1 (reductions, then a streaming output kernel): roofline, warp parity tests; output-kernel occupancy variant
for N in 8192 65536; do echo "minb4 $N $(timeout 300 python tools/k1_run.py $N 2>&1 | tail -1)" | tee -a gpurun_out/r2_k1_2pass.log; done
timeout 900 python -m pytest tests/test_gpu_steps.py -m gpu -x -q 2>&1 | tail -3 | tee -a gpurun_out/r2_k1_2pass.log
cp paper_1205_5351_b200/libtilt_o2.so paper_1205_5351_b200/libtilt.so
for N in 8192 65536; do echo "minb2 $N $(timeout 300 python tools/k1_run.py $N 2>&1 | tail -1)" | tee -a gpurun_out/r2_k1_2pass.log; done
