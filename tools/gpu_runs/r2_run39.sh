# ncu --set full of the standalone K1 (k_warp) on the 1024-patch bench shard
mkdir -p gpurun_out/k1
python tools/k1_run.py > gpurun_out/k1/plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_warp --launch-skip 2 -c 1 -o gpurun_out/k1/k_warp -f python tools/k1_run.py > gpurun_out/k1/ncu.log 2>&1; echo "ncu rc=$?"
cat gpurun_out/k1/plain.log | tail -1
