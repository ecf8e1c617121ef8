timeout 1200 python tools/inner_drift.py --patch 21 > gpurun_out/r2_inner_drift21.log 2>&1; echo "drift rc=$?"
cat gpurun_out/r2_inner_drift21.log
