timeout 900 python tools/inner_drift2.py 21 > gpurun_out/r2_inner_drift2.log 2>&1; echo "drift2 rc=$?"
cat gpurun_out/r2_inner_drift2.log | tail -8
