timeout 900 python tools/inner_trace.py --patch 21 --outer 1 --variants "default;ns=1" > gpurun_out/r2_inner_trace21d.log 2>&1; echo "trace21 rc=$?"
cut -c1-500 gpurun_out/r2_inner_trace21d.log
