python tools/c4_prof.py --batch 256 --outer 1 --inner 30 > gpurun_out/c4_plain.log 2>&1; echo "plain rc=$?"; cat gpurun_out/c4_plain.log
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c4_launches.csv python tools/c4_prof.py --batch 256 --outer 1 --inner 30 > gpurun_out/c4_ncu.log 2>&1; echo "ncu rc=$?"
wc -l gpurun_out/c4_launches.csv
