#!/bin/bash
# Session 4 of round 2: -m gpu suite + smoke at HEAD, and the S56 occupancy probe (5 CTAs/SM variant).
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r2s4_pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/r2s4_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r2s4_smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/r2s4_smoke.log
for i in 1 2; do
  timeout 300 python tools/prof_solve.py --batch 2368 --inner 30 --ns 4 >> gpurun_out/r2s4_probe_default.log 2>&1
  TILT_LIB=build/var/libtilt_m5.so timeout 300 python tools/prof_solve.py --batch 2368 --inner 30 --ns 4 >> gpurun_out/r2s4_probe_minb5.log 2>&1
done
