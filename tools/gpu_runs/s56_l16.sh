#!/bin/bash
# S56 with 16-lane pair units (4 rows per lane, 13 warps) at 2 and 3 CTAs/SM vs the 8-lane default.
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
for i in 1 2; do
  for v in dflt l16m2 l16m3; do
    echo "== $v" >> gpurun_out/r2s4_s56_l16.log
    TILT_LIB=build/var/libtilt_$v.so timeout 300 python tools/prof_solve.py --batch 2368 --inner 30 --ns 4 >> gpurun_out/r2s4_s56_l16.log 2>&1
  done
done
