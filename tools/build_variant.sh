#!/bin/bash
# Build a libtilt variant with overridden compile-time tunables (experiment helper, not product):
#   tools/build_variant.sh NAME -DTILT_S64_L=8 -DTILT_S64_RPL=8 -DTILT_S64_NW=7 -DTILT_S64_MINB=4   (S64 layout)
#   tools/build_variant.sh NAME -DTILT_K1_NT=128 -DTILT_K1_ILP=4 -DTILT_K1_MINB=4                    (K1 shape)
# Output: build/var/libtilt_NAME.so (load with TILT_LIB=...), ptxas report build/var/ptxas_NAME.txt.
set -e
cd "$(dirname "$0")/.."
mkdir -p build/var
NAME=$1; shift
nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -O3 -std=c++17 -Xcompiler -fPIC -Xptxas=-v "$@" \
  -c -o build/var/tilt_$NAME.o paper_1205_5351_b200/csrc/tilt.cu 2> build/var/ptxas_$NAME.txt
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o build/var/libtilt_$NAME.so build/var/tilt_$NAME.o build/obj/tilt_large.o
grep -A2 "k_warp" build/var/ptxas_$NAME.txt | grep -E 'registers|spill' | head -2
