cd $GRAFT_REPO_ROOT
for lib in paper_1205_5351_b200/libtilt.so build/var/libtilt_l4w4.so build/var/libtilt_l4w8.so; do
  for b in 592 2368; do
    echo "$lib b=$b: $(TILT_LIB=$PWD/$lib timeout 300 python tools/prof_solve.py --batch $b --inner 30 --cfg 2 --reps 3 2>&1 | tail -1)"
  done
done
TILT_LIB=$PWD/build/var/libtilt_l4w4.so timeout 600 python -m pytest tests/test_gpu_tilt.py -m gpu -x -q -k "fixed_count_parity or sharding or edge" 2>&1 | tail -3
