cd $GRAFT_REPO_ROOT
for rep in 1 2; do
for lib in paper_1205_5351_b200/libtilt.so build/var/libtilt_nw7.so; do
  echo "$lib: $(TILT_LIB=$PWD/$lib timeout 300 python tools/prof_solve.py --batch 2368 --inner 30 --ns 4 --cfg 2 --reps 3 2>&1 | tail -1)"
done; done
