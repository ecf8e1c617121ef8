cd $GRAFT_REPO_ROOT
echo "base $(timeout 120 python tools/k1_run.py 65536)"
for v in s5 s6 s7 s55; do echo "k1$v $(TILT_LIB=$PWD/build/var/libtilt_k1$v.so timeout 120 python tools/k1_run.py 65536)"; done
echo "base $(timeout 120 python tools/k1_run.py 65536)"
