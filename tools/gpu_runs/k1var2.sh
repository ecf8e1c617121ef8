cd $GRAFT_REPO_ROOT
echo "base $(timeout 120 python tools/k1_run.py 65536)"
for v in g h i j k l g; do echo "k1$v $(TILT_LIB=$PWD/build/var/libtilt_k1$v.so timeout 120 python tools/k1_run.py 65536)"; done
