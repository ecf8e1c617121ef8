cd $GRAFT_REPO_ROOT
nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/cgp tools/experiments/cond_graph_probe.cu && /tmp/cgp
for b in 1 16 256; do timeout 300 python tools/c4_prof.py --batch $b --inner 30 2>&1 | tail -1; done
timeout 900 python -m pytest tests/test_gpu_large.py -m gpu -q -x 2>&1 | tail -2
timeout 900 python tools/configs_bench.py --configs 4 2>&1 | tail -1
