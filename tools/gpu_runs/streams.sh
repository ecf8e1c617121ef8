cd $GRAFT_REPO_ROOT
for ns in 2 3 4; do
  timeout 900 python bench.py --steps 20 --warmup 3 --streams $ns --no-e2e --no-cpu --no-k1 > gpurun_out/streams_$ns.log 2>&1
  echo "streams=$ns $(grep '^{' gpurun_out/streams_$ns.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["ms_per_step"], d["inner_iters_per_s"], d["roofline"]["frac"])')"
done
