# The chunk-kernel sweep of r02be: default vs --chunk-shape 4 on C3 / C2 / C5 / C4 at several F
# (minimal bench, 2 rounds).  usage: bash tools/run_sweep2.sh
python -c "import __graft_entry__ as g; g.build()" > /tmp/build.log 2>&1 || { tail /tmp/build.log; exit 1; }
F="--no-cpu-baseline --no-e2e --no-cusparse --no-traffic --no-graph --no-per-graph --steps 20 --warmup 3"
for r in 1 2; do for c in "--config c3" "--config c2 --F 64" "--config c2 --F 32" "--config c3 --F 32" "--config c5 --F 32" "--config c4 --F 64"; do for o in "" "--chunk-shape 4"; do
  timeout 600 python bench.py $F $c $o > /tmp/b.log 2>&1
  tail -1 /tmp/b.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('[$c $o]', round(d['ms_per_step'],4), round(d['plan_ms'],4), round(d['spmm_only']['ms_per_layer'],4), d['self_check']['ok'])" || tail -3 /tmp/b.log
done; done; done
