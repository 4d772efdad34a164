# A/B of library variants (ab_libs/libagcn_*.so via AGCN_LIBRARY) with the minimal bench, interleaved.
# usage: bash tools/run_ab_libs.sh "c5 c4" "base csr_na csr_ef" ROUNDS
CFGS=${1:-c5}; VARS=${2:-base}; R=${3:-2}
python -c "import __graft_entry__ as g; g.build()" > /tmp/build.log 2>&1 || { tail /tmp/build.log; exit 1; }
F="--no-cpu-baseline --no-e2e --no-cusparse --no-traffic --no-graph --no-per-graph --steps 10 --warmup 3"
for r in $(seq $R); do for c in $CFGS; do for v in $VARS; do
  if [ $v = base ]; then unset AGCN_LIBRARY; else export AGCN_LIBRARY=$PWD/ab_libs/libagcn_$v.so; fi
  timeout 600 python bench.py $F --config $c > /tmp/b.log 2>&1
  tail -1 /tmp/b.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c $v', round(d['ms_per_step'],3), round(d['plan_ms'],3), round(d['spmm_only']['ms_per_layer'],4), d['self_check']['ok'])" || tail -3 /tmp/b.log
done; done; done
