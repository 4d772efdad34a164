# A/B of (library variant, bench flags) pairs, interleaved: bash tools/run_ab_flags.sh CONFIG ROUNDS "var|flags" ...
C=$1; R=$2; shift 2
python -c "import __graft_entry__ as g; g.build()" > /tmp/build.log 2>&1 || { tail /tmp/build.log; exit 1; }
F="--no-cpu-baseline --no-e2e --no-cusparse --no-traffic --no-graph --no-per-graph --steps 10 --warmup 3 --config $C"
for r in $(seq $R); do for vf in "$@"; do
  v=${vf%%|*}; o=${vf#*|}
  if [ "$v" = base ]; then unset AGCN_LIBRARY; else export AGCN_LIBRARY=$PWD/ab_libs/libagcn_$v.so; fi
  timeout 600 python bench.py $F $o > /tmp/b.log 2>&1
  tail -1 /tmp/b.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$C $v [$o]', round(d['ms_per_step'],3), round(d['plan_ms'],3), round(d['spmm_only']['ms_per_layer'],4), d['self_check']['ok'])" || tail -3 /tmp/b.log
done; done
