# usage: tools/run_ab.sh TAG "variant args" ... ; env CONFIGS (default c5), TESTS=1 runs the quick GPU tests
TAG=$1; shift
OUT=gpurun_out/$TAG; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail -20 $OUT/build.log; exit 1; }
if [ -n "$TESTS" ]; then timeout 1200 python -m pytest tests -q -m gpu -x -k "not full_size" > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 $OUT/pytest_gpu.log; fi
for c in ${CONFIGS:-c5}; do for v in "$@"; do
  tag=$(echo "$c $v" | tr ' -' '__')
  timeout 600 python bench.py --config $c --steps ${STEPS:-10} --warmup 3 --no-cpu-baseline --no-e2e --no-cusparse --no-per-graph $v > $OUT/ab_$tag.log 2>&1
  echo "$c [$v]: $(python -c "
import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
g=d.get('spmm_graph') or {}
print(round(d['ms_per_step'],3), 'spmm', round(d['spmm_only']['ms_per_layer'],4), 'graph', round(g.get('ms_per_layer',0),4), 'plan', round(d['plan_ms'],3))" $OUT/ab_$tag.log 2>&1 | tail -1)"
done; done
if [ -n "$NCU_LIST" ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file $OUT/launches.csv python bench.py --profile --steps 2 --warmup 1 $NCU_LIST > $OUT/ncu_list.log 2>&1; echo "ncu_list rc=$?"
  python tools/launches.py $OUT/launches.csv 2>&1 | head -30
fi
