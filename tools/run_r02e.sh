set -x
OUT=gpurun_out/r02e; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail -20 $OUT/build.log; exit 1; }
timeout 1200 python -m pytest tests -q -m gpu -x -k "not full_size" > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -15 $OUT/pytest_gpu.log
for v in "--hot-rows 0" "" "--l2-hint hot_hints" "--l2-hint none" "--hot-rows 160000" "--hot-rows 600000"; do
  timeout 600 python bench.py --config c5 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-cusparse --no-per-graph --no-graph $v > $OUT/ab.log 2>&1
  echo "c5 [$v]: $(python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(round(d['ms_per_step'],3), 'spmm', round(d['spmm_only']['ms_per_layer'],3), 'plan', round(d['plan_ms'],3))" $OUT/ab.log 2>&1 | tail -1)"
done
for c in c4 c3; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-cusparse --no-per-graph --no-graph > $OUT/ab_$c.log 2>&1
  echo "$c: $(python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(round(d['ms_per_step'],3), 'spmm', round(d['spmm_only']['ms_per_layer'],3), 'plan', round(d['plan_ms'],3))" $OUT/ab_$c.log 2>&1 | tail -1)"
done
