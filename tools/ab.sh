#!/bin/bash
# A/B bench runs: tools/ab.sh TAG < spec, spec lines "label|ENV=VAL ...|bench args"
TAG=${1:-ab}; cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
OUT=gpurun_out/$TAG; mkdir -p "$OUT"
while IFS='|' read -r label envs args; do
  [ -z "$label" ] && continue
  env $envs timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-cusparse ${AB_EXTRA:-} $args > "$OUT/ab_$label.log" 2>&1
  echo "$label: $(python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print('step %.3f spmm %.4f plan %.3f frac %.3f graph %s' % (d['ms_per_step'], d['spmm_only']['ms_per_layer'], d['plan_ms'], d['roofline']['frac'], d.get('spmm_graph', {}).get('ms_per_layer', '-')))" "$OUT/ab_$label.log" 2>&1 | tail -1)"
done
