#!/bin/bash
# Config / F / kernel sweep with cuSPARSE and CUDA-graph kernel-only timing:
#   tools/sweep.sh TAG < spec   (spec lines "label|ENV=VAL ...|bench args")
TAG=${1:-sweep}; cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
OUT=gpurun_out/$TAG; mkdir -p "$OUT"
while IFS='|' read -r label envs args; do
  [ -z "$label" ] && continue
  env $envs timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e $args > "$OUT/sw_$label.log" 2>&1
  echo "$label: $(python -c "
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
g=d.get('spmm_graph',{}); c=d.get('cusparse',{})
print('step %.3f spmm %.4f graph %s cusp %s cusp_graph %s plan %.3f' % (d['ms_per_step'], d['spmm_only']['ms_per_layer'], round(g.get('ms_per_layer',-1),4), round(c.get('ms_per_layer',-1),4), round(c.get('graph_ms_per_layer',-1),4), d['plan_ms']))" "$OUT/sw_$label.log" 2>&1 | tail -1)"
done
