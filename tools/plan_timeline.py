#!/usr/bin/env python
"""GPU timeline of one agcn_plan (and optionally the SpMM layers after it) through the CUPTI
activity records of torch.profiler: every kernel / memcpy / memset with its start, duration
and the idle gap before it.   python tools/plan_timeline.py c5 [layers] ['{"hot_rows": 0}']"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import agcn_inputs  # noqa: E402
import paper_2308_11825_b200 as A  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c5"
layers = int(sys.argv[2]) if len(sys.argv) > 2 else 0
kw = dict(max_block_warps=0, max_warp_nzs=0, **(json.loads(sys.argv[3]) if len(sys.argv) > 3 else {}))
w = agcn_inputs.make_config(cfg)
dev = torch.device("cuda:0")
rp, ci = torch.from_numpy(w.rowptr).to(dev), torch.from_numpy(w.colidx).to(dev)
va = torch.from_numpy(w.vals).to(dev)
X = torch.from_numpy(w.X()).to(dev)
Y = [torch.empty_like(X), torch.empty_like(X)]


def step():
    p = A.Plan(rp, ci, w.n, w.nnz, **kw)
    x = X
    for i in range(layers):
        p.spmm(va, x, out=Y[i % 2])
        x = Y[i % 2]
    return p


for _ in range(3):
    step().close()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    p = step()
    torch.cuda.synchronize()
p.close()
evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
evs.sort(key=lambda e: e.time_range.start)
t0 = evs[0].time_range.start
prev_end = t0
busy = 0.0
print(f"{'start_us':>9} {'dur_us':>8} {'gap_us':>7}  name")
for e in evs:
    s, d = e.time_range.start, e.time_range.end - e.time_range.start
    gap = max(0.0, s - prev_end)
    print(f"{s - t0:9.1f} {d:8.1f} {gap:7.1f}  {e.name[:90]}")
    busy += d
    prev_end = max(prev_end, e.time_range.end)
print(f"span {prev_end - t0:.1f} us, busy {busy:.1f} us, idle {prev_end - t0 - busy:.1f} us, {len(evs)} activities")
# host side: CUDA runtime API calls (CUPTI callbacks) on the same clock
api = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CPU and e.name.startswith("cuda")]
api.sort(key=lambda e: e.time_range.start)
print(f"\nhost runtime API calls ({len(api)}), start relative to the first GPU activity:")
print(f"{'start_us':>9} {'dur_us':>8}  name")
for e in api:
    d = e.time_range.end - e.time_range.start
    if d >= 3.0 or e.name.startswith(("cudaStreamSync", "cudaMemcpy", "cudaMalloc", "cudaEventSync")):
        print(f"{e.time_range.start - t0:9.1f} {d:8.1f}  {e.name}")
