#!/usr/bin/env python
"""Plan construction time on a config (CUDA events around agcn_plan_ex on the current stream and
host wall clock), per plan option set:  python tools/plan_time.py c5 '{}' '{"hot_rows": 0}' ..."""
import json
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import agcn_inputs  # noqa: E402
import paper_2308_11825_b200 as A  # noqa: E402

w = agcn_inputs.make_config(sys.argv[1])
dev = torch.device("cuda:0")
rp, ci = torch.from_numpy(w.rowptr).to(dev), torch.from_numpy(w.colidx).to(dev)
for v in sys.argv[2:]:
    kw = dict(max_block_warps=0, max_warp_nzs=0, **json.loads(v))
    for _ in range(3):
        A.Plan(rp, ci, **kw).close()
    torch.cuda.synchronize()
    ev, wall = [], []
    for _ in range(10):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        a.record()
        p = A.Plan(rp, ci, **kw)
        b.record()
        t1 = time.perf_counter()
        torch.cuda.synchronize()
        ev.append(a.elapsed_time(b))
        wall.append(1e3 * (t1 - t0))
        p.close()
    print(f"{sys.argv[1]} {v:30s} events {statistics.median(ev):.3f} ms  host wall {statistics.median(wall):.3f} ms",
          flush=True)
