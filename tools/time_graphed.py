"""Eager vs CUDA-graph-captured propagation (GraphedPropagation) on the small BASELINE graphs."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import agcn_inputs as gen  # noqa: E402
import paper_2308_11825_b200 as A  # noqa: E402

for name, F, layers in (("c1", 16, 2), ("c2", 64, 2), ("c3", 64, 2)):
    w = gen.make_config(name)
    X = torch.from_numpy(w.X(F)).cuda()
    rp, ci, va = (torch.from_numpy(a).cuda() for a in (w.rowptr, w.colidx, w.vals))
    g = A.GraphedPropagation(rp, ci, va, X, layers, max_block_warps=0, max_warp_nzs=0)
    p = g.plan
    reps = 200

    def eager():
        cur = X
        for _ in range(layers):
            cur = p.spmm(va, cur)
        return cur

    for fn, tag in ((eager, "eager"), (g.replay, "graph")):
        for _ in range(10):
            fn()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(reps):
            fn()
        torch.cuda.synchronize()
        print(f"{name} F={F} layers={layers} {tag}: {1e6 * (time.perf_counter() - t0) / reps:.1f} us per propagation")
    g.close()
