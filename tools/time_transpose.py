"""Time agcn_transpose (+ gather_vals + plan of A^T + one backward SpMM) on a config."""
import json
import sys
import os

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import agcn_inputs as gen  # noqa: E402
import paper_2308_11825_b200 as A  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c5"
w = gen.make_config(name)
dev = torch.device("cuda:0")
rp, ci, va = (torch.from_numpy(a).to(dev) for a in (w.rowptr, w.colidx, w.vals))
dY = torch.from_numpy(w.X()).to(dev)
ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
for _ in range(2):
    rt, ct, src = A.transpose(rp, ci, w.n)
torch.cuda.synchronize()
t = {}
a, b, c, d, e = ev(), ev(), ev(), ev(), ev()
a.record()
rt, ct, src = A.transpose(rp, ci, w.n)
b.record()
vt = A.gather_vals(va, src)
c.record()
pt = A.Plan(rt, ct, n_cols=w.n)
d.record()
dX = pt.spmm(vt, dY)
e.record()
torch.cuda.synchronize()
print(json.dumps({"config": name, "nnz": w.nnz, "transpose_ms": a.elapsed_time(b), "gather_vals_ms": b.elapsed_time(c),
                  "plan_t_ms": c.elapsed_time(d), "backward_spmm_ms": d.elapsed_time(e)}))
