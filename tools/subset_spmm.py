#!/usr/bin/env python
"""One agcn_spmm (after 2 warm-up calls) on a row-degree class of a config (the other rows
emptied; same n, X), for ncu:  python tools/subset_spmm.py c5 385 1000000000 [spmm kwargs json]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import agcn_inputs  # noqa: E402
import paper_2308_11825_b200 as agcn  # noqa: E402

name, lo, hi = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
kw = json.loads(sys.argv[4]) if len(sys.argv) > 4 else {}
pk = kw.pop("plan", {})
dev = torch.device("cuda:0")
w = agcn_inputs.make_config(name)
deg = np.diff(w.rowptr)
keep = (deg >= lo) & (deg <= hi)
rp = np.zeros(w.n + 1, np.int64)
rp[1:] = np.cumsum(np.where(keep, deg, 0))
idx = np.repeat(keep, deg)
X = torch.from_numpy(w.X()).to(dev)
p = agcn.Plan(torch.from_numpy(rp.astype(np.int32)).to(dev), torch.from_numpy(w.colidx[idx]).to(dev), **pk)
va = torch.from_numpy(w.vals[idx]).to(dev)
for _ in range(3):
    Y = p.spmm(va, X, **kw)
torch.cuda.synchronize()
print("done", int(keep.sum()), int(idx.sum()))
