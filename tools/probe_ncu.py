#!/usr/bin/env python
"""One launch each of the C5 stream-probe variants and of agcn_spmm (orig / heat layout), for an
ncu capture that compares their DRAM traffic, L2 hit rate and stalls (round 2).

    ncu --set full -k regex:'k_stream|k_spmm' -o gpurun_out/x python tools/probe_ncu.py
"""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

import torch  # noqa: E402

import agcn_inputs  # noqa: E402
import paper_2308_11825_b200 as agcn  # noqa: E402
from stream_probe import build_probe  # noqa: E402


def main():
    lib = build_probe()
    dev = torch.device("cuda:0")
    st = torch.cuda.current_stream().cuda_stream
    w = agcn_inputs.make_config("c5")
    n, nnz, F = w.n, w.nnz, 64
    rp = torch.from_numpy(w.rowptr).to(dev)
    ci = torch.from_numpy(w.colidx).to(dev)
    vals = torch.from_numpy(w.vals).to(dev)
    X = torch.from_numpy(w.X()).to(dev)
    Y = torch.empty_like(X)
    counts = torch.bincount(ci.long(), minlength=n)
    order = torch.argsort(counts, descending=True, stable=True)
    rank = torch.empty(n, dtype=torch.int64, device=dev)
    rank[order] = torch.arange(n, device=dev)
    plan = agcn.Plan(rp, ci)
    sidx = torch.from_numpy(plan.copy("sorted_colidx")).to(dev)
    svals = torch.ones(nnz, dtype=torch.float32, device=dev)
    out_rows = 1 << 22
    out = torch.empty((out_rows, F), dtype=torch.float32, device=dev)
    pidx = rank[sidx.long()].to(torch.int32)
    Xp = X[order].contiguous()
    torch.cuda.synchronize()
    # 1 probe: sorted stream, original X, vals + Y    2 probe: heat-permuted    3 probe bare orig
    lib.probe_stream(0, 0, 0, 1, X.data_ptr(), X.data_ptr(), sidx.data_ptr(), svals.data_ptr(), nnz, 384,
                     out.data_ptr(), out_rows, st)
    lib.probe_stream(0, 0, 0, 1, Xp.data_ptr(), X.data_ptr(), pidx.data_ptr(), svals.data_ptr(), nnz, 384,
                     out.data_ptr(), out_rows, st)
    lib.probe_stream(0, 0, 0, 0, X.data_ptr(), X.data_ptr(), sidx.data_ptr(), svals.data_ptr(), nnz, 384,
                     out.data_ptr(), out_rows, st)
    plan.spmm(vals, X, out=Y)
    ci3 = rank[ci.long()].to(torch.int32)
    with agcn.Plan(rp, ci3) as p3:
        p3.spmm(vals, Xp, out=Y)
    torch.cuda.synchronize()
    print("done")


if __name__ == "__main__":
    main()
