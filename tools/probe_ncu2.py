#!/usr/bin/env python
"""ncu companion of tools/stream_probe.py: one launch each of the compact-hot-buffer variants
(H = 312000 hottest columns = 80 MB): plain, L2 hints (hot evict_last / cold evict_first),
persisting access-policy window over the hot buffer -- does either raise the L2 hit rate?"""
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
    X = torch.from_numpy(w.X()).to(dev)
    counts = torch.bincount(ci.long(), minlength=n)
    order = torch.argsort(counts, descending=True, stable=True)
    plan = agcn.Plan(rp, ci)
    sidx = torch.from_numpy(plan.copy("sorted_colidx")).to(dev)
    svals = torch.ones(nnz, dtype=torch.float32, device=dev)
    out = torch.empty((1 << 22, F), dtype=torch.float32, device=dev)
    H = int(sys.argv[1]) if len(sys.argv) > 1 else 312000
    rank = torch.full((n,), -1, dtype=torch.int64, device=dev)
    rank[order[:H]] = torch.arange(H, device=dev)
    r = rank[sidx.long()]
    e = torch.where(r >= 0, -1 - r, sidx.long()).to(torch.int32)
    Xh = X[order[:H]].contiguous()
    prop = torch.cuda.get_device_properties(0)
    maxp = 82903040
    run = lambda hints: lib.probe_stream(0, 1, hints, 0, X.data_ptr(), Xh.data_ptr(), e.data_ptr(),
                                         svals.data_ptr(), nnz, 384, out.data_ptr(), 1 << 22, st)
    for _ in range(2):
        run(0)
    torch.cuda.synchronize()
    run(0)
    run(1)
    rc = lib.probe_window(ctypes.c_void_p(st), ctypes.c_void_p(Xh.data_ptr()), min(Xh.numel() * 4, maxp), maxp)
    print("window rc", rc)
    run(0)
    run(0)
    lib.probe_window(ctypes.c_void_p(st), None, 0, 0)
    torch.cuda.synchronize()
    print("done")


if __name__ == "__main__":
    main()
