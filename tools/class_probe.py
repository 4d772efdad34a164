#!/usr/bin/env python
"""Where does C5's SpMM time go by row class?  Times agcn_spmm on C5 restricted to row-degree
classes (the other rows emptied, same n, same X), and the zero-row stores alone.

    python tools/class_probe.py [--hot-rows H]
"""
import argparse
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import agcn_inputs  # noqa: E402
import paper_2308_11825_b200 as agcn  # noqa: E402


def timed(fn, reps=10):
    st = torch.cuda.current_stream()
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        fn()
        b.record(st)
        b.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--hot-rows", type=int, default=None)
    ap.add_argument("--mbw", type=int, default=12)
    ap.add_argument("--mwn", type=int, default=32)
    ap.add_argument("--classes", default=None, help="comma list of class names to run")
    args = ap.parse_args()
    dev = torch.device("cuda:0")
    w = agcn_inputs.make_config("c5")
    n, F = w.n, 64
    deg = np.diff(w.rowptr)
    X = torch.from_numpy(w.X()).to(dev)
    Y = torch.empty_like(X)
    classes = [("all", 1, 1 << 30), ("zero rows only", 0, 0), ("deg 1-8", 1, 8), ("deg 9-32", 9, 32),
               ("deg 33-128", 33, 128), ("deg 129-384", 129, 384), ("deg 385-512", 385, 512), ("deg > 512", 513, 1 << 30)]
    tot = deg.sum()
    if args.classes:
        keep_names = set(args.classes.split(","))
        classes = [c for c in classes if c[0] in keep_names]
    for name, lo, hi in classes:
        keep = (deg >= lo) & (deg <= hi)
        rp = np.zeros(n + 1, np.int64)
        rp[1:] = np.cumsum(np.where(keep, deg, 0))
        idx = np.repeat(keep, deg)
        ci = w.colidx[idx]
        va = w.vals[idx]
        p = agcn.Plan(torch.from_numpy(rp.astype(np.int32)).to(dev), torch.from_numpy(ci).to(dev),
                      hot_rows=args.hot_rows, max_block_warps=args.mbw, max_warp_nzs=args.mwn)
        vd = torch.from_numpy(va).to(dev)
        t = timed(lambda: p.spmm(vd, X, out=Y))
        nz = int(keep.sum() if lo > 0 else 0)
        print(f"{name:16s} rows {int(keep.sum()):8d} nnz {ci.size / tot * 100:5.1f}%  {t:.3f} ms  "
              f"{ci.size * 256 / t / 1e9:.2f} TB/s gathered", flush=True)
        p.close()


if __name__ == "__main__":
    main()
