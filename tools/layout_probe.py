#!/usr/bin/env python
"""Does the X-row layout move C5's SpMM?  (round 2, follows tools/stream_probe.py.)

Times the real agcn_spmm on C5 with the same graph and results under three column layouts:
  orig      colidx as generated, X in vertex order;
  compactH  the H hottest columns (by in-degree) relabelled to rows 0..H-1 of X' = [X[hot]; X]
            (the others keep their row, offset by H): a compact hot buffer in front of X;
  heat      every column relabelled by its in-degree rank, X' = X[order].
Y is identical in all three (checked).  Also times the permutation / hot gather itself.

    python tools/layout_probe.py
"""
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

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
    dev = torch.device("cuda:0")
    w = agcn_inputs.make_config("c5")
    n, nnz, F = w.n, w.nnz, 64
    rp = torch.from_numpy(w.rowptr).to(dev)
    ci = torch.from_numpy(w.colidx).to(dev)
    vals = torch.from_numpy(w.vals).to(dev)
    X = torch.from_numpy(w.X()).to(dev)
    counts = torch.bincount(ci.long(), minlength=n)
    order = torch.argsort(counts, descending=True, stable=True)
    rank = torch.empty(n, dtype=torch.int64, device=dev)
    rank[order] = torch.arange(n, device=dev)
    gathered = nnz * F * 4
    Y0 = torch.empty_like(X)
    with agcn.Plan(rp, ci) as p:
        t = timed(lambda: p.spmm(vals, X, out=Y0))
        print(f"orig                 {t:.3f} ms  {gathered / t / 1e9:.2f} TB/s", flush=True)
    for H in (160000, 250000, 312000, 390000, 600000):
        hot = rank < H
        newc = torch.where(hot, rank, torch.arange(n, device=dev) + H)
        ci2 = newc[ci.long()].to(torch.int32)
        X2 = torch.cat([X[order[:H]], X])
        Y = torch.empty_like(X)
        with agcn.Plan(rp, ci2, n_cols=n + H) as p:
            t = timed(lambda: p.spmm(vals, X2, out=Y))
            ok = torch.equal(Y, Y0)
            print(f"compact H={H:7d}   {t:.3f} ms  {gathered / t / 1e9:.2f} TB/s  equal={ok}", flush=True)
        tg = timed(lambda: torch.index_select(X, 0, order[:H], out=X2[:H]))
        print(f"   hot gather {H * F * 4 / 1e6:.0f} MB: {tg * 1e3:.1f} us", flush=True)
        del ci2, X2
    ci3 = rank[ci.long()].to(torch.int32)
    X3 = X[order].contiguous()
    Y = torch.empty_like(X)
    with agcn.Plan(rp, ci3) as p:
        t = timed(lambda: p.spmm(vals, X3, out=Y))
        print(f"heat                 {t:.3f} ms  {gathered / t / 1e9:.2f} TB/s  equal={torch.equal(Y, Y0)}",
              flush=True)
    tp = timed(lambda: torch.index_select(X, 0, order, out=X3))
    print(f"   full permutation (2.15 GB): {tp:.3f} ms", flush=True)


if __name__ == "__main__":
    main()
