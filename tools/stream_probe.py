#!/usr/bin/env python
"""Gather roof for C5's actual column stream ("Next round" item 1).

Builds C5 (R-MAT s23 ef16), its plan, and replays the degree-sorted colidx stream through
tools/stream_probe.cu with the SpMM's access shape (F = 64, 256-B X rows, 8 lanes x 32 B).
Variants: original X; hot columns (top-H by in-degree) relabelled into a compact buffer Xh
(plain / evict_last+evict_first hints / persisting window over Xh); a full heat-order
permutation of X; a shuffled stream (control).  Each bare and with the vals stream + output
stores.  The real agcn_spmm is timed in the same process for comparison.

    python tools/stream_probe.py [--reps 10] [--quick]
"""
import argparse
import ctypes
import os
import statistics
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import agcn_inputs  # noqa: E402
import paper_2308_11825_b200 as agcn  # noqa: E402


def build_probe():
    src = os.path.join(ROOT, "tools", "stream_probe.cu")
    na = os.environ.get("PROBE_NA") == "1"   # loads with .L1::no_allocate (as the kernel's)
    so = "/tmp/stream_probe%s.so" % ("_na" if na else "")
    subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-shared",
                           "-Xcompiler", "-fPIC", "-lineinfo"] + (["-DPROBE_NA"] if na else []) + [src, "-o", so])
    lib = ctypes.CDLL(so)
    lib.probe_stream.argtypes = [ctypes.c_int] * 4 + [ctypes.c_void_p] * 4 + [ctypes.c_int64, ctypes.c_int,
                                                                            ctypes.c_void_p, ctypes.c_int64,
                                                                            ctypes.c_void_p]
    lib.probe_window.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_size_t]
    return lib


def timed(fn, reps):
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
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--quick", action="store_true")
    args = ap.parse_args()
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
    plan = agcn.Plan(rp, ci)
    t_spmm = timed(lambda: plan.spmm(vals, X, out=Y), args.reps)
    gathered = nnz * F * 4
    print(f"C5 n={n} nnz={nnz}  agcn_spmm {t_spmm:.3f} ms  {gathered / t_spmm / 1e9:.2f} TB/s gathered", flush=True)
    sidx = torch.from_numpy(plan.copy("sorted_colidx")).to(dev)
    svals = torch.ones(nnz, dtype=torch.float32, device=dev)
    out_rows = 1 << 22
    out = torch.empty((out_rows, F), dtype=torch.float32, device=dev)
    counts = torch.bincount(ci.long(), minlength=n)
    order = torch.argsort(counts, descending=True, stable=True)
    cum = torch.cumsum(counts[order].double(), 0) / nnz

    def enc_for(H):
        rank = torch.full((n,), -1, dtype=torch.int64, device=dev)
        rank[order[:H]] = torch.arange(H, device=dev)
        r = rank[sidx.long()]
        e = torch.where(r >= 0, -1 - r, sidx.long()).to(torch.int32)
        return e, X[order[:H]].contiguous()

    def row(name, t):
        print(f"{name:64s} {t:7.3f} ms  {gathered / t / 1e9:6.2f} TB/s", flush=True)

    shapes = [(0, "U4x3"), (1, "U2x4"), (2, "U4x4"), (3, "U8x2")]
    if args.quick:
        shapes = shapes[:2]
    CHs = [128, 384] if not args.quick else [384]
    maxp = torch.cuda.get_device_properties(0).persisting_l2_cache_max_size if hasattr(
        torch.cuda.get_device_properties(0), "persisting_l2_cache_max_size") else 82903040
    dummy = X  # unused Xh
    for CH in CHs:
        for sh, sname in shapes:
            for vs in (0, 1):
                tag = f"CH{CH} {sname} {'vals+Y' if vs else 'bare'}"
                t = timed(lambda: lib.probe_stream(sh, 0, 0, vs, X.data_ptr(), dummy.data_ptr(), sidx.data_ptr(),
                                                   svals.data_ptr(), nnz, CH, out.data_ptr(), out_rows, st),
                          args.reps)
                row(f"{tag} original X", t)
    # hot relabel variants at the default shape
    for H in ([312000, 390000] if not args.quick else [312000]):
        e, Xh = enc_for(H)
        print(f"H={H} ({H * 256 / 1e6:.0f} MB) receives {cum[H - 1].item() * 100:.1f}% of references", flush=True)
        for CH in CHs:
            for sh, sname in shapes[:2]:
                for vs in (0, 1):
                    tag = f"CH{CH} {sname} {'vals+Y' if vs else 'bare'} H{H}"
                    for hints in (0, 1):
                        t = timed(lambda: lib.probe_stream(sh, 1, hints, vs, X.data_ptr(), Xh.data_ptr(),
                                                           e.data_ptr(), svals.data_ptr(), nnz, CH, out.data_ptr(),
                                                           out_rows, st), args.reps)
                        row(f"{tag} compact{' +hints' if hints else ''}", t)
                    lib.probe_window(ctypes.c_void_p(st), ctypes.c_void_p(Xh.data_ptr()),
                                     min(Xh.numel() * 4, maxp), maxp)
                    t = timed(lambda: lib.probe_stream(sh, 1, 0, vs, X.data_ptr(), Xh.data_ptr(), e.data_ptr(),
                                                       svals.data_ptr(), nnz, CH, out.data_ptr(), out_rows, st),
                              args.reps)
                    row(f"{tag} compact +window", t)
                    lib.probe_window(ctypes.c_void_p(st), None, 0, 0)
        del e, Xh
    # full heat-order permutation of X (every column relabelled by rank)
    rank = torch.empty(n, dtype=torch.int64, device=dev)
    rank[order] = torch.arange(n, device=dev)
    pidx = rank[sidx.long()].to(torch.int32)
    Xp = X[order].contiguous()
    for vs in (0, 1):
        t = timed(lambda: lib.probe_stream(0, 0, 0, vs, Xp.data_ptr(), dummy.data_ptr(), pidx.data_ptr(),
                                           svals.data_ptr(), nnz, 384, out.data_ptr(), out_rows, st), args.reps)
        row(f"CH384 U4x3 {'vals+Y' if vs else 'bare'} heat-permuted X", t)
    del Xp, pidx
    # shuffled stream (control: order of execution)
    sh_idx = sidx[torch.randperm(nnz, device=dev)]
    t = timed(lambda: lib.probe_stream(0, 0, 0, 0, X.data_ptr(), dummy.data_ptr(), sh_idx.data_ptr(),
                                       svals.data_ptr(), nnz, 384, out.data_ptr(), out_rows, st), args.reps)
    row("CH384 U4x3 bare shuffled stream", t)
    # the original (row-order, unsorted) stream
    t = timed(lambda: lib.probe_stream(0, 0, 0, 0, X.data_ptr(), dummy.data_ptr(), ci.data_ptr(),
                                       svals.data_ptr(), nnz, 384, out.data_ptr(), out_rows, st), args.reps)
    row("CH384 U4x3 bare original row order", t)


if __name__ == "__main__":
    main()
