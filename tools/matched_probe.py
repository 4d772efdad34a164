#!/usr/bin/env python
"""The roof of the C5 SpMM's own access stream (round 2, follows tools/stream_probe.py).

Rebuilds, from the plan the bench uses (auto Alg. 1 parameters, hot rows), the exact stream of
(column, val) pairs the SpMM walks -- the degree-sorted CSR order of the small-row descriptors,
then the oversized chunks in the plan's column-position execution order -- with the plan's hot
encoding (hot columns read from a compact buffer of 524K rows, evict_last; cold evict_first),
and replays it through probe_stream_full: the same gather shape as k_spmm_wide (F = 64, 8 lanes
x 32 B, U = 4, 24 warps/SM) plus the vals stream and ALL n output-row stores (incl. the
degree-0 rows), but none of the SpMM's bookkeeping (descriptors, row offsets, row boundaries,
partial rows).  Interleaved timing against agcn_spmm on the same plan and inputs.

    python tools/matched_probe.py [--rounds 15]
"""
import argparse
import ctypes
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import agcn_inputs  # noqa: E402
import paper_2308_11825_b200 as agcn  # noqa: E402
from stream_probe import build_probe  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rounds", type=int, default=15)
    args = ap.parse_args()
    lib = build_probe()
    lib.probe_stream_full.argtypes = [ctypes.c_void_p] * 4 + [ctypes.c_int64, ctypes.c_int, ctypes.c_void_p,
                                                              ctypes.c_int64, ctypes.c_int64, ctypes.c_int,
                                                              ctypes.c_void_p]
    dev = torch.device("cuda:0")
    st = torch.cuda.current_stream()
    w = agcn_inputs.make_config("c5")
    n, nnz, F = w.n, w.nnz, 64
    rp = torch.from_numpy(w.rowptr).to(dev)
    ci = torch.from_numpy(w.colidx).to(dev)
    va = torch.from_numpy(w.vals).to(dev)
    X = torch.from_numpy(w.X()).to(dev)
    Y = torch.empty_like(X)
    plan = agcn.Plan(rp, ci, max_block_warps=0, max_warp_nzs=0)
    stt = plan.stats()
    H, db = stt["hot_rows"], stt["deg_bound"]
    perm = plan.copy("perm").astype(np.int64)
    srp = plan.copy("sorted_rowptr").astype(np.int64)
    rso = plan.copy("row_src_off").astype(np.int64)
    blocks = plan.copy("blocks").astype(np.int64)
    nb_small = int((blocks[:, 0] <= db).sum())
    # entry offsets (into the caller's CSR) in sorted-CSR order
    sdeg = np.diff(srp)
    src = np.repeat(rso - srp[:-1], sdeg) + np.arange(nnz, dtype=np.int64)
    # oversized chunks in the plan's execution order: bucket of (j + 0.5) / nc, stable
    ch = blocks[nb_small:]
    j = (ch[:, 1] - srp[ch[:, 2]]) // db
    nc = (ch[:, 0] + db - 1) // db
    key = np.minimum(63, ((2 * j + 1) * 64) // (2 * nc))
    order = np.argsort(key, kind="stable")
    ov0 = int(srp[n - stt["n_oversized_rows"]]) if stt["n_oversized_rows"] else nnz
    segs = [np.arange(ov0)] + [np.arange(ch[o, 1], ch[o, 1] + ch[o, 3]) for o in order]
    pos = np.concatenate(segs)
    assert pos.size == nnz
    src = src[pos]
    # the plan's hot encoding: hot vertices = the H highest-degree rows, slots in column order
    hot_cols = np.sort(perm[n - H:])
    slot = np.full(n, -1, np.int64)
    slot[hot_cols] = np.arange(H)
    c = w.colidx[src].astype(np.int64)
    enc = np.where(slot[c] >= 0, -1 - slot[c], c).astype(np.int32)
    print(f"C5 plan ({stt['max_block_warps']},{stt['max_warp_nzs']}) hot rows {H}: "
          f"{100.0 * (slot[c] >= 0).mean():.1f}% of entries hot", flush=True)
    idx = torch.from_numpy(enc).to(dev)
    vals = torch.from_numpy(w.vals[src]).to(dev)
    Xh = X[torch.from_numpy(hot_cols).to(dev)].contiguous()
    out = torch.empty_like(X)
    runs = {"agcn_spmm": lambda: plan.spmm(va, X, out=Y)}
    for CH in (256, 384, 512):
        zero = max(0, n - 4 * ((nnz + CH - 1) // CH))
        runs[f"probe CH{CH} (+vals, all {n} Y rows)"] = (
            lambda CH=CH, zero=zero: lib.probe_stream_full(X.data_ptr(), Xh.data_ptr(), idx.data_ptr(),
                                                           vals.data_ptr(), nnz, CH, out.data_ptr(), n, zero, 1,
                                                           st.cuda_stream))
    for f in runs.values():
        for _ in range(3):
            f()
    torch.cuda.synchronize()
    times = {k: [] for k in runs}
    for _ in range(args.rounds):
        for k, f in runs.items():
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(st)
            f()
            b.record(st)
            b.synchronize()
            times[k].append(a.elapsed_time(b))
    for k, v in times.items():
        t = statistics.median(v)
        print(f"{k:44s} median {t:.3f} ms  min {min(v):.3f}  {nnz * F * 4 / t / 1e9:.2f} TB/s gathered", flush=True)


if __name__ == "__main__":
    main()
