#!/usr/bin/env python
"""Interleaved A/B of agcn_spmm variants on one config (same process, same GPU, same inputs):
every round times each variant once (CUDA events), R rounds, median per variant.

    python tools/ab_spmm.py c5 '{"hot_rows": 0}' '{}' '{"spmm": {"chunk_shape": -1}}' [--rounds 15]

A variant is a JSON object; keys "plan" / "spmm" hold kwargs of agcn.Plan / Plan.spmm (other
top-level keys are Plan kwargs).  Plans with equal plan kwargs are shared.
"""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import agcn_inputs  # noqa: E402
import paper_2308_11825_b200 as agcn  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config")
    ap.add_argument("variants", nargs="+")
    ap.add_argument("--rounds", type=int, default=15)
    ap.add_argument("--F", type=int, default=None)
    ap.add_argument("--flush", action="store_true", help="write 512 MB before every timed call (cold L2)")
    args = ap.parse_args()
    dev = torch.device("cuda:0")
    w = agcn_inputs.make_config(args.config)
    F = args.F or w.F
    rp = torch.from_numpy(w.rowptr).to(dev)
    ci = torch.from_numpy(w.colidx).to(dev)
    va = torch.from_numpy(w.vals).to(dev)
    X = torch.from_numpy(w.X(F)).to(dev)
    Y = torch.empty((w.n, F), dtype=torch.float32, device=dev)
    scratch = torch.empty(512 << 18, dtype=torch.float32, device=dev) if args.flush else None
    plans, runs = {}, []
    for v in args.variants:
        d = json.loads(v)
        pk = dict(d.get("plan", {}), **{k: x for k, x in d.items() if k not in ("plan", "spmm")})
        key = json.dumps(pk, sort_keys=True)
        if key not in plans:
            plans[key] = agcn.Plan(rp, ci, **pk)
        runs.append((v, plans[key], d.get("spmm", {})))
    st = torch.cuda.current_stream()
    for _, p, sk in runs:
        for _ in range(3):
            p.spmm(va, X, out=Y, **sk)
    torch.cuda.synchronize()
    times = {v: [] for v, _, _ in runs}
    for _ in range(args.rounds):
        for v, p, sk in runs:
            if scratch is not None:
                scratch.fill_(1.0)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(st)
            p.spmm(va, X, out=Y, **sk)
            b.record(st)
            b.synchronize()
            times[v].append(a.elapsed_time(b))
    gathered = w.nnz * F * 4
    for v in times:
        t = statistics.median(times[v])
        print(f"{args.config} {v:50s} median {t:.4f} ms  min {min(times[v]):.4f}  {gathered / t / 1e9:.2f} TB/s gathered",
              flush=True)


if __name__ == "__main__":
    main()
