#!/usr/bin/env python
"""Benchmark of the Accel-GCN hot path on B200: plan (degree sort + block partition) and
stacked SpMM propagation layers Y = A.X, row-sharded over N GPUs with an in-place NCCL
all-gather between layers.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c5] [--impl agcn|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...

One step = one pass of the whole hot path over one synthetic graph:
agcn_plan (a1-a5) -> for each layer: agcn_spmm (a6-a8) [-> all-gather (a9)].
Rank 0 prints ONE JSON line.  See DESIGN.md "Measurement" for the byte model.
"""
from __future__ import annotations

import argparse
import json
import os
import re
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "A·X SpMM GFLOP/s and HBM GB/s (% of ~8 TB/s) per graph at 1/2/4/8 B200"
UNIT = "GFLOP/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["agcn", "reference"], default="agcn")
    ap.add_argument("--config", default="c5", choices=["c1", "c2", "c3", "c4", "c5"])
    ap.add_argument("--F", type=int, default=None)
    ap.add_argument("--layers", type=int, default=None)
    ap.add_argument("--partition", choices=["block", "warp"], default="block")
    ap.add_argument("--kernel", choices=["auto", "general", "looped", "wide"], default="auto")
    ap.add_argument("--mbw", type=int, default=0, help="Alg. 1 max_block_warps (P:318; the paper's storage "
                    "example: 12); 0 with --mwn 0 (default): agcn_auto_partition's per-graph choice")
    ap.add_argument("--mwn", type=int, default=0, help="Alg. 1 max_warp_nzs (P:318; SPEC default 32)")
    ap.add_argument("--l2-hint", default=None,
                    choices=["auto", "none", "keep_all", "hot_window", "hot_hints"],
                    help="agcn_l2_hint_t (default auto: hot_window for plans with hot rows)")
    ap.add_argument("--hot-rows", type=int, default=None, help="agcn_opts_t.hot_rows (None: auto)")
    ap.add_argument("--hot-mb", type=int, default=None, help="agcn_spmm_opts_t.hot_mb (None: device max)")
    ap.add_argument("--chunk-shape", type=int, default=0, help="agcn_spmm_opts_t.chunk_shape (0: auto)")
    ap.add_argument("--chunk-order", type=int, default=0, help="agcn_spmm_opts_t.chunk_order (0: bucketed, -1: off)")
    ap.add_argument("--e2e-steps", type=int, default=10)
    ap.add_argument("--pipe-depth", type=int, default=2, help="e2e: agcn_pipe buffer slots")
    ap.add_argument("--cpu-seconds", type=float, default=12.0, help="CPU-oracle sample budget")
    ap.add_argument("--ref-seconds", type=float, default=120.0,
                    help="--impl reference: total CPU budget over warm-up + timed steps")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cusparse", action="store_true", help="skip the protocol / cuSPARSE arm on this config")
    ap.add_argument("--no-traffic", action="store_true", help="skip the live ncu DRAM-traffic capture")
    ap.add_argument("--no-graph", action="store_true", help="skip the CUDA-graph kernel-only timing")
    ap.add_argument("--no-per-graph", action="store_true",
                    help="skip the kernel-only per-graph table of the other BASELINE configs")
    ap.add_argument("--aggregation", choices=["sum", "mean"], default="sum",
                    help="sum: GCN (the metric's workload); mean: GraphSAGE-mean (P:126)")
    ap.add_argument("--gin-eps", type=float, default=None, help="GIN self term (1 + eps) x_i (square A)")
    ap.add_argument("--bias-relu", action="store_true", help="fused bias + ReLU epilogue")
    ap.add_argument("--fused-allgather", action="store_true",
                    help="N>1: the SpMM epilogue stores rows into every rank's X (CUDA IPC / NVLink) "
                         "instead of an all-gather collective (SURVEY 8(f1))")
    ap.add_argument("--overlap-chunks", type=int, default=1,
                    help="K > 1: column-chunked propagation, the all-gather of chunk k overlapping the "
                         "SpMM of chunk k+1 (SURVEY 8(f1)); 1: one SpMM + one all-gather per layer")
    ap.add_argument("--dist-backend", choices=["nccl", "gloo"], default="nccl",
                    help="gloo: test mode, every rank on cuda:0, all-gather staged through the host")
    ap.add_argument("--profile", action="store_true",
                    help="short run for ncu: no clocks/e2e/cpu/cusparse legs")
    return ap.parse_args()


# ---------------------------------------------------------------- helpers
def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return {"hbm_gbs": float(d["hbm_gbs"]), "source": "measured (MEASURED_PEAKS.json)"}
    return {"hbm_gbs": 6650.0, "source": "fallback (B200_PROFILING.md)"}


def build_hash() -> str:
    """sha256 (16 hex) of the CUDA sources + C ABI header this bench runs (the library build)."""
    import hashlib
    h = hashlib.sha256()
    cdir = os.path.join(ROOT, "paper_2308_11825_b200", "csrc")
    for f in sorted(os.listdir(cdir)):
        if f.endswith((".cu", ".h", ".cuh")):
            h.update(f.encode())
            h.update(open(os.path.join(cdir, f), "rb").read())
    h.update(open(os.path.join(ROOT, "include", "agcn.h"), "rb").read())
    return h.hexdigest()[:16]


def git_sha() -> str | None:
    """HEAD of the repo: `git rev-parse` where .git exists, else the `.git_sha` file a post-commit
    hook writes at the repo root (the GPU box gets the tree without .git)."""
    try:
        sha = subprocess.run(["git", "-C", ROOT, "rev-parse", "HEAD"], capture_output=True, text=True,
                             timeout=10).stdout.strip()
        if sha:
            return sha
    except Exception:
        pass
    try:
        return open(os.path.join(ROOT, ".git_sha")).read().strip() or None
    except OSError:
        return None


TRAFFIC_KERNELS = "regex:k_spmm_wide|k_spmm_chunks|k_spmm_block|k_gather_hot|k_ov_reduce_h"


def live_traffic(args, timeout_s: float = 420.0):
    """DRAM bytes per agcn_spmm call of THIS build, measured now: ncu (dram__bytes_read.sum +
    dram__bytes_write.sum, Nsight Compute's default cache control = cold per kernel) over every
    kernel of the SpMM calls of a short `bench.py --profile` run with the same options, summed
    and divided by the number of calls.  Returns (bytes, source) or (None, reason)."""
    import csv
    import io
    import shutil
    ncu = shutil.which("ncu") or "/usr/local/cuda/bin/ncu"
    if not os.path.exists(ncu):
        return None, "ncu not found"
    logf = tempfile.NamedTemporaryFile(suffix=".csv", delete=False).name
    cmd = [ncu, "--metrics", "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum",
           "--clock-control", "none", "-k", TRAFFIC_KERNELS, "--csv", "--log-file", logf,
           sys.executable, os.path.abspath(__file__), "--profile", "--config", args.config,
           "--steps", "1", "--warmup", "3", "--kernel", args.kernel, "--chunk-shape", str(args.chunk_shape),
           "--chunk-order", str(args.chunk_order),
           "--mbw", str(args.mbw), "--mwn", str(args.mwn), "--partition", args.partition]
    for k in ("F", "layers", "hot_rows", "hot_mb", "l2_hint"):
        v = getattr(args, k)
        if v is not None:
            cmd += ["--" + k.replace("_", "-"), str(v)]
    try:
        r = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout_s)
        text = open(logf).read()
    except Exception as e:
        return None, f"ncu failed: {str(e)[:120]}"
    finally:
        try:
            os.unlink(logf)
        except OSError:
            pass
    rows = list(csv.reader(io.StringIO(text)))
    start = next((i for i, x in enumerate(rows) if x and x[0] == "ID"), None)
    if start is None:
        return None, f"ncu gave no metrics (rc {r.returncode}): {r.stderr.strip()[-160:]}"
    hdr = rows[start]
    rows = [hdr] + [x for x in rows[start + 1:] if len(x) == len(hdr)]
    iid, ik, im, iu, iv = (hdr.index(c) for c in ("ID", "Kernel Name", "Metric Name", "Metric Unit", "Metric Value"))
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    total, calls, kt = 0.0, set(), {}
    for x in rows[1:]:
        if x[im].startswith("dram__bytes_"):
            b = float(x[iv].replace(",", "")) * scale.get(x[iu], 1.0)
            total += b
            mm = re.search(r"(k_\w+)", x[ik])
            name = mm.group(1) if mm else x[ik][:40]
            kt[name] = kt.get(name, 0.0) + b
            if name in ("k_spmm_wide", "k_spmm_block"):
                calls.add(x[iid])
    if not calls:
        return None, "ncu captured no SpMM kernel"
    per = {k: v / len(calls) for k, v in kt.items()}
    return total / len(calls), {"source": f"live ncu capture of this build ({build_hash()}), "
                                          f"{len(calls)} agcn_spmm calls, cold cache per kernel",
                                "per_kernel_bytes": per}


def load_traffic(config: str, F: int):
    """Fallback: DRAM bytes per agcn_spmm call from a committed capture of this exact build
    (profiles/ncu_traffic_<build hash>.json), else None."""
    name = f"ncu_traffic_{build_hash()}.json"
    path = os.path.join(ROOT, "profiles", name)
    if os.path.exists(path):
        d = json.load(open(path))
        key = f"{config}_F{F}"
        if key in d:
            return d[key], {"source": f"profiles/{name} (committed capture of this build)"}
    return None, {"source": "none: no live capture and no committed capture of this build"}


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(index), f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "200"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except FileNotFoundError:
            self.p = None

    def stop(self):
        if self.p is None:
            return None
        time.sleep(0.25)
        self.p.terminate()
        try:
            self.p.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.p.kill()
        self.f.flush()
        rows = []
        for line in open(self.f.name):
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                rows.append((float(parts[1]), float(parts[2]), parts[5:9]))
            except ValueError:
                continue
        os.unlink(self.f.name)
        if not rows:
            return None
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for _, _, r in rows for i, v in enumerate(r) if v == "Active"})
        return {"sm_mhz": statistics.median(r[0] for r in rows), "sm_max_mhz": max(r[1] for r in rows),
                "reasons": reasons, "samples": len(rows)}


class NvmlClockSampler:
    """SM clock and clock-event reasons sampled every `period` s by NVML from a thread, only
    while the timed region runs (start() right before it, stop() right after the closing
    synchronize).  The nvidia-smi sampler above is the fallback when NVML is unavailable."""

    BITS = {"hw_slowdown": "nvmlClocksEventReasonHwSlowdown",
            "hw_thermal_slowdown": "nvmlClocksEventReasonHwThermalSlowdown",
            "sw_thermal_slowdown": "nvmlClocksEventReasonSwThermalSlowdown",
            "sw_power_cap": "nvmlClocksEventReasonSwPowerCap"}

    def __init__(self, cuda_index: int, period: float = 0.005):
        import threading
        import pynvml as N
        N.nvmlInit()
        self.N, self.period, self.rows = N, period, []
        h = None
        try:
            import torch
            uuid = str(torch.cuda.get_device_properties(cuda_index).uuid)
            h = N.nvmlDeviceGetHandleByUUID(uuid if uuid.startswith("GPU-") else "GPU-" + uuid)
        except Exception:
            vis = os.environ.get("CUDA_VISIBLE_DEVICES", "")
            ids = [x for x in vis.split(",") if x.strip().isdigit()]
            h = N.nvmlDeviceGetHandleByIndex(int(ids[cuda_index]) if cuda_index < len(ids) else cuda_index)
        self.h = h
        self.max_mhz = N.nvmlDeviceGetMaxClockInfo(h, N.NVML_CLOCK_SM)
        self.bits = {k: getattr(N, v) for k, v in self.BITS.items()}
        self.stop_ev = threading.Event()
        self.t = threading.Thread(target=self._run, daemon=True)
        self.t.start()

    def _run(self):
        N = self.N
        while not self.stop_ev.is_set():
            try:
                mhz = N.nvmlDeviceGetClockInfo(self.h, N.NVML_CLOCK_SM)
                rs = N.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                self.rows.append((mhz, rs))
            except Exception:
                pass
            time.sleep(self.period)

    def stop(self):
        self.stop_ev.set()
        self.t.join(timeout=2)
        if not self.rows:
            return None
        reasons = sorted(k for k, b in self.bits.items() if any(rs & b for _, rs in self.rows))
        return {"sm_mhz": statistics.median(r[0] for r in self.rows), "sm_max_mhz": self.max_mhz,
                "reasons": reasons, "samples": len(self.rows), "sampler": "nvml 5 ms, timed region only"}


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def _pct(xs, q):
    """q-th percentile (nearest rank) of the samples xs."""
    xs = sorted(xs)
    return xs[min(len(xs) - 1, max(0, int(round(q / 100.0 * (len(xs) - 1)))))]


def graph_protocol(A, torch, dev, w, F, rp, ci, va, X, scratch, hbm_gbs, plan_kw, reps=20, cpu=False):
    """The measurement protocol of SURVEY.md 8(d4) for one graph (kernel time,
    preprocessing excluded, against cuSPARSE):
      * agcn_spmm COLD (primary, Nsight Compute's cache control): 512 MB scratch written and
        persisting L2 reset before every rep, CUDA events around one agcn_spmm call;
      * agcn_spmm WARM: 20 calls captured in one CUDA graph, replayed 10 times (no launch gaps);
        a sample = one replay / 20;
      * cusparseSpMM directly (baseline/cusparse_spmm.cu) for ALG_DEFAULT and CSR_ALG1/2/3,
        bufferSize + preprocess outside timing, the same cold / warm reps; its output is
        checked against the fp64 oracle on a row sample; speedups against the best algorithm;
      * cpu=True (C1, C2): the oracle on 1 thread and on all host cores (full layer).
    Medians (and p10 / p90) over `reps` (>= 20)."""
    import baseline
    import oracle
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    n, nnz = w.n, w.nnz
    Y = torch.empty((n, F), dtype=torch.float32, device=dev)
    S = torch.cuda.Stream()
    with torch.cuda.stream(S):
        A.Plan(rp, ci, stream=S, **plan_kw).close()  # warm the allocator
        a, b = ev(), ev()
        a.record(S)
        plan = A.Plan(rp, ci, stream=S, **plan_kw)
        b.record(S)
    torch.cuda.synchronize()
    plan_ms = a.elapsed_time(b)
    st = plan.stats()
    run = lambda: plan.spmm(va, X, out=Y, stream=S)  # noqa: E731
    for _ in range(3):
        run()
    torch.cuda.synchronize()
    cold = []
    for _ in range(reps):
        baseline.l2_flush(scratch, S)
        a, b = ev(), ev()
        with torch.cuda.stream(S):
            a.record(S)
            run()
            b.record(S)
        b.synchronize()
        cold.append(a.elapsed_time(b))
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=S):
        for _ in range(20):
            run()
    g.replay()
    torch.cuda.synchronize()
    warms = []
    for _ in range(10):
        a, b = ev(), ev()
        with torch.cuda.stream(S):
            a.record(S)
            g.replay()
            b.record(S)
        b.synchronize()
        warms.append(a.elapsed_time(b) / 20)
    warm = statistics.median(warms)
    del g
    cold_ms = statistics.median(cold)
    bc = 4 * (n + 1) + 8 * nnz + 8 * n * F
    row = {"n": n, "nnz": nnz, "F": F, "max_block_warps": st["max_block_warps"],
           "max_warp_nzs": st["max_warp_nzs"], "hot_rows": st["hot_rows"], "plan_ms": plan_ms,
           "cold_ms": cold_ms, "warm_ms": warm, "spmm_ms": cold_ms, "cold_reps": len(cold),
           "cold_p10_ms": _pct(cold, 10), "cold_p90_ms": _pct(cold, 90),
           "warm_p10_ms": _pct(warms, 10), "warm_p90_ms": _pct(warms, 90),
           "gflops_cold": 2.0 * nnz * F / (cold_ms * 1e-3) / 1e9,
           "b_comp_frac_of_hbm_cold": bc / (cold_ms * 1e-3) / 1e9 / hbm_gbs,
           "b_comp_frac_of_hbm_warm": bc / (warm * 1e-3) / 1e9 / hbm_gbs}
    plan.close()
    # cuSPARSE, every CSR algorithm (rowptr rebased to 0 for the library)
    rp0 = rp - rp[0] if int(rp[0]) != 0 else rp
    cs, best = {}, None
    Yc = torch.empty_like(Y)
    for alg in baseline.ALGS:
        r = {}
        for mode in ("cold", "warm"):
            ms, rc, bb = baseline.cusparse_spmm_times(rp0, ci, va, X, Yc, alg, reps, mode == "cold", scratch, S)
            if ms is None:
                r = {"status": rc}
                break
            r[f"{mode}_ms"] = statistics.median(ms)
            r[f"{mode}_p10_ms"], r[f"{mode}_p90_ms"] = _pct(ms, 10), _pct(ms, 90)
            r["buffer_bytes"] = bb
        cs[alg] = r
        if "cold_ms" in r and (best is None or r["cold_ms"] < cs[best]["cold_ms"]):
            best = alg
    row["cusparse"] = cs
    if best:
        # parity of the baseline itself (the best algorithm's output) on a row sample
        ms, rc, _ = baseline.cusparse_spmm_times(rp0, ci, va, X, Yc, best, 1, False, scratch, S)
        rows = np.unique(np.concatenate([np.arange(min(n, 64)), np.argsort(np.diff(w.rowptr))[-16:],
                                         np.random.default_rng(0).integers(0, n, 500)])).astype(np.int64)
        chk = oracle.spmm_check(w.rowptr, w.colidx, w.vals, X.cpu().numpy(), Yc[torch.from_numpy(rows).to(dev)].cpu().numpy(),
                                rows=rows)
        row.update({"cusparse_best_alg": best, "cusparse_best_cold_ms": cs[best]["cold_ms"],
                    "cusparse_best_warm_ms": cs[best]["warm_ms"],
                    "speedup_vs_cusparse_best_cold": cs[best]["cold_ms"] / cold_ms,
                    "speedup_vs_cusparse_best_warm": cs[best]["warm_ms"] / warm,
                    "cusparse_parity": {"rows": chk["rows"], "nfail": chk["nfail"],
                                        "max_ratio": chk["max_ratio"]}})
    if cpu:
        Xh = X.cpu().numpy()
        for nt, key in ((1, "cpu_1thread_ms"), (os.cpu_count() or 1, "cpu_all_cores_ms")):
            ts = []
            for _ in range(3):
                t0 = time.perf_counter()
                oracle.spmm(w.rowptr, w.colidx, w.vals, Xh, nthreads=nt, with_abs=False)
                ts.append(time.perf_counter() - t0)
            row[key] = 1e3 * statistics.median(ts)
        row["cpu_threads"] = os.cpu_count() or 1
    return row


def per_graph_table(A, gen, torch, dev, skip: str, hbm_gbs: float, scratch):
    """The protocol of graph_protocol for the other BASELINE graphs (C1-C4 and C2's F sweep),
    with the library's per-graph Alg. 1 parameters (agcn_auto_partition)."""
    out = {}
    cases = [("c1", None), ("c2", 16), ("c2", 32), ("c2", 64), ("c2", 128), ("c3", None), ("c4", None)]
    for name, Fo in cases:
        if name == skip:
            continue
        key = name if Fo is None else f"{name}_F{Fo}"
        try:
            w = gen.make_config(name)
            F = Fo or w.F
            rp = torch.from_numpy(w.rowptr).to(dev)
            ci = torch.from_numpy(w.colidx).to(dev)
            va = torch.from_numpy(w.vals).to(dev)
            X = torch.from_numpy(w.X(F)).to(dev)
            out[key] = graph_protocol(A, torch, dev, w, F, rp, ci, va, X, scratch, hbm_gbs,
                                      dict(max_block_warps=0, max_warp_nzs=0),
                                      cpu=(key in ("c1", "c2_F16")))
            del rp, ci, va, X
        except Exception as e:  # pragma: no cover
            out[key] = {"error": str(e)[:160]}
    return out


def clock_sampler(cuda_index: int):
    try:
        return NvmlClockSampler(cuda_index)
    except Exception:
        return ClockSampler(cuda_index)


def cpu_sample_gflops(w, X, budget_s: float):
    """Time the fp64 CPU oracle (as it stands) on a bounded contiguous row sample."""
    import oracle
    n, F = w.n, X.shape[1]
    cores = os.cpu_count() or 1
    # calibrate on ~0.2% of nnz, then size the sample for `budget_s`
    def run(lo, hi):
        rp = w.rowptr[lo:hi + 1]
        t0 = time.perf_counter()
        oracle.spmm(rp, w.colidx, w.vals, X, nthreads=cores, with_abs=False)
        return time.perf_counter() - t0, int(rp[-1] - rp[0])
    target = max(1, w.nnz // 500)
    hi = int(np.searchsorted(w.rowptr, target))
    t, nz = run(0, max(hi, 1))
    rate = nz / max(t, 1e-6)
    want_nnz = int(min(w.nnz, rate * budget_s))
    lo = n // 3
    hi = int(np.searchsorted(w.rowptr, w.rowptr[lo] + want_nnz))
    hi = max(lo + 1, min(hi, n))
    t, nz = run(lo, hi)
    passes = 1
    while t < 0.9 * budget_s:        # the sample is capped at 2/3 of the graph: repeat it
        dt, dn = run(lo, hi)
        t, nz, passes = t + dt, nz + dn, passes + 1
    return {"value": 2.0 * nz * F / t / 1e9, "unit": UNIT, "cores": cores, "kind": "oracle",
            "sample": f"rows [{lo},{hi}) of {w.name} ({nz // passes} nnz = "
                      f"{100.0 * nz / passes / w.nnz:.2f}% of nnz) x {passes} passes, "
                      f"one fp64 SpMM layer each, F={F}, {t:.1f} s"}, t


# ---------------------------------------------------------------- reference arm (the oracle)
def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import agcn_inputs as gen
    w = gen.make_config(args.config)
    F = args.F or w.F
    X = w.X(F)
    times, vals = [], []
    budget = max(min(2.0, args.ref_seconds), args.ref_seconds / max(1, args.steps + args.warmup))
    for i in range(args.warmup + args.steps):
        cb, t = cpu_sample_gflops(w, X, budget)
        if i >= args.warmup:
            times.append(t)
            vals.append(cb["value"])
    v = statistics.median(vals)
    layers = args.layers or w.layers
    line = {"metric": METRIC, "value": v, "unit": UNIT, "n_gpus": 0, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * statistics.median(times),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "impl": "reference",
            "config": {"workload": w.meta["desc"], "name": w.name, "F": F, "layers": layers,
                       "sample": cb["sample"]},
            "cpu_baseline": dict(cb, value=v),
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- the B200 arm
def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist

    import agcn_inputs as gen
    import paper_2308_11825_b200 as A
    from paper_2308_11825_b200.dist import (PeerBuffers, ShardLayout, chunk_widths, join_columns,
                                            make_all_gather, make_all_gather_async, propagate,
                                            propagate_chunked, propagate_fused, split_columns)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.dist_backend == "gloo":  # test mode: all ranks share cuda:0 (no NCCL, no NVLink)
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group("gloo")
    P = world
    A.library_path()

    w = gen.make_config(args.config)
    F = args.F or w.F
    layers = args.layers or w.layers
    n, nnz = w.n, w.nnz
    X_host = w.X(F)

    # resident inputs
    rp_d = torch.from_numpy(w.rowptr).to(dev)
    ci_d = torch.from_numpy(w.colidx).to(dev)
    va_d = torch.from_numpy(w.vals).to(dev)
    bounds = A.shard_bounds(rp_d, P)
    lay = ShardLayout(bounds, rank)
    S = lay.slot_rows
    rp_local = rp_d[lay.lo:lay.hi + 1].contiguous()
    X0 = torch.zeros((lay.padded_rows, F), dtype=torch.float32, device=dev)
    lay.pad(torch.from_numpy(X_host).to(dev), X0)
    bufs = [torch.empty_like(X0) for _ in range(min(layers, 2))]
    plan_kw = dict(n_cols=n, max_block_warps=args.mbw, max_warp_nzs=args.mwn, partition=args.partition,
                   hot_rows=args.hot_rows)
    if P > 1:
        plan_kw.update(col_bounds=bounds, col_slot_rows=S)

    bias_d = torch.linspace(-0.5, 0.5, F, device=dev) if args.bias_relu else None

    def epi_kw(Xin):  # aggregation variant / epilogue of agcn_spmm; default: plain GCN sum
        kw = {"aggregation": args.aggregation}
        if args.gin_eps is not None:
            if P > 1:
                raise SystemExit("--gin-eps: single GPU only (the self rows are the rank's own rows)")
            kw.update(self_x=Xin, self_scale=1.0 + args.gin_eps)
        if args.bias_relu:
            kw.update(bias=bias_d, relu=True)
        return kw

    stream = torch.cuda.current_stream()
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    rec = {"plan": [], "spmm": [], "ag": []}

    gather = make_all_gather(args.dist_backend) if P > 1 else None
    fused = args.fused_allgather and P > 1
    K = max(1, args.overlap_chunks)
    if K > 1 and fused:
        raise SystemExit("--overlap-chunks and --fused-allgather are alternatives")
    if K > 1:   # chunk-major layout: K contiguous [P*S, w_k] buffers per X / Y
        widths = chunk_widths(F, K)
        X0c = split_columns(X0, widths)
        bufs_c = [[torch.empty_like(c) for _ in range(min(layers, 2))] for c in X0c]
        gather_async = make_all_gather_async(args.dist_backend) if P > 1 else None
    peers = PeerBuffers(lay, F) if fused else None

    def fused_barrier():  # the peers' stores of this layer are complete everywhere
        e0, e1 = ev(), ev()
        e0.record(stream)
        torch.cuda.current_stream().synchronize()
        dist.barrier()
        e1.record(stream)
        rec["ag"].append((e0, e1))

    def all_gather(full, slot):
        e0, e1 = ev(), ev()
        e0.record(stream)
        gather(full, slot)
        e1.record(stream)
        rec["ag"].append((e0, e1))

    def step(record: bool):
        e0, e1 = ev(), ev()
        e0.record(stream)
        plan = A.Plan(rp_local, ci_d, **plan_kw)
        e1.record(stream)
        if record:
            rec["plan"].append((e0, e1))

        def spmm(Xin, out_rows):
            s0, s1 = ev(), ev()
            s0.record(stream)
            plan.spmm(va_d, Xin, out=out_rows, kernel=args.kernel, l2_hint=args.l2_hint,
                      hot_mb=args.hot_mb, chunk_shape=args.chunk_shape, chunk_order=args.chunk_order, **epi_kw(Xin))
            s1.record(stream)
            if record:
                rec["spmm"].append((s0, s1))
        if fused:
            def spmm_f(Xin, out_rows, peer_out):
                s0, s1 = ev(), ev()
                s0.record(stream)
                plan.spmm(va_d, Xin, out=out_rows, kernel=args.kernel, l2_hint=args.l2_hint,
                          hot_mb=args.hot_mb, chunk_shape=args.chunk_shape, chunk_order=args.chunk_order, peer_out=peer_out,
                          **epi_kw(Xin))
                s1.record(stream)
                if record:
                    rec["spmm"].append((s0, s1))
            out = propagate_fused(lay, spmm_f, X0, peers, layers, fused_barrier)
        elif K > 1:
            out = join_columns(propagate_chunked(lay, spmm, X0c, bufs_c, layers, gather_async))
        else:
            out = propagate(lay, spmm, X0, bufs, layers, all_gather if P > 1 else None)
        return plan, out  # plans stay alive until after the timed region (closed below)

    def barrier():
        if P > 1:
            dist.barrier()

    # warm-up (plans are destroyed stream-ordered at the end of every step, as a user would)
    for _ in range(max(3, args.warmup)):
        plan, _ = step(False)
        plan.close()
    torch.cuda.synchronize()
    rec = {"plan": [], "spmm": [], "ag": []}

    barrier()
    torch.cuda.synchronize()
    clocks = None if args.profile else clock_sampler(local)
    l0 = A.launch_count()
    t_start, t_end = ev(), ev()
    t_start.record(stream)
    st_plan = None
    for i in range(args.steps):
        plan, out = step(True)
        if i == args.steps - 1:
            st_plan = plan.stats()
        plan.close()
    t_end.record(stream)
    torch.cuda.synchronize()
    clk = clocks.stop() if clocks else None
    barrier()
    launches = A.launch_count() - l0
    ms_local = t_start.elapsed_time(t_end) / args.steps
    spmm_ms = [a.elapsed_time(b) for a, b in rec["spmm"]]
    plan_ms = [a.elapsed_time(b) for a, b in rec["plan"]]
    ag_ms = [a.elapsed_time(b) for a, b in rec["ag"]]
    spmm_avg = sum(spmm_ms) / max(1, len(spmm_ms)) * K      # per layer (K chunk SpMMs per layer)
    vec = torch.tensor([ms_local, spmm_avg, sum(plan_ms) / max(1, len(plan_ms)),
                        sum(ag_ms) / max(1, len(ag_ms)) if ag_ms else 0.0], device=dev)
    if P > 1:
        dist.all_reduce(vec, op=dist.ReduceOp.MAX)
    ms_step, spmm_max, plan_max, ag_max = [float(x) for x in vec.tolist()]

    # correctness guard on the timed output (a few rows vs a host fp64 recomputation is the
    # test suite's job; here: finite and the right shape)
    # (N > 1: the last layer's output stays row-sharded -- all-gathers run between layers only)
    Yfinal = lay.own_rows(out) if P > 1 else out
    assert Yfinal.shape == (lay.rows, F) and bool(torch.isfinite(Yfinal[: min(lay.rows, 4096)]).all())

    flops_layer = 2.0 * nnz * F
    value = flops_layer * layers / (ms_step * 1e-3) / 1e9

    # byte model: B_comp per SpMM launch on this rank
    n_p, nnz_p = lay.rows, int(w.rowptr[lay.hi] - w.rowptr[lay.lo])
    b_comp = 4 * (n_p + 1) + 8 * nnz_p + 4 * n * F + 4 * n_p * F
    b_gather = 4 * (n_p + 1) + 8 * nnz_p + 4 * nnz_p * F + 4 * n_p * F
    peaks = load_peaks()
    achieved = b_comp / (spmm_max * 1e-3) / 1e9
    traffic, traffic_src = None, {"source": "not measured (--profile / N > 1)"}

    line = None
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": P, "steps": args.steps,
            "warmup": max(3, args.warmup), "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "strong" if P > 1 else "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic",
            "config": {"workload": w.meta["desc"], "name": w.name, "n": n, "nnz": nnz, "F": F,
                       "layers": layers, "partition": args.partition, "kernel": args.kernel,
                       "aggregation": args.aggregation, "gin_eps": args.gin_eps, "bias_relu": args.bias_relu,
                       "allgather": ("fused (SpMM epilogue peer stores)" if fused else
                                     f"{args.dist_backend} all_gather_into_tensor" +
                                     (f", {K} column chunks overlapped with the SpMM" if K > 1 else ""))
                                    if P > 1 else None, "parallelism": f"row-shard{P}",
                       "overlap_chunks": K,
                       "max_block_warps": st_plan["max_block_warps"], "max_warp_nzs": st_plan["max_warp_nzs"],
                       "partition_params": "auto (agcn_auto_partition)" if args.mbw == 0 and args.mwn == 0
                                           else "given",
                       "l2": "inputs larger than L2 (CSR + X > 126 MB)" if
                             (8 * nnz + 4 * n * F) > 126e6 else "inputs fit in L2 (warm)",
                       "step": "agcn_plan + layers x agcn_spmm (+ an all-gather between layers if N>1; "
                               "the last layer's output stays row-sharded)"},
            "spmm_only": {"ms_per_layer": spmm_max, "gflops": flops_layer / (spmm_max * 1e-3) / 1e9,
                          "b_comp_gbs": achieved, "b_gather_gbs": b_gather / (spmm_max * 1e-3) / 1e9},
            "plan_ms": plan_max, "allgather_ms": ag_max if P > 1 else 0.0,
            "plan_stats": {k: st_plan[k] for k in ("nblocks", "n_zero_rows", "n_oversized_rows",
                                                   "n_oversized_blocks", "max_deg")},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                         "frac": achieved / peaks["hbm_gbs"], "traffic": traffic,
                         # the DRAM bytes ncu measured for this kernel, moved in the event time
                         "traffic_gbs": traffic / (spmm_max * 1e-3) / 1e9 if traffic else None,
                         "traffic_frac": traffic / (spmm_max * 1e-3) / 1e9 / peaks["hbm_gbs"] if traffic else None,
                         "kernel": "agcn_spmm: every kernel of one call (%s)" % (
                             "[k_gather_hot] + [k_spmm_chunks] + k_spmm_wide + k_ov_reduce_h"
                             if args.kernel in ("auto", "wide") and F % 8 == 0 and F <= 256
                             else "[k_gather_hot] + k_spmm_block + k_ov_reduce_h"),
                         "bytes_per_launch": b_comp, "peak_source": peaks["source"],
                         "traffic_source": traffic_src},
            "gpu_launches": int(launches),
            "clocks": clk,
            "build": {"hash": build_hash(), "git_sha": git_sha()},
        }

    # ---- parity of what was timed (outside the timed region, N = 1): the same plan options
    # and kernel, layer by layer; output rows of every layer vs the fp64 oracle fed the GPU's
    # own layer input (north_star tolerance); the re-run's last layer is bitwise the timed output
    if rank == 0 and P == 1 and not args.profile:
        import oracle
        if args.aggregation != "sum" or args.gin_eps is not None or args.bias_relu:
            line["self_check"] = {"skipped": "epilogue variant (covered by tests/test_gpu_parity.py)"}
        else:
            deg = np.diff(w.rowptr)
            rng = np.random.default_rng(7)
            rows = np.unique(np.concatenate([np.argsort(deg, kind="stable")[-16:], np.flatnonzero(deg == 0)[:8],
                                             rng.integers(0, n, 2000)])).astype(np.int64)
            rows_d = torch.from_numpy(rows).to(dev)
            chk = []
            with A.Plan(rp_local, ci_d, **plan_kw) as pc:
                Xin = X0
                kw = dict(kernel=args.kernel, l2_hint=args.l2_hint, hot_mb=args.hot_mb, chunk_shape=args.chunk_shape, chunk_order=args.chunk_order)
                for l in range(layers):
                    if K > 1:   # the same column chunks as the timed run
                        Yl = join_columns([pc.spmm(va_d, c, **kw) for c in split_columns(Xin, widths)])
                    else:
                        Yl = pc.spmm(va_d, Xin, **kw)
                    r = oracle.spmm_check(w.rowptr, w.colidx, w.vals, Xin.cpu().numpy(), Yl[rows_d].cpu().numpy(),
                                          rows=rows)
                    chk.append({"layer": l + 1, "rows": r["rows"], "nfail": r["nfail"], "max_ratio": r["max_ratio"]})
                    Xin = Yl
                same = bool(torch.equal(Yl, Yfinal))
            line["self_check"] = {"layers": chk, "bitwise_equal_to_timed_output": same,
                                  "ok": same and all(c["nfail"] == 0 for c in chk)}

    # ---- the measurement protocol on this config: agcn_spmm
    # cold-L2 (primary) and warm (CUDA graph), cusparseSpMM per algorithm (cold / warm), N = 1
    scratch = None
    if rank == 0 and P == 1 and not args.profile:
        scratch = torch.empty(512 << 18, dtype=torch.float32, device=dev)   # 512 MB > L2
    if rank == 0 and P == 1 and not args.profile and not args.no_cusparse:
        try:
            pk = dict(plan_kw)
            pr = graph_protocol(A, torch, dev, w, F, rp_local, ci_d, va_d, X0, scratch, peaks["hbm_gbs"], pk)
            line["protocol"] = pr
            line["spmm_graph"] = {"ms_per_layer": pr["warm_ms"], "gflops": flops_layer / (pr["warm_ms"] * 1e-3) / 1e9,
                                  "how": "20 agcn_spmm in one CUDA graph, replayed 3x (warm L2)"}
            line["spmm_cold"] = {"ms_per_layer": pr["cold_ms"], "gflops": pr["gflops_cold"],
                                 "how": "512 MB scratch written + persisting L2 reset before each call, events"}
            if "cusparse_best_alg" in pr:
                line["cusparse"] = {"best_alg": pr["cusparse_best_alg"], "cold_ms": pr["cusparse_best_cold_ms"],
                                    "warm_ms": pr["cusparse_best_warm_ms"],
                                    "speedup_cold": pr["speedup_vs_cusparse_best_cold"],
                                    "speedup_warm": pr["speedup_vs_cusparse_best_warm"],
                                    "via": "cusparseSpMM (CSR, row-major X/Y; bufferSize + preprocess "
                                           "outside timing; baseline/cusparse_spmm.cu)",
                                    "algs": pr["cusparse"]}
        except Exception as e:  # pragma: no cover
            line["protocol"] = {"error": str(e)[:200]}

    # ---- end to end through the C ABI on HOST buffers (copies inside the timed region)
    if not args.no_e2e and not args.profile:
        e2e = None
        if P == 1:
            pin = lambda a: torch.from_numpy(a).pin_memory()  # noqa: E731
            rp_h, ci_h, va_h, X_h = pin(w.rowptr), pin(w.colidx), pin(w.vals), pin(X_host)
            Y_h = torch.empty((n, F), dtype=torch.float32).pin_memory()
            A.propagate_host(rp_h, ci_h, va_h, X_h, layers, out=Y_h)   # warm-up
            ts = []
            for _ in range(args.e2e_steps):
                t0 = time.perf_counter()
                A.propagate_host(rp_h, ci_h, va_h, X_h, layers, out=Y_h)
                ts.append(time.perf_counter() - t0)
            t_sync = statistics.median(ts)
            # the serving path: agcn_pipe_* overlaps job k's copy-in with job k-1's copy-out;
            # every job still copies its CSR + X in and its Y out (host wall clock, K jobs)
            Y_h2 = torch.empty((n, F), dtype=torch.float32).pin_memory()
            with A.Pipeline(depth=args.pipe_depth, max_block_warps=args.mbw, max_warp_nzs=args.mwn) as pipe:
                for k in range(max(2, args.pipe_depth)):   # warm-up: every slot's buffers exist
                    pipe.submit(rp_h, ci_h, va_h, X_h, layers, out=(Y_h, Y_h2)[k & 1])
                pipe.wait()
                t0 = time.perf_counter()
                for k in range(args.e2e_steps):
                    pipe.submit(rp_h, ci_h, va_h, X_h, layers, out=(Y_h, Y_h2)[k & 1])
                pipe.wait()
                t = (time.perf_counter() - t0) / args.e2e_steps
            # what the host got back is the device path's timed output, bit for bit (outside timing)
            y_last = (Y_h, Y_h2)[(args.e2e_steps - 1) & 1]
            same_out = bool(torch.equal(torch.as_tensor(y_last).reshape(n, F), Yfinal.cpu())) \
                if (args.aggregation == "sum" and args.gin_eps is None and not args.bias_relu) else None
            e2e = {"value": flops_layer * layers / t / 1e9, "unit": UNIT, "ms_per_step": 1e3 * t,
                   "h2d_bytes_per_step": 4 * (n + 1) + 8 * nnz + 4 * n * F,
                   "d2h_bytes_per_step": 4 * n * F, "output_equals_timed_device_output": same_out,
                   "api": "agcn_pipe_submit x steps + agcn_pipe_wait (C ABI, pinned host buffers)",
                   "jobs": args.e2e_steps, "sync_call_ms_per_step": 1e3 * t_sync,
                   "sync_call_api": "agcn_propagate_host (one blocking call per step)"}
        else:
            pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()  # noqa: E731
            lo, hi = lay.lo, lay.hi
            a0, a1 = int(w.rowptr[lo]), int(w.rowptr[hi])
            rp_h = pin(w.rowptr[lo:hi + 1] - a0)
            ci_h, va_h = pin(w.colidx[a0:a1]), pin(w.vals[a0:a1])
            X_h = pin(X_host)
            Y_h = torch.empty((lay.rows, F), dtype=torch.float32).pin_memory()
            ts = []
            for it in range(args.e2e_steps + 1):
                barrier()
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                rp_e, ci_e, va_e = (rp_h.to(dev, non_blocking=True), ci_h.to(dev, non_blocking=True),
                                    va_h.to(dev, non_blocking=True))
                Xe = torch.empty((lay.padded_rows, F), dtype=torch.float32, device=dev)
                lay.pad(X_h.to(dev, non_blocking=True), Xe)
                pe = A.Plan(rp_e, ci_e, **plan_kw)
                bufs_e = [torch.empty_like(Xe) for _ in range(min(layers, 2))]
                oute = propagate(lay, lambda Xin, o: pe.spmm(va_e, Xin, out=o), Xe, bufs_e, layers,
                                 gather)
                Y_h.copy_(lay.own_rows(oute))
                torch.cuda.synchronize()
                dt = torch.tensor([time.perf_counter() - t0], device=dev)
                dist.all_reduce(dt, op=dist.ReduceOp.MAX)
                pe.close()
                if it > 0:
                    ts.append(float(dt.item()))
            t = statistics.median(ts)
            e2e = {"value": flops_layer * layers / t / 1e9, "unit": UNIT, "ms_per_step": 1e3 * t,
                   "h2d_bytes_per_step": 4 * (lay.rows + 1) + 8 * (a1 - a0) + 4 * n * F,
                   "d2h_bytes_per_step": 4 * lay.rows * F, "api": "Plan/spmm + NCCL (python)"}
        if rank == 0:
            line["e2e"] = e2e

    # ---- CPU oracle baseline (rank 0, N=1 only)
    if rank == 0 and P == 1 and not args.no_cpu_baseline and not args.profile:
        cb, _ = cpu_sample_gflops(w, X_host, args.cpu_seconds)
        cb["cpu_model"] = cpu_model()
        cb["threads"] = cb["cores"]
        line["cpu_baseline"] = cb

    # ---- kernel-only table of the other BASELINE graphs (N=1)
    if rank == 0 and P == 1 and not args.profile and not args.no_per_graph:
        line["per_graph"] = per_graph_table(A, gen, torch, dev, args.config if args.F is None else "",
                                            peaks["hbm_gbs"], scratch)

    # ---- roofline.traffic: DRAM bytes of THIS build's SpMM calls (live ncu capture; outside
    # every timed region; N = 1), or a committed capture of the same build
    if rank == 0 and P == 1 and not args.profile:
        traffic, traffic_src = (None, None) if args.no_traffic else live_traffic(args)
        if traffic is None:
            why = traffic_src
            traffic, traffic_src = load_traffic(args.config, F)
            traffic_src = dict(traffic_src, live_error=why)
        rl = line["roofline"]
        rl["traffic"] = traffic
        rl["traffic_gbs"] = traffic / (spmm_max * 1e-3) / 1e9 if traffic else None
        rl["traffic_frac"] = rl["traffic_gbs"] / peaks["hbm_gbs"] if traffic else None
        rl["traffic_over_algorithmic"] = traffic / b_comp if traffic else None
        rl["traffic_source"] = traffic_src

    if rank == 0:
        print(json.dumps(line), flush=True)
    if P > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
