"""Seeded synthetic inputs shared by the oracle and the CUDA path.

This package manufactures inputs only (graphs shaped like PAPER.md Table I, lines
453-468, dense features and values).  It holds none of the method's arithmetic and
imports neither ``oracle`` nor ``paper_2308_11825_b200``.  The heavy generators are
plain C (``gen.c``), built on first use with gcc; every random number is counter based,
so outputs are bit-identical for any thread count.  Recipes: DESIGN.md "Input recipe".
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "gen.c")
_LIB = os.path.join(_HERE, "libagcn_inputs.so")
_lib = None

I32P = ctypes.POINTER(ctypes.c_int32)
F32P = ctypes.POINTER(ctypes.c_float)


def build(force: bool = False) -> str:
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O3", "-std=c11", "-fPIC", "-shared", "-pthread",
                               _SRC, "-o", tmp, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        lib = ctypes.CDLL(build())
        lib.gen_uniform_f32.argtypes = [ctypes.c_uint64, ctypes.c_int64, ctypes.c_float,
                                        ctypes.c_float, F32P, ctypes.c_int]
        lib.gen_int_f32.argtypes = [ctypes.c_uint64, ctypes.c_int64, ctypes.c_int, ctypes.c_int,
                                    F32P, ctypes.c_int]
        lib.gen_gcn_vals.argtypes = [ctypes.c_int64, I32P, I32P, F32P, ctypes.c_int]
        lib.gen_permutation.argtypes = [ctypes.c_uint64, ctypes.c_int64, I32P]
        lib.gen_chung_lu_alpha.argtypes = [ctypes.c_int64, ctypes.c_double]
        lib.gen_chung_lu_alpha.restype = ctypes.c_double
        lib.gen_chung_lu.argtypes = [ctypes.c_int64, ctypes.c_int64, ctypes.c_double,
                                     ctypes.c_uint64, ctypes.c_int, I32P, I32P, ctypes.c_int]
        lib.gen_chung_lu.restype = ctypes.c_double
        lib.gen_rmat.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_double, ctypes.c_double,
                                 ctypes.c_double, ctypes.c_uint64, I32P, I32P, ctypes.c_int]
        _lib = lib
    return _lib


def _p(a: np.ndarray, t):
    return a.ctypes.data_as(t)


def uniform_f32(seed: int, shape, lo=-1.0, hi=1.0, nthreads=0) -> np.ndarray:
    out = np.empty(shape, dtype=np.float32)
    _load().gen_uniform_f32(seed, out.size, lo, hi, _p(out, F32P), nthreads)
    return out


def int_f32(seed: int, shape, lo=-4, hi=4, nthreads=0) -> np.ndarray:
    out = np.empty(shape, dtype=np.float32)
    _load().gen_int_f32(seed, out.size, lo, hi, _p(out, F32P), nthreads)
    return out


def gcn_vals(rowptr: np.ndarray, colidx: np.ndarray, nthreads=0) -> np.ndarray:
    n = rowptr.size - 1
    out = np.empty(colidx.size, dtype=np.float32)
    _load().gen_gcn_vals(n, _p(rowptr, I32P), _p(colidx, I32P), _p(out, F32P), nthreads)
    return out


def permutation(seed: int, n: int) -> np.ndarray:
    out = np.empty(n, dtype=np.int32)
    _load().gen_permutation(seed, n, _p(out, I32P))
    return out


def chung_lu(n: int, nnz: int, max_over_mean: float, seed: int, relabel=True, nthreads=0):
    """Chung-Lu power-law CSR (n x n, exactly nnz, distinct sorted columns)."""
    rowptr = np.empty(n + 1, dtype=np.int32)
    colidx = np.empty(nnz, dtype=np.int32)
    alpha = _load().gen_chung_lu(n, nnz, max_over_mean, seed, 1 if relabel else 0,
                                 _p(rowptr, I32P), _p(colidx, I32P), nthreads)
    return rowptr, colidx, alpha


def rmat(scale: int, edge_factor: int, seed: int, a=0.57, b=0.19, c=0.19, nthreads=0):
    """Graph500 R-MAT CSR: 2^scale rows, edge_factor*2^scale nnz (duplicates kept)."""
    n = 1 << scale
    rowptr = np.empty(n + 1, dtype=np.int32)
    colidx = np.empty(n * edge_factor, dtype=np.int32)
    _load().gen_rmat(scale, edge_factor, a, b, c, seed, _p(rowptr, I32P), _p(colidx, I32P),
                     nthreads)
    return rowptr, colidx


# ---------------------------------------------------------------- BASELINE.json configs
@dataclass
class Workload:
    name: str
    rowptr: np.ndarray
    colidx: np.ndarray
    vals: np.ndarray
    F: int
    x_seed: int
    layers: int = 1
    meta: dict = field(default_factory=dict)

    @property
    def n(self) -> int:
        return self.rowptr.size - 1

    @property
    def nnz(self) -> int:
        return int(self.colidx.size)

    def X(self, F: int | None = None, nthreads=0) -> np.ndarray:
        F = self.F if F is None else F
        return uniform_f32(self.x_seed, (self.n, F), -1.0, 1.0, nthreads)


# (name, generator args, F, seeds graph/X/vals) -- SURVEY.md section 8(d1), BASELINE.md section 3
CONFIGS = {
    "c1": dict(kind="cl", n=2708, nnz=10556, mom=66.0, F=16, seeds=(1, 101, 201),
               desc="Cora-shaped Chung-Lu, F=16"),
    "c2": dict(kind="cl", n=19717, nnz=88648, mom=66.0, F=16, seeds=(2, 102, 202),
               desc="Pubmed-shaped Chung-Lu, F sweep 16/32/64/128"),
    "c3": dict(kind="cl", n=169343, nnz=1166243, mom=66.0, F=64, seeds=(3, 103, 203),
               desc="ogbn-arxiv-shaped Chung-Lu, F=64"),
    "c4": dict(kind="cl", n=232965, nnz=114615891, mom=44.0, F=128, seeds=(4, 104, 204),
               desc="Reddit-shaped dense-hub Chung-Lu, F=128"),
    "c5": dict(kind="rmat", scale=23, ef=16, F=64, seeds=(5, 105, 205), layers=2,
               desc="R-MAT scale 23 edge factor 16, F=64, 2-layer propagation"),
}


def make_config(name: str, nthreads=0, vals_kind: str = "gcn") -> Workload:
    cfg = CONFIGS[name]
    gseed, xseed, vseed = cfg["seeds"]
    if cfg["kind"] == "cl":
        rowptr, colidx, alpha = chung_lu(cfg["n"], cfg["nnz"], cfg["mom"], gseed, True, nthreads)
        meta = {"alpha": alpha}
    else:
        rowptr, colidx = rmat(cfg["scale"], cfg["ef"], gseed, nthreads=nthreads)
        meta = {"scale": cfg["scale"], "edge_factor": cfg["ef"]}
    if vals_kind == "gcn":
        vals = gcn_vals(rowptr, colidx, nthreads)
    elif vals_kind == "uniform":
        vals = uniform_f32(vseed, colidx.size, -1.0, 1.0, nthreads)
    elif vals_kind == "int":
        vals = int_f32(vseed, colidx.size, -4, 4, nthreads)
    elif vals_kind == "ones":
        vals = np.ones(colidx.size, dtype=np.float32)
    else:
        raise ValueError(vals_kind)
    meta["desc"] = cfg["desc"]
    return Workload(name, rowptr, colidx, vals, cfg["F"], xseed, cfg.get("layers", 1), meta)


# ---------------------------------------------------------------- small random CSRs (tests)
def random_csr(n: int, n_cols: int, seed: int, max_deg: int | None = None,
               p_zero: float = 0.2, dup: bool = False):
    """Small random CSR with a heavy-tailed degree mix, zero rows, optional duplicates."""
    rng = np.random.default_rng(seed)
    max_deg = n_cols if max_deg is None else max_deg
    degs = np.minimum(rng.zipf(1.6, size=n) - 1, max_deg).astype(np.int64)
    degs[rng.random(n) < p_zero] = 0
    if not dup:
        degs = np.minimum(degs, n_cols)
    rowptr = np.zeros(n + 1, dtype=np.int32)
    rowptr[1:] = np.cumsum(degs)
    cols = []
    for d in degs:
        if dup:
            c = rng.integers(0, n_cols, size=d)
        else:
            c = rng.choice(n_cols, size=d, replace=False)
        cols.append(np.sort(c))
    colidx = np.concatenate(cols).astype(np.int32) if cols else np.zeros(0, np.int32)
    return rowptr, colidx
