"""CPU oracle for the Accel-GCN hot path (arXiv 2308.11825) -- TEST INFRASTRUCTURE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  The product path
(``paper_2308_11825_b200``) never imports it and shares no code with it.

The arithmetic lives in plain C (``oracle.c``, fp64 accumulation) and is wrapped here with
ctypes; each function cites the PAPER.md passage it follows (P:n = PAPER.md line n).
Pins: tests/test_oracle.py (Fig. 3 worked example, closed forms, dense brute force,
invariants).  Readings of ambiguous passages: DESIGN.md "Readings" (Q-numbers).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None

I32P = ctypes.POINTER(ctypes.c_int32)
I64P = ctypes.POINTER(ctypes.c_int64)
U32P = ctypes.POINTER(ctypes.c_uint32)
F32P = ctypes.POINTER(ctypes.c_float)
F64P = ctypes.POINTER(ctypes.c_double)

# BASELINE.json north_star: |y - y_ref| <= 1e-5 * sum_j |a_ij x_jk| + 1e-7
REL_TOL = 1e-5
ABS_TOL = 1e-7


def build(force: bool = False) -> str:
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-pthread",
                               _SRC, "-o", tmp, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        lib = ctypes.CDLL(build())
        lib.orc_spmm.argtypes = [ctypes.c_int64, I32P, I32P, F32P, F32P, ctypes.c_int64,
                                 F64P, F64P, ctypes.c_int]
        lib.orc_spmm_check.argtypes = [ctypes.c_int64, I32P, I32P, F32P, F32P, ctypes.c_int64,
                                       F32P, I64P, ctypes.c_int64, ctypes.c_double,
                                       ctypes.c_double, F64P, I64P, ctypes.c_int]
        lib.orc_spmm_check.restype = ctypes.c_int64
        lib.orc_degree_sort.argtypes = [ctypes.c_int64, I32P, I32P]
        lib.orc_degree_sort.restype = ctypes.c_int64
        lib.orc_sorted_csr.argtypes = [ctypes.c_int64, I32P, I32P, I32P, I32P, I32P, I32P]
        lib.orc_patterns.argtypes = [ctypes.c_int32, ctypes.c_int32, I32P, I32P]
        lib.orc_patterns.restype = ctypes.c_int64
        lib.orc_block_partition.argtypes = [ctypes.c_int64, I32P, ctypes.c_int32, ctypes.c_int32,
                                            U32P, ctypes.c_int64]
        lib.orc_block_partition.restype = ctypes.c_int64
        lib.orc_warp_partition.argtypes = [ctypes.c_int64, I32P, ctypes.c_int32, U32P,
                                           ctypes.c_int64]
        lib.orc_warp_partition.restype = ctypes.c_int64
        lib.orc_shard_bounds.argtypes = [ctypes.c_int64, I32P, ctypes.c_int32, I64P]
        _lib = lib
    return _lib


def _c(a: np.ndarray, dtype) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=dtype)


def _p(a, t):
    return a.ctypes.data_as(t)


# ---------------------------------------------------------------- result oracle
def spmm(rowptr, colidx, vals, X, nthreads: int = 0, with_abs: bool = True):
    """Y = A.X in fp64: returns (y_ref, s) with s = sum_p |a_p x| (None if not with_abs)."""
    rowptr = _c(rowptr, np.int32); colidx = _c(colidx, np.int32)
    vals = _c(vals, np.float32); X = _c(X, np.float32)
    n = rowptr.size - 1
    F = X.shape[1] if X.ndim == 2 else 1
    y = np.empty((n, F), dtype=np.float64)
    s = np.empty((n, F), dtype=np.float64) if with_abs else None
    _load().orc_spmm(n, _p(rowptr, I32P), _p(colidx, I32P), _p(vals, F32P), _p(X, F32P), F,
                     _p(y, F64P), _p(s, F64P) if s is not None else None, nthreads)
    return y, s


def spmm_check(rowptr, colidx, vals, X, Y, rows=None, rel=REL_TOL, abs_tol=ABS_TOL,
               nthreads: int = 0):
    """Streaming tolerance check of a candidate fp32 Y against the fp64 definition.

    rows=None: Y is the full n x F output.  Otherwise Y[t] is output row rows[t].
    Returns dict(max_ratio, worst=(row, col), nfail, rows checked); pass iff nfail == 0 (ratio <= 1).
    """
    rowptr = _c(rowptr, np.int32); colidx = _c(colidx, np.int32)
    vals = _c(vals, np.float32); X = _c(X, np.float32); Y = _c(Y, np.float32)
    n = rowptr.size - 1
    F = X.shape[1] if X.ndim == 2 else 1
    mr = ctypes.c_double(0.0)
    worst = np.zeros(2, dtype=np.int64)
    if rows is not None:
        rows = _c(rows, np.int64)
        assert Y.shape[0] == rows.size
        nf = _load().orc_spmm_check(n, _p(rowptr, I32P), _p(colidx, I32P), _p(vals, F32P),
                                    _p(X, F32P), F, _p(Y, F32P), _p(rows, I64P), rows.size,
                                    rel, abs_tol, ctypes.byref(mr), _p(worst, I64P), nthreads)
    else:
        assert Y.shape[0] == n
        nf = _load().orc_spmm_check(n, _p(rowptr, I32P), _p(colidx, I32P), _p(vals, F32P),
                                    _p(X, F32P), F, _p(Y, F32P), None, 0, rel, abs_tol,
                                    ctypes.byref(mr), _p(worst, I64P), nthreads)
    return {"max_ratio": mr.value, "worst": (int(worst[0]), int(worst[1])), "nfail": int(nf),
            "rows": int(n if rows is None else rows.size)}


def spmm_epilogue(rowptr, colidx, vals, X, aggregation="sum", self_x=None, self_scale=0.0,
                  bias=None, relu=False):
    """The aggregation variants of P:126 on top of the fp64 definition (reading Q34):
    y_i = (sum_j a_ij x_j) * (1 / deg_i if aggregation == "mean", 0 for deg_i = 0)
          + self_scale * self_x[i] + bias;  y = max(y, 0) if relu.
    GCN: sum; GraphSAGE-mean: mean; GIN: sum with self_x = X, self_scale = 1 + eps.
    Returns (y_ref, tol_scale): fp64 result and the magnitude the tolerance is relative to,
    (scale_i * sum_j |a_ij x_jk| + |self_scale * self_x[i,k]| + |bias_k|)."""
    y, sabs = spmm(rowptr, colidx, vals, X)
    deg = np.diff(np.asarray(rowptr, dtype=np.int64)).astype(np.float64)
    if aggregation == "mean":
        sc = np.where(deg > 0, 1.0 / np.maximum(deg, 1.0), 0.0)[:, None]
        y = y * sc
        sabs = sabs * sc
    elif aggregation != "sum":
        raise ValueError(aggregation)
    if self_scale != 0.0:
        t = float(np.float32(self_scale)) * np.asarray(self_x, dtype=np.float64)
        y = y + t
        sabs = sabs + np.abs(t)
    if bias is not None:
        b = np.asarray(bias, dtype=np.float64)[None, :]
        y = y + b
        sabs = sabs + np.abs(b)
    if relu:
        y = np.maximum(y, 0.0)
    return y, sabs


def check_epilogue(Y, y_ref, tol_scale, rel=REL_TOL, abs_tol=ABS_TOL):
    """|Y - y_ref| <= rel * tol_scale + abs_tol per element (NaN fails); ReLU is 1-Lipschitz, so
    the bound of the pre-activation carries over.  Returns dict(max_ratio, nfail)."""
    Y = np.asarray(Y, dtype=np.float64)
    err = np.abs(Y - y_ref)
    ratio = err / (rel * tol_scale + abs_tol)
    ratio[~np.isfinite(Y)] = np.inf
    return {"max_ratio": float(ratio.max()) if ratio.size else 0.0, "nfail": int((~(ratio <= 1.0)).sum())}


def gcn_layer(rowptr, colidx, vals, X, W, bias=None, relu=True):
    """One GCN layer in fp64 (X' = sigma(A' Y), Y = X W; sigma = ReLU, plus a bias):
    Y = X W (numpy matmul, the library step), then y_i = sum_p a_p Y[col_p] (the SpMM
    definition written out with np.add.reduceat), + bias, ReLU.  Returns (y_ref, tol_scale)
    with tol_scale = sum_p |a_p| sum_k |x_{col_p,k}| |w_kc| (+ |bias|): the magnitude the
    fp32 tolerance (1e-5 relative) applies to for either evaluation order."""
    rowptr = np.asarray(rowptr, dtype=np.int64)
    base = int(rowptr[0])
    nnz = int(rowptr[-1] - base)
    cols = np.asarray(colidx, dtype=np.int64)[base:base + nnz]
    a = np.asarray(vals, dtype=np.float64)[base:base + nnz]
    X64, W64 = np.asarray(X, dtype=np.float64), np.asarray(W, dtype=np.float64)
    T = X64 @ W64
    Tabs = np.abs(X64) @ np.abs(W64)
    n, Fo = rowptr.size - 1, W64.shape[1]
    y = np.zeros((n, Fo))
    t = np.zeros((n, Fo))
    nz = np.flatnonzero(np.diff(rowptr) > 0)
    if nnz:
        starts = (rowptr[:-1] - base)[nz]
        y[nz] = np.add.reduceat(a[:, None] * T[cols], starts, axis=0)
        t[nz] = np.add.reduceat(np.abs(a)[:, None] * Tabs[cols], starts, axis=0)
    if bias is not None:
        b = np.asarray(bias, dtype=np.float64)[None, :]
        y = y + b
        t = t + np.abs(b)
    if relu:
        y = np.maximum(y, 0.0)
    return y, t


def transpose(rowptr, colidx, n_cols: int):
    """CSR of A^T (backward pass, dX = A^T dY): (rowptr_t, colidx_t, src) with
    row j of A^T = the rows i holding column j in increasing i (a stable sort of the entries
    by column: np.argsort(kind="stable") is the library step); entry k of A^T is entry
    src[k] of A (rowptr-relative)."""
    rowptr = np.asarray(rowptr, dtype=np.int64)
    base = int(rowptr[0])
    nnz = int(rowptr[-1] - base)
    cols = np.asarray(colidx, dtype=np.int64)[base:base + nnz]
    src = np.argsort(cols, kind="stable").astype(np.int32)
    rows = np.repeat(np.arange(rowptr.size - 1, dtype=np.int32), np.diff(rowptr))
    rowptr_t = np.zeros(n_cols + 1, dtype=np.int32)
    rowptr_t[1:] = np.cumsum(np.bincount(cols, minlength=n_cols))
    return rowptr_t, rows[src], src


# ---------------------------------------------------------------- preprocessing
def degree_sort(rowptr):
    """Stable ascending counting sort of rows by degree -> perm (sorted_to_orig)."""
    rowptr = _c(rowptr, np.int32)
    n = rowptr.size - 1
    perm = np.empty(n, dtype=np.int32)
    maxd = _load().orc_degree_sort(n, _p(rowptr, I32P), _p(perm, I32P))
    if maxd < 0:
        raise ValueError("malformed rowptr")
    return perm


def sorted_csr(rowptr, colidx, perm):
    """(sorted_rowptr, sorted_colidx, row_src_off) for the degree-sorted row order."""
    rowptr = _c(rowptr, np.int32); colidx = _c(colidx, np.int32); perm = _c(perm, np.int32)
    n = rowptr.size - 1
    nnz = int(rowptr[-1] - rowptr[0]) if n > 0 else 0
    srp = np.empty(n + 1, dtype=np.int32)
    sci = np.empty(nnz, dtype=np.int32)
    rso = np.empty(n, dtype=np.int32)
    _load().orc_sorted_csr(n, _p(rowptr, I32P), _p(colidx, I32P), _p(perm, I32P),
                           _p(srp, I32P), _p(sci, I32P), _p(rso, I32P))
    return srp, sci, rso


def patterns(max_block_warps: int, max_warp_nzs: int):
    """Algorithm 1: arrays block_rows[d], warp_nzs[d] for d in 0..deg_bound (index 0 unused)."""
    db = max_block_warps * max_warp_nzs
    br = np.zeros(db + 1, dtype=np.int32)
    wn = np.zeros(db + 1, dtype=np.int32)
    _load().orc_patterns(max_block_warps, max_warp_nzs, _p(br, I32P), _p(wn, I32P))
    return br, wn


def block_partition(sorted_deg, max_block_warps: int = 12, max_warp_nzs: int = 32):
    """Algorithm 2 -> uint32 array (nblocks, 4) of (deg, loc, row, info) descriptors."""
    sd = _c(sorted_deg, np.int32)
    lib = _load()
    nd = lib.orc_block_partition(sd.size, _p(sd, I32P), max_block_warps, max_warp_nzs, None, 0)
    if nd == -1:
        raise ValueError("input rows are not degree-sorted")
    if nd == -2:
        raise OverflowError("block_rows or warp_nzs does not fit 16 bits")
    out = np.zeros((max(nd, 0), 4), dtype=np.uint32)
    nd2 = lib.orc_block_partition(sd.size, _p(sd, I32P), max_block_warps, max_warp_nzs,
                                  _p(out, U32P), nd)
    assert nd2 == nd
    return out


def warp_partition(rowptr, max_warp_nzs: int = 32):
    """Fig. 3(b) warp-level metadata -> uint32 array (ntasks, 4) of (row, col, len, 0)."""
    rowptr = _c(rowptr, np.int32)
    n = rowptr.size - 1
    lib = _load()
    nt = lib.orc_warp_partition(n, _p(rowptr, I32P), max_warp_nzs, None, 0)
    out = np.zeros((nt, 4), dtype=np.uint32)
    lib.orc_warp_partition(n, _p(rowptr, I32P), max_warp_nzs, _p(out, U32P), nt)
    return out


def shard_bounds(rowptr, nranks: int):
    rowptr = _c(rowptr, np.int32)
    n = rowptr.size - 1
    b = np.zeros(nranks + 1, dtype=np.int64)
    _load().orc_shard_bounds(n, _p(rowptr, I32P), nranks, _p(b, I64P))
    return b


def plan(rowptr, colidx, max_block_warps: int = 12, max_warp_nzs: int = 32):
    """The whole preprocessing of P:295 + Alg. 1/2 as a dict of integer arrays."""
    rowptr = _c(rowptr, np.int32)
    perm = degree_sort(rowptr)
    srp, sci, rso = sorted_csr(rowptr, colidx, perm)
    sdeg = np.diff(srp).astype(np.int32)
    blocks = block_partition(sdeg, max_block_warps, max_warp_nzs)
    return {"perm": perm, "sorted_rowptr": srp, "sorted_colidx": sci, "row_src_off": rso,
            "sorted_deg": sdeg, "blocks": blocks,
            "deg_bound": max_block_warps * max_warp_nzs}


# ---------------------------------------------------------------- small closed forms
def combined_warp(F: int):
    """c = ceil(F / 32) warps per combined warp, round_dim = 32 c."""
    c = (F + 31) // 32
    return c, 32 * c


def storage_ratio(nblocks: int, ntasks: int) -> float:
    """Eq. (1): S_B / S_W with equal 128-bit records = nblocks / ntasks."""
    if ntasks == 0:
        raise ZeroDivisionError("empty warp partition")
    return nblocks / ntasks
