"""Comparison arms of the measurement protocol, not the product.

``cusparse_spmm.cu`` -> ``libcusparse_bench.so`` (built with nvcc on first use / by
``__graft_entry__.build()``): cusparseSpMM per algorithm with bufferSize / preprocess outside
timing, cold or warm L2, and the L2 flush helper both bench arms use.
"""
from __future__ import annotations

import ctypes
import os
import shutil
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "cusparse_spmm.cu")
LIB = os.path.join(HERE, "libcusparse_bench.so")
ALGS = {"ALG_DEFAULT": 0, "CSR_ALG1": 4, "CSR_ALG2": 6, "CSR_ALG3": 12}
_lib = None


def build(force: bool = False) -> str:
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        nvcc = next(c for c in ("/usr/local/cuda/bin/nvcc", shutil.which("nvcc")) if c and os.path.exists(c))
        tmp = LIB + f".tmp{os.getpid()}"
        subprocess.check_call([nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-shared",
                               "-Xcompiler", "-fPIC", SRC, "-o", tmp, "-lcusparse"])
        os.replace(tmp, LIB)
    return LIB


def lib():
    global _lib
    if _lib is None:
        L = ctypes.CDLL(build())
        vp, i32, i64, sz = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_size_t
        L.bl_l2_flush.argtypes = [vp, sz, vp]
        L.bl_l2_flush.restype = ctypes.c_int
        L.bl_cusparse_spmm.argtypes = [vp, vp, vp, i64, i64, i64, vp, i32, vp, i32, i32, i32, vp, sz,
                                       ctypes.POINTER(ctypes.c_float), ctypes.POINTER(sz), vp]
        L.bl_cusparse_spmm.restype = ctypes.c_int
        _lib = L
    return _lib


def l2_flush(scratch, stream) -> None:
    """Cold L2 before a timed call: write `scratch` (a CUDA tensor larger than L2) and reset
    persisting lines, on `stream` (a torch.cuda.Stream)."""
    if lib().bl_l2_flush(scratch.data_ptr(), scratch.numel() * scratch.element_size(), stream.cuda_stream) != 0:
        raise RuntimeError("bl_l2_flush failed")


def cusparse_spmm_times(rowptr, colidx, vals, X, Y, alg: str, reps: int, cold: bool, scratch, stream):
    """Per-call ms of cusparseSpMM (algorithm `alg`) on device tensors; None if the algorithm
    does not accept the problem (status returned instead)."""
    ms = (ctypes.c_float * reps)()
    bb = ctypes.c_size_t(0)
    n, F = Y.shape
    rc = lib().bl_cusparse_spmm(rowptr.data_ptr(), colidx.data_ptr(), vals.data_ptr(), n, X.shape[0],
                                colidx.numel(), X.data_ptr(), F, Y.data_ptr(), ALGS[alg], reps, int(cold),
                                scratch.data_ptr() if scratch is not None else None,
                                scratch.numel() * 4 if scratch is not None else 0, ms, ctypes.byref(bb),
                                stream.cuda_stream)
    if rc != 0:
        return None, rc, bb.value
    return list(ms), 0, bb.value
