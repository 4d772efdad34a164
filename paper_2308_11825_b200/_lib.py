"""ctypes declarations of include/agcn.h.  Argument marshalling only."""
from __future__ import annotations

import ctypes
import os

from . import _build

c_i32, c_i64, c_u64, c_size, c_vp = (ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64,
                                     ctypes.c_size_t, ctypes.c_void_p)

STATUS = {0: "AGCN_OK", 1: "AGCN_ERR_INVALID_ARG", 2: "AGCN_ERR_BAD_CSR", 3: "AGCN_ERR_OOM",
          4: "AGCN_ERR_CUDA", 5: "AGCN_ERR_OVERFLOW", 6: "AGCN_ERR_UNSUPPORTED"}
FIELDS = {"perm": 0, "blocks": 1, "sorted_colidx": 2, "row_src_off": 3, "tasks": 4,
          "sorted_rowptr": 5, "hot_cols": 6}


class Opts(ctypes.Structure):
    _fields_ = [("max_block_warps", c_i32), ("max_warp_nzs", c_i32), ("partition", c_i32),
                ("validate", c_i32), ("n_cols", c_i64), ("stream", c_vp),
                ("col_bounds", ctypes.POINTER(c_i64)), ("col_nparts", c_i32),
                ("col_slot_rows", c_i64), ("hot_rows", c_i64), ("small_plan", c_i32),
                ("chunk_buckets", c_i32)]


KERNELS = {"auto": 0, "general": 1, "looped": 2, "wide": 3}
L2_HINTS = {None: -1, "auto": -1, "none": 0, 0: 0, "keep_all": 1, 1: 1, "hot_window": 2, 2: 2,
            "hot_hints": 3, 3: 3}


class SpmmOpts(ctypes.Structure):
    _fields_ = [("kernel", c_i32), ("l2_hint", c_i32), ("hot_mb", c_i32),
                ("aggregation", c_i32), ("self_scale", ctypes.c_float), ("relu", c_i32),
                ("self", c_vp), ("bias", c_vp), ("peer_out", c_vp * 8), ("npeer", c_i32),
                ("chunk_shape", c_i32), ("chunk_order", c_i32), ("pad0_", c_i32),
                ("reserved", c_i64 * 2)]


class Stats(ctypes.Structure):
    _fields_ = [("n", c_i64), ("n_cols", c_i64), ("nnz", c_i64), ("nblocks", c_i64),
                ("ntasks", c_i64), ("deg_bound", c_i64), ("max_deg", c_i64),
                ("n_zero_rows", c_i64), ("n_oversized_rows", c_i64),
                ("n_oversized_blocks", c_i64), ("max_block_warps", c_i32),
                ("max_warp_nzs", c_i32), ("partition", c_i32), ("reserved", c_i32),
                ("device_bytes", c_size), ("hot_rows", c_i64)]


_lib = None


def lib():
    """Load libagcn.so (building it with nvcc first if it is missing or stale).

    There is no fallback: if the library cannot be built or loaded this raises.
    """
    global _lib
    if _lib is not None:
        return _lib
    path = os.environ.get("AGCN_LIBRARY") or _build.build()  # AGCN_LIBRARY: A/B of builds
    L = ctypes.CDLL(path, mode=os.RTLD_LOCAL)
    L.agcn_default_opts.argtypes = [ctypes.POINTER(Opts)]
    L.agcn_default_opts.restype = None
    L.agcn_plan.argtypes = [c_vp, c_vp, c_i64, c_i64]
    L.agcn_plan.restype = c_vp
    L.agcn_plan_ex.argtypes = [c_vp, c_vp, c_i64, c_i64, ctypes.POINTER(Opts)]
    L.agcn_plan_ex.restype = c_vp
    L.agcn_spmm.argtypes = [c_vp, c_vp, c_vp, c_i32, c_vp, c_vp]
    L.agcn_spmm.restype = c_i32
    L.agcn_default_spmm_opts.argtypes = [ctypes.POINTER(SpmmOpts)]
    L.agcn_default_spmm_opts.restype = None
    L.agcn_spmm_ex.argtypes = [c_vp, c_vp, c_vp, c_i32, c_vp, c_vp, ctypes.POINTER(SpmmOpts)]
    L.agcn_spmm_ex.restype = c_i32
    L.agcn_plan_destroy.argtypes = [c_vp]
    L.agcn_plan_destroy.restype = c_i32
    L.agcn_plan_stats.argtypes = [c_vp, ctypes.POINTER(Stats)]
    L.agcn_plan_stats.restype = c_i32
    L.agcn_plan_copy.argtypes = [c_vp, c_i32, c_vp, c_size]
    L.agcn_plan_copy.restype = c_i32
    L.agcn_auto_partition.argtypes = [c_i64, c_i64, c_i32, ctypes.POINTER(c_i32), ctypes.POINTER(c_i32)]
    L.agcn_auto_partition.restype = c_i32
    L.agcn_shard_bounds.argtypes = [c_vp, c_i64, c_i32, ctypes.POINTER(c_i64), c_vp]
    L.agcn_shard_bounds.restype = c_i32
    L.agcn_propagate_host.argtypes = [c_vp, c_vp, c_vp, c_i64, c_i64, c_vp, c_i32, c_i32, c_vp,
                                      ctypes.POINTER(Opts)]
    L.agcn_propagate_host.restype = c_i32
    L.agcn_graph_create.argtypes = [c_vp, c_vp, c_vp, c_i32, c_i32, c_vp, c_vp]
    L.agcn_graph_create.restype = c_vp
    L.agcn_graph_launch.argtypes = [c_vp, c_vp]
    L.agcn_graph_launch.restype = c_i32
    L.agcn_graph_destroy.argtypes = [c_vp]
    L.agcn_graph_destroy.restype = c_i32
    L.agcn_pipe_create.argtypes = [c_i32, ctypes.POINTER(Opts)]
    L.agcn_pipe_create.restype = c_vp
    L.agcn_pipe_submit.argtypes = [c_vp, c_vp, c_vp, c_vp, c_i64, c_i64, c_vp, c_i32, c_i32, c_vp]
    L.agcn_pipe_submit.restype = c_i32
    L.agcn_pipe_wait.argtypes = [c_vp]
    L.agcn_pipe_wait.restype = c_i32
    L.agcn_pipe_destroy.argtypes = [c_vp]
    L.agcn_pipe_destroy.restype = c_i32
    L.agcn_transpose.argtypes = [c_vp, c_vp, c_i64, c_i64, c_i64, c_vp, c_vp, c_vp, c_vp]
    L.agcn_transpose.restype = c_i32
    L.agcn_gather_vals.argtypes = [c_vp, c_vp, c_i64, c_vp, c_vp]
    L.agcn_gather_vals.restype = c_i32
    L.agcn_gemm_xw.argtypes = [c_vp, c_i64, c_i32, c_vp, c_i32, c_vp, c_vp, c_i32, c_vp]
    L.agcn_gemm_xw.restype = c_i32
    L.agcn_gemm_xw_ex.argtypes = [c_vp, c_i64, c_i32, c_vp, c_i32, c_vp, c_vp, c_i32, c_i32, c_vp]
    L.agcn_gemm_xw_ex.restype = c_i32
    L.agcn_device_alloc.argtypes = [c_size, ctypes.POINTER(c_vp)]
    L.agcn_device_alloc.restype = c_i32
    L.agcn_device_free.argtypes = [c_vp]
    L.agcn_device_free.restype = c_i32
    L.agcn_ipc_export.argtypes = [c_vp, c_vp]
    L.agcn_ipc_export.restype = c_i32
    L.agcn_ipc_open.argtypes = [c_vp, ctypes.POINTER(c_vp)]
    L.agcn_ipc_open.restype = c_i32
    L.agcn_ipc_close.argtypes = [c_vp]
    L.agcn_ipc_close.restype = c_i32
    L.agcn_last_status.argtypes = []
    L.agcn_last_status.restype = c_i32
    L.agcn_last_error.argtypes = []
    L.agcn_last_error.restype = ctypes.c_char_p
    L.agcn_launch_count.argtypes = []
    L.agcn_launch_count.restype = c_u64
    L.agcn_version.argtypes = []
    L.agcn_version.restype = ctypes.c_char_p
    _lib = L
    return L


EXPORTS = ["agcn_default_opts", "agcn_plan", "agcn_plan_ex", "agcn_spmm", "agcn_default_spmm_opts",
           "agcn_spmm_ex", "agcn_plan_destroy",
           "agcn_plan_stats", "agcn_plan_copy", "agcn_auto_partition", "agcn_shard_bounds", "agcn_propagate_host",
           "agcn_pipe_create", "agcn_pipe_submit", "agcn_pipe_wait", "agcn_pipe_destroy",
           "agcn_graph_create", "agcn_graph_launch", "agcn_graph_destroy",
           "agcn_transpose", "agcn_gather_vals", "agcn_gemm_xw", "agcn_gemm_xw_ex", "agcn_device_alloc", "agcn_device_free", "agcn_ipc_export",
           "agcn_ipc_open", "agcn_ipc_close", "agcn_last_status", "agcn_last_error", "agcn_launch_count", "agcn_version"]
