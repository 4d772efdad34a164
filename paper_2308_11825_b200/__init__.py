"""B200-native (sm_100a) Accel-GCN aggregation SpMM, Y = A.X (arXiv 2308.11825).

Thin Python binding over the C ABI in ``include/agcn.h`` (argument marshalling only; every
step of the path runs in the CUDA kernels of ``csrc/``).  PyTorch supplies device memory,
streams and process groups.  There is no CPU fallback: if ``libagcn.so`` cannot be built or
loaded, or a tensor is not on a CUDA device, the call raises.

    plan = Plan(rowptr, colidx)            # agcn_plan: degree sort + block partition (Alg. 1/2)
    Y = plan.spmm(vals, X)                 # agcn_spmm: combined-warp SpMM
"""
from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from ._lib import FIELDS, STATUS

__all__ = ["Plan", "AgcnError", "agcn_plan", "agcn_spmm", "agcn_spmm_ex", "transpose", "gather_vals", "gemm_xw", "DeviceBuffer", "ipc_open", "ipc_close", "shard_bounds", "propagate_host", "Pipeline", "GraphedPropagation",
           "launch_count", "version", "library_path"]


class AgcnError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{STATUS.get(code, code)}: {msg}")
        self.code = code
        self.status = STATUS.get(code, str(code))


def _raise_last():
    L = _lib.lib()
    code = L.agcn_last_status()
    msg = L.agcn_last_error().decode(errors="replace")
    raise AgcnError(code, msg)


def _check(code: int):
    if code != 0:
        _raise_last()


def _torch():
    import torch
    return torch


def _dev_ptr(t, dtype_name: str, what: str) -> int:
    torch = _torch()
    if not isinstance(t, torch.Tensor):
        raise TypeError(f"{what} must be a torch.Tensor on a CUDA device")
    if not t.is_cuda:
        raise TypeError(f"{what} must be on a CUDA device (no CPU fallback)")
    want = {"int32": torch.int32, "float32": torch.float32}[dtype_name]
    if t.dtype != want:
        raise TypeError(f"{what} must be {dtype_name}, got {t.dtype}")
    if not t.is_contiguous():
        raise ValueError(f"{what} must be contiguous")
    return t.data_ptr()


def _stream_handle(stream) -> int:
    torch = _torch()
    if stream is None:
        stream = torch.cuda.current_stream()
    if isinstance(stream, torch.cuda.Stream):
        return stream.cuda_stream
    return int(stream)


def library_path() -> str:
    from . import _build
    _lib.lib()
    return _build.LIB


def version() -> str:
    return _lib.lib().agcn_version().decode()


def launch_count() -> int:
    """Kernels launched by libagcn.so in this process (monotone)."""
    return int(_lib.lib().agcn_launch_count())


class Plan:
    """agcn_plan_ex: degree-sort + block-partition metadata on the current CUDA device.

    rowptr: int32 [n+1] CUDA tensor (rowptr[0] may be nonzero for a row shard; colidx is
    then indexed by the rowptr values).  colidx: int32 CUDA tensor.
    partition: "block" (the method) or "warp" (the ablation arm, Fig. 3(b)).
    col_bounds / col_slot_rows: optional padded-layout column relabel (multi-GPU).
    """

    def __init__(self, rowptr, colidx, n: int | None = None, nnz: int | None = None, *,
                 n_cols: int | None = None, max_block_warps: int = 12, max_warp_nzs: int = 32,
                 partition: str = "block", col_bounds=None, col_slot_rows: int | None = None,
                 hot_rows: int | None = None, small_plan: bool = True, chunk_buckets: int = 0, stream=None):
        L = _lib.lib()
        rp = _dev_ptr(rowptr, "int32", "rowptr")
        ci = _dev_ptr(colidx, "int32", "colidx") if colidx.numel() else 0
        if n is None:
            n = rowptr.numel() - 1
        if nnz is None:  # agcn_plan_ex reads rowptr[0], rowptr[n] itself (one readback)
            nnz = -1
        opts = _lib.Opts()
        L.agcn_default_opts(ctypes.byref(opts))
        opts.max_block_warps = max_block_warps
        opts.max_warp_nzs = max_warp_nzs
        opts.partition = {"block": 0, "warp": 1}[partition]
        opts.n_cols = 0 if n_cols is None else int(n_cols)
        opts.stream = _stream_handle(stream)
        opts.hot_rows = -1 if hot_rows is None else int(hot_rows)
        opts.small_plan = int(bool(small_plan))
        opts.chunk_buckets = int(chunk_buckets)
        self._bounds_keep = None
        if col_bounds is not None:
            b = np.ascontiguousarray(col_bounds, dtype=np.int64)
            self._bounds_keep = b
            opts.col_bounds = b.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))
            opts.col_nparts = b.size - 1
            opts.col_slot_rows = int(col_slot_rows)
        h = L.agcn_plan_ex(rp or None, ci or None, int(n), int(nnz), ctypes.byref(opts))
        if not h:
            _raise_last()
        self._h = h
        self.partition = partition
        st = self.stats()
        self.n, self.n_cols, self.nnz = st["n"], st["n_cols"], st["nnz"]
        self.x_rows = (opts.col_nparts * opts.col_slot_rows) if col_bounds is not None else self.n_cols

    @property
    def handle(self) -> int:
        if not self._h:
            raise ValueError("plan is closed")
        return self._h

    def stats(self) -> dict:
        st = _lib.Stats()
        _check(_lib.lib().agcn_plan_stats(self.handle, ctypes.byref(st)))
        return {k: getattr(st, k) for k, _ in _lib.Stats._fields_ if k != "reserved"}

    def copy(self, field: str) -> np.ndarray:
        st = self.stats()
        shapes = {"perm": (st["n"],), "blocks": (st["nblocks"], 4),
                  "sorted_colidx": (st["nnz"],), "row_src_off": (st["n"],),
                  "tasks": (st["ntasks"], 4), "sorted_rowptr": (st["n"] + 1,),
                  "hot_cols": (st["hot_rows"],)}
        dt = np.uint32 if field in ("blocks", "tasks") else np.int32
        out = np.zeros(shapes[field], dtype=dt)
        _check(_lib.lib().agcn_plan_copy(self.handle, FIELDS[field],
                                         out.ctypes.data or None, out.nbytes))
        return out

    def spmm(self, vals, X, out=None, stream=None, kernel: str = "auto", l2_hint=None,
             hot_mb: int | None = None, aggregation: str = "sum", self_x=None,
             self_scale: float = 0.0, bias=None, relu: bool = False, peer_out=(), chunk_shape: int = 0,
             chunk_order: int = 0):
        """Y = A.X (asynchronous on `stream`, default the current torch stream).

        kernel: "auto" | "general" | "looped" | "wide" (agcn_kernel_t).  l2_hint
        (agcn_l2_hint_t): None / "auto", "none", "keep_all" (evict_last on every X row),
        "hot_window" (the plan's hot rows in a compact buffer under a persisting L2 window),
        "hot_hints" (same buffer, evict_last / evict_first hints).  hot_mb: MiB of hot rows
        kept resident (None: the device's persisting-L2 maximum).
        Epilogue (agcn_spmm_opts_t): y_i = agg_i + self_scale * self_x[i] + bias, then ReLU if
        relu; aggregation "sum" (GCN) or "mean" (GraphSAGE-mean, / deg_i); GIN: self_x = X,
        self_scale = 1 + eps.
        """
        torch = _torch()
        F = X.shape[1] if X.dim() == 2 else 1
        if out is None:
            out = torch.empty((self.n, F), dtype=torch.float32, device=X.device)
        if X.dim() != 2 or X.shape[0] != self.x_rows:
            raise ValueError(f"X must be [{self.x_rows}, F], got {tuple(X.shape)}")
        if out.shape != (self.n, F):
            raise ValueError(f"out must be [{self.n}, {F}]")
        v = _dev_ptr(vals, "float32", "vals") if vals.numel() else 0
        x = _dev_ptr(X, "float32", "X") if X.numel() else 0
        y = _dev_ptr(out, "float32", "out") if out.numel() else 0
        opts = _spmm_opts(kernel, l2_hint, hot_mb, aggregation, self_x, self_scale, bias, relu,
                          shape=(self.n, F), peer_out=peer_out, chunk_shape=chunk_shape,
                          chunk_order=chunk_order)
        _check(_lib.lib().agcn_spmm_ex(self.handle, v or None, x or None, int(F), y or None,
                                       _stream_handle(stream), opts))
        return out

    def close(self):
        if getattr(self, "_h", None):
            _lib.lib().agcn_plan_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()


def _spmm_opts(kernel: str = "auto", l2_hint=None, hot_mb: int | None = None,
               aggregation: str = "sum", self_x=None, self_scale: float = 0.0, bias=None,
               relu: bool = False, shape=None, peer_out=(), chunk_shape: int = 0, chunk_order: int = 0):
    o = _lib.SpmmOpts()
    _lib.lib().agcn_default_spmm_opts(ctypes.byref(o))
    o.kernel = _lib.KERNELS[kernel]
    o.l2_hint = _lib.L2_HINTS[l2_hint] if l2_hint is None or isinstance(l2_hint, str) else int(l2_hint)
    o.hot_mb = 0 if hot_mb is None else int(hot_mb)
    o.chunk_shape = int(chunk_shape)
    o.chunk_order = int(chunk_order)
    o.aggregation = {"sum": 0, "mean": 1}[aggregation]
    o.relu = int(bool(relu))
    o.self_scale = float(self_scale)
    if self_x is not None:
        if shape is not None and tuple(self_x.shape) != tuple(shape):
            raise ValueError(f"self_x must be {tuple(shape)}, got {tuple(self_x.shape)}")
        o.self = _dev_ptr(self_x, "float32", "self_x")
    if bias is not None:
        if shape is not None and tuple(bias.shape) != (shape[1],):
            raise ValueError(f"bias must be [{shape[1]}]")
        o.bias = _dev_ptr(bias, "float32", "bias")
    if len(peer_out) > 8:
        raise ValueError("at most 8 peer_out pointers")
    for q, ptr in enumerate(peer_out):   # fused all-gather targets (device addresses)
        o.peer_out[q] = int(ptr)
    o.npeer = len(peer_out)
    return ctypes.byref(o)


# ---------------------------------------------------------------- C-ABI-named functions
def agcn_plan(rowptr, colidx, n: int, nnz: int) -> Plan:
    return Plan(rowptr, colidx, n, nnz)


def agcn_spmm(plan: Plan, vals, X, F: int, Y, stream=None) -> None:
    v = _dev_ptr(vals, "float32", "vals") if vals.numel() else 0
    x = _dev_ptr(X, "float32", "X") if X.numel() else 0
    y = _dev_ptr(Y, "float32", "Y") if Y.numel() else 0
    _check(_lib.lib().agcn_spmm(plan.handle, v or None, x or None, int(F), y or None,
                                _stream_handle(stream)))


def agcn_spmm_ex(plan: Plan, vals, X, F: int, Y, stream=None, kernel: str = "auto",
                 l2_hint=None, hot_mb: int | None = None) -> None:
    v = _dev_ptr(vals, "float32", "vals") if vals.numel() else 0
    x = _dev_ptr(X, "float32", "X") if X.numel() else 0
    y = _dev_ptr(Y, "float32", "Y") if Y.numel() else 0
    _check(_lib.lib().agcn_spmm_ex(plan.handle, v or None, x or None, int(F), y or None,
                                   _stream_handle(stream), _spmm_opts(kernel, l2_hint, hot_mb)))


def transpose(rowptr, colidx, n_cols: int, stream=None):
    """agcn_transpose: (rowptr_t, colidx_t, src) of A^T on the device (dX = A^T . dY).

    Row j of A^T lists the rows i with a_ij != 0 in increasing i; entry k of A^T is entry
    src[k] of A, so vals_t = gather_vals(vals, src).
    """
    torch = _torch()
    n = rowptr.numel() - 1
    nnz = int(rowptr[-1].item() - rowptr[0].item()) if n >= 0 else 0
    dev = rowptr.device
    rowptr_t = torch.empty(n_cols + 1, dtype=torch.int32, device=dev)
    colidx_t = torch.empty(nnz, dtype=torch.int32, device=dev)
    src = torch.empty(nnz, dtype=torch.int32, device=dev)
    _check(_lib.lib().agcn_transpose(_dev_ptr(rowptr, "int32", "rowptr"),
                                     _dev_ptr(colidx, "int32", "colidx") if colidx.numel() else None,
                                     n, int(n_cols), nnz, rowptr_t.data_ptr(),
                                     colidx_t.data_ptr() if nnz else None, src.data_ptr() if nnz else None,
                                     _stream_handle(stream)))
    return rowptr_t, colidx_t, src


def gather_vals(vals, src, out=None, stream=None):
    """agcn_gather_vals: out[k] = vals[src[k]] (values of A^T from those of A)."""
    torch = _torch()
    if out is None:
        out = torch.empty(src.numel(), dtype=torch.float32, device=src.device)
    if src.numel():
        _check(_lib.lib().agcn_gather_vals(_dev_ptr(vals, "float32", "vals"), _dev_ptr(src, "int32", "src"),
                                           src.numel(), _dev_ptr(out, "float32", "out"),
                                           _stream_handle(stream)))
    return out


def gemm_xw(X, Wt, bias=None, relu: bool = False, out=None, stream=None, precision: str = "tf32"):
    """agcn_gemm_xw_ex: Y = X . W (+ bias, ReLU) on the tcgen05 tensor cores.

    precision "tf32" (TF32 operands) or "fp32" (3xTF32 split operands, fp32 accuracy; CUDA-core
    FFMA for shapes whose split W does not fit in shared memory).
    X: [M, K] float32 CUDA; Wt: W transposed, [N, K] float32 CUDA (contiguous)."""
    torch = _torch()
    M, K = X.shape
    N = Wt.shape[0]
    if Wt.shape[1] != K:
        raise ValueError("Wt must be [N, K]")
    if out is None:
        out = torch.empty((M, N), dtype=torch.float32, device=X.device)
    b = _dev_ptr(bias, "float32", "bias") if bias is not None else None
    prec = {"fp32": 0, "tf32": 1}[precision]
    _check(_lib.lib().agcn_gemm_xw_ex(_dev_ptr(X, "float32", "X"), int(M), int(K), _dev_ptr(Wt, "float32", "Wt"),
                                      int(N), _dev_ptr(out, "float32", "out"), b, int(bool(relu)), prec,
                                      _stream_handle(stream)))
    return out


class DeviceBuffer:
    """A cudaMalloc'd fp32 [rows, cols] buffer from libagcn (agcn_device_alloc): exportable to
    other processes (agcn_ipc_export); ``.tensor`` views it as a torch CUDA tensor (zero copy,
    via __cuda_array_interface__)."""

    def __init__(self, rows: int, cols: int):
        torch = _torch()
        ptr = ctypes.c_void_p()
        _check(_lib.lib().agcn_device_alloc(max(1, rows * cols) * 4, ctypes.byref(ptr)))
        self.ptr = int(ptr.value)
        self.shape = (rows, cols)
        self.__cuda_array_interface__ = {"shape": self.shape, "typestr": "<f4", "data": (self.ptr, False),
                                         "version": 3, "strides": None}
        self.tensor = torch.as_tensor(self, device="cuda")

    def export(self) -> bytes:
        h = ctypes.create_string_buffer(64)
        _check(_lib.lib().agcn_ipc_export(self.ptr, h))
        return h.raw

    def close(self):
        if self.ptr:
            self.tensor = None
            _lib.lib().agcn_device_free(self.ptr)
            self.ptr = 0


def ipc_open(handle: bytes) -> int:
    """Map another process's DeviceBuffer (agcn_ipc_open); returns the device address."""
    ptr = ctypes.c_void_p()
    _check(_lib.lib().agcn_ipc_open(ctypes.create_string_buffer(handle, 64), ctypes.byref(ptr)))
    return int(ptr.value)


def ipc_close(ptr: int):
    _check(_lib.lib().agcn_ipc_close(ptr))


def auto_partition(n: int, nnz: int, sms: int = 0) -> tuple[int, int]:
    """agcn_auto_partition: the (max_block_warps, max_warp_nzs) a plan built with (0, 0) uses
    (host-only rule; sms <= 0 means the current device's SM count)."""
    mbw, mwn = ctypes.c_int32(0), ctypes.c_int32(0)
    _check(_lib.lib().agcn_auto_partition(int(n), int(nnz), int(sms), ctypes.byref(mbw), ctypes.byref(mwn)))
    return mbw.value, mwn.value


def shard_bounds(rowptr, nranks: int, stream=None) -> np.ndarray:
    """agcn_shard_bounds: nnz-balanced row shard bounds (int64 [nranks+1])."""
    rp = _dev_ptr(rowptr, "int32", "rowptr")
    out = np.zeros(nranks + 1, dtype=np.int64)
    _check(_lib.lib().agcn_shard_bounds(rp, rowptr.numel() - 1, int(nranks),
                                        out.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
                                        _stream_handle(stream)))
    return out


def _host_ptr(a, dtype):
    torch = _torch()
    if isinstance(a, torch.Tensor):
        if a.is_cuda:
            raise TypeError("propagate_host takes HOST buffers")
        if a.dtype != {np.int32: torch.int32, np.float32: torch.float32}[dtype]:
            raise TypeError("wrong dtype")
        if not a.is_contiguous():
            raise ValueError("must be contiguous")
        return a.data_ptr()
    if not (isinstance(a, np.ndarray) and a.dtype == dtype and a.flags.c_contiguous):
        raise TypeError(f"expected a contiguous {np.dtype(dtype).name} numpy array")
    return a.ctypes.data


def propagate_host(rowptr, colidx, vals, X, layers: int = 1, out=None, *, max_block_warps=12,
                   max_warp_nzs=32, partition="block", stream=None):
    """agcn_propagate_host: HOST buffers in, HOST result out (H2D, plan, layers x SpMM, D2H)."""
    n = (rowptr.shape[0] if hasattr(rowptr, "shape") else len(rowptr)) - 1
    nnz = int(rowptr[-1]) - int(rowptr[0])
    F = X.shape[1]
    if out is None:
        out = np.empty((n, F), dtype=np.float32)
    L = _lib.lib()
    opts = _lib.Opts()
    L.agcn_default_opts(ctypes.byref(opts))
    opts.max_block_warps, opts.max_warp_nzs = max_block_warps, max_warp_nzs
    opts.partition = {"block": 0, "warp": 1}[partition]
    opts.n_cols = X.shape[0]
    opts.stream = _stream_handle(stream) if stream is not None else 0
    _check(L.agcn_propagate_host(_host_ptr(rowptr, np.int32), _host_ptr(colidx, np.int32) or None,
                                 _host_ptr(vals, np.float32) or None, n, nnz,
                                 _host_ptr(X, np.float32), int(F), int(layers),
                                 _host_ptr(out, np.float32), ctypes.byref(opts)))
    return out


class Pipeline:
    """agcn_pipe_*: pipelined executor of propagate_host jobs (copy-in of job k overlaps the
    copy-out of job k-1 on the full-duplex PCIe link; results identical to propagate_host).

    submit() returns once the job's inputs are on the device and its plan is built; the host
    arrays of every submitted job are kept referenced here until wait() (the caller must not
    modify them, nor read `out`, before wait()).  Pinned host memory gives the overlap."""

    def __init__(self, depth: int = 2, *, n_cols: int = 0, max_block_warps=12, max_warp_nzs=32,
                 partition="block"):
        L = _lib.lib()
        opts = _lib.Opts()
        L.agcn_default_opts(ctypes.byref(opts))
        opts.max_block_warps, opts.max_warp_nzs = max_block_warps, max_warp_nzs
        opts.partition = {"block": 0, "warp": 1}[partition]
        opts.n_cols = int(n_cols)
        h = L.agcn_pipe_create(int(depth), ctypes.byref(opts))
        if not h:
            _raise_last()
        self._h = h
        self._keep = []

    def submit(self, rowptr, colidx, vals, X, layers: int = 1, out=None):
        n = (rowptr.shape[0] if hasattr(rowptr, "shape") else len(rowptr)) - 1
        nnz = int(rowptr[-1]) - int(rowptr[0])
        F = X.shape[1]
        if out is None:
            out = np.empty((n, F), dtype=np.float32)
        args = (rowptr, colidx, vals, X, out)
        _check(_lib.lib().agcn_pipe_submit(self._h, _host_ptr(rowptr, np.int32),
                                           _host_ptr(colidx, np.int32) or None,
                                           _host_ptr(vals, np.float32) or None, n, nnz,
                                           _host_ptr(X, np.float32), int(F), int(layers),
                                           _host_ptr(out, np.float32)))
        self._keep.append(args)
        return out

    def wait(self):
        _check(_lib.lib().agcn_pipe_wait(self._h))
        self._keep.clear()

    def close(self):
        if self._h:
            h, self._h = self._h, None
            _check(_lib.lib().agcn_pipe_destroy(h))
            self._keep.clear()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class GraphedPropagation:
    """agcn_graph_*: `layers` x agcn_spmm (Y_{l+1} = A.Y_l, Y_0 = X) captured once in a CUDA graph
    and replayed with one launch -- small graphs are bound by launch latency, not by the GPU.
    The graph reads `self.X` and `vals` at their captured addresses: write new features into
    `self.X` in place, then `replay()`.  layers > 1 needs a square A."""

    def __init__(self, rowptr, colidx, vals, X, layers: int = 2, **plan_kw):
        torch = _torch()
        self.X, self.vals, self.layers = X, vals, int(layers)
        self.plan = Plan(rowptr, colidx, **plan_kw)
        n, F = self.plan.stats()["n"], X.shape[1]
        self.bufs = [torch.empty((n, F), dtype=torch.float32, device=X.device)
                     for _ in range(min(self.layers, 2))]
        self.out = self.bufs[(self.layers - 1) % 2]
        h = _lib.lib().agcn_graph_create(self.plan.handle, _dev_ptr(vals, "float32", "vals") if vals.numel() else None,
                                         _dev_ptr(X, "float32", "X"), int(F), self.layers,
                                         self.bufs[0].data_ptr(),
                                         self.bufs[1].data_ptr() if len(self.bufs) > 1 else None)
        if not h:
            _raise_last()
        self._h = h

    def replay(self, stream=None):
        """One launch of the captured layers on `stream` (default: the current torch stream);
        returns the output buffer."""
        _check(_lib.lib().agcn_graph_launch(self._h, _stream_handle(stream)))
        return self.out

    def close(self):
        if getattr(self, "_h", None):
            h, self._h = self._h, None
            _check(_lib.lib().agcn_graph_destroy(h))
        if getattr(self, "plan", None) is not None:
            self.plan.close()
            self.plan = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
