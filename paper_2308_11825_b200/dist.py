"""Multi-GPU row sharding for stacked propagation layers (BASELINE.json north_star).

A is split into contiguous row shards with balanced nnz (agcn_shard_bounds); X is
replicated.  Rank p owns rows [b_p, b_{p+1}); its plan relabels columns into the padded
layout j -> q*S + (j - b_q) (q = owner of j, S = max shard rows), so one in-place
``all_gather_into_tensor`` of the S-row slots (NCCL over NVLink) IS the next layer's X.
No other collective is on the data path.

This module holds the host-side bookkeeping only; the SpMM is the C-ABI call.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass
class ShardLayout:
    bounds: np.ndarray   # int64 [P+1]
    rank: int

    @property
    def P(self) -> int:
        return int(self.bounds.size - 1)

    @property
    def slot_rows(self) -> int:
        """S = max shard rows (every rank's slot in the padded layout has S rows)."""
        return int(np.diff(self.bounds).max()) if self.P > 0 else 0

    @property
    def lo(self) -> int:
        return int(self.bounds[self.rank])

    @property
    def hi(self) -> int:
        return int(self.bounds[self.rank + 1])

    @property
    def rows(self) -> int:
        return self.hi - self.lo

    @property
    def padded_rows(self) -> int:
        return self.P * self.slot_rows

    def slot(self, buf, q: int | None = None):
        """Rows of rank q's slot in a padded [P*S, F] buffer (default: this rank)."""
        q = self.rank if q is None else q
        S = self.slot_rows
        return buf[q * S:(q + 1) * S]

    def own_rows(self, buf):
        """The rows this rank computes (first `rows` rows of its slot)."""
        return self.slot(buf)[:self.rows]

    def pad(self, X, out):
        """Copy a full [n, F] matrix into the padded layout `out` ([P*S, F])."""
        S = self.slot_rows
        for q in range(self.P):
            a, b = int(self.bounds[q]), int(self.bounds[q + 1])
            out[q * S:q * S + (b - a)] = X[a:b]
        return out

    def unpad(self, buf):
        """Padded [P*S, F] -> the [n, F] rows in original order (a copy)."""
        S = self.slot_rows
        parts = [buf[q * S:q * S + int(self.bounds[q + 1] - self.bounds[q])] for q in range(self.P)]
        if hasattr(buf, "new_empty"):  # torch
            import torch
            return torch.cat(parts, 0)
        return np.concatenate(parts, 0)

    def relabel(self, colidx: np.ndarray) -> np.ndarray:
        """Host reference of the plan's column relabel (the CUDA path does it on device)."""
        q = np.searchsorted(self.bounds, colidx, side="right") - 1
        return (q * self.slot_rows + (colidx - self.bounds[q])).astype(np.int64)


def propagate(layout: ShardLayout, spmm, X0, bufs, layers: int, all_gather=None, final_gather: bool = False):
    """Run `layers` propagation layers.

    spmm(Xin_padded, out_rows) computes this rank's rows of A.Xin into out_rows (a view of
    this rank's slot); all_gather(full_buf, slot_view) fills every slot (in place) BETWEEN
    layers (the next layer reads every rank's rows); the last layer's output stays row-sharded
    (each rank holds its own rows) unless final_gather.
    bufs: list of padded buffers to rotate through (>= 1, must not include X0).
    Returns the padded buffer holding the last layer's output.
    """
    cur = X0
    for layer in range(layers):
        nxt = bufs[layer % len(bufs)]
        spmm(cur, layout.own_rows(nxt))
        if all_gather is not None and layout.P > 1 and (layer < layers - 1 or final_gather):
            all_gather(nxt, layout.slot(nxt))
        cur = nxt
    return cur


def chunk_widths(F: int, K: int) -> list:
    """Column chunks of the overlapped propagation: K widths summing to F, multiples of 8 where
    possible (the WIDE kernel's 32-byte lanes), the earlier chunks never narrower."""
    if K < 1 or K > F:
        raise ValueError(f"need 1 <= K <= F, got K={K}, F={F}")
    q = F // K
    base = (q // 8) * 8 if q >= 8 else q
    widths = [base] * K
    rest = F - base * K
    i = 0
    while rest > 0:                        # hand out the remainder in steps of 8 (or 1)
        step = 8 if rest >= 8 and base >= 8 else 1
        widths[i % K] += step
        rest -= step
        i += 1
    return widths


def split_columns(X, widths):
    """[rows, F] -> K contiguous [rows, w_k] column blocks (the chunk-major layout)."""
    out, c = [], 0
    for wk in widths:
        out.append(X[:, c:c + wk].contiguous())
        c += wk
    return out


def join_columns(chunks):
    import torch
    return torch.cat(chunks, 1)


def propagate_chunked(layout: ShardLayout, spmm, X0_chunks, bufs_chunks, layers: int, all_gather_async=None,
                      final_gather: bool = False):
    """Column-chunked propagation with the all-gather of chunk k overlapping the SpMM of chunk
    k + 1.  The SpMM is column-separable -- (A X)[:, c] = A X[:, c] -- so every
    layer runs as K narrower SpMMs over contiguous chunk buffers ([P*S, w_k] each, the chunk-
    major layout), and a chunk's all-gather only has to finish before the NEXT layer's SpMM of
    the same chunk reads it:

        layer l:  SpMM_0  SpMM_1  SpMM_2 ...            (compute stream)
                        AG_0    AG_1    AG_2 ...        (communicator's stream, async)
        layer l+1: wait(AG_0) SpMM_0, wait(AG_1) SpMM_1, ...

    spmm(Xin_chunk, out_rows_chunk) as in ``propagate``; all_gather_async(full, slot) starts an
    in-place all-gather and returns a handle with .wait() (device-side ordering of the current
    stream after the collective, e.g. torch.distributed async work); None for one rank.
    bufs_chunks: per chunk a list of >= 1 padded buffers (not X0's).  The last layer's output
    stays row-sharded unless final_gather.  Returns the list of the last layer's chunk buffers;
    every pending all-gather has been waited for."""
    K = len(X0_chunks)
    cur = list(X0_chunks)
    pending = [None] * K
    for layer in range(layers):
        nxt = [bufs_chunks[k][layer % len(bufs_chunks[k])] for k in range(K)]
        for k in range(K):
            if pending[k] is not None:      # this chunk's input of the previous layer is complete
                pending[k].wait()
                pending[k] = None
            spmm(cur[k], layout.own_rows(nxt[k]))
            if all_gather_async is not None and layout.P > 1 and (layer < layers - 1 or final_gather):
                pending[k] = all_gather_async(nxt[k], layout.slot(nxt[k]))
        cur = nxt
    for k in range(K):
        if pending[k] is not None:
            pending[k].wait()
    return cur


def make_all_gather_async(backend: str):
    """all_gather_async(full, slot) -> handle with .wait(): nccl: torch.distributed async work
    (runs on the communicator's stream; .wait() orders the current stream after it, no host
    block); gloo (test mode): the host-staged all-gather, done before returning."""
    import torch.distributed as dist

    if backend == "nccl":
        return lambda full, slot: dist.all_gather_into_tensor(full, slot, async_op=True)
    sync = make_all_gather("gloo")

    class _Done:
        def wait(self):
            pass

    def ag(full, slot):
        sync(full, slot)
        return _Done()

    return ag


def make_all_gather(backend: str):
    """In-place all-gather of the S-row slots of a padded [P*S, F] buffer.

    nccl: one ``all_gather_into_tensor`` on the device buffer (NVLink / NVSwitch).
    gloo: the same collective staged through host memory -- only for testing the multi-rank
    path with several ranks on one GPU (gloo has no device all-gather).
    """
    import torch.distributed as dist

    if backend == "nccl":
        return lambda full, slot: dist.all_gather_into_tensor(full, slot)

    def gloo_all_gather(full, slot):
        h_full = full.cpu()
        n = slot.shape[0]
        rank = dist.get_rank()
        dist.all_gather_into_tensor(h_full, h_full[rank * n:(rank + 1) * n].clone())
        full.copy_(h_full)

    return gloo_all_gather


class PeerBuffers:
    """Fused all-gather: ``n_bufs`` padded [P*S, F] next-layer X buffers per rank,
    allocated by libagcn (DeviceBuffer) and mapped into every other rank (CUDA IPC).  The SpMM of
    rank p stores each finished output row into its own slot AND into slot p of every peer's
    buffer (agcn_spmm_opts_t.peer_out: NVLink peer stores from the kernel's epilogue), so no
    separate collective runs between layers -- only a barrier."""

    def __init__(self, layout: ShardLayout, F: int, n_bufs: int = 2):
        import torch.distributed as dist

        from . import DeviceBuffer, ipc_open
        self.layout, self.F = layout, F
        self.local = [DeviceBuffer(layout.padded_rows, F) for _ in range(n_bufs)]
        handles = [b.export() for b in self.local]
        everyone = [None] * layout.P
        dist.all_gather_object(everyone, handles)
        self.mapped = []       # mapped[b][q]: device address of rank q's buffer b (0 = own)
        for b in range(n_bufs):
            self.mapped.append([0 if q == layout.rank else ipc_open(everyone[q][b]) for q in range(layout.P)])
        dist.barrier()

    def tensor(self, b: int):
        return self.local[b].tensor

    def peer_out(self, b: int):
        """Addresses of this rank's slot in every peer's buffer b."""
        off = self.layout.rank * self.layout.slot_rows * self.F * 4
        return [self.mapped[b][q] + off for q in range(self.layout.P) if q != self.layout.rank]

    def close(self):
        from . import ipc_close
        for row in self.mapped:
            for q, ptr in enumerate(row):
                if ptr:
                    ipc_close(ptr)
        for b in self.local:
            b.close()


def propagate_fused(layout: ShardLayout, spmm, X0, peers: PeerBuffers, layers: int, barrier,
                    final_gather: bool = False):
    """``layers`` propagation layers with the fused all-gather: spmm(Xin, out_rows, peer_out)
    writes this rank's rows locally and into every peer (not for the last layer unless
    final_gather: its output stays row-sharded); ``barrier()`` orders the peers' stores before
    the next layer reads them.  Returns the padded buffer of the last layer."""
    cur = X0
    nb = len(peers.local)
    for layer in range(layers):
        nxt = peers.tensor(layer % nb)
        last = layer == layers - 1 and not final_gather
        spmm(cur, layout.own_rows(nxt), [] if last else peers.peer_out(layer % nb))
        if not last:
            barrier()
        cur = nxt
    return cur
