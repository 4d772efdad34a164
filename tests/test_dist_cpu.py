"""Multi-process (gloo, world_size 2 and 3, CPU) test of the row-sharded propagation host logic
in paper_2308_11825_b200/dist.py: nnz-balanced shard bounds, the padded slot layout, the
column relabel and the in-place all-gather between layers.  The per-shard SpMM is the CPU
oracle here (the CUDA kernel is covered by tests/test_gpu_parity.py on one GPU); the
sharded 2-layer result must equal the unsharded one bitwise (same per-row summation order).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import agcn_inputs as gen
import oracle
from paper_2308_11825_b200.dist import ShardLayout, propagate


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        w = gen.make_config("c2")
        F, layers = 16, 2
        X = w.X(F)
        bounds = oracle.shard_bounds(w.rowptr, world)
        lay = ShardLayout(bounds, rank)
        rp = w.rowptr[lay.lo:lay.hi + 1]
        ci_relabel = lay.relabel(w.colidx).astype(np.int32)   # the plan does this on device
        X0 = torch.zeros((lay.padded_rows, F))
        lay.pad(torch.from_numpy(X), X0)
        bufs = [torch.zeros_like(X0) for _ in range(2)]

        def spmm(Xin, out_rows):
            y, _ = oracle.spmm(rp, ci_relabel, w.vals, Xin.numpy(), with_abs=False)
            out_rows.copy_(torch.from_numpy(y.astype(np.float32)))

        ag = lambda full, slot: dist.all_gather_into_tensor(full, slot.clone())  # noqa: E731
        out = propagate(lay, spmm, X0, bufs, layers, ag, final_gather=True)
        Y = lay.unpad(out).numpy()
        # without the final all-gather (the bench's default): this rank's rows are the same
        own = lay.own_rows(propagate(lay, spmm, X0, [torch.zeros_like(X0) for _ in range(2)], layers, ag)).numpy()
        own_ok = bool(np.array_equal(own, Y[lay.lo:lay.hi]))
        if rank == 0:
            y1, _ = oracle.spmm(w.rowptr, w.colidx, w.vals, X, with_abs=False)
            y2, _ = oracle.spmm(w.rowptr, w.colidx, w.vals, y1.astype(np.float32), with_abs=False)
            q.put(("ok", bool(np.array_equal(Y, y2.astype(np.float32))) and own_ok,
                   int(lay.slot_rows), bounds.tolist()))
    except Exception as e:  # pragma: no cover
        q.put(("err", repr(e), 0, []))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_two_layer_propagation_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    status, ok, slot, bounds = q.get(timeout=240)
    for p in procs:
        p.join(timeout=120)
    assert status == "ok", ok
    assert ok
    w = gen.make_config("c2")
    nnz = w.nnz
    # nnz-balanced: every shard within one max-degree of nnz / P
    shard_nnz = [int(w.rowptr[bounds[i + 1]] - w.rowptr[bounds[i]]) for i in range(world)]
    assert max(abs(s - nnz / world) for s in shard_nnz) <= np.diff(w.rowptr).max() + 1
    assert slot == max(np.diff(bounds))


def test_layout_relabel_roundtrip():
    bounds = np.array([0, 3, 3, 10, 12], np.int64)       # includes an empty shard
    lay = ShardLayout(bounds, 2)
    assert lay.slot_rows == 7 and lay.padded_rows == 28 and (lay.lo, lay.hi) == (3, 10)
    j = np.arange(12)
    r = lay.relabel(j)
    X = np.arange(12 * 2, dtype=np.float32).reshape(12, 2)
    P = np.full((28, 2), -1, np.float32)
    lay.pad(X, P)
    assert np.array_equal(P[r], X)                        # relabelled rows read the same data
    assert np.array_equal(lay.unpad(P), X)


def _worker_chunked(rank, world, port, K, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2308_11825_b200.dist import (chunk_widths, join_columns, make_all_gather_async,
                                                propagate_chunked, split_columns)
        w = gen.make_config("c2")
        F, layers = 40, 3
        X = w.X(F)
        bounds = oracle.shard_bounds(w.rowptr, world)
        lay = ShardLayout(bounds, rank)
        rp = w.rowptr[lay.lo:lay.hi + 1]
        ci_relabel = lay.relabel(w.colidx).astype(np.int32)
        X0 = torch.zeros((lay.padded_rows, F))
        lay.pad(torch.from_numpy(X), X0)
        widths = chunk_widths(F, K)
        X0c = split_columns(X0, widths)
        bufs = [[torch.zeros_like(c) for _ in range(2)] for c in X0c]
        order = []

        def spmm(Xin, out_rows):
            order.append(Xin.shape[1])
            y, _ = oracle.spmm(rp, ci_relabel, w.vals, Xin.numpy(), with_abs=False)
            out_rows.copy_(torch.from_numpy(y.astype(np.float32)))

        ag = make_all_gather_async("gloo")
        out = propagate_chunked(lay, spmm, X0c, bufs, layers, ag, final_gather=True)
        Y = lay.unpad(join_columns(out)).numpy()
        if rank == 0:
            ref = X
            for _ in range(layers):
                ref = oracle.spmm(w.rowptr, w.colidx, w.vals, ref, with_abs=False)[0].astype(np.float32)
            q.put(("ok", bool(np.array_equal(Y, ref)), order == widths * layers, widths))
    except Exception as e:  # pragma: no cover
        q.put(("err", repr(e), False, []))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,K", [(2, 3), (3, 2)])
def test_chunked_overlapped_propagation_gloo(world, K):
    """the column-chunked propagation (all-gather of chunk k overlapping the SpMM of
    chunk k+1) equals the unsharded, unchunked 3-layer propagation bitwise (column-separable
    SpMM; per-element summation order unchanged) at world size 2 and 3."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_chunked, args=(r, world, port, K, q)) for r in range(world)]
    for p in procs:
        p.start()
    status, ok, order_ok, widths = q.get(timeout=240)
    for p in procs:
        p.join(timeout=120)
    assert status == "ok", ok
    assert ok and order_ok and sum(widths) == 40


def test_chunk_widths():
    from paper_2308_11825_b200.dist import chunk_widths
    for F in range(1, 300):
        for K in (1, 2, 3, 4, 7):
            if K > F:
                continue
            w = chunk_widths(F, K)
            assert len(w) == K and sum(w) == F and min(w) >= 1
            if F % (8 * K) == 0:
                assert all(x % 8 == 0 for x in w)
