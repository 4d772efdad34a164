"""Row-sharded multi-rank propagation with the CUDA kernels (gpu): two ranks on cuda:0 with
the gloo backend (the all-gather staged through the host: make_all_gather("gloo")), so the
whole multi-GPU code path -- shard bounds, per-rank plans over rowptr slices with the
padded-layout column relabel, SpMM into the rank's slot, in-place all-gather, next layer --
runs through libagcn.so on the one GPU a gpurun box has.  Each layer is checked against the
fp64 oracle fed the layer's actual fp32 input; and the bench's multi-rank
mode runs under torchrun.
"""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

import agcn_inputs as gen
import oracle

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, F, q, fused=False):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2308_11825_b200 as A
        from paper_2308_11825_b200.dist import ShardLayout, make_all_gather, propagate
        dev = torch.device("cuda:0")
        w = gen.make_config("c3")
        X = w.X(F)
        rp_d = torch.from_numpy(w.rowptr).to(dev)
        ci_d = torch.from_numpy(w.colidx).to(dev)
        va_d = torch.from_numpy(w.vals).to(dev)
        bounds = A.shard_bounds(rp_d, world)
        assert np.array_equal(bounds, oracle.shard_bounds(w.rowptr, world))
        lay = ShardLayout(bounds, rank)
        plan = A.Plan(rp_d[lay.lo:lay.hi + 1].contiguous(), ci_d, n_cols=w.n,
                      col_bounds=bounds, col_slot_rows=lay.slot_rows)
        X0 = torch.zeros((lay.padded_rows, F), dtype=torch.float32, device=dev)
        lay.pad(torch.from_numpy(X).to(dev), X0)
        bufs = [torch.empty_like(X0) for _ in range(2)]
        layers_out = []

        def spmm(Xin, out_rows):
            plan.spmm(va_d, Xin, out=out_rows)
            layers_out.append(Xin)

        if fused is True:   # the SpMM epilogue stores every row into all ranks' buffers (CUDA IPC)
            from paper_2308_11825_b200.dist import PeerBuffers, propagate_fused
            peers = PeerBuffers(lay, F)

            def spmm_f(Xin, out_rows, peer_out):
                plan.spmm(va_d, Xin, out=out_rows, peer_out=peer_out)
                layers_out.append(Xin)

            def barrier():
                torch.cuda.synchronize()
                dist.barrier()

            out = propagate_fused(lay, spmm_f, X0, peers, 2, barrier, final_gather=True)
        elif fused == "chunks":   # column chunks, all-gather of chunk k overlapping SpMM k+1
            from paper_2308_11825_b200.dist import (chunk_widths, join_columns, make_all_gather_async,
                                                    propagate_chunked, split_columns)
            widths = chunk_widths(F, 3)
            X0c = split_columns(X0, widths)
            bufs_c = [[torch.empty_like(c) for _ in range(2)] for c in X0c]
            seen = []

            def spmm_c(Xin, out_rows):
                plan.spmm(va_d, Xin, out=out_rows)
                seen.append(Xin)

            outc = propagate_chunked(lay, spmm_c, X0c, bufs_c, 2, make_all_gather_async("gloo"), final_gather=True)
            out = join_columns(outc)
            layers_out = [join_columns(seen[:3]), join_columns(seen[3:6])]
        else:
            out = propagate(lay, spmm, X0, bufs, 2, make_all_gather("gloo"), final_gather=True)
        torch.cuda.synchronize()
        if rank == 0:
            Y1 = lay.unpad(layers_out[1]).cpu().numpy()     # layer-2 input = layer-1 output
            Y2 = lay.unpad(out).cpu().numpy()
            r1 = oracle.spmm_check(w.rowptr, w.colidx, w.vals, X, Y1)
            r2 = oracle.spmm_check(w.rowptr, w.colidx, w.vals, Y1, Y2)
            q.put(("ok", r1["nfail"], r2["nfail"], r1["max_ratio"], r2["max_ratio"]))
        dist.barrier()
        if fused is True:
            peers.close()
        plan.close()
    except Exception as e:  # pragma: no cover
        q.put(("err", repr(e), 0, 0, 0))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,F,fused", [(2, 64, False), (3, 16, False), (2, 64, True), (3, 128, True),
                                           (2, 64, "chunks"), (3, 40, "chunks")])
def test_sharded_propagation_on_gpu(world, F, fused):
    """fused=True: the fused all-gather -- peer stores from the SpMM epilogue
    into IPC-mapped buffers of every rank instead of a collective.  fused="chunks": the
    column-chunked propagation (3 chunks; the all-gather of chunk k overlaps the SpMM of chunk
    k+1), every layer checked against the oracle."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, F, q, fused)) for r in range(world)]
    for p in procs:
        p.start()
    status, n1, n2, m1, m2 = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
    assert status == "ok", n1
    assert n1 == 0 and n2 == 0, (m1, m2)


@pytest.mark.parametrize("fused", [False, True, "chunks"])
def test_bench_multi_rank_mode(fused):
    """bench.py under torchrun, 2 ranks (gloo test mode on one GPU): one JSON line from rank 0."""
    port = _free_port()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "bench.py"),
           "--gpus", "2", "--steps", "2", "--warmup", "3", "--config", "c3", "--layers", "2", "--dist-backend", "gloo",
           "--e2e-steps", "1"] + (["--fused-allgather"] if fused is True else []) + \
          (["--overlap-chunks", "2"] if fused == "chunks" else [])
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["gpu_launches"] > 0
    assert (d["allgather_ms"] > 0 or fused == "chunks") and d["e2e"]["value"] > 0
