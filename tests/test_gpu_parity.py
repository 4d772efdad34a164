"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle.

Integer metadata (degree order, sorted CSR, descriptors, warp tasks, shard bounds) must be
bit-exact.  fp32 output must satisfy |y - y_ref| <= 1e-5 * sum|a x| + 1e-7 per element
(BASELINE.json north_star), checked by oracle.spmm_check.
"""
import json
import os

import numpy as np
import pytest

import agcn_inputs as gen
import oracle

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2308_11825_b200 as A  # noqa: E402

GOLD = os.path.join(os.path.dirname(__file__), "golden")
DEV = torch.device("cuda:0")


def cu(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(DEV)


def make_plan(rowptr, colidx, **kw):
    return A.Plan(cu(rowptr.astype(np.int32)), cu(colidx.astype(np.int32)), **kw)


def check_plan_vs_oracle(rowptr, colidx, mbw=12, mwn=32, n_cols=None, **kw):
    p = make_plan(rowptr, colidx, max_block_warps=mbw, max_warp_nzs=mwn, n_cols=n_cols, **kw)
    o = oracle.plan(rowptr, colidx, mbw, mwn)
    assert np.array_equal(p.copy("perm"), o["perm"])
    assert np.array_equal(p.copy("sorted_rowptr"), o["sorted_rowptr"])
    assert np.array_equal(p.copy("row_src_off"), o["row_src_off"])
    assert np.array_equal(p.copy("sorted_colidx"), o["sorted_colidx"])
    assert np.array_equal(p.copy("blocks"), o["blocks"])
    st = p.stats()
    assert st["nblocks"] == o["blocks"].shape[0]
    assert st["n_zero_rows"] == int((o["sorted_deg"] == 0).sum())
    assert st["n_oversized_rows"] == int((o["sorted_deg"] > mbw * mwn).sum())
    return p


def check_spmm(p, rowptr, colidx, vals, X, Y=None, kernel="auto"):
    if Y is None:
        Y = p.spmm(cu(vals), cu(X), kernel=kernel).cpu().numpy()
    r = oracle.spmm_check(rowptr, colidx, vals, X, Y)
    assert r["nfail"] == 0, r
    return Y


# ---------------------------------------------------------------- metadata
def test_fig3_golden_on_gpu():
    g = json.load(open(os.path.join(GOLD, "fig3.json")))
    rowptr, colidx = np.array(g["rowptr"], np.int32), np.array(g["colidx"], np.int32)
    p = make_plan(rowptr, colidx, max_block_warps=2, max_warp_nzs=2, n_cols=g["n_cols"])
    assert p.copy("perm").tolist() == g["perm"]
    assert p.copy("blocks").tolist() == g["blocks"]
    w = make_plan(rowptr, colidx, max_block_warps=2, max_warp_nzs=2, n_cols=4, partition="warp")
    t = w.copy("tasks")
    assert t.shape[0] == g["n_warp_tasks"] and t[0].tolist() == g["warp_tasks_first"]


@pytest.mark.parametrize("name", ["c1", "c2", "c3"])
def test_metadata_bit_exact_configs(name):
    w = gen.make_config(name)
    check_plan_vs_oracle(w.rowptr, w.colidx)


@pytest.mark.parametrize("seed", range(300))
def test_metadata_bit_exact_random(seed):
    rng = np.random.default_rng(seed)
    mbw, mwn = [(1, 1), (2, 2), (12, 32), (16, 64), (3, 5), (12, 1), (4, 7)][seed % 7]
    n = int(rng.integers(1, 3000))
    nc = int(rng.integers(1, 3000))
    rowptr, colidx = gen.random_csr(n, nc, seed, max_deg=int(rng.choice([8, 100, 1500, 2500])),
                                    dup=bool(seed % 2))
    check_plan_vs_oracle(rowptr, colidx, mbw, mwn, n_cols=nc)


def _plan_fields(p):
    return {f: p.copy(f) for f in ("perm", "sorted_rowptr", "row_src_off", "blocks", "sorted_colidx")}, p.stats()


@pytest.mark.parametrize("seed", range(24))
def test_small_plan_equals_general_plan(seed):
    """The one-CTA plan (graphs of <= 32768 rows) and the general multi-kernel plan give
    identical metadata (both are also checked against the oracle), incl. the fallback when a
    small graph has more than 1024 oversized rows."""
    rng = np.random.default_rng(1000 + seed)
    mbw, mwn = [(12, 32), (2, 2), (1, 1), (4, 16), (8, 16), (3, 5)][seed % 6]
    if seed % 8 == 7:          # > 1024 oversized rows: the small path falls back
        degs = np.concatenate([np.full(1500, mbw * mwn + 1), rng.integers(0, 5, 300)])
        rowptr, colidx = _rows_csr(rng.permutation(degs), 500, seed)
        nc = 500
    else:
        n, nc = int(rng.integers(1, 32768)), int(rng.integers(1, 5000))
        rowptr, colidx = gen.random_csr(n, nc, seed, max_deg=int(rng.choice([4, 60, 700])),
                                        dup=bool(seed % 2))
    got = {}
    for small in (True, False):
        p = check_plan_vs_oracle(rowptr, colidx, mbw, mwn, n_cols=nc, small_plan=small)
        got[small] = _plan_fields(p)
    for f in got[True][0]:
        assert np.array_equal(got[True][0][f], got[False][0][f]), f
    s1, s0 = got[True][1], got[False][1]
    for k in ("nblocks", "n_zero_rows", "n_oversized_rows", "n_oversized_blocks", "max_deg", "deg_bound"):
        assert s1[k] == s0[k], k


def _rows_csr(degs, n_cols, seed=0):
    rng = np.random.default_rng(seed)
    rowptr = np.concatenate([[0], np.cumsum(degs)]).astype(np.int32)
    colidx = rng.integers(0, n_cols, size=int(rowptr[-1])).astype(np.int32)
    return rowptr, colidx


@pytest.mark.parametrize("n", [1, 4095, 4096, 4097, 32 * 4096, 33 * 4096 + 1, 300001])
def test_scan_tile_boundaries(n):
    """The plan's single-pass look-back scans (bucket table, sorted rowptr fused with
    row_src_off, chunk starts) at lengths around the 4096-element tile and beyond the 32-tile
    look-back window: metadata bit-exact against the oracle on the general plan."""
    rng = np.random.default_rng(n)
    degs = rng.integers(0, 6, n)
    degs[rng.integers(0, n, 3)] = [900, 400, 5000]
    rowptr, colidx = _rows_csr(degs, 777, n)
    check_plan_vs_oracle(rowptr, colidx, n_cols=777, small_plan=False)


@pytest.mark.parametrize("degs", [
    [384], [383], [385], [768], [769], [384 * 5, 1, 0, 384 * 5 + 7],   # around deg_bound
    [0, 0, 0], [0], [70000, 3, 0, 65536, 65537],                        # zero rows, deg >= 2^16
    [1] * 5000 + [2] * 3000 + [33] * 100,                               # many full blocks
])
def test_metadata_edge_cases(degs):
    rowptr, colidx = _rows_csr(np.array(degs), 1000)
    p = check_plan_vs_oracle(rowptr, colidx, n_cols=1000)
    vals = gen.uniform_f32(3, colidx.size)
    X = gen.uniform_f32(4, (1000, 64))
    check_spmm(p, rowptr, colidx, vals, X)


@pytest.mark.parametrize("F", [37, 132, 1040])
def test_oversized_merge_shapes(F):
    """The level-3 merge of oversized rows at column counts that need several passes: rows of
    few chunks (one warp each) and rows of more than 16 chunks (one CTA each), F/4 or F
    vector columns above 32 and above 256."""
    rowptr, colidx = _rows_csr(np.array([5, 9, 40, 3, 200, 0, 17, 64, 1]), 300, F)
    rng = np.random.default_rng(F)
    vals = rng.uniform(-1, 1, colidx.size).astype(np.float32)
    X = rng.uniform(-1, 1, (300, F)).astype(np.float32)
    for mbw, mwn in [(2, 2), (1, 1), (12, 32)]:
        p = make_plan(rowptr, colidx, max_block_warps=mbw, max_warp_nzs=mwn, n_cols=300)
        check_spmm(p, rowptr, colidx, vals, X)


@pytest.mark.parametrize("name", ["c1", "c2", "c3"])
def test_auto_partition_plans(name):
    """max_block_warps = max_warp_nzs = 0: the plan takes agcn_auto_partition's parameters,
    reports them in its stats, and its metadata and SpMM match the oracle at those values."""
    w = gen.make_config(name, vals_kind="uniform")
    p = make_plan(w.rowptr, w.colidx, max_block_warps=0, max_warp_nzs=0)
    st = p.stats()
    mbw, mwn = A.auto_partition(w.n, w.rowptr[-1])
    assert (st["max_block_warps"], st["max_warp_nzs"]) == (mbw, mwn)
    check_plan_vs_oracle(w.rowptr, w.colidx, mbw, mwn)
    for F in (16, 64, 128):
        check_spmm(p, w.rowptr, w.colidx, w.vals, w.X(F))


def test_empty_plans():
    for rowptr in (np.zeros(1, np.int32), np.zeros(5, np.int32)):
        p = make_plan(rowptr, np.zeros(0, np.int32), n_cols=3)
        assert p.stats()["nblocks"] == 0
        Y = p.spmm(cu(np.zeros(0, np.float32)), cu(np.ones((3, 8), np.float32))).cpu().numpy()
        assert Y.shape == (rowptr.size - 1, 8) and not Y.any()


def test_warp_tasks_bit_exact():
    for seed in range(10):
        rowptr, colidx = gen.random_csr(2000, 500, seed, max_deg=300)
        for mwn in (1, 2, 32):
            p = make_plan(rowptr, colidx, partition="warp", max_warp_nzs=mwn, n_cols=500)
            assert np.array_equal(p.copy("tasks"), oracle.warp_partition(rowptr, mwn))


# ---------------------------------------------------------------- SpMM parity
def test_spmm_c2_F_sweep():
    """Pubmed-shaped graph over a sweep of F (F = 1..128 on C1/C2)."""
    w = gen.make_config("c2", vals_kind="uniform")
    p = make_plan(w.rowptr, w.colidx)
    for F in list(range(1, 129, 7)) + [64, 128]:
        check_spmm(p, w.rowptr, w.colidx, w.vals, w.X(F))


def test_spmm_c1_all_F():
    w = gen.make_config("c1")
    p = make_plan(w.rowptr, w.colidx)
    for F in range(1, 129):
        X = w.X(F)
        check_spmm(p, w.rowptr, w.colidx, w.vals, X)


@pytest.mark.parametrize("F", [16, 32, 64, 128, 96, 100, 3, 256, 520])
def test_spmm_c2_F(F):
    w = gen.make_config("c2", vals_kind="uniform")
    p = make_plan(w.rowptr, w.colidx)
    check_spmm(p, w.rowptr, w.colidx, w.vals, w.X(F))


KERNEL_F = [("general", F) for F in (3, 4, 16, 64, 128, 100)] + \
    [("looped", F) for F in (1, 16, 33, 64, 100, 128)] + \
    [("wide", F) for F in (8, 16, 24, 32, 40, 64, 96, 128, 200, 248, 256)]


@pytest.mark.parametrize("kernel,F", KERNEL_F)
def test_spmm_every_kernel(kernel, F):
    """Every SpMM kernel variant (agcn_spmm_opts_t.kernel) against the oracle."""
    w = gen.make_config("c2", vals_kind="uniform")
    p = make_plan(w.rowptr, w.colidx)
    check_spmm(p, w.rowptr, w.colidx, w.vals, w.X(F), kernel=kernel)
    rowptr, colidx = _rows_csr(np.array([0, 1, 2, 3, 5, 31, 33, 64, 97, 130, 200, 383, 384, 385, 768,
                                         769, 2000, 0, 7]), 500, 11)
    rng = np.random.default_rng(F)
    vals = rng.uniform(-1, 1, colidx.size).astype(np.float32)
    X = rng.uniform(-1, 1, (500, F)).astype(np.float32)
    for mbw, mwn in [(12, 32), (2, 2), (1, 1), (32, 8), (5, 7)]:
        p = make_plan(rowptr, colidx, max_block_warps=mbw, max_warp_nzs=mwn, n_cols=500)
        check_spmm(p, rowptr, colidx, vals, X, kernel=kernel)


def _hub_graph(n, seed, F):
    """Square power-law CSR with hubs (rows of degree > deg_bound), X and vals."""
    rng = np.random.default_rng(seed)
    degs = np.minimum(rng.zipf(1.4, size=n) - 1, 3 * n).astype(np.int64)
    degs[rng.random(n) < 0.3] = 0
    degs[rng.integers(0, n, 3)] = [2000, 900, 385]
    rowptr = np.zeros(n + 1, dtype=np.int32)
    rowptr[1:] = np.cumsum(degs)
    w = 1.0 / np.arange(1, n + 1) ** 0.8
    w = w[rng.permutation(n)]
    colidx = rng.choice(n, size=int(rowptr[-1]), p=w / w.sum()).astype(np.int32)
    vals = rng.uniform(-1, 1, colidx.size).astype(np.float32)
    X = rng.uniform(-1, 1, (n, F)).astype(np.float32)
    return rowptr, colidx, vals, X


@pytest.mark.parametrize("F", [8, 40, 64, 128, 256, 100, 3])
def test_hot_rows_every_mode(F):
    """Hot X rows (agcn_opts_t.hot_rows): the plan re-encodes the columns of its hot vertices
    (tail of the degree order) and agcn_spmm reads them from a compact gathered buffer.  Every
    hot count x L2 mode x kernel gives the oracle's result, bitwise equal to the plan without
    hot rows (the summation order does not change); the sorted colidx copy decodes exactly."""
    rowptr, colidx, vals, X = _hub_graph(3000, F, F)
    o = oracle.plan(rowptr, colidx, 12, 32)
    ref = make_plan(rowptr, colidx, hot_rows=0)
    assert ref.stats()["hot_rows"] == 0
    Y0 = check_spmm(ref, rowptr, colidx, vals, X)
    kernels = ["auto", "general"] + (["wide"] if F % 8 == 0 else [])
    for H in (1, 17, 500, 10 ** 9):
        p = make_plan(rowptr, colidx, hot_rows=H)
        live = int((np.diff(rowptr) > 0).sum())
        assert p.stats()["hot_rows"] == min(H, live)
        assert np.array_equal(p.copy("sorted_colidx"), o["sorted_colidx"])
        assert np.array_equal(p.copy("blocks"), o["blocks"])
        for kernel in kernels:
            for l2 in ("auto", "none", "keep_all", "hot_window", "hot_hints"):
                for hot_mb in (None, 1):
                    Y = p.spmm(cu(vals), cu(X), kernel=kernel, l2_hint=l2, hot_mb=hot_mb).cpu().numpy()
                    if kernel == "general":
                        check_spmm(p, rowptr, colidx, vals, X, Y)
                    else:
                        assert np.array_equal(Y, Y0), (H, kernel, l2, hot_mb)


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_hot_set_is_the_degree_tail(seed):
    """The hot set (agcn_opts_t.hot_rows, reading Q35) is exactly the tail of the oracle's
    stable degree order (the H largest (degree, row) keys), on both plan paths and for every H,
    including H among the oversized rows and ties inside a degree bucket.  Metadata, the decoded
    colidx copy and the SpMM are bitwise the same for every H."""
    rowptr, colidx, vals, X = _hub_graph(5000 + 777 * seed, 30 + seed, 64)
    n = rowptr.size - 1
    deg = np.diff(rowptr)
    live = int((deg > 0).sum())
    o = oracle.plan(rowptr, colidx, 4, 8)                  # deg_bound 32: many oversized rows
    n_ov = int((deg > 32).sum())
    assert 1 < n_ov < live
    Y0 = None
    for H in (1, n_ov - 1, n_ov, n_ov + 1, n_ov + 37, live - 1, live, 10 ** 9):
        want = np.sort(o["perm"][n - min(H, live):])
        for small in (True, False):
            p = make_plan(rowptr, colidx, max_block_warps=4, max_warp_nzs=8, hot_rows=H, small_plan=small)
            assert p.stats()["hot_rows"] == min(H, live)
            assert np.array_equal(p.copy("hot_cols"), want), (H, small)
            assert np.array_equal(p.copy("perm"), o["perm"])
            assert np.array_equal(p.copy("blocks"), o["blocks"])
            assert np.array_equal(p.copy("sorted_colidx"), o["sorted_colidx"])
            Y = p.spmm(cu(vals), cu(X)).cpu().numpy()
            if Y0 is None:
                Y0 = check_spmm(p, rowptr, colidx, vals, X, Y)
            assert np.array_equal(Y, Y0), (H, small)


@pytest.mark.parametrize("partition,small", [("block", False), ("block", True), ("warp", False)])
def test_plan_does_not_read_caller_arrays_after_return(partition, small):
    """agcn_plan returns while its last kernels still run (the general block plan waits for
    events, not the stream); none of them may read the caller's rowptr / colidx.  The caller's
    arrays are overwritten on another stream right after the call, without any ordering: the
    plan's metadata and SpMM must still match the oracle."""
    w = gen.make_config("c3", vals_kind="uniform")
    o = oracle.plan(w.rowptr, w.colidx, 12, 32)
    other = torch.cuda.Stream()
    for rep in range(3):
        rp, ci = cu(w.rowptr), cu(w.colidx)
        torch.cuda.synchronize()
        p = A.Plan(rp, ci, hot_rows=20000, small_plan=small, partition=partition)
        with torch.cuda.stream(other):
            ci.fill_(-7)
            rp.fill_(3)
        torch.cuda.synchronize()
        if partition == "block":
            assert np.array_equal(p.copy("perm"), o["perm"])
            assert np.array_equal(p.copy("blocks"), o["blocks"])
            assert np.array_equal(p.copy("sorted_colidx"), o["sorted_colidx"])
            assert np.array_equal(p.copy("hot_cols"), np.sort(o["perm"][w.n - p.stats()["hot_rows"]:]))
        check_spmm(p, w.rowptr, w.colidx, w.vals, w.X())


@pytest.mark.parametrize("F", [32, 64, 128, 256, 40])
def test_chunk_kernel_writes_zero_rows(F):
    """Plans with more than 16384 oversized chunks run them in k_spmm_chunks, which also writes
    the degree-0 rows (one batch of 32 after every chunk, the rest after its last chunk):
    bitwise the same Y as the single-kernel path (chunk_shape -1), every row checked against
    the oracle, zero rows exactly 0."""
    rng = np.random.default_rng(F)
    n = 70000
    degs = np.zeros(n, np.int64)
    live = rng.permutation(n)[:30000]
    degs[live[:12000]] = rng.integers(5, 9, 12000)      # deg_bound 4: 2 chunks each -> > 16384 chunks
    degs[live[12000:]] = rng.integers(1, 5, 18000)
    rowptr, colidx = _rows_csr(degs, n, F)
    vals = rng.uniform(-1, 1, colidx.size).astype(np.float32)
    X = rng.uniform(-1, 1, (n, F)).astype(np.float32)
    p = make_plan(rowptr, colidx, max_block_warps=1, max_warp_nzs=4, small_plan=False)
    assert p.stats()["n_oversized_blocks"] > 16384
    Y = p.spmm(cu(vals), cu(X)).cpu().numpy()
    Y1 = p.spmm(cu(vals), cu(X), chunk_shape=-1).cpu().numpy()
    assert np.array_equal(Y, Y1)
    assert not Y[degs == 0].any()
    check_spmm(p, rowptr, colidx, vals, X, Y)


def test_hot_rows_auto_rule():
    """hot_rows = -1: on for square graphs with n >= 2^19, off otherwise and for padded layouts."""
    rowptr = np.zeros(2 ** 19 + 1, dtype=np.int32)
    rowptr[1:] = np.arange(1, 2 ** 19 + 1)
    colidx = (np.arange(2 ** 19, dtype=np.int64) * 7919 % 2 ** 19).astype(np.int32)
    p = make_plan(rowptr, colidx)
    assert p.stats()["hot_rows"] == 2 ** 19
    p2 = make_plan(rowptr, colidx, n_cols=2 ** 19 + 5)
    assert p2.stats()["hot_rows"] == 0
    vals = np.ones(colidx.size, np.float32)
    X = np.random.default_rng(0).uniform(-1, 1, (2 ** 19, 8)).astype(np.float32)
    Y = p.spmm(cu(vals), cu(X)).cpu().numpy()
    assert np.array_equal(Y, X[colidx])


def test_plan_copies_colidx():
    """the caller may free or change rowptr / colidx after agcn_plan returns."""
    w = gen.make_config("c2", vals_kind="uniform")
    X = w.X(64)
    for part in ("block", "warp"):
        rp, ci = cu(w.rowptr), cu(w.colidx)
        p = A.Plan(rp, ci, partition=part)
        ci.fill_(-7)
        rp.fill_(0)
        del rp, ci
        torch.cuda.empty_cache()
        check_spmm(p, w.rowptr, w.colidx, w.vals, X)


def test_spmm_kernel_unsupported_is_reported():
    w = gen.make_config("c1")
    p = make_plan(w.rowptr, w.colidx)
    with pytest.raises(A.AgcnError) as e:
        p.spmm(cu(w.vals), cu(w.X(100)), kernel="wide")
    assert e.value.status == "AGCN_ERR_UNSUPPORTED"
    with pytest.raises(A.AgcnError):
        p.spmm(cu(w.vals), cu(w.X(64)), kernel="wide", l2_hint=7)


def test_wide_kernel_nonfinite_x_rows_not_referenced():
    """Rows of X that A never references may hold inf/nan: they must not leak into Y."""
    rowptr = np.array([0, 3, 3, 8], dtype=np.int32)
    colidx = np.array([1, 2, 3, 1, 2, 3, 4, 5], dtype=np.int32)
    vals = np.ones(8, dtype=np.float32)
    X = np.ones((7, 64), dtype=np.float32)
    X[0] = np.inf
    X[6] = np.nan
    for kernel in ("auto", "general", "looped", "wide"):
        p = make_plan(rowptr, colidx, n_cols=7)
        Y = p.spmm(cu(vals), cu(X), kernel=kernel).cpu().numpy()
        assert np.isfinite(Y).all(), kernel
        check_spmm(p, rowptr, colidx, vals, X, Y)


def test_spmm_c3_both_partitions():
    w = gen.make_config("c3")
    X = w.X()
    Yb = check_spmm(make_plan(w.rowptr, w.colidx), w.rowptr, w.colidx, w.vals, X)
    Yw = check_spmm(make_plan(w.rowptr, w.colidx, partition="warp"), w.rowptr, w.colidx, w.vals, X)
    assert Yb.shape == Yw.shape


@pytest.mark.parametrize("seed", range(40))
def test_spmm_random(seed):
    rng = np.random.default_rng(100 + seed)
    mbw, mwn = [(12, 32), (2, 2), (1, 1), (16, 64), (3, 5), (6, 8)][seed % 6]
    n, nc = int(rng.integers(1, 1500)), int(rng.integers(1, 1500))
    F = int(rng.choice([1, 2, 4, 7, 16, 24, 33, 64, 96, 128, 200]))
    rowptr, colidx = gen.random_csr(n, nc, seed, max_deg=int(rng.choice([10, 400, 1400])),
                                    dup=bool(seed % 3 == 0))
    vals = rng.uniform(-1, 1, colidx.size).astype(np.float32)
    X = rng.uniform(-1, 1, (nc, F)).astype(np.float32)
    part = "warp" if seed % 4 == 3 else "block"
    p = make_plan(rowptr, colidx, max_block_warps=mbw, max_warp_nzs=mwn, n_cols=nc, partition=part)
    check_spmm(p, rowptr, colidx, vals, X)


@pytest.mark.parametrize("F", [64, 40, 96, 200])
def test_spmm_integer_exact_and_deterministic(F):
    rng = np.random.default_rng(5)
    rowptr, colidx = _rows_csr(np.array([0, 1, 5, 40, 384, 385, 2000, 3, 900]), 300, 5)
    vals = rng.integers(-4, 5, colidx.size).astype(np.float32)
    X = rng.integers(-4, 5, (300, F)).astype(np.float32)
    p = make_plan(rowptr, colidx, n_cols=300)
    Y1 = p.spmm(cu(vals), cu(X)).cpu().numpy()
    Y2 = p.spmm(cu(vals), cu(X)).cpu().numpy()
    y, _ = oracle.spmm(rowptr, colidx, vals, X)
    assert np.array_equal(Y1.astype(np.float64), y)    # exact: |partial sums| < 2^24
    assert np.array_equal(Y1, Y2)                      # deterministic order, bitwise


def test_spmm_unaligned_scalar_path():
    w = gen.make_config("c1")
    p = make_plan(w.rowptr, w.colidx)
    Xbig = cu(w.X(65))
    X = Xbig[:, 1:]                                    # stride 65: not contiguous -> copy
    Xs = torch.empty(w.n * 64 + 1, device=DEV)[1:].view(w.n, 64)   # 4-byte offset
    Xs.copy_(X)
    out = torch.empty(w.n * 64 + 1, device=DEV)[1:].view(w.n, 64)
    p.spmm(cu(w.vals), Xs, out=out)
    check_spmm(p, w.rowptr, w.colidx, w.vals, Xs.cpu().numpy(), out.cpu().numpy())


# ---------------------------------------------------------------- full BASELINE sizes (sampled)
def _sample_rows(rowptr, k, seed):
    deg = np.diff(rowptr)
    rng = np.random.default_rng(seed)
    top = np.argsort(deg, kind="stable")[-16:]
    zero = np.flatnonzero(deg == 0)[:8]
    rnd = rng.choice(deg.size, size=min(k, deg.size), replace=False)
    return np.unique(np.concatenate([top, zero, rnd])).astype(np.int64)


@pytest.mark.parametrize("name", ["c4", "c5"])
def test_full_size_every_row(name):
    """BASELINE configs C4 and C5 at full size: metadata bit-exact, and EVERY output row of every
    layer within the north_star tolerance of the fp64 oracle (streaming check),
    through the default path (C5: hot rows on); the plan without hot rows gives bitwise the same Y."""
    w = gen.make_config(name)
    rp, ci, va = cu(w.rowptr), cu(w.colidx), cu(w.vals)
    p = A.Plan(rp, ci, max_block_warps=0, max_warp_nzs=0)   # the bench's (auto) Alg. 1 parameters
    st = p.stats()
    o = oracle.plan(w.rowptr, w.colidx, st["max_block_warps"], st["max_warp_nzs"])  # bit-exact at full size
    for field in ("perm", "sorted_rowptr", "row_src_off", "blocks", "sorted_colidx"):
        assert np.array_equal(p.copy(field), o[field]), field
    del o
    X = w.X()
    Xd = cu(X)
    Y = p.spmm(va, Xd)
    Yh = Y.cpu().numpy()
    r = oracle.spmm_check(w.rowptr, w.colidx, w.vals, X, Yh)
    assert r["nfail"] == 0 and r["rows"] == w.n, r
    if p.stats()["hot_rows"] > 0:
        p0 = A.Plan(rp, ci, hot_rows=0, max_block_warps=0, max_warp_nzs=0)
        assert torch.equal(p0.spmm(va, Xd), Y)
        p0.close()
    if w.layers > 1:                                   # layer 2 on the GPU's own layer-1 output
        Y2 = p.spmm(va, Y).cpu().numpy()
        r = oracle.spmm_check(w.rowptr, w.colidx, w.vals, Yh, Y2)
        assert r["nfail"] == 0 and r["rows"] == w.n, r
    # properties at full size: all-ones X gives row sums of vals
    ones = torch.ones((w.n, 4), device=DEV)
    Ys = p.spmm(va, ones).cpu().numpy()
    rs = np.add.reduceat(w.vals.astype(np.float64), w.rowptr[:-1].clip(max=w.nnz - 1))
    rs[np.diff(w.rowptr) == 0] = 0.0
    s_abs = np.add.reduceat(np.abs(w.vals).astype(np.float64), w.rowptr[:-1].clip(max=w.nnz - 1))
    s_abs[np.diff(w.rowptr) == 0] = 0.0
    assert np.all(np.abs(Ys[:, 0] - rs) <= 1e-5 * s_abs + 1e-7)


# ---------------------------------------------------------------- shards, relabel, host API
def test_shard_bounds_and_sharded_plans():
    w = gen.make_config("c3")
    rp = cu(w.rowptr)
    X = w.X(32)
    Y_full, _ = oracle.spmm(w.rowptr, w.colidx, w.vals, X, with_abs=False)
    ci, va, Xd = cu(w.colidx), cu(w.vals), cu(X)
    for P in (1, 2, 3, 8):
        b = A.shard_bounds(rp, P)
        assert b.tolist() == oracle.shard_bounds(w.rowptr, P).tolist()
        outs = []
        for q in range(P):
            lo, hi = int(b[q]), int(b[q + 1])
            sub = rp[lo:hi + 1].contiguous()
            ps = A.Plan(sub, ci, n_cols=w.n)
            o = oracle.plan(w.rowptr[lo:hi + 1], w.colidx)
            assert np.array_equal(ps.copy("blocks"), o["blocks"])
            assert np.array_equal(ps.copy("row_src_off"), o["row_src_off"])
            outs.append(ps.spmm(va, Xd).cpu().numpy())
        Y = np.concatenate(outs)
        r = oracle.spmm_check(w.rowptr, w.colidx, w.vals, X, Y)
        assert r["nfail"] == 0


def test_padded_column_relabel():
    w = gen.make_config("c2")
    P = 3
    b = oracle.shard_bounds(w.rowptr, P)
    slot = int(np.diff(b).max()) + 5
    X = w.X(16)
    Xpad = np.zeros((P * slot, 16), np.float32)
    for q in range(P):
        Xpad[q * slot:q * slot + b[q + 1] - b[q]] = X[b[q]:b[q + 1]]
    p = A.Plan(cu(w.rowptr), cu(w.colidx), col_bounds=b, col_slot_rows=slot)
    Y = p.spmm(cu(w.vals), cu(Xpad)).cpu().numpy()
    check_spmm(p, w.rowptr, w.colidx, w.vals, X, Y)


def test_propagate_host_two_layers():
    w = gen.make_config("c3")
    X = w.X(16)
    Y2 = A.propagate_host(w.rowptr, w.colidx, w.vals, X, layers=2)
    Y1 = A.propagate_host(w.rowptr, w.colidx, w.vals, X, layers=1)
    check_spmm(A.Plan(cu(w.rowptr), cu(w.colidx)), w.rowptr, w.colidx, w.vals, X, Y1)
    r = oracle.spmm_check(w.rowptr, w.colidx, w.vals, Y1, Y2)
    assert r["nfail"] == 0


def test_bad_csr_is_reported():
    rowptr = np.array([0, 3, 2, 5], np.int32)
    with pytest.raises(A.AgcnError) as e:
        make_plan(rowptr, np.zeros(5, np.int32))
    assert e.value.status == "AGCN_ERR_BAD_CSR"
    # a bogus huge degree (the one-CTA plan must not emit its oversized chunks
    # before the check), decreasing or with the wrong total, on both plan paths
    for rp, nnz in (([0, 1000000, 5], 5), ([0, 1000000], 5), ([0, 5, 1000000, 5], 5)):
        for small in (True, False):
            with pytest.raises(A.AgcnError) as e:
                A.Plan(cu(np.array(rp, np.int32)), cu(np.zeros(8, np.int32)), len(rp) - 1, nnz,
                       small_plan=small)
            assert e.value.status == "AGCN_ERR_BAD_CSR", (rp, small)
    torch.cuda.synchronize()  # the device is still healthy (no out-of-bounds write happened)
    with pytest.raises(A.AgcnError) as e:
        make_plan(np.array([0, 1, 2], np.int32), np.array([0, 7], np.int32), n_cols=3)
    assert e.value.status == "AGCN_ERR_BAD_CSR"
    p = make_plan(np.array([0, 1, 2], np.int32), np.array([0, 1], np.int32))
    X = cu(np.ones((2, 4), np.float32))
    with pytest.raises(A.AgcnError) as e:
        A.agcn_spmm(p, cu(np.ones(2, np.float32)), X, 4, X)
    assert e.value.status == "AGCN_ERR_INVALID_ARG"


def test_launch_counter_moves():
    w = gen.make_config("c1")
    p = make_plan(w.rowptr, w.colidx)
    c0 = A.launch_count()
    p.spmm(cu(w.vals), cu(w.X()))
    assert A.launch_count() > c0


# ---------------------------------------------------------------- aggregation variants / epilogue
EPI_CASES = [
    dict(aggregation="mean"),
    dict(self_scale=1.5, self_x=True),                       # GIN, eps = 0.5
    dict(bias=True, relu=True),
    dict(aggregation="mean", self_scale=-0.75, self_x=True, bias=True, relu=True),
]


@pytest.mark.parametrize("kernel,F", [("auto", 64), ("wide", 128), ("wide", 40), ("general", 100), ("general", 64),
                                      ("looped", 16)])
@pytest.mark.parametrize("case", range(len(EPI_CASES)))
def test_spmm_epilogue(kernel, F, case):
    """GCN / GraphSAGE-mean / GIN aggregation with bias and ReLU vs the oracle, through
    the fused epilogue (WIDE, oversized-row reduction) and the separate pass (other kernels)."""
    ep = dict(EPI_CASES[case])
    rowptr, colidx = _rows_csr(np.array([0, 1, 2, 3, 5, 31, 33, 64, 97, 130, 200, 383, 384, 385,
                                         768, 769, 2000, 0, 7]), 19, 11)
    n = rowptr.size - 1
    rng = np.random.default_rng(case * 10 + F)
    vals = rng.uniform(-1, 1, colidx.size).astype(np.float32)
    X = rng.uniform(-1, 1, (n, F)).astype(np.float32)
    bias = rng.uniform(-1, 1, F).astype(np.float32)
    p = make_plan(rowptr, colidx, hot_rows=5 if case % 2 else 0)   # odd cases: hot-row encoding too
    kw = {"aggregation": ep.get("aggregation", "sum"), "self_scale": ep.get("self_scale", 0.0),
          "relu": ep.get("relu", False)}
    if ep.get("self_x"):
        kw["self_x"] = cu(X)
    if ep.get("bias"):
        kw["bias"] = cu(bias)
    Y = p.spmm(cu(vals), cu(X), kernel=kernel, **kw).cpu().numpy()
    y, t = oracle.spmm_epilogue(rowptr, colidx, vals, X, aggregation=kw["aggregation"],
                                self_x=X if ep.get("self_x") else None,
                                self_scale=kw["self_scale"], bias=bias if ep.get("bias") else None,
                                relu=kw["relu"])
    r = oracle.check_epilogue(Y, y, t)
    assert r["nfail"] == 0, r


def test_spmm_epilogue_warp_partition_and_sharded_rows():
    w = gen.make_config("c2", vals_kind="uniform")
    X = w.X(64)
    b = np.linspace(-1, 1, 64).astype(np.float32)
    y, t = oracle.spmm_epilogue(w.rowptr, w.colidx, w.vals, X, aggregation="mean", bias=b, relu=True)
    for part in ("warp", "block"):
        p = make_plan(w.rowptr, w.colidx, partition=part)
        Y = p.spmm(cu(w.vals), cu(X), aggregation="mean", bias=cu(b), relu=True).cpu().numpy()
        assert oracle.check_epilogue(Y, y, t)["nfail"] == 0, part


# ---------------------------------------------------------------- transpose / backward (8(f4))
@pytest.mark.parametrize("name", ["c1", "c3"])
def test_transpose_bit_exact_and_backward(name):
    w = gen.make_config(name, vals_kind="uniform")
    rp, ci = cu(w.rowptr), cu(w.colidx)
    rt, ct, src = A.transpose(rp, ci, w.n)
    ort, oct_, osrc = oracle.transpose(w.rowptr, w.colidx, w.n)
    assert np.array_equal(rt.cpu().numpy(), ort)
    assert np.array_equal(ct.cpu().numpy(), oct_)
    assert np.array_equal(src.cpu().numpy(), osrc)
    vt = A.gather_vals(cu(w.vals), src)
    assert np.array_equal(vt.cpu().numpy(), w.vals[osrc])
    dY = w.X(64)                                           # backward: dX = A^T dY
    pt = A.Plan(rt, ct, n_cols=w.n)
    dX = pt.spmm(vt, cu(dY)).cpu().numpy()
    check_spmm(pt, ort, oct_, w.vals[osrc], dY, dX)


def test_transpose_rectangular_shard_and_empty():
    rowptr, colidx = _rows_csr(np.array([0, 3, 0, 7, 1, 0]), 9, 4)
    base = 5                                               # a row shard: rowptr[0] != 0
    rp = np.concatenate([[0], rowptr + base]).astype(np.int32)[1:]
    ci = np.concatenate([np.zeros(base, np.int32), colidx]).astype(np.int32)
    rt, ct, src = A.transpose(cu(rp), cu(ci), 9)
    ort, oct_, osrc = oracle.transpose(rp, ci, 9)
    assert np.array_equal(rt.cpu().numpy(), ort) and np.array_equal(ct.cpu().numpy(), oct_)
    assert np.array_equal(src.cpu().numpy(), osrc)
    rt, ct, src = A.transpose(cu(np.zeros(4, np.int32)), cu(np.zeros(0, np.int32)), 3)
    assert np.array_equal(rt.cpu().numpy(), np.zeros(4, np.int32)) and ct.numel() == 0


# ---------------------------------------------------------------- GCN layer (8(f3))
@pytest.mark.parametrize("fin,fout,prec", [(64, 16, "fp32"), (16, 64, "fp32"), (128, 128, "fp32"),
                                           (32, 8, "fp32"), (256, 64, "fp32"), (64, 256, "fp32"),
                                           (64, 16, "tf32"), (16, 64, "tf32"), (128, 128, "tf32")])
def test_gcn_layer(fin, fout, prec):
    """fp32: the north-star tolerance (1e-5 relative); tf32 (tcgen05 X.W): 2^-9 relative."""
    from paper_2308_11825_b200.layer import GCNLayer
    w = gen.make_config("c2", vals_kind="uniform")
    rng = np.random.default_rng(fin + fout)
    X = w.X(fin)
    W = rng.uniform(-0.5, 0.5, (fin, fout)).astype(np.float32)
    b = rng.uniform(-0.5, 0.5, fout).astype(np.float32)
    layer = GCNLayer(make_plan(w.rowptr, w.colidx), cu(w.vals), cu(W), cu(b), relu=True, precision=prec)
    Y = layer(cu(X)).cpu().numpy()
    y, t = oracle.gcn_layer(w.rowptr, w.colidx, w.vals, X, W, b, relu=True)
    r = oracle.check_epilogue(Y, y, t, rel=1e-5 if prec == "fp32" else 2.0 ** -9)
    assert r["nfail"] == 0, (layer.order, r)


# ---------------------------------------------------------------- tcgen05 GEMM (8(f3))
@pytest.mark.parametrize("M,K,N", [(1, 4, 16), (127, 32, 16), (300, 64, 64), (1000, 100, 32),
                                   (4097, 128, 128), (513, 256, 64), (257, 64, 256), (70000, 64, 64)])
@pytest.mark.parametrize("epi", [False, True])
def test_gemm_xw_tcgen05_tf32(M, K, N, epi):
    """agcn_gemm_xw (tcgen05 kind::tf32) vs the fp64 product: |y - y_ref| <= 2^-9 sum|x w| + 1e-6
    (TF32 operands: 10-bit mantissa, fp32 accumulation)."""
    rng = np.random.default_rng(M + K + N)
    X = rng.uniform(-1, 1, (M, K)).astype(np.float32)
    W = rng.uniform(-1, 1, (K, N)).astype(np.float32)
    b = rng.uniform(-1, 1, N).astype(np.float32) if epi else None
    Y = A.gemm_xw(cu(X), cu(np.ascontiguousarray(W.T)), bias=cu(b) if epi else None, relu=epi).cpu().numpy()
    ref = X.astype(np.float64) @ W.astype(np.float64)
    mag = np.abs(X).astype(np.float64) @ np.abs(W).astype(np.float64)
    if epi:
        ref = np.maximum(ref + b, 0.0)
    err = np.abs(Y - ref)
    assert np.all(err <= 2.0 ** -9 * mag + 1e-6), float((err / (2.0 ** -9 * mag + 1e-6)).max())
    assert err.mean() > 1e-7 or M * N < 100            # it really is TF32 (not an fp32 fallback)


@pytest.mark.parametrize("M,K,N", [(1, 4, 16), (127, 32, 16), (300, 64, 64), (1000, 100, 32),
                                   (4097, 128, 128), (513, 256, 64), (257, 64, 256), (70000, 64, 64),
                                   (100, 16, 8), (300, 256, 256), (33, 12, 20)])
@pytest.mark.parametrize("epi", [False, True])
def test_gemm_xw_fp32(M, K, N, epi):
    """agcn_gemm_xw_ex(AGCN_GEMM_FP32): 3xTF32 on tcgen05 (or the CUDA-core kernel where the split
    W does not fit) vs the fp64 product within the layer tolerance 1e-5 sum|x w| + 1e-7, and at
    least 50x more accurate than the TF32 path on the same data (the split is really applied)."""
    rng = np.random.default_rng(M + K + N + 7)
    X = rng.uniform(-1, 1, (M, K)).astype(np.float32)
    W = rng.uniform(-1, 1, (K, N)).astype(np.float32)
    b = rng.uniform(-1, 1, N).astype(np.float32) if epi else None
    Wt = cu(np.ascontiguousarray(W.T))
    Y = A.gemm_xw(cu(X), Wt, bias=cu(b) if epi else None, relu=epi, precision="fp32").cpu().numpy()
    ref = X.astype(np.float64) @ W.astype(np.float64)
    mag = np.abs(X).astype(np.float64) @ np.abs(W).astype(np.float64)
    if epi:
        ref = np.maximum(ref + b, 0.0)
        mag = mag + np.abs(b)
    err = np.abs(Y - ref)
    assert np.all(err <= 1e-5 * mag + 1e-7), float((err / (1e-5 * mag + 1e-7)).max())
    if N in (16, 32, 64, 128, 256) and M * N >= 100 and K * N <= 128 * 128:   # tf32 and 3xTF32 both run
        Yt = A.gemm_xw(cu(X), Wt, bias=cu(b) if epi else None, relu=epi, precision="tf32").cpu().numpy()
        assert np.abs(Yt - ref).mean() > 50 * err.mean()


def test_pipeline_matches_propagate_host():
    """agcn_pipe_*: interleaved jobs of different graphs, widths and layer counts through a
    depth-2 executor (slots reused, buffers grown) give exactly propagate_host's Y, and the
    single-layer jobs pass the oracle check."""
    jobs = []
    for name, F, layers in (("c1", 16, 2), ("c2", 64, 1), ("c3", 32, 2), ("c1", 8, 1),
                            ("c2", 128, 2), ("c3", 64, 1), ("c1", 16, 1)):
        w = gen.make_config(name)
        jobs.append((w, w.X(F), layers))
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()  # noqa: E731
    with A.Pipeline(depth=2) as pipe:
        outs = []
        for w, X, layers in jobs:
            Y = torch.empty((w.n, X.shape[1]), dtype=torch.float32).pin_memory()
            pipe.submit(pin(w.rowptr), pin(w.colidx), pin(w.vals), pin(X), layers, out=Y)
            outs.append(Y)
        pipe.wait()
    for (w, X, layers), Y in zip(jobs, outs):
        ref = A.propagate_host(w.rowptr, w.colidx, w.vals, X, layers)
        assert np.array_equal(Y.numpy(), ref)
        if layers == 1:
            assert oracle.spmm_check(w.rowptr, w.colidx, w.vals, X, Y.numpy())["nfail"] == 0


@pytest.mark.parametrize("depth", [1, 3])
def test_pipeline_many_jobs_random_sizes(depth):
    """20 jobs of random size / width / layer count (buffers grow and shrink) through one
    executor: every Y equals agcn_propagate_host's."""
    rng = np.random.default_rng(77 + depth)
    jobs = []
    for i in range(20):
        n = int(rng.integers(1, 40000))
        rowptr, colidx = gen.random_csr(n, n, 500 + i, max_deg=int(rng.choice([3, 50, 700])))
        F = int(rng.choice([8, 16, 40, 64, 100]))
        vals = rng.uniform(-1, 1, colidx.size).astype(np.float32)
        X = rng.uniform(-1, 1, (n, F)).astype(np.float32)
        jobs.append((rowptr, colidx, vals, X, int(rng.integers(1, 3))))
    with A.Pipeline(depth=depth) as pipe:
        outs = [pipe.submit(*j) for j in jobs]
        pipe.wait()
    for (rowptr, colidx, vals, X, layers), Y in zip(jobs, outs):
        assert np.array_equal(Y, A.propagate_host(rowptr, colidx, vals, X, layers))


def test_pipeline_degenerate_jobs():
    """Edgeless graphs (Y = 0) and a 1-row graph through the executor, between real jobs."""
    w = gen.make_config("c1")
    X = w.X(16)
    with A.Pipeline(depth=2) as pipe:
        Y0 = np.full((7, 16), 5.0, np.float32)
        pipe.submit(np.zeros(8, np.int32), np.zeros(0, np.int32), np.zeros(0, np.float32),
                    np.ones((7, 16), np.float32), 2, out=Y0)
        Y1 = pipe.submit(w.rowptr, w.colidx, w.vals, X, 1)
        Yr = pipe.submit(np.array([0, 2], np.int32), np.array([0, 0], np.int32),
                         np.array([1.5, -0.5], np.float32), np.full((1, 16), 2.0, np.float32), 3)
        pipe.wait()
    assert not Y0.any()
    assert np.array_equal(Y1, A.propagate_host(w.rowptr, w.colidx, w.vals, X, 1))
    assert np.allclose(Yr, 2.0)                        # (1.5 - 0.5) ** 3 * 2


def test_pipeline_error_leaves_executor_usable():
    w = gen.make_config("c1")
    X = w.X(16)
    pipe = A.Pipeline(depth=1)
    bad = w.colidx.copy()
    bad[5] = w.n + 3                                   # column out of range: plan rejects it
    pipe.submit(w.rowptr, bad, w.vals, X, 1)          # the plan (worker) finds it
    with pytest.raises(A.AgcnError) as e:
        pipe.wait()
    assert e.value.status == "AGCN_ERR_BAD_CSR"
    from paper_2308_11825_b200 import _lib
    Yb = np.empty((w.n, 16), np.float32)               # rowptr[n] - rowptr[0] != nnz
    assert _lib.lib().agcn_pipe_submit(pipe._h, w.rowptr.ctypes.data, w.colidx.ctypes.data,
                                       w.vals.ctypes.data, w.n, w.nnz + 1, X.ctypes.data, 16, 1,
                                       Yb.ctypes.data) == 2
    Y = pipe.submit(w.rowptr, w.colidx, w.vals, X, 1)
    pipe.wait()
    ref = A.propagate_host(w.rowptr, w.colidx, w.vals, X, 1)
    assert np.array_equal(Y, ref)
    # a good job and a bad job in one batch: the failing wait still returns only after the good
    # job's Y is written
    w3 = gen.make_config("c3")
    X3 = w3.X(64)
    Yg = pipe.submit(w3.rowptr, w3.colidx, w3.vals, X3, 2)
    pipe.submit(w.rowptr, bad, w.vals, X, 1)
    with pytest.raises(A.AgcnError) as e:
        pipe.wait()
    assert e.value.status == "AGCN_ERR_BAD_CSR"
    assert np.array_equal(Yg, A.propagate_host(w3.rowptr, w3.colidx, w3.vals, X3, 2))
    pipe.close()


@pytest.mark.parametrize("name,F,layers", [("c1", 16, 2), ("c2", 64, 3), ("c3", 40, 1)])
def test_graphed_propagation(name, F, layers):
    """Layers captured in a CUDA graph give exactly the eager layers; replay after writing new
    features into the captured X buffer recomputes from them."""
    w = gen.make_config(name)
    X = cu(w.X(F))
    rp, ci, va = cu(w.rowptr), cu(w.colidx), cu(w.vals)
    g = A.GraphedPropagation(rp, ci, va, X, layers)
    p = A.Plan(rp, ci)
    ref = X
    for _ in range(layers):
        ref = p.spmm(va, ref)
    torch.cuda.synchronize()
    assert torch.equal(g.out, ref)
    X2 = torch.from_numpy(gen.uniform_f32(9, (w.n, F))).to(DEV)
    g.X.copy_(X2)
    torch.cuda.synchronize()
    Y = g.replay()
    torch.cuda.synchronize()
    ref = X2
    for _ in range(layers):
        ref = p.spmm(va, ref)
    torch.cuda.synchronize()
    assert torch.equal(Y, ref)
    if layers == 1:
        assert oracle.spmm_check(w.rowptr, w.colidx, w.vals, X2.cpu().numpy(), Y.cpu().numpy())["nfail"] == 0
    g.close()


def test_graph_scratch_guard():
    """While a captured graph holds a plan's scratch, an SpMM that would grow it is refused
    (ADVICE r01); smaller F works; after the graph is destroyed the plan grows normally."""
    w = gen.make_config("c3")  # has oversized rows: level-3 scratch
    rp, ci, va = cu(w.rowptr), cu(w.colidx), cu(w.vals)
    X16 = cu(w.X(16))
    g = A.GraphedPropagation(rp, ci, va, X16, 2)
    p = g.plan
    X64 = cu(w.X(64))
    with pytest.raises(A.AgcnError) as e:
        p.spmm(va, X64)
    assert e.value.status == "AGCN_ERR_UNSUPPORTED"
    Y8 = p.spmm(va, cu(w.X(8))).cpu().numpy()
    check_spmm(p, w.rowptr, w.colidx, w.vals, w.X(8), Y8)
    s = torch.cuda.Stream()
    g.replay(stream=s)           # launch on another stream: the plan's destroy is ordered after it
    _lib_destroy = A._lib.lib().agcn_graph_destroy(g._h)
    assert _lib_destroy == 0
    g._h = None
    Y64 = p.spmm(va, X64).cpu().numpy()
    check_spmm(p, w.rowptr, w.colidx, w.vals, w.X(64), Y64)
    g.close()


@pytest.mark.parametrize("F", [8, 40, 64, 128, 256])
def test_chunk_order_and_chunk_kernel(F):
    """The oversized chunks in column-position order (agcn_spmm_opts_t.chunk_order, plan option
    chunk_buckets) and in the separate chunk kernel (chunk_shape) give bitwise the result of
    descriptor order in the main kernel, which passes the oracle."""
    rowptr, colidx, vals, X = _hub_graph(4000, 100 + F, F)
    ref = None
    for mbw, mwn in ((2, 8), (12, 32)):
        for buckets in (0, 3, 1000):
            p = make_plan(rowptr, colidx, max_block_warps=mbw, max_warp_nzs=mwn, chunk_buckets=buckets, hot_rows=0)
            Y0 = p.spmm(cu(vals), cu(X), kernel="wide", chunk_order=-1, chunk_shape=-1).cpu().numpy()
            if ref is None:
                check_spmm(p, rowptr, colidx, vals, X, Y0)
            for order in (0, -1):
                for shape in (-1, 0, 3, 4, 6):
                    Y = p.spmm(cu(vals), cu(X), kernel="wide", chunk_order=order, chunk_shape=shape).cpu().numpy()
                    assert np.array_equal(Y, Y0), (mbw, mwn, buckets, order, shape)
            ref = Y0


def test_c_example_runs(tmp_path):
    """examples/spmm_c.c on the GPU: plan + SpMM from plain C, checked against a double loop
    (north_star tolerance), the caller's colidx freed after agcn_plan, and equal to
    agcn_propagate_host on host buffers."""
    import subprocess
    import sys
    sys.path.insert(0, os.path.dirname(__file__))
    from test_abi_cpu import _build_c_example
    exe = str(tmp_path / "spmm_c")
    r = _build_c_example(exe)
    assert r.returncode == 0, r.stderr
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and r.stdout.startswith("ok"), r.stdout + r.stderr
