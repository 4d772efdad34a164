"""Pins for the CPU oracle (oracle/), run without a GPU.

Each pin is something other than the oracle itself: a value PAPER.md prints for its worked
example (tests/golden/), a closed form, dense brute force, an invariant, or a special case
that reduces to a library routine.  Chosen so that a dropped term, a wrong sign or index,
a transposed operand, an off-by-one bound or an unstable sort fails at least one of them.
"""
import json
import os

import numpy as np
import pytest

import agcn_inputs as gen
import oracle

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def _dense(rowptr, colidx, vals, n_cols):
    n = rowptr.size - 1
    A = np.zeros((n, n_cols), dtype=np.float64)
    for i in range(n):
        for p in range(rowptr[i], rowptr[i + 1]):
            A[i, colidx[p]] += float(vals[p])  # duplicates add (Q26)
    return A


# ---------------------------------------------------------------- Fig. 3 worked example
def test_fig3_golden():
    g = _gold("fig3.json")
    rowptr = np.array(g["rowptr"], np.int32)
    colidx = np.array(g["colidx"], np.int32)
    mbw, mwn = g["max_block_warps"], g["max_warp_nzs"]
    plan = oracle.plan(rowptr, colidx, mbw, mwn)
    assert plan["perm"].tolist() == g["perm"]
    assert plan["blocks"].tolist() == g["blocks"]
    tasks = oracle.warp_partition(rowptr, mwn)
    assert tasks.shape[0] == g["n_warp_tasks"]
    assert tasks[0].tolist() == g["warp_tasks_first"]
    assert oracle.storage_ratio(plan["blocks"].shape[0], tasks.shape[0]) == g["storage_ratio"]
    # BP-1's two warps start at nnz offsets loc + w*deg = 0 and 2, 2 nnz each
    deg, loc, row, info = plan["blocks"][0]
    assert [loc + w * deg for w in range(info & 0xFFFF)] == [0, 2]
    assert [int(info >> 16)] * 2 == g["warp_nnz_bp1"]


# ---------------------------------------------------------------- Algorithm 1
def _closed_form_pattern(d, mbw, mwn):
    f = min(f for f in range(1, mbw + 1) if mbw % f == 0 and f * mwn >= d)
    return mbw // f, -(-d // f)


@pytest.mark.parametrize("mbw,mwn", [(2, 2), (1, 1), (12, 32), (16, 64), (6, 5), (7, 3), (12, 1),
                                     (30, 4), (1, 17)])
def test_patterns_closed_form(mbw, mwn):
    br, wn = oracle.patterns(mbw, mwn)
    db = mbw * mwn
    assert br.size == db + 1
    for d in range(1, db + 1):
        assert (br[d], wn[d]) == _closed_form_pattern(d, mbw, mwn), d
        assert mbw % br[d] == 0 and (mbw // br[d]) * wn[d] >= d and wn[d] <= mwn


def test_patterns_hand_traces():
    # S:209-211 hand traces of Alg. 1 with factors [1, 2]
    br, wn = oracle.patterns(2, 2)
    assert [(br[d], wn[d]) for d in (1, 2, 3, 4)] == [(2, 1), (2, 2), (1, 2), (1, 2)]
    br, wn = oracle.patterns(1, 1)
    assert (br[1], wn[1]) == (1, 1)
    # (12,32) buckets 1-32 ->(12,d); 33-64 ->(6,ceil d/2); 65-96 ->(4, ceil d/3);
    # 97-128 ->(3, ceil d/4); 129-192 ->(2, ceil d/6); 193-384 ->(1, ceil d/12)
    br, wn = oracle.patterns(12, 32)
    for lo, hi, rows, f in [(1, 32, 12, 1), (33, 64, 6, 2), (65, 96, 4, 3), (97, 128, 3, 4),
                            (129, 192, 2, 6), (193, 384, 1, 12)]:
        for d in range(lo, hi + 1):
            assert br[d] == rows and wn[d] == -(-d // f)
    assert _gold("paper_values.json")["deg_bound_12_32"]["value"] == 12 * 32


# ---------------------------------------------------------------- Algorithm 2
def test_oversized_row_hand_trace():
    # one row of degree 9 at (2,2) (deg_bound 4) -> infos 4,4,1 at locs 0,4,8
    b = oracle.block_partition(np.array([9], np.int32), 2, 2)
    assert b.tolist() == [[9, 0, 0, 4], [9, 4, 0, 4], [9, 8, 0, 1]]


def test_block_partition_rejects_unsorted():
    with pytest.raises(ValueError):
        oracle.block_partition(np.array([3, 1], np.int32), 2, 2)


def test_block_partition_empty_and_zero_rows():
    assert oracle.block_partition(np.zeros(0, np.int32)).shape == (0, 4)
    assert oracle.block_partition(np.zeros(7, np.int32)).shape == (0, 4)
    b = oracle.block_partition(np.array([0, 0, 1], np.int32), 12, 32)
    assert b.tolist() == [[1, 0, 2, (1 << 16) | 1]]   # row cursor skips the 2 zero rows


def _check_blocks(sdeg, blocks, mbw, mwn):
    """Invariants + per-bucket closed form (SURVEY section 7 'Parallel Alg. 2 emission')."""
    db = mbw * mwn
    nnz = int(sdeg.sum())
    srp = np.concatenate([[0], np.cumsum(sdeg)])
    covered = np.zeros(nnz, np.int32)
    br, wn = oracle.patterns(mbw, mwn)
    for deg, loc, row, info in blocks.astype(np.int64):
        if deg <= db:
            rows = info & 0xFFFF
            assert info >> 16 == wn[deg] and 1 <= rows <= br[deg]
            assert np.all(sdeg[row:row + rows] == deg)
            assert srp[row] == loc
            covered[loc:loc + rows * deg] += 1
        else:
            assert 1 <= info <= db and sdeg[row] == deg
            assert srp[row] <= loc and loc + info <= srp[row + 1]
            covered[loc:loc + info] += 1
    assert np.all(covered == 1)          # descriptors tile [0, nnz) exactly once
    # closed form: bucket d with cnt rows starting at rowstart -> ceil(cnt/br) blocks
    small = blocks[blocks[:, 0] <= db]
    for d in np.unique(sdeg[(sdeg > 0) & (sdeg <= db)]):
        rs = np.flatnonzero(sdeg == d)
        cnt, r0 = rs.size, rs[0]
        bd = small[small[:, 0] == d]
        nb = -(-cnt // br[d])
        assert bd.shape[0] == nb
        for b in range(nb):
            assert bd[b, 2] == r0 + b * br[d]
            assert bd[b, 1] == srp[r0] + b * br[d] * d
            assert bd[b, 3] & 0xFFFF == min(br[d], cnt - b * br[d])
    big = np.flatnonzero(sdeg > db)
    assert blocks.shape[0] - small.shape[0] == int(sum(-(-int(sdeg[r]) // db) for r in big))


@pytest.mark.parametrize("seed", range(40))
def test_block_partition_random(seed):
    rng = np.random.default_rng(seed)
    mbw = int(rng.choice([1, 2, 3, 4, 6, 12, 16]))
    mwn = int(rng.choice([1, 2, 5, 32, 64]))
    n = int(rng.integers(0, 400))
    deg = np.minimum(rng.zipf(1.5, size=n) - 1, 5000).astype(np.int32)
    sdeg = np.sort(deg).astype(np.int32)
    _check_blocks(sdeg, oracle.block_partition(sdeg, mbw, mwn), mbw, mwn)


def test_block_partition_many_configs():
    # AC4: 1000 random (matrix, cfg) instances tile [0, nnz) exactly
    rng = np.random.default_rng(1234)
    for _ in range(1000):
        mbw = int(rng.integers(1, 17)); mwn = int(rng.integers(1, 40))
        sdeg = np.sort(np.minimum(rng.zipf(1.7, size=int(rng.integers(0, 60))) - 1, 900))
        sdeg = sdeg.astype(np.int32)
        b = oracle.block_partition(sdeg, mbw, mwn)
        db = mbw * mwn
        sz = np.where(b[:, 0] <= db, (b[:, 3] & 0xFFFF).astype(np.int64) * b[:, 0], b[:, 3])
        assert int(sz.sum()) == int(sdeg.sum())
        if b.shape[0]:
            assert b[0, 1] == 0 and np.all(b[1:, 1] == b[:-1, 1] + sz[:-1])


def test_block_partition_field_overflow():
    # block_rows = max_block_warps / 1 >= 2^16 does not fit the 16-bit info half
    with pytest.raises(OverflowError):
        oracle.block_partition(np.array([1], np.int32), 65536, 1)


# ---------------------------------------------------------------- storage ratio (Eq. 1)
def test_storage_ratio_full_blocks():
    gv = _gold("paper_values.json")["storage_ratio_mbw12"]
    mbw, mwn = gv["max_block_warps"], gv["max_warp_nzs"]
    deg = mbw * mwn                                     # every block is one full row of 12 warps
    rowptr = np.arange(0, deg * 50 + 1, deg, dtype=np.int32)
    plan_blocks = oracle.block_partition(np.diff(rowptr).astype(np.int32), mbw, mwn)
    tasks = oracle.warp_partition(rowptr, mwn)
    assert oracle.storage_ratio(plan_blocks.shape[0], tasks.shape[0]) == gv["ratio"]
    # rows of degree 32 -> 12 rows per block, one task per row: again exactly 1/12
    rowptr = np.arange(0, 32 * 120 + 1, 32, dtype=np.int32)
    b = oracle.block_partition(np.diff(rowptr).astype(np.int32), mbw, mwn)
    assert oracle.storage_ratio(b.shape[0], oracle.warp_partition(rowptr, mwn).shape[0]) == gv["ratio"]


def test_storage_ratio_power_law():
    lim = _gold("paper_values.json")["storage_ratio_typical_max"]["value"]
    rowptr, colidx, _ = gen.chung_lu(100000, 700000, 66.0, seed=9)
    p = oracle.plan(rowptr, colidx)
    r = oracle.storage_ratio(p["blocks"].shape[0], oracle.warp_partition(rowptr).shape[0])
    assert r <= lim


# ---------------------------------------------------------------- degree sort
def test_degree_sort_is_stable_argsort():
    for seed in range(20):
        rowptr, _ = gen.random_csr(int(np.random.default_rng(seed).integers(1, 500)), 64, seed)
        deg = np.diff(rowptr)
        assert np.array_equal(oracle.degree_sort(rowptr), np.argsort(deg, kind="stable"))


def test_degree_sort_identity_when_sorted():
    rowptr = np.concatenate([[0], np.cumsum([0, 0, 1, 1, 2, 5, 5, 9])]).astype(np.int32)
    assert oracle.degree_sort(rowptr).tolist() == list(range(8))


def test_sorted_csr_rows_preserved():
    rowptr, colidx = gen.random_csr(300, 80, seed=3)
    perm = oracle.degree_sort(rowptr)
    srp, sci, rso = oracle.sorted_csr(rowptr, colidx, perm)
    assert np.all(np.diff(np.diff(srp)) >= 0)
    for k, r in enumerate(perm):
        assert np.array_equal(sci[srp[k]:srp[k + 1]], colidx[rowptr[r]:rowptr[r + 1]])
        assert rso[k] == rowptr[r]


# ---------------------------------------------------------------- SpMM result oracle
@pytest.mark.parametrize("seed", range(200))
def test_spmm_vs_dense_brute_force(seed):
    # AC3: 200 random tiny CSRs vs dense A @ X
    rng = np.random.default_rng(seed)
    n, nc, F = int(rng.integers(1, 65)), int(rng.integers(1, 65)), int(rng.integers(1, 129))
    rowptr, colidx = gen.random_csr(n, nc, seed, dup=bool(seed % 3 == 0))
    vals = rng.uniform(-1, 1, colidx.size).astype(np.float32)
    X = rng.uniform(-1, 1, (nc, F)).astype(np.float32)
    y, s = oracle.spmm(rowptr, colidx, vals, X)
    A = _dense(rowptr, colidx, vals, nc)
    np.testing.assert_allclose(y, A @ X.astype(np.float64), rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(s, _dense(rowptr, colidx, np.abs(vals), nc) @ np.abs(X).astype(np.float64),
                               rtol=1e-12, atol=1e-12)


def test_spmm_integer_exact():
    rng = np.random.default_rng(7)
    rowptr, colidx = gen.random_csr(200, 150, 7, dup=True)
    vals = rng.integers(-4, 5, colidx.size).astype(np.float32)
    X = rng.integers(-4, 5, (150, 33)).astype(np.float32)
    y, _ = oracle.spmm(rowptr, colidx, vals, X)
    Ai = np.zeros((200, 150), np.int64)
    for i in range(200):
        for p in range(rowptr[i], rowptr[i + 1]):
            Ai[i, colidx[p]] += int(vals[p])
    assert np.array_equal(y, (Ai @ X.astype(np.int64)).astype(np.float64))


def test_spmm_identity_and_ones():
    n, F = 97, 19
    rowptr = np.arange(n + 1, dtype=np.int32)
    colidx = np.arange(n, dtype=np.int32)
    X = gen.uniform_f32(5, (n, F))
    y, _ = oracle.spmm(rowptr, colidx, np.ones(n, np.float32), X)
    assert np.array_equal(y, X.astype(np.float64))           # A = I -> Y = X
    rowptr, colidx = gen.random_csr(120, 120, 11)
    vals = gen.uniform_f32(6, colidx.size)
    y, _ = oracle.spmm(rowptr, colidx, vals, np.ones((120, 4), np.float32))
    rs = np.array([vals[rowptr[i]:rowptr[i + 1]].astype(np.float64).sum() for i in range(120)])
    np.testing.assert_allclose(y, np.repeat(rs[:, None], 4, 1), rtol=0, atol=1e-12)


def test_spmm_row_permutation_and_linearity():
    rowptr, colidx = gen.random_csr(150, 90, 21)
    vals = gen.uniform_f32(7, colidx.size)
    X = gen.uniform_f32(8, (90, 24)); Z = gen.uniform_f32(9, (90, 24))
    y, _ = oracle.spmm(rowptr, colidx, vals, X)
    # (P A) X = P (A X), bitwise (each row is summed in the same order)
    perm = gen.permutation(3, 150)
    d = np.diff(rowptr)
    prp = np.concatenate([[0], np.cumsum(d[perm])]).astype(np.int32)
    pci = np.concatenate([colidx[rowptr[r]:rowptr[r + 1]] for r in perm]).astype(np.int32)
    pva = np.concatenate([vals[rowptr[r]:rowptr[r + 1]] for r in perm]).astype(np.float32)
    yp, _ = oracle.spmm(prp, pci, pva, X)
    assert np.array_equal(yp, y[perm])
    yz, _ = oracle.spmm(rowptr, colidx, vals, Z)
    W = (2.0 * X.astype(np.float64) - 3.0 * Z.astype(np.float64)).astype(np.float32)
    yw, sw = oracle.spmm(rowptr, colidx, vals, W)
    np.testing.assert_allclose(yw, 2.0 * y - 3.0 * yz, atol=1e-6)


def test_spmm_conservation_integer():
    rng = np.random.default_rng(4)
    rowptr, colidx = gen.random_csr(100, 60, 4)
    vals = rng.integers(-4, 5, colidx.size).astype(np.float32)
    X = rng.integers(-4, 5, (60, 10)).astype(np.float32)
    y, _ = oracle.spmm(rowptr, colidx, vals, X)
    rhs = sum(float(vals[p]) * float(X[colidx[p]].sum()) for p in range(colidx.size))
    assert y.sum() == rhs                                     # S:334 conservation


def test_spmm_shard_rowptr_base():
    rowptr, colidx = gen.random_csr(80, 50, 5)
    vals = gen.uniform_f32(3, colidx.size); X = gen.uniform_f32(4, (50, 8))
    y, _ = oracle.spmm(rowptr, colidx, vals, X)
    ys, _ = oracle.spmm(rowptr[30:61], colidx, vals, X)      # rowptr slice, global colidx/vals
    assert np.array_equal(ys, y[30:60])


def test_spmm_check_sensitivity():
    rowptr, colidx = gen.random_csr(60, 60, 2)
    vals = gen.uniform_f32(1, colidx.size); X = gen.uniform_f32(2, (60, 16))
    y, s = oracle.spmm(rowptr, colidx, vals, X)
    Y = y.astype(np.float32)
    r = oracle.spmm_check(rowptr, colidx, vals, X, Y)
    assert r["nfail"] == 0 and r["max_ratio"] <= 1.0
    i = int(np.argmax(np.diff(rowptr)))
    bad = Y.copy(); bad[i, 3] += np.float32(3 * (1e-5 * s[i, 3] + 1e-7))
    r = oracle.spmm_check(rowptr, colidx, vals, X, bad)
    assert r["nfail"] == 1 and r["worst"] == (i, 3)
    bad = Y.copy(); bad[0, 0] = np.nan
    assert oracle.spmm_check(rowptr, colidx, vals, X, bad)["nfail"] >= 1
    rows = np.array([i, 0, 5], np.int64)
    r = oracle.spmm_check(rowptr, colidx, vals, X, Y[rows], rows=rows)
    assert r["nfail"] == 0


# ---------------------------------------------------------------- warp partition, shards
def test_warp_partition_coverage():
    rowptr, colidx = gen.random_csr(500, 400, 8)
    for mwn in (1, 2, 7, 32):
        t = oracle.warp_partition(rowptr, mwn).astype(np.int64)
        assert t[:, 2].sum() == rowptr[-1] and np.all(t[:, 2] <= mwn) and np.all(t[:, 3] == 0)
        for i in range(500):
            ti = t[t[:, 0] == i]
            d = rowptr[i + 1] - rowptr[i]
            assert ti.shape[0] == -(-d // mwn)
            if ti.shape[0]:
                assert np.array_equal(ti[:, 1], np.arange(0, d, mwn))


@pytest.mark.parametrize("P", [1, 2, 3, 4, 8])
def test_shard_bounds_closed_form(P):
    rowptr, _ = gen.random_csr(1000, 100, 12)
    b = oracle.shard_bounds(rowptr, P)
    nnz = int(rowptr[-1])
    want = [0] + [int(np.searchsorted(rowptr, (p * nnz) // P, side="left")) for p in range(1, P)] + [1000]
    assert b.tolist() == want


# ---------------------------------------------------------------- combined warp
def test_combined_warp_values():
    for e in _gold("paper_values.json")["combined_warp"]:
        assert oracle.combined_warp(e["F"]) == (e["c"], e["round_dim"])
    for F in range(1, 129):
        c, rd = oracle.combined_warp(F)
        lanes = np.arange(rd)
        active = lanes < F                                    # lanes >= F truncated
        assert active.sum() == F and rd % 32 == 0 and rd - F < 32


# ---------------------------------------------------------------- aggregation variants
def test_epilogue_mean_is_neighbour_mean():
    """GraphSAGE-mean with unit values = the arithmetic mean of the neighbours' rows (dense)."""
    rng = np.random.default_rng(7)
    n, nc, F = 40, 30, 5
    rowptr, colidx = gen.random_csr(n, nc, 7, max_deg=9, dup=False)
    vals = np.ones(colidx.size, np.float32)
    X = rng.uniform(-1, 1, (nc, F)).astype(np.float32)
    y, _ = oracle.spmm_epilogue(rowptr, colidx, vals, X, aggregation="mean")
    for i in range(n):
        nb = colidx[rowptr[i]:rowptr[i + 1]]
        want = X[nb].astype(np.float64).mean(0) if nb.size else np.zeros(F)
        assert np.allclose(y[i], want, rtol=1e-12, atol=1e-12)


def test_epilogue_gin_self_term_bias_relu():
    """GIN on an edgeless graph reduces to (1 + eps) * x; bias broadcasts; ReLU clips."""
    rng = np.random.default_rng(8)
    n, F = 12, 6
    rowptr = np.zeros(n + 1, np.int32)
    colidx = np.zeros(0, np.int32)
    X = rng.uniform(-1, 1, (n, F)).astype(np.float32)
    b = rng.uniform(-1, 1, F).astype(np.float32)
    y, t = oracle.spmm_epilogue(rowptr, colidx, np.zeros(0, np.float32), X, self_x=X,
                                self_scale=1.25, bias=b)
    assert np.allclose(y, 1.25 * X.astype(np.float64) + b, rtol=0, atol=1e-12)
    assert np.allclose(t, np.abs(1.25 * X.astype(np.float64)) + np.abs(b), rtol=0, atol=1e-12)
    yr, _ = oracle.spmm_epilogue(rowptr, colidx, np.zeros(0, np.float32), X, self_x=X,
                                 self_scale=1.25, bias=b, relu=True)
    assert np.array_equal(yr, np.maximum(y, 0.0))
    r = oracle.check_epilogue((y + 1e-3).astype(np.float32), y, t)   # planted error fails
    assert r["nfail"] > 0


# ---------------------------------------------------------------- transpose (backward, 8(f4))
@pytest.mark.parametrize("seed", range(6))
def test_transpose_dense_and_involution(seed):
    rng = np.random.default_rng(seed)
    n, nc = int(rng.integers(1, 60)), int(rng.integers(1, 60))
    rowptr, colidx = gen.random_csr(n, nc, seed, max_deg=20, dup=bool(seed % 2))
    vals = rng.uniform(-1, 1, colidx.size)
    rt, ct, src = oracle.transpose(rowptr, colidx, nc)
    D = np.zeros((n, nc))
    np.add.at(D, (np.repeat(np.arange(n), np.diff(rowptr)), colidx), vals)
    Dt = np.zeros((nc, n))
    np.add.at(Dt, (np.repeat(np.arange(nc), np.diff(rt)), ct), vals[src])
    assert np.array_equal(Dt, D.T)                         # dense brute force
    for j in range(nc):                                    # rows of A^T ascending (stable)
        assert np.all(np.diff(ct[rt[j]:rt[j + 1]]) >= 0)
    r2, c2, s2 = oracle.transpose(rt, ct, n)               # (A^T)^T = A, entry for entry
    assert np.array_equal(r2, rowptr.astype(np.int32)) and np.array_equal(c2, colidx)
    assert np.array_equal(src[s2], np.arange(colidx.size))


# ---------------------------------------------------------------- GCN layer (8(f3))
def test_gcn_layer_reduces_to_spmm_and_dense():
    rng = np.random.default_rng(9)
    n, F = 30, 6
    rowptr, colidx = gen.random_csr(n, n, 9, max_deg=8, dup=True)
    vals = rng.uniform(-1, 1, colidx.size).astype(np.float32)
    X = rng.uniform(-1, 1, (n, F)).astype(np.float32)
    y, _ = oracle.gcn_layer(rowptr, colidx, vals, X, np.eye(F), relu=False)   # W = I: the SpMM
    y0, _ = oracle.spmm(rowptr, colidx, vals, X)
    assert np.allclose(y, y0, rtol=1e-13, atol=1e-13)
    W = rng.uniform(-1, 1, (F, 4))
    b = rng.uniform(-1, 1, 4)
    eye = np.arange(n + 1, dtype=np.int32)                                  # A = I: dense layer
    y1, _ = oracle.gcn_layer(eye, np.arange(n, dtype=np.int32), np.ones(n, np.float32), X, W, b)
    assert np.allclose(y1, np.maximum(X.astype(np.float64) @ W + b, 0), rtol=1e-13, atol=1e-13)
