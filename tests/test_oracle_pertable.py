"""Pins: NEXT-2 per-table independent families (reading C3, "L independent
hash tables of m-sized hash codes"; SURVEY 8(c) A1 "table{t}/" labels).

Each check is fixed by the mathematics, not by retyping the oracle:
hand-computed pipeline values, a brute-force dense matrix, the unbiased inner
product of a count sketch, independence of the tables' hashes, the K = 1 closed
form and the collision law (Thm CS_Eucl_LSH_property P:580 with m -> K).
"""
import math

import numpy as np
import pytest

from oracle import lsh, rng, theory


def _p(scheme="CS_E2LSH", d=12, L=3, K=4, w=2.0, seed=7):
    return lsh.Params(scheme, d=d, m=L * K, L=L, K=K, w=w, seed=seed, per_table=True)


def test_hand_computed_pipeline():
    # d = 3, one table of K = 2: h = (0, 1, 1), s = (+1, -1, +1), b = (0.5, 0.25), w = 1
    # x = (1, 2, 4): y = (1, -2 + 4) = (1, 2); codes floor(sqrt(2) y + b) = (1, 3)
    p = lsh.Params("CS_E2LSH", d=3, m=2, L=1, K=2, w=1.0, per_table=True)
    t = lsh.Tables(h=[np.array([0, 1, 1])], s=[np.array([1, -1, 1])], b=np.array([0.5, 0.25], np.float32))
    out = lsh.hash_points(p, t, np.array([[1.0, 2.0, 4.0]], np.float32))
    assert out["proj"].tolist() == [[1.0, 2.0]]
    assert out["codes"].tolist() == [[1, 3]]
    # SRP on the same sketch: bits (1, 1) -> key 0b11; x -> -x flips both
    ps = lsh.Params("CS_SRP", d=3, m=2, L=1, K=2, per_table=True)
    assert lsh.hash_points(ps, t, np.array([[1.0, 2.0, 4.0]], np.float32))["keys"].tolist() == [[3]]
    assert lsh.hash_points(ps, t, np.array([[-1.0, -2.0, -4.0]], np.float32))["keys"].tolist() == [[0]]


def test_dense_matrix_bruteforce_block_layout():
    # y[:, tK:(t+1)K] = S_t x with S_t[k, i] = s_t(i) [h_t(i) = k], assembled entry by entry
    p = _p(d=9, L=3, K=4)
    t = lsh.make_tables(p)
    S = np.zeros((p.m, p.d))
    for tt in range(p.L):
        for i in range(p.d):
            S[tt * p.K + int(t.h[tt][i]), i] += float(t.s[tt][i])
    X = np.random.default_rng(0).standard_normal((5, p.d)).astype(np.float32)
    np.testing.assert_allclose(lsh.project(p, t, X), X.astype(np.float64) @ S.T, rtol=0, atol=1e-12)
    # every column of every block has exactly one +-1
    for tt in range(p.L):
        blk = S[tt * p.K:(tt + 1) * p.K]
        assert (np.abs(blk).sum(axis=0) == 1).all()


def test_tables_use_their_own_streams():
    p = _p(d=64, L=4, K=8)
    t = lsh.make_tables(p)
    # table t's family is the stream labelled "table{t}/mode0/bucket" (not the shared one)
    shared = rng.bucket_table(p.seed, 0, p.d, p.K)
    for tt in range(p.L):
        assert not np.array_equal(t.h[tt], shared)
        for u in range(tt):
            assert not np.array_equal(t.h[tt], t.h[u])
            assert not np.array_equal(t.s[tt], t.s[u])
    assert len({float(v) for v in t.b}) == p.m   # offsets drawn per table, all distinct


def test_inner_product_unbiased_across_tables():
    # E[<S_t x, S_t x'>] = <x, x'> for a count sketch with random signs; a dropped or
    # shared sign would add sum_{i != j} x_i x'_j P[h(i) = h(j)]
    g = np.random.default_rng(1)
    d, K, L = 24, 4, 3000
    x = g.standard_normal(d)
    xp = x + 0.8 * g.standard_normal(d) + 0.5
    p = lsh.Params("CS_SRP", d=d, m=L * K, L=L, K=K, seed=3, per_table=True)
    t = lsh.make_tables(p)
    Y = lsh.project(p, t, np.stack([x, xp]).astype(np.float32)).reshape(2, L, K)
    est = (Y[0] * Y[1]).sum(axis=1)
    xs, xps = x.astype(np.float32).astype(np.float64), xp.astype(np.float32).astype(np.float64)
    se = est.std(ddof=1) / math.sqrt(L)
    assert abs(est.mean() - xs @ xps) < 4 * se
    # and the squared norm (Var of the estimate is O(||x||^4 / K))
    nrm = (Y[0] ** 2).sum(axis=1)
    assert abs(nrm.mean() - xs @ xs) < 4 * nrm.std(ddof=1) / math.sqrt(L)


def test_bins_independent_across_tables():
    # for a fixed coordinate, h_t(i) over many tables is uniform on [K] (chi-square),
    # and two coordinates collide in a table with rate 1/K
    d, K, L = 6, 8, 4000
    p = lsh.Params("CS_SRP", d=d, m=L * K, L=L, K=K, seed=11, per_table=True)
    t = lsh.make_tables(p)
    H = np.stack(t.h)           # [L][d]
    cnt = np.bincount(H[:, 2], minlength=K)
    chi2 = ((cnt - L / K) ** 2 / (L / K)).sum()
    assert chi2 < 30.0          # 7 dof: P[chi2 > 30] ~ 1e-4
    coll = (H[:, 0] == H[:, 1]).mean()
    assert abs(coll - 1 / K) < 4 * math.sqrt((1 / K) * (1 - 1 / K) / L)


def test_k1_closed_form():
    # K = 1: every coordinate lands in the single bin, y_t = sum_i s_t(i) x_i
    p = lsh.Params("CS_SRP", d=10, m=5, L=5, K=1, seed=2, per_table=True)
    t = lsh.make_tables(p)
    x = np.arange(1, 11, dtype=np.float32)
    y = lsh.project(p, t, x[None])[0]
    for tt in range(p.L):
        assert y[tt] == float(sum(int(t.s[tt][i]) * (i + 1) for i in range(10)))


@pytest.mark.slow
def test_per_table_collision_law_mc():
    # Thm CS_Eucl_LSH_property per table: sqrt(K) CS_t(p)_k is asymptotically
    # N(0, ||p||^2), so Pr[g_t(p)_k = g_t(q)_k] -> p(R) with R = ||p - q||
    g = np.random.default_rng(5)
    d, K, L, w = 4000, 4, 600, 4.0
    e = g.standard_normal(d); e /= np.linalg.norm(e)
    pt = g.standard_normal(d); pt /= np.linalg.norm(pt)
    X = np.stack([pt, pt + 1.0 * e]).astype(np.float32)
    p = lsh.Params("CS_E2LSH", d=d, m=L * K, L=L, K=K, w=w, seed=9, per_table=True)
    c = lsh.hash_points(p, lsh.make_tables(p), X)["codes"]
    R = float(np.linalg.norm(X[0].astype(np.float64) - X[1]))
    pr = theory.p_collision_e2lsh(R, w)
    rate = (c[0] == c[1]).mean()
    assert abs(rate - pr) < 0.03


def test_work_and_space_are_o_l_d():
    p = _p(d=20, L=3, K=4)
    t = lsh.make_tables(p)
    assert lsh.projection_op_count(p, t, np.ones(20)) == 3 * 20
    assert lsh.param_count(p) == 2 * 20 * 3 + p.m
    with pytest.raises(ValueError):
        lsh.Params("HCS_SRP", d=8, m=4, L=2, K=2, mode_d=(2, 4), mode_m=(2, 2), per_table=True)
