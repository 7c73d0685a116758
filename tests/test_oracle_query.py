"""Pins of the oracle's query completion."""
import numpy as np
import pytest

from oracle import lsh


def _keys(L, n, g, vals=6):
    return g.integers(0, vals, (L, n)).astype(np.uint64)


def test_candidates_equal_brute_force_union():
    g = np.random.default_rng(0)
    L, n = 5, 400
    keys = _keys(L, n, g)
    tables = lsh.group(keys, id_base=0)
    for q in range(0, n, 37):
        qk = keys[:, q]
        got = lsh.query_candidates(tables, qk, max_cand=10 ** 9)
        want = np.flatnonzero((keys == qk[:, None]).any(axis=0))   # points sharing a bucket in some table
        assert np.array_equal(got, want)
        assert q in got                                             # self-retrieval


def test_candidate_cap_is_table_order_prefix():
    # table 0 bucket of key 1 = ids {0, 2}; table 1 bucket of key 7 = ids {1, 2, 3}
    keys = np.array([[1, 0, 1, 0], [5, 7, 7, 7]], dtype=np.uint64)
    tables = lsh.group(keys)
    q = np.array([1, 7], dtype=np.uint64)
    assert lsh.query_candidates(tables, q, 10).tolist() == [0, 1, 2, 3]
    assert lsh.query_candidates(tables, q, 3).tolist() == [0, 1, 2]     # entries 0, 2, 1 (then 2, 3 cut)
    assert lsh.query_candidates(tables, q, 2).tolist() == [0, 2]
    assert lsh.query_candidates(tables, np.array([9, 9], np.uint64), 10).tolist() == []


@pytest.mark.parametrize("metric", ["l2", "cosine"])
def test_rerank_matches_independent_library(metric):
    from scipy.spatial.distance import cdist
    g = np.random.default_rng(1)
    X = g.standard_normal((300, 17))
    X[5] = 0.0                                  # zero vector: cosine score 0 by reading C2
    q = g.standard_normal(17)
    cand = np.sort(g.choice(300, 120, replace=False))
    cand = np.union1d(cand, [5])
    ids, sc = lsh.rerank(X[cand], q, cand, 10, metric)
    if metric == "l2":
        d = cdist(q[None, :], X[cand], "sqeuclidean")[0]
        want = cand[np.lexsort((cand, d))][:10]
        assert np.allclose(sc, np.sort(d)[:10], rtol=1e-12)
    else:
        d = 1.0 - cdist(q[None, :], X[cand], "cosine")[0]
        d = np.where(np.isnan(d), 0.0, d)
        want = cand[np.lexsort((cand, -d))][:10]
        assert np.allclose(sc, np.sort(d)[::-1][:10], rtol=1e-12)
    assert np.array_equal(ids, want)


def test_rerank_pads_missing():
    X = np.eye(3)
    ids, sc = lsh.rerank(X[[2]], np.ones(3), np.array([2]), 3, "l2")
    assert ids.tolist() == [2, -1, -1] and np.isinf(sc[1:]).all()
