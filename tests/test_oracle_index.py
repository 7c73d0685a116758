"""Pins for grouping into buckets, lookup and the sharded-count arithmetic."""
import numpy as np

from oracle import lsh


def _build(scheme="CS_E2LSH", n=1000, d=64, m=16, L=2, K=8, dup=True):
    p = lsh.Params(scheme, d=d, m=m, L=L, K=K, w=4.0, seed=0)
    t = lsh.make_tables(p)
    X = np.random.default_rng(0).random((n, d)).astype(np.float32)
    if dup:
        X[10:20] = X[5]  # duplicates land in identical buckets
    out = lsh.hash_points(p, t, X)
    return p, t, X, out, lsh.group(out["keys"])


def test_each_id_once_per_table_and_soundness():
    for scheme in ("CS_E2LSH", "CS_SRP"):
        p, t, X, out, idx = _build(scheme)
        for tt, tix in enumerate(idx):
            assert sorted(tix.ids.tolist()) == list(range(1000))
            for b in range(tix.ukeys.size):
                mem = tix.ids[tix.offs[b]:tix.offs[b + 1]]
                assert np.all(out["keys"][tt, mem] == tix.ukeys[b])
                assert np.all(np.diff(mem.astype(np.int64)) > 0)  # ids ascending in bucket
            assert np.all(np.diff(tix.ukeys.astype(object)) > 0) if tix.ukeys.size > 1 else True


def test_sort_grouping_equals_dict_grouping():
    p, t, X, out, idx = _build()
    for tt in range(p.L):
        byk = {}
        for i, k in enumerate(out["keys"][tt].tolist()):
            byk.setdefault(k, []).append(i)
        assert {int(k): tix for k, tix in zip(idx[tt].ukeys.tolist(), range(idx[tt].ukeys.size))}.keys() == byk.keys()
        for b, k in enumerate(idx[tt].ukeys.tolist()):
            assert idx[tt].ids[idx[tt].offs[b]:idx[tt].offs[b + 1]].tolist() == byk[k]
        # buckets by fingerprint == buckets by exact K-tuple
        tup = lsh.group_by_tuple(out["codes"][:, tt * p.K:(tt + 1) * p.K])
        assert sorted(map(tuple, tup.values())) == sorted(map(tuple, byk.values()))


def test_duplicates_share_buckets_and_self_query():
    p, t, X, out, idx = _build()
    for tt in range(p.L):
        ks = out["keys"][tt]
        assert np.all(ks[10:20] == ks[5])
        for i in range(0, 1000, 37):
            b, e = lsh.lookup(idx[tt], int(ks[i]))
            assert i in idx[tt].ids[b:e].tolist()


def test_absent_key_empty_range():
    p, t, X, out, idx = _build()
    tix = idx[0]
    present = set(tix.ukeys.tolist())
    k = 12345
    while k in present:
        k += 1
    b, e = lsh.lookup(tix, k)
    assert b == e
    assert b == int(tix.offs[np.searchsorted(tix.ukeys, np.uint64(k))])


def test_empty_input():
    tix = lsh.group_table(np.zeros(0, np.uint64))
    assert tix.ids.size == 0 and tix.ukeys.size == 0 and tix.offs.tolist() == [0]
    assert lsh.lookup(tix, 5) == (0, 0)


def test_sharded_concatenation_equals_global():
    # §8(e): per-bucket rank-order concatenation of shard runs equals the G=1 run
    p, t, X, out, idx = _build(n=1000)
    G = 3
    bounds = [0, 300, 650, 1000]
    shards = [lsh.group(out["keys"][:, bounds[r]:bounds[r + 1]], id_base=bounds[r]) for r in range(G)]
    for tt in range(p.L):
        for b, k in enumerate(idx[tt].ukeys.tolist()):
            cat = []
            for r in range(G):
                bb, ee = lsh.lookup(shards[r][tt], k)
                cat += shards[r][tt].ids[bb:ee].tolist()
            assert cat == idx[tt].ids[idx[tt].offs[b]:idx[tt].offs[b + 1]].tolist()
    B = 4
    tot = sum(lsh.coarse_counts(p, out["keys"][:, bounds[r]:bounds[r + 1]], B) for r in range(G))
    assert np.array_equal(tot, lsh.coarse_counts(p, out["keys"], B))
    assert np.all(tot.sum(axis=1) == 1000)


def test_coarse_bins_monotone_in_key_order():
    p, t, X, out, idx = _build()
    for tix in idx:
        bins = [lsh.coarse_bin(k, 64, 12) for k in tix.ukeys.tolist()]
        assert bins == sorted(bins)
