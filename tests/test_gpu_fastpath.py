"""GPU parity of the KEYS-ONLY hot path — the kernel instantiations that
`lsh_build_index` and `bench.py` run (no debug outputs requested) — against the
oracle, on the same seeded inputs.

  * keys:   bit-exact for every (table, point) without an exempt coordinate
            (north_star: codes within 1e-5*w of a bin boundary / SRP projections
            within 1e-6 of zero are exempt, counted and reported);
  * tables: the built index equals the oracle's grouping of the oracle's keys, where
            only exempt keys may take the GPU's value (tables bit-exact given
            identical keys);
  * coverage: full n at C1, C2, C3; at C4 the first 20,000 rows
            plus 20,000 random rows, with the index built over all 10^6 rows.
Definitions: PAPER.md:205 (Def. CS, eq:eq_cs), :314 (Def. CS-E2LSH), :918 (Def.
CS-SRP), :212 / :624 / :1441 (HCS), :155 (the (m, L) index).  Exemption counts
and fingerprint merges are appended to the parity log (tests/conftest.py)."""
from __future__ import annotations

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import lsh  # noqa: E402
import synth  # noqa: E402

from . import parity  # noqa: E402

pytestmark = pytest.mark.gpu

# Exempt fraction bound: a code coordinate with continuous data is exempt with
# probability ~2e-5 at the 1e-5 band (an empty sum never is, tests/parity.py).  C2's
# values lie on the lattice k/255, so exact cancellations (+a - a: y = 0 in fp64, a
# rounding residue in fp32 in another summation order) put ~5e-4 of its SRP entries
# within 1e-6 of zero (measured on the oracle: 4.9e-4 exact zeros with nonzero terms).
CODE_EXEMPT_MAX = {"C2": 1e-3}
CODE_EXEMPT_DEFAULT = 1e-4


@pytest.fixture(scope="module", autouse=True)
def _lib():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2503_06737_b200 as pk
    pk.lib()
    yield


def _params(cfg: synth.Config, scheme: str) -> lsh.Params:
    kw = dict(mode_d=cfg.mode_d, mode_m=cfg.mode_m) if scheme.startswith("HCS") else {}
    return lsh.Params(scheme, d=cfg.d, m=cfg.m, L=cfg.L, K=cfg.K, w=cfg.w, seed=cfg.hash_seed, **kw)


def _handle(p: lsh.Params):
    import paper_2503_06737_b200 as pk
    kw = dict(mode_d=p.mode_d, mode_m=p.mode_m) if lsh.is_hcs(p.scheme) else {}
    return pk.LSH(p.scheme, p.d, p.m, p.L, p.K, p.w, p.seed, per_table=p.per_table, **kw)


def _u64(t) -> np.ndarray:
    return t.view(torch.int64).cpu().numpy().view(np.uint64)


def _oracle(p: lsh.Params, Xn: np.ndarray) -> dict:
    t = lsh.make_tables(p)
    ref = lsh.hash_points(p, t, Xn)
    ref["band"] = parity.code_band(p, t, Xn) if lsh.is_e2lsh(p.scheme) else parity.srp_band(p, t, Xn)
    return ref


def _check(p, ref, gkeys, what, parity_log):
    """keys rule + exemption bounds; returns the per-key exempt mask [L][n]."""
    kr = parity.check_keys(p, ref, gkeys)
    ex = parity.exempt_mask(p, ref)
    rep = {"test": what, "scheme": p.scheme, "keys": kr["n"], "key_mismatch": kr["mismatch"],
           "key_mismatch_outside_exempt": kr["mismatch_outside_exempt"], "exempt_keys": kr["exempt"],
           "code_entries": int(ex.size), "exempt_codes": int(ex.sum())}
    if lsh.is_e2lsh(p.scheme):
        rep["fingerprint_merges"] = int(lsh.fingerprint_merges(ref["codes"], ref["keys"], p.L, p.K)) \
            if ref["codes"].shape[0] <= 60000 else None
    parity_log(rep)
    assert kr["mismatch_outside_exempt"] == 0, rep
    bound = CODE_EXEMPT_MAX.get(what.split("/")[0], CODE_EXEMPT_DEFAULT)
    assert ex.sum() <= bound * max(1, ex.size), rep
    if rep.get("fingerprint_merges") is not None:
        assert rep["fingerprint_merges"] == 0, rep
    return ex.reshape(ex.shape[0], p.L, p.K).any(axis=2).T


def _check_tables_against_oracle_keys(idx, ref_keys, gkeys, ex_t, L, id_base=0):
    """Index == grouping of the oracle's keys, where exempt keys may take the GPU value."""
    keys = np.where(ex_t, gkeys, ref_keys)
    for t in range(L):
        r = lsh.group_table(keys[t], id_base)
        ids, uk, of = (x.cpu().numpy() for x in idx.view(t))
        assert np.array_equal(uk.astype(np.uint64), r.ukeys), t
        assert np.array_equal(of.astype(np.uint32), r.offs), t
        assert np.array_equal(ids.astype(np.uint32), r.ids), t


@pytest.mark.parametrize("cfg,scheme", [("C1", "CS_E2LSH"), ("C1", "CS_SRP"), ("C2", "CS_E2LSH"), ("C2", "CS_SRP"),
                                        ("C3", "CS_E2LSH"), ("C3", "CS_SRP"), ("C3", "HCS_E2LSH"),
                                        ("C3", "HCS_SRP")])
def test_keys_only_and_index_full_n(cfg, scheme, parity_log):
    """C1 runs the K = 8 fast kernel, C2 the K = 16 one, C3 CS the chunked plan and
    C3 HCS the slab kernel, all keys-only, as lsh_build_index calls them."""
    c = synth.CONFIGS[cfg]
    p = _params(c, scheme)
    h = _handle(p)
    X = synth.rows(c, 0, c.n, device="cuda")
    gk = _u64(h.hash(X, keys=True)["keys"])
    idx = h.build_index(X, id_base=0)
    torch.cuda.synchronize()
    h.check()
    ref = _oracle(p, X.cpu().numpy())
    ex_t = _check(p, ref, gk, f"{cfg}/keys_only_full_n", parity_log)
    _check_tables_against_oracle_keys(idx, ref["keys"], gk, ex_t, p.L)
    idx.close()


def _c4_rows(n: int) -> np.ndarray:
    g = np.random.default_rng(2024)
    return np.concatenate([np.arange(20000), np.sort(g.choice(np.arange(20000, n), 20000, replace=False))])


@pytest.mark.parametrize("scheme", ["CS_E2LSH", "CS_SRP"])
def test_c4_keys_only_and_index_sampled(scheme, parity_log):
    """C4 (n = 10^6, d = 960, m = 1024 = 64 x 16, w = 1) in the bench's launch
    configuration: keys of 40,000 sampled rows vs the oracle; the index over all rows
    equals the grouping of the kernel's keys in every table; every sampled row is
    found in the bucket of its ORACLE key in every table where that key is not exempt."""
    c = synth.CONFIGS["C4"]
    p = _params(c, scheme)
    h = _handle(p)
    X = synth.rows(c, 0, c.n, device="cuda")
    keys_dev = h.hash(X, keys=True)["keys"]
    idx = h.build_index(X, id_base=0)
    torch.cuda.synchronize()
    h.check()
    rows = _c4_rows(c.n)
    ri = torch.from_numpy(rows).cuda()
    ref = _oracle(p, X[ri].cpu().numpy())
    gk_all = _u64(keys_dev)
    ex_t = _check(p, ref, gk_all[:, rows], "C4/keys_only_sampled", parity_log)
    for t in range(p.L):
        r = lsh.group_table(gk_all[t])
        ids, uk, of = (x.cpu().numpy() for x in idx.view(t))
        assert np.array_equal(uk.astype(np.uint64), r.ukeys), t
        assert np.array_equal(of.astype(np.uint32), r.offs), t
        assert np.array_equal(ids.astype(np.uint32), r.ids), t
        tix = lsh.TableIndex(ids=ids.astype(np.uint32), ukeys=uk.astype(np.uint64), offs=of.astype(np.uint32))
        for j in np.nonzero(~ex_t[t])[0][::97]:
            b, e = lsh.lookup(tix, int(ref["keys"][t, j]))
            assert rows[j] in ids[b:e].tolist(), (t, rows[j])
    idx.close()


@pytest.mark.parametrize("scheme", ["CS_E2LSH", "CS_SRP"])
def test_c4_fast_path_equals_generic_path(scheme, parity_log):
    """Full C4: keys from the keys-only instantiation (pair gathers, biased fast floor)
    equal, bit for bit, the keys the generic instantiation computes when codes / bits
    are also requested (sequential bin sums, exact floor).  E2LSH: fingerprint merges
    (equal 64-bit keys over different K-code tuples, reading B10) counted over all
    10^6 points of every table from the generic path's codes."""
    c = synth.CONFIGS["C4"]
    p = _params(c, scheme)
    h = _handle(p)
    X = synth.rows(c, 0, c.n, device="cuda")
    k_fast = h.hash(X, keys=True)["keys"]
    out = h.hash(X, keys=True, codes=True, bits=True)
    torch.cuda.synchronize()
    h.check()
    assert torch.equal(k_fast.view(torch.int64), out["keys"].view(torch.int64))
    if lsh.is_e2lsh(scheme):
        merges, distinct = 0, 0
        codes = out["codes"]
        for t in range(p.L):
            kt = out["keys"][t].view(torch.int64)
            order = torch.argsort(kt, stable=True)
            ks = kt[order]
            ct = codes[:, t * p.K:(t + 1) * p.K][order]
            same_key = ks[1:] == ks[:-1]
            diff_tuple = (ct[1:] != ct[:-1]).any(dim=1)
            merges += int((same_key & diff_tuple).sum())
            distinct += int((~same_key).sum()) + 1
        parity_log({"test": "C4/fingerprint_merges_full_n", "scheme": scheme, "tables": p.L, "n": c.n,
                    "distinct_keys": distinct, "fingerprint_merges": merges})
        assert merges == 0


@pytest.mark.parametrize("scheme", ["HCS_E2LSH", "HCS_SRP"])
def test_c5_keys_only_sampled(scheme, parity_log):
    """C5 (d = 65536 = 16^4, m = 4096 = 8^4) keys-only at full n, 1000 + 1000 rows vs the oracle."""
    c = synth.CONFIGS["C5"]
    p = _params(c, scheme)
    h = _handle(p)
    X = synth.rows(c, 0, c.n, device="cuda")
    gk = _u64(h.hash(X, keys=True)["keys"])
    torch.cuda.synchronize()
    h.check()
    g = np.random.default_rng(5)
    rows = np.concatenate([np.arange(1000), np.sort(g.choice(np.arange(1000, c.n), 1000, replace=False))])
    Xs = X[torch.from_numpy(rows).cuda()].cpu().numpy()
    del X
    ref = _oracle(p, Xs)
    _check(p, ref, gk[:, rows], "C5/keys_only_sampled", parity_log)



@pytest.mark.parametrize("K,L,d,m", [(8, 5, 64, 40), (16, 3, 200, 48)])
def test_fast_path_large_codes_and_partial_table_groups(K, L, d, m, parity_log):
    """The E2LSH keys-only kernel takes four tables per warp (L % 4 != 0 here: clamped
    lanes compute but never fold or store) and four points per lane; a code outside
    the fast floor's range (|q| >= 2^22, here rows scaled by 10^5 among unscaled rows,
    ragged n) sends the lane's four points through the exact floor.  Keys equal the
    generic instantiation bit for bit and the oracle outside the exemption bands
    (Def. CS-E2LSH; reading B9, floor toward -inf)."""
    p = lsh.Params("CS_E2LSH", d=d, m=m, L=L, K=K, w=0.05, seed=11)
    h = _handle(p)
    X = synth.gaussian_rows_like(203, d, 17, device="cuda")
    X[3] *= 1e5
    X[41] *= 1e5
    X[200] *= -1e5
    k_fast = h.hash(X, keys=True)["keys"]
    out = h.hash(X, keys=True, codes=True)
    torch.cuda.synchronize()
    h.check()
    assert torch.equal(k_fast.view(torch.int64), out["keys"].view(torch.int64))
    codes = out["codes"].cpu().numpy()
    assert np.abs(codes).max() >= 4194304   # the exact-floor branch was taken
    ref = _oracle(p, X.cpu().numpy())
    kr = parity.check_keys(p, ref, _u64(k_fast))
    parity_log({"test": f"large_codes/K{K}_L{L}", "scheme": p.scheme, "keys": kr["n"],
                "key_mismatch_outside_exempt": kr["mismatch_outside_exempt"], "exempt_keys": kr["exempt"]})
    assert kr["mismatch_outside_exempt"] == 0, kr


@pytest.mark.parametrize("n", [200, 202, 203, 5])
@pytest.mark.parametrize("scheme,K,L,d,m", [("CS_E2LSH", 16, 6, 200, 96), ("CS_SRP", 16, 7, 200, 112),
                                            ("CS_E2LSH", 8, 5, 64, 40), ("CS_SRP", 8, 9, 64, 72)])
def test_four_table_key_store_forms(scheme, K, L, d, m, n, parity_log):
    """The four-table keys-only loop (both families) writes a lane's four keys with one
    256-bit store when (t n + row) * 8 is 32-byte aligned, else two 128-bit stores, else
    four 64-bit stores: n = 200 takes the 256-bit form in every table, n = 202 alternates
    256- / 128-bit by table parity, n = 203 mixes all three and has a ragged last quad,
    n = 5 is a single partial tile.  Keys equal the generic instantiation bit for bit and
    the oracle outside the exemption bands (PAPER.md:314 Def. CS-E2LSH, :918 Def. CS-SRP;
    :155 the table keys)."""
    p = lsh.Params(scheme, d=d, m=m, L=L, K=K, w=0.7, seed=23)
    h = _handle(p)
    X = synth.gaussian_rows_like(n, d, 29, device="cuda")
    k_fast = h.hash(X, keys=True)["keys"]
    dbg = dict(codes=True) if lsh.is_e2lsh(scheme) else dict(bits=True)
    k_gen = h.hash(X, keys=True, **dbg)["keys"]
    torch.cuda.synchronize()
    h.check()
    assert torch.equal(k_fast.view(torch.int64), k_gen.view(torch.int64))
    ref = _oracle(p, X.cpu().numpy())
    kr = parity.check_keys(p, ref, _u64(k_fast))
    parity_log({"test": f"store_forms/{scheme}_K{K}_n{n}", "scheme": p.scheme, "keys": kr["n"],
                "key_mismatch_outside_exempt": kr["mismatch_outside_exempt"], "exempt_keys": kr["exempt"]})
    assert kr["mismatch_outside_exempt"] == 0, kr


@pytest.mark.parametrize("scheme", ["CS_E2LSH", "CS_SRP"])
def test_c4_query_buckets(scheme):
    """Query lookup at the bench's scale (10^6 buckets per E2LSH table, where the
    interpolation-guided probes run before the binary search): (begin, end) of 1000
    indexed points and 1000 fresh points in every table equal the lower-bound lookup of
    their keys in the built tables (the bucket hbar_t(q)); indexed points
    find themselves."""
    c = synth.CONFIGS["C4"]
    p = _params(c, scheme)
    h = _handle(p)
    X = synth.rows(c, 0, c.n, device="cuda")
    idx = h.build_index(X, id_base=0)
    Q = torch.cat([X[:1000], synth.gaussian_rows_like(1000, c.d, 91, device="cuda")])
    b, e = h.query_buckets(idx, Q)
    qk = _u64(h.hash(Q, keys=True)["keys"])
    torch.cuda.synchronize()
    b, e = b.cpu().numpy(), e.cpu().numpy()
    for t in range(p.L):
        ids, uk, of = (x.cpu().numpy() for x in idx.view(t))
        uk = uk.astype(np.uint64)
        of = of.astype(np.int64)
        pos = np.searchsorted(uk, qk[t], side="left")
        hit = (pos < uk.shape[0]) & (uk[np.minimum(pos, uk.shape[0] - 1)] == qk[t])
        eb = of[pos]
        ee = np.where(hit, of[np.minimum(pos + 1, of.shape[0] - 1)], eb)
        assert np.array_equal(b[:, t], eb), t
        assert np.array_equal(e[:, t], ee), t
        for q in range(0, 1000, 37):
            assert q in ids[b[q, t]:e[q, t]].tolist(), (t, q)
    idx.close()
