"""GPU parity: the CUDA path (through the C ABI) against the oracle, element by
element on the same seeded inputs.  Marked `gpu`: runs on a B200 only."""
from __future__ import annotations

import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import lsh  # noqa: E402
import synth  # noqa: E402

from . import parity  # noqa: E402

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _lib():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2503_06737_b200 as pk
    pk.lib()
    yield


def _handle(p: lsh.Params):
    import paper_2503_06737_b200 as pk
    kw = dict(mode_d=p.mode_d, mode_m=p.mode_m) if lsh.is_hcs(p.scheme) else {}
    return pk.LSH(p.scheme, p.d, p.m, p.L, p.K, p.w, p.seed, per_table=p.per_table, **kw)


def _params(cfg: synth.Config, scheme: str) -> lsh.Params:
    kw = dict(mode_d=cfg.mode_d, mode_m=cfg.mode_m) if scheme.startswith("HCS") else {}
    return lsh.Params(scheme, d=cfg.d, m=cfg.m, L=cfg.L, K=cfg.K, w=cfg.w, seed=cfg.hash_seed, **kw)


def _compare(p: lsh.Params, X_dev, X_np, h=None, rows=None, report=None):
    """Hash X_dev on the GPU, compare proj / codes|bits / keys with the oracle on X_np."""
    h = h or _handle(p)
    out = h.hash(X_dev, keys=True, codes=True, bits=True, proj=True)
    torch.cuda.synchronize()
    h.check()
    sel = slice(None) if rows is None else rows
    gk = out["keys"].cpu().numpy()[:, sel]
    gp = out["proj"].cpu().numpy()[sel]
    t = lsh.make_tables(p)
    ref = lsh.hash_points(p, t, X_np)
    pr = parity.check_proj(gp, ref["proj"], parity.sigma(p, t, X_np))
    assert pr["bad"] == 0 and pr["bad_empty"] == 0, pr
    ref["band"] = parity.code_band(p, t, X_np) if lsh.is_e2lsh(p.scheme) else parity.srp_band(p, t, X_np)
    if lsh.is_e2lsh(p.scheme):
        cr = parity.check_codes(p, ref, gpu_codes=out["codes"].cpu().numpy()[sel])
    else:
        cr = parity.check_codes(p, ref, gpu_bits=parity.unpack_bits(out["bits"].cpu().numpy()[sel], p.m))
    assert cr["mismatch_outside_exempt"] == 0, cr
    kr = parity.check_keys(p, ref, gk)
    assert kr["mismatch_outside_exempt"] == 0, kr
    if report is not None:
        report.update(proj=pr, codes=cr, keys=kr)
    return h, out, ref


@pytest.mark.parametrize("cfg,scheme", [("C1", "CS_E2LSH"), ("C1", "CS_SRP"), ("C2", "CS_E2LSH"),
                                        ("C2", "CS_SRP"), ("C2", "E2LSH"), ("C2", "SRP"),
                                        ("C3", "HCS_E2LSH"), ("C3", "HCS_SRP"), ("C3", "CS_E2LSH"),
                                        ("C3", "CS_SRP")])
def test_config_full_n(cfg, scheme):
    c = synth.CONFIGS[cfg]
    p = _params(c, scheme)
    X = synth.rows(c, 0, c.n, device="cuda")
    _compare(p, X, X.cpu().numpy())


@pytest.mark.parametrize("scheme", ["CS_E2LSH", "CS_SRP"])
def test_c4_full_size_sampled(scheme):
    """C4 at full n=1e6 in the bench's launch configuration; oracle on sampled rows."""
    c = synth.CONFIGS["C4"]
    p = _params(c, scheme)
    X = synth.rows(c, 0, c.n, device="cuda")
    h = _handle(p)
    out = h.hash(X, keys=True, codes=True, bits=True, proj=True)
    torch.cuda.synchronize()
    g = np.random.default_rng(0)
    rows = np.concatenate([np.arange(4096), np.sort(g.choice(np.arange(4096, c.n), 4096, replace=False))])
    Xs = X[torch.from_numpy(rows).cuda()].cpu().numpy()
    t = lsh.make_tables(p)
    ref = lsh.hash_points(p, t, Xs)
    pr = parity.check_proj(out["proj"][torch.from_numpy(rows).cuda()].cpu().numpy(), ref["proj"],
                           parity.sigma(p, t, Xs))
    assert pr["bad"] == 0 and pr["bad_empty"] == 0, pr
    kr = parity.check_keys(p, ref, out["keys"].view(torch.int64)[:, torch.from_numpy(rows).cuda()].cpu().numpy()
                           .view(np.uint64))
    assert kr["mismatch_outside_exempt"] == 0, kr


@pytest.mark.parametrize("n", [0, 1, 31, 33, 1000])
@pytest.mark.parametrize("scheme,d,m,L,K,kw", [
    ("CS_E2LSH", 64, 16, 2, 8, {}),
    ("CS_SRP", 50, 24, 3, 8, {}),                                   # d % 4 != 0: scalar staging path
    ("HCS_E2LSH", 60, 24, 3, 8, dict(mode_d=(4, 4, 4), mode_m=(2, 3, 4))),   # zero padding, unequal modes
    ("CS_E2LSH", 1500, 64, 4, 16, {}),                              # multi-chunk, ragged last chunk
    ("SRP", 37, 40, 5, 8, {}),
])
def test_edge_shapes(n, scheme, d, m, L, K, kw):
    p = lsh.Params(scheme, d=d, m=m, L=L, K=K, w=2.5, seed=7, **kw)
    X = synth.gaussian_rows_like(n, d, 3, device="cuda")
    if n == 0:
        h = _handle(p)
        out = h.hash(X, keys=True)
        assert out["keys"].shape == (L, 0)
        return
    _compare(p, X, X.cpu().numpy())


def test_padded_rows_and_unaligned_pointer():
    p = lsh.Params("CS_E2LSH", d=64, m=16, L=2, K=8, w=4.0, seed=1)
    big = synth.gaussian_rows_like(300, 72, 5, device="cuda")
    X = big[:, :64]                     # ld = 72 > d
    _compare(p, X, X.cpu().numpy())
    X2 = big.view(-1)[1:1 + 299 * 72].view(299, 72)[:, :64]  # misaligned base -> scalar path
    _compare(p, X2, X2.cpu().numpy())


def test_zero_and_duplicate_points():
    for scheme in ("CS_E2LSH", "CS_SRP", "HCS_SRP"):
        kw = dict(mode_d=(8, 8), mode_m=(4, 4)) if scheme.startswith("HCS") else {}
        p = lsh.Params(scheme, d=64, m=16, L=1, K=16, w=4.0, seed=2, **kw)
        X = synth.gaussian_rows_like(100, 64, 9, device="cuda")
        X[0:10] = 0
        X[20:40] = X[19]
        _h, out, ref = _compare(p, X, X.cpu().numpy())
        keys = out["keys"].cpu().numpy()
        assert np.all(keys[:, 20:40] == keys[:, 19:20])


def test_overflow_flag():
    import paper_2503_06737_b200 as pk
    p = lsh.Params("CS_E2LSH", d=64, m=16, L=2, K=8, w=1e-6, seed=1)
    h = _handle(p)
    X = torch.full((32, 64), 1e6, device="cuda")
    h.hash(X, keys=True)
    with pytest.raises(pk.LshError) as e:
        h.check()
    assert e.value.status == 5
    h.check()  # sticky flag cleared


def test_device_params_equal_oracle():
    for scheme, kw in [("CS_E2LSH", {}), ("HCS_SRP", dict(mode_d=(16, 16, 16), mode_m=(8, 8, 8))),
                       ("E2LSH", {})]:
        d = 4096 if scheme.startswith("HCS") else 784
        p = lsh.Params(scheme, d=d, m=512 if scheme.startswith("HCS") else 160,
                       L=32 if scheme.startswith("HCS") else 10, K=16, w=4.0, seed=3, **kw)
        h = _handle(p)
        t = lsh.make_tables(p)
        assert np.array_equal(h.get_params("offsets").view(np.uint32), t.b.view(np.uint32))
        if lsh.is_dense(scheme):
            got = (h.get_params("gaussian").astype(np.uint32) << 16).view(np.float32)
            assert np.array_equal(got, t.R.astype(np.float32).ravel())
        else:
            for k in range(p.N):
                assert np.array_equal(h.get_params("bucket", k), t.h[k])
                assert np.array_equal(h.get_params("sign", k), t.s[k])


# ---------------------------------------------------------------- grouping --

def _check_index(idx, ref_tables, L):
    for tt in range(L):
        ids, uk, of = (x.cpu().numpy() for x in idx.view(tt))
        r = ref_tables[tt]
        assert np.array_equal(uk.astype(np.uint64), r.ukeys), tt
        assert np.array_equal(of.astype(np.uint32), r.offs), tt
        assert np.array_equal(ids.astype(np.uint32), r.ids), tt


@pytest.mark.parametrize("scheme,K,n", [("CS_E2LSH", 16, 60000), ("CS_SRP", 16, 60000), ("CS_SRP", 8, 5000),
                                        ("CS_SRP", 24, 20000), ("CS_E2LSH", 8, 1)])
def test_group_keys_bit_exact_given_oracle_keys(scheme, K, n):
    L = 4
    p = lsh.Params(scheme, d=64, m=L * K, L=L, K=K, w=4.0, seed=0)
    h = _handle(p)
    g = np.random.default_rng(1)
    if lsh.is_e2lsh(scheme):
        keys = g.integers(0, 2 ** 63, (L, n), dtype=np.int64).astype(np.uint64) * np.uint64(2) + \
            g.integers(0, 2, (L, n)).astype(np.uint64)
        keys[:, : n // 3] = keys[:, :1]          # a large equal-key bucket
        keys[:, n // 2: n // 2 + 100] = (keys[:, n // 2: n // 2 + 100] >> np.uint64(40)) << np.uint64(40)
    else:
        keys = g.integers(0, 1 << K, (L, n)).astype(np.uint64)
        keys[:, ::7] = 5                          # skewed bucket
    idx = h.group_keys(torch.from_numpy(keys.view(np.int64)).cuda().view(torch.uint64), id_base=17)
    ref = lsh.group(keys, id_base=17)
    _check_index(idx, ref, L)
    h.check()


@pytest.mark.parametrize("cfg,scheme", [("C2", "CS_E2LSH"), ("C2", "CS_SRP"), ("C3", "HCS_SRP"),
                                        ("C1", "CS_E2LSH")])
def test_build_index_and_query(cfg, scheme):
    c = synth.CONFIGS[cfg]
    p = _params(c, scheme)
    h = _handle(p)
    X = synth.rows(c, 0, c.n, device="cuda")
    keys = h.hash(X, keys=True)["keys"].cpu().numpy()
    idx = h.build_index(X, id_base=0)
    _check_index(idx, lsh.group(keys), p.L)
    # queries: a subset of the indexed points plus fresh points
    Q = torch.cat([X[:500], synth.gaussian_rows_like(100, c.d, 77, device="cuda").abs()])
    b, e = h.query_buckets(idx, Q)
    qk = h.hash(Q, keys=True)["keys"].cpu().numpy()
    ref = lsh.group(keys)
    b, e = b.cpu().numpy(), e.cpu().numpy()
    for q in range(Q.shape[0]):
        for tt in range(p.L):
            assert (b[q, tt], e[q, tt]) == lsh.lookup(ref[tt], int(qk[tt, q]))
    for q in range(500):  # self-retrieval
        for tt in range(p.L):
            ids = idx.view(tt)[0].cpu().numpy()[b[q, tt]:e[q, tt]]
            assert q in ids.tolist()
    # coarse counts (multi-GPU exchange)
    for B in (4, 12):
        cnt = idx.counts(B).cpu().numpy().astype(np.uint32)
        assert np.array_equal(cnt, lsh.coarse_counts(p, keys, B))


def test_empty_index():
    p = lsh.Params("CS_SRP", d=64, m=16, L=2, K=8, seed=0)
    h = _handle(p)
    idx = h.build_index(torch.zeros((0, 64), device="cuda"))
    ids, uk, of = idx.view(0)
    assert ids.numel() == 0 and uk.numel() == 0 and of.cpu().tolist() == [0]


@pytest.mark.parametrize("scheme", ["HCS_E2LSH", "HCS_SRP"])
def test_c5_full_size_sampled(scheme):
    """C5 (d = 65536 = 16^4, m = 4096 = 8^4): chunked/grouped plan at full n, sampled rows."""
    c = synth.CONFIGS["C5"]
    p = _params(c, scheme)
    h = _handle(p)
    X = synth.rows(c, 0, c.n, device="cuda")
    keys = h.hash(X, keys=True)["keys"]
    torch.cuda.synchronize()
    h.check()
    g = np.random.default_rng(5)
    rows = np.concatenate([np.arange(96), np.sort(g.choice(np.arange(96, c.n), 96, replace=False))])
    ridx = torch.from_numpy(rows).cuda()
    Xs = X[ridx].contiguous()
    del X
    # full debug comparison on the sampled rows (same kernels, smaller launch)
    _h, out, ref = _compare(p, Xs, Xs.cpu().numpy(), h=h)
    kr = parity.check_keys(p, ref, keys.view(torch.int64)[:, ridx].cpu().numpy().view(np.uint64))
    assert kr["mismatch_outside_exempt"] == 0, kr


@pytest.mark.parametrize("scheme,d,m,L,K", [("CS_E2LSH", 2100, 2048, 128, 16), ("CS_SRP", 3000, 4096, 256, 16),
                                            ("HCS_SRP", 6000, 1024, 64, 16)])
def test_grouped_chunked_plans(scheme, d, m, L, K):
    kw = dict(mode_d=(10, 25, 25), mode_m=(8, 8, 16)) if scheme.startswith("HCS") else {}
    p = lsh.Params(scheme, d=d, m=m, L=L, K=K, w=3.0, seed=11, **kw)
    X = synth.gaussian_rows_like(333, d, 21, device="cuda")
    _compare(p, X, X.cpu().numpy())


@pytest.mark.parametrize("G,L,B", [(1, 3, 4), (4, 7, 12), (8, 64, 12), (3, 2, 20)])
def test_global_offsets_kernel(G, L, B):
    import paper_2503_06737_b200 as pk
    g = np.random.default_rng(G * 100 + B)
    allc = g.integers(0, 1000, (G, L, 1 << B)).astype(np.int32)
    dev = torch.from_numpy(allc).cuda()
    for r in range(G):
        got = pk.global_offsets(dev, r).cpu().numpy()
        assert np.array_equal(got, lsh.global_coarse_offsets(allc, r)), r


def test_build_index_sharded_single_rank():
    from paper_2503_06737_b200.dist import build_index_sharded
    c = synth.CONFIGS["C2"]
    p = _params(c, "CS_SRP")
    h = _handle(p)
    X = synth.rows(c, 0, 5000, device="cuda")
    sh = build_index_sharded(h, X, id_base=0, B=8)
    keys = h.hash(X, keys=True)["keys"].cpu().numpy()
    assert np.array_equal(sh.counts.cpu().numpy().astype(np.uint32), lsh.coarse_counts(p, keys, 8))
    assert np.array_equal(sh.offsets.cpu().numpy(), lsh.global_coarse_offsets(sh.all_counts.cpu().numpy(), 0))


def test_c5_dense_e2lsh_tensor_core_sampled():
    """Dense E2LSH baseline at C5 shape (d = 65536, m = 4096): tcgen05 bf16x3 GEMM."""
    c = synth.CONFIGS["C5"]
    p = lsh.Params("E2LSH", d=c.d, m=c.m, L=c.L, K=c.K, w=c.w, seed=c.hash_seed)
    rows = np.concatenate([np.arange(40), np.array([5000, 77777, 99999])])
    Xs = synth.sample_rows(c, rows, device="cuda")
    _compare(p, Xs, Xs.cpu().numpy())


@pytest.mark.parametrize("m,L,K", [(160, 10, 16), (256, 16, 16), (520, 65, 8), (48, 3, 16)])
def test_dense_tensor_core_shapes(m, L, K):
    """Tile-edge shapes of the tcgen05 GEMM: m not a multiple of the N tile, d not of 64."""
    for scheme in ("E2LSH", "SRP"):
        p = lsh.Params(scheme, d=300, m=m, L=L, K=K, w=2.0, seed=9)
        X = synth.gaussian_rows_like(333, 300, 4, device="cuda")
        _compare(p, X, X.cpu().numpy())


def test_group_long_equal_prefix_segments():
    """Many keys sharing their top 16 bits (long segments -> CTA radix path), ties by id."""
    p = lsh.Params("CS_E2LSH", d=64, m=32, L=2, K=16, w=4.0, seed=0)
    h = _handle(p)
    g = np.random.default_rng(3)
    n = 50000
    keys = g.integers(0, 2 ** 62, (2, n), dtype=np.int64).astype(np.uint64)
    pref = np.uint64(0xABCD) << np.uint64(48)
    keys[0, :30000] = pref | g.integers(0, 50, 30000).astype(np.uint64)          # 50 distinct low parts
    keys[1, 10000:20000] = pref | (g.integers(0, 3, 10000).astype(np.uint64) << np.uint64(40))
    keys[1, 30000:39000] = keys[1, 30000]                                             # all equal
    idx = h.group_keys(torch.from_numpy(keys.view(np.int64)).cuda().view(torch.uint64), id_base=5)
    _check_index(idx, lsh.group(keys, id_base=5), 2)
    h.check()


def _structured_keys(kind: str, L: int, n: int, g) -> np.ndarray:
    u64 = np.uint64
    if kind == "uniform":
        return g.integers(0, 2 ** 63, (L, n), dtype=np.int64).astype(u64) * u64(2) + g.integers(0, 2, (L, n)).astype(u64)
    if kind == "smem_long_segments":
        # inside one L1 bin: > 64 keys sharing the next 16 bits but differing below (and duplicates)
        k = _structured_keys("uniform", L, n, g)
        pref = u64(0x5A5A5) << u64(44)
        k[:, 100:700] = pref | g.integers(0, 40, (L, 600)).astype(u64) << u64(3)
        k[:, 900:1000] = pref | u64(7)
        return k
    if kind == "big_bin_no_dominant":
        # one L1 bin far larger than shared memory, keys spread (no 3-way split)
        k = g.integers(0, 2 ** 62, (L, n), dtype=np.int64).astype(u64)
        k[:, : n // 2] = (u64(3) << u64(60)) | g.integers(0, 2 ** 20, (L, n // 2)).astype(u64) << u64(7)
        return k
    if kind == "all_equal":
        return np.full((L, n), 0xDEADBEEF12345678, dtype=u64)
    if kind == "two_values":
        return np.where(g.integers(0, 2, (L, n)) == 1, u64(2 ** 63 + 5), u64(5)).astype(u64)
    raise ValueError(kind)


@pytest.mark.parametrize("kind,n", [("uniform", 4097), ("uniform", 300001), ("smem_long_segments", 6000),
                                    ("big_bin_no_dominant", 40000), ("all_equal", 20000), ("two_values", 9000)])
def test_group_keys_structures(kind, n):
    """L1 MSD scatter + per-bin sort paths: shared-memory bins with long equal-prefix
    segments, bins larger than shared memory with and without a dominant key, ragged tiles."""
    L = 3
    p = lsh.Params("CS_E2LSH", d=64, m=L * 16, L=L, K=16, w=4.0, seed=0)
    h = _handle(p)
    keys = _structured_keys(kind, L, n, np.random.default_rng(n))
    idx = h.group_keys(torch.from_numpy(keys.view(np.int64)).cuda().view(torch.uint64), id_base=3)
    _check_index(idx, lsh.group(keys, id_base=3), L)
    h.check()


@pytest.mark.parametrize("K,n", [(1, 5000), (3, 70000), (11, 100000), (40, 30000)])
def test_group_keys_srp_widths(K, n):
    """SRP keys are K bits wide: the L1 digit never exceeds the key width."""
    L = 2
    p = lsh.Params("CS_SRP", d=64, m=L * K, L=L, K=K, w=4.0, seed=0)
    h = _handle(p)
    g = np.random.default_rng(K)
    keys = g.integers(0, 2 ** min(K, 62), (L, n), dtype=np.int64).astype(np.uint64)
    keys[:, ::5] = keys[0, 0]
    idx = h.group_keys(torch.from_numpy(keys.view(np.int64)).cuda().view(torch.uint64), id_base=0)
    _check_index(idx, lsh.group(keys, id_base=0), L)


@pytest.mark.parametrize("scheme", ["HCS_E2LSH", "HCS_SRP"])
@pytest.mark.parametrize("n,mode_d,mode_m,K", [
    (333, (16, 16, 16), (8, 8, 8), 16),          # C3 shape: slab 256, block 64 bins = 4 tables
    (65, (8, 8, 4, 2), (4, 4, 2, 2), 8),         # N = 4, slab 64, block 16 bins
    (97, (4, 16, 8, 3), (8, 8, 3, 2), 16),       # unequal outer modes (empty blocks likely)
    (31, (16, 8, 2, 2, 3), (4, 8, 2, 2, 2), 16), # N = 5, block 32 bins
])
def test_hcs_slab_kernel(scheme, n, mode_d, mode_m, K):
    """HCS slab kernel (Kronecker-structured staging): every shape it accepts,
    ragged tiles, both families; compared with the oracle like every other path."""
    d = int(np.prod(mode_d))
    m = int(np.prod(mode_m))
    p = lsh.Params(scheme, d=d, m=m, L=m // K, K=K, w=2.0, seed=13, mode_d=mode_d, mode_m=mode_m)
    X = synth.gaussian_rows_like(n, d, 8, device="cuda")
    _compare(p, X, X.cpu().numpy())


def test_hcs_slab_matches_generic_fallback(monkeypatch):
    """The generic chunked plan (fallback for unaligned inputs) gives the same keys."""
    c = synth.CONFIGS["C3"]
    p = _params(c, "HCS_E2LSH")
    h = _handle(p)
    X = synth.rows(c, 0, 2000, device="cuda")
    k1 = h.hash(X, keys=True)["keys"].cpu().numpy()
    monkeypatch.setenv("LSH_NO_HCS_SLAB", "1")
    k2 = h.hash(X, keys=True)["keys"].cpu().numpy()
    ref = lsh.hash_points(p, lsh.make_tables(p), X.cpu().numpy())
    r1 = parity.check_keys(p, ref, k1.view(np.uint64))
    r2 = parity.check_keys(p, ref, k2.view(np.uint64))
    assert r1["mismatch_outside_exempt"] == 0 and r2["mismatch_outside_exempt"] == 0, (r1, r2)


@pytest.mark.parametrize("cfg,scheme,tables", [("C4", "CS_E2LSH", (0, 17, 63)), ("C4", "CS_SRP", (0, 31, 63)),
                                               ("C5", "HCS_E2LSH", (0, 1, 128, 255))])
def test_full_size_index_tables(cfg, scheme, tables):
    """Index build at full n in the bench's launch configuration: selected tables are
    bit-exact against the oracle's grouping of the same keys (tables rule, §5), and
    bucket lookups of sampled points return their own buckets."""
    c = synth.CONFIGS[cfg]
    p = _params(c, scheme)
    h = _handle(p)
    X = synth.rows(c, 0, c.n, device="cuda")
    idx = h.build_index(X, id_base=0)
    keys = h.hash(X, keys=True)["keys"]
    torch.cuda.synchronize()
    h.check()
    for tt in tables:
        kt = keys[tt].view(torch.int64).cpu().numpy().view(np.uint64)[None, :]
        ref = lsh.group(kt)[0]
        ids, uk, of = (x.cpu().numpy() for x in idx.view(tt))
        assert np.array_equal(uk.astype(np.uint64), ref.ukeys), tt
        assert np.array_equal(of.astype(np.uint32), ref.offs), tt
        assert np.array_equal(ids.astype(np.uint32), ref.ids), tt
    rows = torch.from_numpy(np.random.default_rng(1).choice(c.n, 64, replace=False)).cuda()
    b, e = h.query_buckets(idx, X[rows].contiguous())
    b, e = b.cpu().numpy(), e.cpu().numpy()
    for tt in tables:
        ids = idx.view(tt)[0].cpu().numpy()
        for qi, r in enumerate(rows.cpu().numpy()):
            assert r in ids[b[qi, tt]:e[qi, tt]].tolist()
    idx.close()


def _knn_check(p, X, Q, k, max_cand, rtol=1e-4):
    """GPU query_knn vs the oracle's union/rerank on the same keys (NEXT-1)."""
    h = _handle(p)
    idx = h.build_index(X, id_base=0)
    ids, sc, nc = h.query_knn(idx, X, Q, k, max_cand=max_cand)
    torch.cuda.synchronize()
    keys = h.hash(X, keys=True)["keys"].view(torch.int64).cpu().numpy().view(np.uint64)
    qkeys = h.hash(Q, keys=True)["keys"].view(torch.int64).cpu().numpy().view(np.uint64)
    tables = lsh.group(keys, id_base=0)
    Xn, Qn = X.cpu().numpy(), Q.cpu().numpy()
    ids, sc, nc = ids.cpu().numpy(), sc.cpu().numpy(), nc.cpu().numpy()
    metric = lsh.metric_of(p)
    stats = {"queries": Q.shape[0], "empty": 0, "ties": 0}
    for qi in range(Q.shape[0]):
        cand = lsh.query_candidates(tables, qkeys[:, qi], max_cand)
        assert nc[qi] == len(cand), qi
        if len(cand) == 0:
            stats["empty"] += 1
            assert (ids[qi] == -1).all()
            continue
        rid, rsc = lsh.rerank(Xn[cand], Qn[qi], cand, k, metric)
        kk = min(k, len(cand))
        assert (ids[qi, kk:] == -1).all() and (ids[qi, :kk] >= 0).all(), qi
        assert set(ids[qi, :kk].tolist()) <= set(cand.tolist()), qi
        # every reported score is the exact score of that id within the fp32 tolerance
        aid, asc = lsh.rerank(Xn[cand], Qn[qi], cand, len(cand), metric)
        full = dict(zip(aid.tolist(), asc.tolist()))
        for j in range(kk):
            ref = full[int(ids[qi, j])]
            assert abs(sc[qi, j] - ref) <= rtol * max(1.0, abs(ref)), (qi, j, sc[qi, j], ref)
        # same top-k except near-ties at the k-th score
        kth = rsc[kk - 1]
        band = rtol * max(1.0, abs(kth))
        sure = {int(i) for i, s in zip(cand.tolist(), [full[c] for c in cand.tolist()])
                if (s < kth - band if metric == "l2" else s > kth + band)}
        got = set(ids[qi, :kk].tolist())
        assert sure <= got, (qi, sure - got)
        stats["ties"] += int(got != set(rid[:kk].tolist()))
    idx.close()
    return stats


@pytest.mark.parametrize("cfg,scheme,k,max_cand", [("C2", "CS_E2LSH", 10, 4096), ("C2", "CS_SRP", 20, 512),
                                                   ("C3", "HCS_E2LSH", 10, 2048), ("C3", "HCS_SRP", 5, 8192),
                                                   ("C1", "CS_E2LSH", 7, 64)])
def test_query_knn_matches_oracle(cfg, scheme, k, max_cand):
    """NEXT-1 query completion: union of the L buckets (table order, capped), distinct ids,
    exact re-rank, top-k (squared L2 for E2LSH, cosine for SRP), ties by id."""
    c = synth.CONFIGS[cfg]
    p = _params(c, scheme)
    n = min(c.n, 8000)
    X = synth.rows(c, 0, n, device="cuda")
    g = torch.Generator(device="cuda").manual_seed(11)
    Q = torch.cat([X[:40], X[100:140] + 0.01 * torch.randn((40, c.d), device="cuda", generator=g),
                   synth.gaussian_rows_like(8, c.d, 123, device="cuda") * 50.0]).contiguous()
    st = _knn_check(p, X, Q, k, max_cand)
    assert st["empty"] < Q.shape[0]


def test_query_knn_self_is_first_and_errors():
    import paper_2503_06737_b200 as pk
    c = synth.CONFIGS["C2"]
    p = _params(c, "CS_E2LSH")
    h = _handle(p)
    X = synth.rows(c, 0, 3000, device="cuda")
    idx = h.build_index(X, id_base=0)
    ids, sc, nc = h.query_knn(idx, X, X[:64].contiguous(), 3)
    ids, sc = ids.cpu().numpy(), sc.cpu().numpy()
    # a point's own row is at distance 0: first unless another row is identical (lower id)
    for q in range(64):
        assert sc[q, 0] == 0.0 and (ids[q, 0] == q or (X[ids[q, 0]] == X[q]).all().item())
    with pytest.raises(pk.LshError):
        h.query_knn(idx, X, X[:2].contiguous(), 9000, max_cand=9000)
    idx.close()


# ---- NEXT-2: per-table independent families (reading C3) --------------------------

def _pt_params(cfg: synth.Config, scheme: str) -> lsh.Params:
    return lsh.Params(scheme, d=cfg.d, m=cfg.m, L=cfg.L, K=cfg.K, w=cfg.w, seed=cfg.hash_seed, per_table=True)


@pytest.mark.parametrize("cfg,scheme", [("C1", "CS_E2LSH"), ("C1", "CS_SRP"), ("C2", "CS_E2LSH"), ("C2", "CS_SRP")])
def test_per_table_config_full_n(cfg, scheme):
    c = synth.CONFIGS[cfg]
    p = _pt_params(c, scheme)
    X = synth.rows(c, 0, c.n, device="cuda")
    _compare(p, X, X.cpu().numpy())


@pytest.mark.parametrize("n", [1, 33, 1000])
@pytest.mark.parametrize("scheme,d,L,K", [("CS_E2LSH", 300, 5, 8), ("CS_SRP", 37, 3, 16), ("CS_E2LSH", 64, 24, 1)])
def test_per_table_edge_shapes(n, scheme, d, L, K):
    """m not a multiple of the GEMM's N tile, d not of 64, K = 1 (one bin per table)."""
    p = lsh.Params(scheme, d=d, m=L * K, L=L, K=K, w=2.5, seed=7, per_table=True)
    X = synth.gaussian_rows_like(n, d, 3, device="cuda")
    _compare(p, X, X.cpu().numpy())


def test_per_table_differs_from_shared_sketch():
    """The flag really switches families: same seed, different keys than the shared sketch."""
    c = synth.CONFIGS["C1"]
    X = synth.rows(c, 0, 256, device="cuda")
    kp = _handle(_pt_params(c, "CS_SRP")).hash(X, keys=True)["keys"].cpu().numpy()
    ks = _handle(_params(c, "CS_SRP")).hash(X, keys=True)["keys"].cpu().numpy()
    assert (kp != ks).mean() > 0.5


@pytest.mark.parametrize("scheme", ["CS_E2LSH", "CS_SRP"])
def test_per_table_build_index_and_knn(scheme):
    c = synth.CONFIGS["C2"]
    p = _pt_params(c, scheme)
    h = _handle(p)
    X = synth.rows(c, 0, c.n, device="cuda")
    keys = h.hash(X, keys=True)["keys"].cpu().numpy()
    idx = h.build_index(X, id_base=0)
    _check_index(idx, lsh.group(keys), p.L)
    idx.close()
    _knn_check(p, X, X[:64], 10, 1024)


@pytest.mark.parametrize("scheme", ["CS_E2LSH", "CS_SRP"])
def test_per_table_c4_full_size_sampled(scheme):
    """C4 shape (n = 1e6, d = 960, L = 64, K = 16) with per-table families, sampled rows."""
    c = synth.CONFIGS["C4"]
    p = _pt_params(c, scheme)
    X = synth.rows(c, 0, c.n, device="cuda")
    h = _handle(p)
    out = h.hash(X, keys=True, proj=True)
    torch.cuda.synchronize()
    rows = np.concatenate([np.arange(512), np.array([131071, 500000, 999999])])
    ri = torch.from_numpy(rows).cuda()
    Xs = X[ri].cpu().numpy()
    t = lsh.make_tables(p)
    ref = lsh.hash_points(p, t, Xs)
    pr = parity.check_proj(out["proj"][ri].cpu().numpy(), ref["proj"], parity.sigma(p, t, Xs))
    assert pr["bad"] == 0 and pr["bad_empty"] == 0, pr
    ref["band"] = parity.code_band(p, t, Xs) if lsh.is_e2lsh(p.scheme) else parity.srp_band(p, t, Xs)
    kr = parity.check_keys(p, ref, out["keys"].view(torch.int64)[:, ri].cpu().numpy().view(np.uint64))
    assert kr["mismatch_outside_exempt"] == 0, kr


@pytest.mark.parametrize("scheme,d,m,L,K,per_table", [
    ("E2LSH", 300, 160, 10, 16, False), ("SRP", 300, 48, 6, 8, False), ("E2LSH", 200, 1024, 64, 16, False),
    ("CS_E2LSH", 960, 1024, 64, 16, True), ("CS_SRP", 100, 40, 10, 4, True), ("CS_E2LSH", 64, 24, 24, 1, True)])
def test_fused_key_epilogue_equals_materialised(scheme, d, m, L, K, per_table):
    """Keys from the GEMM's fused TMEM epilogue == keys from the materialised projection
    (same accumulators, same discretisation), and == the oracle outside the bands."""
    p = lsh.Params(scheme, d=d, m=m, L=L, K=K, w=2.0, seed=5, per_table=per_table)
    h = _handle(p)
    X = synth.gaussian_rows_like(1000, d, 4, device="cuda")
    kf = h.hash(X, keys=True)["keys"].view(torch.int64).cpu().numpy()
    km = h.hash(X, keys=True, proj=True)["keys"].view(torch.int64).cpu().numpy()
    h.check()
    assert np.array_equal(kf, km)
    t = lsh.make_tables(p)
    Xn = X.cpu().numpy()
    ref = lsh.hash_points(p, t, Xn)
    ref["band"] = parity.code_band(p, t, Xn) if lsh.is_e2lsh(p.scheme) else parity.srp_band(p, t, Xn)
    kr = parity.check_keys(p, ref, kf.view(np.uint64))
    assert kr["mismatch_outside_exempt"] == 0, kr


def test_group_path_overflow_fallback_and_hint():
    """Wide keys take the fixed-capacity L1 scatter (lsh_group_path 0) until a bin
    overflows — here 30,000 identical points, one bucket per table — then the gated
    histogram path redoes the grouping in the same build and the hint keeps the next
    builds on it (path > 0); the index equals the oracle's grouping of the kernel's keys
    on every build, whichever path ran (DESIGN.md §7 K3)."""
    c = synth.CONFIGS["C2"]
    p = _params(c, "CS_E2LSH")
    h = _handle(p)
    X = synth.rows(c, 0, c.n, device="cuda")
    Xdup = X.clone()
    Xdup[:30000] = X[0]
    for step, (Xs, want) in enumerate([(X, 0), (Xdup, 1), (X, 1)]):
        keys = h.hash(Xs, keys=True)["keys"].cpu().numpy()
        idx = h.build_index(Xs, id_base=0)
        torch.cuda.synchronize()
        path = h.group_path()
        assert (path > 0) == bool(want), (step, path)
        _check_index(idx, lsh.group(keys), p.L)
        idx.close()


def test_hcs_register_fed_kernel_equals_tma_kernel(tmp_path):
    """K2's register-fed slab kernel (used when X cannot be described by a tensor map;
    forced here with LSH_HCS_NO_TMA=1 in a fresh process — the switch is read once per
    process) and the TMA-fed default give the same keys bit for bit at full C3 n for both
    HCS families, and the oracle's on the first 1000 rows."""
    import subprocess
    import sys
    import os
    c = synth.CONFIGS["C3"]
    for scheme in ("HCS_E2LSH", "HCS_SRP"):
        p = _params(c, scheme)
        h = _handle(p)
        X = synth.rows(c, 0, c.n, device="cuda")
        k_tma = h.hash(X, keys=True)["keys"].view(torch.int64).cpu().numpy()
        out = tmp_path / f"{scheme}.npy"
        code = (
            "import sys, numpy as np, torch; sys.path.insert(0, %r)\n"
            "import paper_2503_06737_b200 as pk, synth\n"
            "c = synth.CONFIGS['C3']\n"
            "h = pk.LSH(%r, c.d, c.m, c.L, c.K, c.w, c.hash_seed, mode_d=c.mode_d, mode_m=c.mode_m)\n"
            "X = synth.rows(c, 0, c.n, device='cuda')\n"
            "np.save(%r, h.hash(X, keys=True)['keys'].view(torch.int64).cpu().numpy())\n"
        ) % (os.path.dirname(os.path.dirname(os.path.abspath(__file__))), scheme, str(out))
        env = dict(os.environ, LSH_HCS_NO_TMA="1")
        r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        k_reg = np.load(out)
        assert np.array_equal(k_reg, k_tma), scheme
        ref = lsh.hash_points(p, lsh.make_tables(p), X[:1000].cpu().numpy())
        ref["band"] = parity.code_band(p, lsh.make_tables(p), X[:1000].cpu().numpy()) if lsh.is_e2lsh(scheme) \
            else parity.srp_band(p, lsh.make_tables(p), X[:1000].cpu().numpy())
        kr = parity.check_keys(p, ref, k_tma[:, :1000].view(np.uint64))
        assert kr["mismatch_outside_exempt"] == 0, kr
