"""NEXT-3: GPU Monte-Carlo validation of the paper's collision laws through the
CUDA path (test ideas from SPEC acceptance criteria 1-4).

The laws are closed forms (oracle/theory.py, pinned against the paper's integral
in tests/test_oracle_laws.py); the samples come from the GPU hashers at the
paper's regime d = 10^4:
  * Thm ubiased_cssrp / Thm hcssrp_lsh_property: Pr[bit equal] = 1 - theta/pi
  * Thm CS_Eucl_LSH_property / Thm HCS_Eucl_LSH_property: Pr[code equal] = p(R)
  * eq:eq201022: the K-coordinate code collides with probability p(R)^K
  * Thm uni_cs (P:531ff): CS(p)_l ~ N(0, ||p||^2 / m), coordinates uncorrelated.
Independent trials come from the per-table families (NEXT-2: every table its own
(h_t, s_t, b_t)), from fresh seeds (HCS) and from the rows of R (dense).
"""
import math

import numpy as np
import pytest
import torch

from oracle import theory

pytestmark = pytest.mark.gpu

D = 10_000


@pytest.fixture(scope="module", autouse=True)
def _lib():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2503_06737_b200 as pk
    pk.lib()
    yield


def _unit(g, d):
    v = g.standard_normal(d)
    return v / np.linalg.norm(v)


def _angle_rows(g, thetas):
    u = _unit(g, D)
    rows = [u]
    for th in thetas:
        v = g.standard_normal(D)
        v -= (v @ u) * u
        v /= np.linalg.norm(v)
        rows.append(math.cos(th) * u + math.sin(th) * v)
    return torch.from_numpy(np.stack(rows).astype(np.float32)).cuda()


def _distance_rows(g, Rs):
    p = _unit(g, D)
    return torch.from_numpy(np.stack([p] + [p + R * _unit(g, D) for R in Rs]).astype(np.float32)).cuda()


def _bits(h, X, m):
    w = h.hash(X, keys=False, bits=True)["bits"].cpu().numpy().astype(np.uint32)
    out = np.zeros((X.shape[0], m), dtype=np.uint8)
    for l in range(m):
        out[:, l] = (w[:, l >> 5] >> np.uint32(l & 31)) & 1
    return out


def _codes(h, X):
    return h.hash(X, keys=False, codes=True)["codes"].cpu().numpy()


THETAS = (math.pi / 6, math.pi / 3, math.pi / 2)
RS = (0.5, 1.0, 2.0, 4.0)
TRIALS = 20_000


def _hcs(scheme, seed, w=4.0):
    import paper_2503_06737_b200 as pk
    return pk.LSH(scheme, D, 16, 1, 16, w, seed, mode_d=(100, 100), mode_m=(4, 4))


@pytest.mark.parametrize("family", ["SRP", "CS_SRP_per_table", "HCS_SRP_seeds"])
def test_cosine_collision_law(family):
    import paper_2503_06737_b200 as pk
    X = _angle_rows(np.random.default_rng(1), THETAS)
    if family == "SRP":
        B = _bits(pk.LSH("SRP", D, TRIALS, TRIALS // 16, 16, 4.0, 3), X, TRIALS)
    elif family == "CS_SRP_per_table":
        L = TRIALS // 16
        B = _bits(pk.LSH("CS_SRP", D, TRIALS, L, 16, 4.0, 3, per_table=True), X, TRIALS)
    else:
        B = np.concatenate([_bits(_hcs("HCS_SRP", s), X, 16) for s in range(TRIALS // 16)], axis=1)
    for j, th in enumerate(THETAS):
        rate = float((B[0] == B[j + 1]).mean())
        assert abs(rate - theory.p_collision_srp(th)) < 0.015, (family, th, rate)


@pytest.mark.parametrize("family", ["E2LSH", "CS_E2LSH_per_table", "HCS_E2LSH_seeds"])
def test_euclidean_collision_law(family):
    import paper_2503_06737_b200 as pk
    X = _distance_rows(np.random.default_rng(2), RS)
    if family == "E2LSH":
        C = _codes(pk.LSH("E2LSH", D, TRIALS, TRIALS // 16, 16, 4.0, 5), X)
    elif family == "CS_E2LSH_per_table":
        C = _codes(pk.LSH("CS_E2LSH", D, TRIALS, TRIALS // 16, 16, 4.0, 5, per_table=True), X)
    else:
        C = np.concatenate([_codes(_hcs("HCS_E2LSH", s), X) for s in range(TRIALS // 16)], axis=1)
    for j, R in enumerate(RS):
        rate = float((C[0] == C[j + 1]).mean())
        assert abs(rate - theory.p_collision_e2lsh(R, 4.0)) < 0.02, (family, R, rate)


def test_product_law_full_code():
    """eq:eq201022: a table's K = 4 codes all collide with probability p(R)^4 (keys compared)."""
    import paper_2503_06737_b200 as pk
    L = 8000
    h = pk.LSH("CS_E2LSH", D, 4 * L, L, 4, 4.0, 8, per_table=True)
    X = _distance_rows(np.random.default_rng(3), (0.5, 1.0))
    k = h.hash(X, keys=True)["keys"].view(torch.int64).cpu().numpy()   # [L][3]
    c = _codes(h, X)
    for j, R in enumerate((0.5, 1.0)):
        full = float((k[:, 0] == k[:, j + 1]).mean())
        single = float((c[0] == c[j + 1]).mean())
        assert abs(full - theory.p_collision_e2lsh(R, 4.0) ** 4) < 0.02, (R, full)
        assert abs(full - single ** 4) < 0.02, (R, full, single)


def test_sketch_normality_and_independence():
    """Thm uni_cs: Var CS(p)_l = ||p||^2 / K per table (within 5%), coordinates uncorrelated."""
    import paper_2503_06737_b200 as pk
    L, K = 5000, 16
    g = np.random.default_rng(4)
    p = (10.0 * _unit(g, D)).astype(np.float32)      # ||p||^2 = 100
    h = pk.LSH("CS_SRP", D, K * L, L, K, 4.0, 13, per_table=True)
    y = h.hash(torch.from_numpy(p[None]).cuda(), keys=False, proj=True)["proj"].cpu().numpy().reshape(L, K)
    nrm2 = float(p.astype(np.float64) @ p)
    var = (y.astype(np.float64) ** 2).mean(axis=0)    # E y = 0 by the random signs
    assert np.all(np.abs(var / (nrm2 / K) - 1) < 0.05), var
    corr = np.corrcoef(y.T)
    off = np.abs(corr[~np.eye(K, dtype=bool)])
    assert off.max() < 5.0 / math.sqrt(L), off.max()
    # p = 0: the sketch is exactly 0
    z = h.hash(torch.zeros((1, D), device="cuda"), keys=False, proj=True)["proj"]
    assert int((z != 0).sum()) == 0
