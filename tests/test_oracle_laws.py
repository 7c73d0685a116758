"""Pins: collision-probability laws (closed forms vs quadrature, Monte-Carlo)."""
import math

import numpy as np
import pytest

from oracle import lsh, theory


def test_closed_form_matches_paper_integral(golden):
    ex = golden["spec_worked_examples"]["p_collision_e2lsh"]
    assert abs(theory.p_collision_e2lsh(ex["R"], ex["w"]) - ex["expect"]) < ex["tol"]
    for R in np.logspace(-2, 2, 40):
        for w in (1.0, 4.0, 10.0):
            assert abs(theory.p_collision_e2lsh(R, w) - theory.p_collision_e2lsh_integral(R, w)) < 1e-8


def test_p_r_monotone_and_scale():
    vals = [theory.p_collision_e2lsh(R, 4.0) for R in (0.5, 1, 2, 4)]
    assert vals == sorted(vals, reverse=True)
    assert abs(theory.p_collision_e2lsh(1.0, 1.0) - theory.p_collision_e2lsh(4.0, 4.0)) < 1e-14
    assert abs(theory.p_collision_e2lsh(1e-9, 4.0) - 1.0) < 1e-6


def test_srp_law_values():
    assert theory.p_collision_srp(0) == 1 and theory.p_collision_srp(math.pi) == 0
    assert theory.p_collision_srp(math.pi / 2) == 0.5
    for th in np.linspace(0, math.pi, 11):
        assert abs(theory.p_collision_srp(th) + theory.p_collision_srp(math.pi - th) - 1) < 1e-15


def _pair_at_distance(g, d, R):
    p = g.standard_normal(d); p /= np.linalg.norm(p)
    e = g.standard_normal(d); e /= np.linalg.norm(e)
    return p, p + R * e


def _pair_at_angle(g, d, th):
    u = g.standard_normal(d); u /= np.linalg.norm(u)
    v = g.standard_normal(d); v -= (v @ u) * u; v /= np.linalg.norm(v)
    return u, math.cos(th) * u + math.sin(th) * v


def test_dense_e2lsh_collision_law_mc():
    # p(R) is exact for any d for the dense hash; oracle's own seeded draws
    g = np.random.default_rng(0)
    T = 6000
    for R in (0.5, 2.0):
        pt, qt = _pair_at_distance(g, 8, R)
        X = np.stack([pt, qt])
        hits = 0
        for seed in range(T):
            p = lsh.Params("E2LSH", d=8, m=1, L=1, K=1, w=4.0, seed=seed)
            c = lsh.hash_points(p, lsh.make_tables(p), X)["codes"]
            hits += c[0, 0] == c[1, 0]
        pr = theory.p_collision_e2lsh(R, 4.0)
        assert abs(hits / T - pr) < 3 * math.sqrt(pr * (1 - pr) / T) + 1e-3


def test_dense_srp_collision_law_mc():
    g = np.random.default_rng(1)
    T = 6000
    for th in (math.pi / 3, math.pi / 2):
        u, v = _pair_at_angle(g, 8, th)
        X = np.stack([u, v])
        hits = 0
        for seed in range(T):
            p = lsh.Params("SRP", d=8, m=1, L=1, K=1, seed=seed)
            b = lsh.hash_points(p, lsh.make_tables(p), X)["bits"]
            hits += b[0, 0] == b[1, 0]
        pr = theory.p_collision_srp(th)
        assert abs(hits / T - pr) < 3 * math.sqrt(pr * (1 - pr) / T) + 1e-3


def _cs_coord0(H, S, x):
    # CS(x)_0 for many independent (h, s) draws: sum_{h(i)=0} s(i) x_i
    return ((H == 0) * S) @ x


@pytest.mark.slow
def test_cs_e2lsh_and_cs_srp_laws_mc():
    # Thm CS_Eucl_LSH_property and Thm ubiased_cssrp: asymptotic laws at d=1e4
    g = np.random.default_rng(2)
    d, m, T = 10_000, 16, 3000
    H = g.integers(0, m, (T, d)).astype(np.int16)
    S = g.choice(np.array([-1.0, 1.0]), (T, d))
    b = g.uniform(0, 4.0, T)
    for R in (1.0, 2.0):
        p, q = _pair_at_distance(g, d, R)
        zp = np.floor((math.sqrt(m) * _cs_coord0(H, S, p) + b) / 4.0)
        zq = np.floor((math.sqrt(m) * _cs_coord0(H, S, q) + b) / 4.0)
        assert abs((zp == zq).mean() - theory.p_collision_e2lsh(R, 4.0)) < 0.02  # S:693 tolerance
    for th in (math.pi / 3, math.pi / 2):
        u, v = _pair_at_angle(g, d, th)
        assert abs(((_cs_coord0(H, S, u) > 0) == (_cs_coord0(H, S, v) > 0)).mean() - theory.p_collision_srp(th)) < 0.03


def test_cs_law_through_oracle_sketch():
    # Same law through the oracle's own cs_sketch / e2lsh_codes on a moderate d
    g = np.random.default_rng(3)
    d, m, T = 2000, 4, 1500
    p, q = _pair_at_distance(g, d, 1.0)
    X = np.stack([p, q])
    hits = 0
    for _ in range(T):
        h = g.integers(0, m, d); s = g.choice([-1, 1], d)
        b = g.uniform(0, 4.0, m).astype(np.float32)
        z = lsh.e2lsh_codes(lsh.cs_sketch(X, h, s, m), b, 4.0, math.sqrt(m))
        hits += int(z[0, 0] == z[1, 0])
    assert abs(hits / T - theory.p_collision_e2lsh(1.0, 4.0)) < 0.035


@pytest.mark.slow
def test_product_law_full_code():
    # Eq. eq201022: Pr[all m codes equal] = p(R)^m at m=4, d=1e4
    g = np.random.default_rng(4)
    d, m, T = 10_000, 4, 3000
    p, q = _pair_at_distance(g, d, 0.5)
    allc = 0
    H = g.integers(0, m, (T, d)).astype(np.int16)
    S = g.choice(np.array([-1.0, 1.0]), (T, d))
    B = g.uniform(0, 4.0, (T, m))
    eq = np.ones(T, bool)
    for l in range(m):
        yp = ((H == l) * S) @ p
        yq = ((H == l) * S) @ q
        eq &= np.floor((math.sqrt(m) * yp + B[:, l]) / 4) == np.floor((math.sqrt(m) * yq + B[:, l]) / 4)
    assert abs(eq.mean() - theory.p_collision_e2lsh(0.5, 4.0) ** m) < 0.03
