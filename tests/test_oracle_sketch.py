"""Pins for the oracle's projection, discretisation and keys (oracle/lsh.py)."""
import itertools
import math
from fractions import Fraction

import numpy as np
import pytest

from oracle import lsh, rng


def test_cs_worked_example(golden):
    ex = golden["spec_worked_examples"]["cs_apply"]
    y = lsh.cs_sketch(np.array([ex["p"]], float), np.array(ex["h"]), np.array(ex["s"]), ex["m"])
    assert y[0].tolist() == ex["expect"]
    e2 = golden["spec_worked_examples"]["cs_e2lsh"]
    codes = lsh.e2lsh_codes(y, np.array(e2["b"], np.float32), e2["w"], math.sqrt(ex["m"]))
    assert codes[0].tolist() == e2["expect"]
    assert lsh.srp_bits(y)[0].tolist() == golden["spec_worked_examples"]["cs_srp"]["expect"]


def test_hcs_worked_example(golden):
    ex = golden["spec_worked_examples"]["hcs_apply"]
    h = [np.array(v) for v in ex["h"]]
    s = [np.array(v) for v in ex["s"]]
    y = lsh.hcs_sketch(np.array([ex["p"]], float), ex["mode_d"], ex["mode_m"], h, s)
    assert y[0].tolist() == ex["expect"]
    e2 = golden["spec_worked_examples"]["hcs_e2lsh"]
    codes = lsh.e2lsh_codes(y, np.array(e2["b"], np.float32), e2["w"], 1.0)  # m = 1 -> sqrt(m) = 1
    assert codes[0].tolist() == e2["expect"]


def test_discretize_examples(golden):
    for x, b, w, want in golden["spec_worked_examples"]["discretize"]["cases"]:
        assert lsh.e2lsh_codes(np.array([[x]]), np.array([b], np.float32), w, 1.0)[0, 0] == want


def test_floor_shift_identity():
    g = np.random.default_rng(1)
    y = g.uniform(-50, 50, (1, 2000))
    b = g.uniform(0, 4, 2000).astype(np.float32)
    z0 = lsh.e2lsh_codes(y, b, 4.0, 1.0)
    z1 = lsh.e2lsh_codes(y + 4.0, b, 4.0, 1.0)
    assert np.array_equal(z1, z0 + 1)


def _rand_cs(g, d, m):
    return g.integers(0, m, d), g.choice([-1, 1], d)


def test_cs_basis_vectors_one_nonzero_per_column():
    # CS(e_i) = s(i) e_{h(i)}: each input coordinate lands in exactly one bin
    p = lsh.Params("CS_E2LSH", d=50, m=8, L=2, K=4, seed=9)
    t = lsh.make_tables(p)
    Y = lsh.cs_sketch(np.eye(50), t.h[0], t.s[0], 8)
    for i in range(50):
        nz = np.nonzero(Y[i])[0]
        assert nz.tolist() == [t.h[0][i]] and Y[i, nz[0]] == t.s[0][i]


def test_cs_dense_matrix_bruteforce():
    g = np.random.default_rng(2)
    for d in (1, 5, 16):
        for m in (1, 3, 8):
            h, s = _rand_cs(g, d, m)
            S = np.zeros((m, d))
            S[h, np.arange(d)] = s
            X = g.standard_normal((7, d))
            assert np.allclose(lsh.cs_sketch(X, h, s, m), X @ S.T, rtol=0, atol=1e-12)


def test_cs_linearity():
    g = np.random.default_rng(3)
    h, s = _rand_cs(g, 300, 16)
    p, q = g.standard_normal((2, 300))
    a, b = 1.7, -0.3
    lhs = lsh.cs_sketch((a * p + b * q)[None], h, s, 16)
    rhs = a * lsh.cs_sketch(p[None], h, s, 16) + b * lsh.cs_sketch(q[None], h, s, 16)
    assert np.allclose(lhs, rhs, rtol=1e-12, atol=1e-12)


def test_cs_exact_variance_by_enumeration(golden):
    ex = golden["spec_worked_examples"]["exact_variance_cs"]
    p = np.array(ex["p"], float)
    d, m = len(p), ex["m"]
    s1 = s2 = s11 = Fraction(0)
    count = 0
    for hv in itertools.product(range(m), repeat=d):
        for sv in itertools.product((-1, 1), repeat=d):
            y = lsh.cs_sketch(p[None], np.array(hv), np.array(sv), m)[0]
            y0, y1 = Fraction(y[0]), Fraction(y[1])
            s1 += y0
            s2 += y0 * y0
            s11 += y0 * y1
            count += 1
    mean = s1 / count
    assert mean == 0
    assert s2 / count == Fraction(ex["var_num"], ex["var_den"])
    assert s2 / count == Fraction(sum(Fraction(v) ** 2 for v in p)) / m
    assert s11 / count == 0  # Cov(CS_0, CS_1) = 0 exactly


def test_hcs_exact_variance_by_enumeration():
    # Thm hcs_normality proof: Var[vec(HCS(p))_l] = ||p||^2/m exactly
    p = np.array([[1.0, -2.0, 3.0, 0.5, 2.0, -1.0]])
    mode_d, mode_m = (2, 3), (2, 2)
    acc = Fraction(0)
    cnt = 0
    for h1 in itertools.product(range(2), repeat=2):
        for h2 in itertools.product(range(2), repeat=3):
            for s1 in itertools.product((-1, 1), repeat=2):
                for s2 in itertools.product((-1, 1), repeat=3):
                    y = lsh.hcs_sketch(p, mode_d, mode_m, [np.array(h1), np.array(h2)],
                                       [np.array(s1), np.array(s2)])[0]
                    acc += Fraction(y[3]) ** 2
                    cnt += 1
    assert acc / cnt == Fraction(sum(Fraction(v) ** 2 for v in p[0])) / 4


def test_hcs_kronecker_bruteforce():
    # vec(HCS(x)) = (S_N kron ... kron S_1) x  (P:59-60 matrix view, column-major vec)
    g = np.random.default_rng(4)
    for mode_d, mode_m in [((4, 3, 5), (2, 3, 2)), ((16, 16), (8, 8)), ((3, 4), (3, 2)), ((2, 2, 2, 2), (2, 1, 2, 2))]:
        d = int(np.prod(mode_d))
        h = [g.integers(0, mk, dk) for dk, mk in zip(mode_d, mode_m)]
        s = [g.choice([-1, 1], dk) for dk in mode_d]
        mats = []
        for k in range(len(mode_d)):
            S = np.zeros((mode_m[k], mode_d[k]))
            S[h[k], np.arange(mode_d[k])] = s[k]
            mats.append(S)
        big = mats[-1]
        for S in reversed(mats[:-1]):
            big = np.kron(big, S)
        X = g.standard_normal((3, d))
        assert np.allclose(lsh.hcs_sketch(X, mode_d, mode_m, h, s), X @ big.T, atol=1e-12)


def test_hcs_order2_is_left_right_countsketch():
    # For N=2: HCS(P) = S_1 P S_2^T with P the d1 x d2 reshaping
    g = np.random.default_rng(5)
    d1, d2, m1, m2 = 6, 5, 3, 2
    h = [g.integers(0, m1, d1), g.integers(0, m2, d2)]
    s = [g.choice([-1, 1], d1), g.choice([-1, 1], d2)]
    S1 = np.zeros((m1, d1)); S1[h[0], np.arange(d1)] = s[0]
    S2 = np.zeros((m2, d2)); S2[h[1], np.arange(d2)] = s[1]
    x = g.standard_normal(d1 * d2)
    P = x.reshape(d2, d1).T  # column-major reshape: P[i1, i2] = x[i1 + d1*i2]
    want = (S1 @ P @ S2.T).T.ravel()  # vec column-major
    got = lsh.hcs_sketch(x[None], (d1, d2), (m1, m2), h, s)[0]
    assert np.allclose(got, want, atol=1e-12)


def test_hcs_order1_equals_cs_bit_identical():
    p = lsh.Params("CS_SRP", d=200, m=16, L=2, K=8, seed=21)
    t = lsh.make_tables(p)
    X = np.random.default_rng(6).standard_normal((5, 200))
    a = lsh.cs_sketch(X, t.h[0], t.s[0], 16)
    b = lsh.hcs_sketch(X, (200,), (16,), t.h, t.s)
    assert np.array_equal(a, b)


def test_hcs_zero_padding():
    # d not factorable: pad with zeros; sketch of x equals sketch of padded x
    g = np.random.default_rng(7)
    mode_d, mode_m = (4, 4, 4), (2, 2, 2)
    h = [g.integers(0, 2, 4) for _ in range(3)]
    s = [g.choice([-1, 1], 4) for _ in range(3)]
    x = g.standard_normal((2, 50))
    xp = np.concatenate([x, np.zeros((2, 14))], axis=1)
    assert np.array_equal(lsh.hcs_sketch(x, mode_d, mode_m, h, s), lsh.hcs_sketch(xp, mode_d, mode_m, h, s))


@pytest.mark.parametrize("scheme", lsh.SCHEMES)
def test_zero_vector_gives_zero_codes(scheme):
    kw = dict(mode_d=(4, 4, 4), mode_m=(2, 2, 4)) if lsh.is_hcs(scheme) else {}
    p = lsh.Params(scheme, d=64, m=16, L=2, K=8, w=4.0, seed=3, **kw)
    t = lsh.make_tables(p)
    out = lsh.hash_points(p, t, np.zeros((2, 64)))
    if lsh.is_e2lsh(scheme):
        assert np.all(out["codes"] == 0)   # floor(b/w) = 0 for b in [0, w)
    else:
        assert np.all(out["bits"] == 0)    # sgn(0) = 0


@pytest.mark.parametrize("scheme", ["SRP", "CS_SRP", "HCS_SRP"])
def test_srp_positive_scale_invariance(scheme):
    kw = dict(mode_d=(8, 8), mode_m=(4, 4)) if lsh.is_hcs(scheme) else {}
    p = lsh.Params(scheme, d=64, m=16, L=1, K=16, seed=4, **kw)
    t = lsh.make_tables(p)
    X = np.random.default_rng(8).standard_normal((20, 64))
    a = lsh.hash_points(p, t, X)["keys"]
    b = lsh.hash_points(p, t, 3.25 * X)["keys"]
    assert np.array_equal(a, b)


def test_param_count_examples(golden):
    for scheme, d, m, mode_d, mode_m, want in golden["spec_worked_examples"]["param_count"]["cases"]:
        kw = dict(mode_d=tuple(mode_d), mode_m=tuple(mode_m)) if lsh.is_hcs(scheme) else {}
        p = lsh.Params(scheme, d=d, m=m, L=1, K=m, **kw)
        assert lsh.param_count(p) == want


def test_work_is_o_d_for_sketches_and_o_md_for_dense():
    # Table 1: CS/HCS O(d) time independent of m; E2LSH O(md)
    x = np.random.default_rng(9).standard_normal(64)
    for m in (4, 16, 64):
        for scheme, kw in [("CS_E2LSH", {}), ("HCS_E2LSH", dict(mode_d=(8, 8), mode_m=(m // 4 if m > 4 else 2, 4 if m > 4 else 2)))]:
            p = lsh.Params(scheme, d=64, m=m, L=1, K=m, **kw)
            assert lsh.projection_op_count(p, lsh.make_tables(p), x) == 64
        p = lsh.Params("E2LSH", d=64, m=m, L=1, K=m)
        assert lsh.projection_op_count(p, lsh.make_tables(p), x) == 64 * m


def test_fingerprint_special_cases():
    # Reading B10 reduces to the SplitMix64 finaliser (pinned by its published vectors)
    # on inputs whose two polynomial lanes are known without evaluating the lanes:
    # all-zero codes give lanes (0, 0); a single code u gives lanes (u, u).
    assert lsh.fingerprint([0] * 16) == rng.fmix64(0) == 0
    assert lsh.fingerprint([1]) == rng.fmix64((1 << 32) | 1)
    assert lsh.fingerprint([-1]) == rng.fmix64(0xFFFFFFFFFFFFFFFF)     # two's complement word
    assert lsh.fingerprint([-(1 << 31)]) == rng.fmix64(0x8000000080000000)
    # leading zero codes leave both Horner lanes at 0 (the polynomial is in u_{K-1} last)
    assert lsh.fingerprint([0, 0, 0, 5]) == lsh.fingerprint([5])
    # a code in front is multiplied by the lane's multiplier once per later code
    A, B = lsh.FP_A, lsh.FP_B
    assert lsh.fingerprint([1, 0]) == rng.fmix64((A << 32) | B)
    assert lsh.fingerprint([1, 0, 0]) == rng.fmix64(((A * A % 2 ** 32) << 32) | (B * B % 2 ** 32))


def _lane_values(mult: int, K: int, radius: int, lo: int, hi: int) -> np.ndarray:
    """sum_{k in [lo,hi)} delta_k * mult^(K-1-k) mod 2^32 over every delta in [-r, r]^(hi-lo)."""
    out = np.zeros(1, dtype=np.int64)
    for k in range(lo, hi):
        c = pow(mult, K - 1 - k, 1 << 32)
        out = np.concatenate([out + j * c for j in range(-radius, radius + 1)])
    return out % (1 << 32)


@pytest.mark.parametrize("K", [8, 16])
def test_fingerprint_separates_nearby_code_tuples(K):
    """No two K-code tuples that differ by at most 2 in every coordinate share a key.

    Near neighbours of an E2LSH code differ by small amounts in a few coordinates
    (adjacent bins), so those are the merges that would matter.  Key equality
    of z and z' = both lanes agree = P_A(z - z') = P_B(z - z') = 0 mod 2^32 (fmix64 is
    a bijection); checked exhaustively over all 5^K differences by meet in the middle.
    """
    M = 1 << 32
    h = K // 2
    la = _lane_values(lsh.FP_A, K, 2, 0, h)
    ra = (-_lane_values(lsh.FP_A, K, 2, h, K)) % M
    lb = _lane_values(lsh.FP_B, K, 2, 0, h)
    rb = _lane_values(lsh.FP_B, K, 2, h, K)
    order = np.argsort(ra, kind="stable")
    rs = ra[order]
    p0 = np.searchsorted(rs, la, side="left")
    p1 = np.searchsorted(rs, la, side="right")
    both = 0
    for i in np.nonzero(p1 > p0)[0]:
        for q in range(p0[i], p1[i]):
            if (lb[i] + rb[order[q]]) % M == 0:
                both += 1
    assert both == 1   # only the zero difference (z == z')


def test_fingerprint_separates_two_coordinate_changes():
    """No two tuples differing in exactly two coordinates by up to 4096 each share a key
    (d_i A^p + d_j A^q = 0 mod 2^32 would need d_i = -d_j A^(q-p))."""
    M = 1 << 32
    R = 4096
    d = np.arange(-R, R + 1, dtype=np.int64)
    d = d[d != 0]
    for mult in (lsh.FP_A, lsh.FP_B):
        for r in range(1, 16):
            v = (d * pow(mult, r, M)) % M
            v = np.where(v >= M // 2, v - M, v)
            assert not np.any(np.abs(v) <= R), (hex(mult), r)


def test_fingerprint_merges_counts_forced_collisions():
    """fingerprint_merges counts the rows whose K-tuple differs from the first tuple filed
    under the same (table, key): forced collisions (keys chosen equal for different codes)
    must be counted, equal tuples under one key must not."""
    codes = np.array([[1, 2, 0, 0], [1, 2, 0, 1], [3, 4, 0, 0], [1, 2, 5, 5], [3, 4, 5, 5]])
    # table 0 = columns 0..1, table 1 = columns 2..3
    keys = np.array([[7, 7, 9, 7, 7],          # t0: rows 0,1,3 are (1,2) under 7: fine; row 4 (3,4) under 7: merge
                     [1, 2, 1, 3, 3]], dtype=np.uint64)   # t1: row 2 (0,0) under 1 with row 0: fine; row 4 (5,5) = row 3: fine
    assert lsh.fingerprint_merges(codes, keys, 2, 2) == 1
    keys[1, 1] = 1                               # (0,1) under the key of (0,0): a second merge
    assert lsh.fingerprint_merges(codes, keys, 2, 2) == 2
    assert lsh.fingerprint_merges(codes, lsh.e2lsh_keys(codes, 2, 2), 2, 2) == 0


def test_srp_key_packing():
    bits = np.array([[1, 0, 1, 1, 0, 0, 0, 1]])
    assert lsh.srp_keys(bits, 2, 4).tolist() == [[0b1101], [0b1000]]


def test_no_fingerprint_merges_on_sample():
    p = lsh.Params("CS_E2LSH", d=64, m=16, L=2, K=8, w=4.0, seed=0)
    t = lsh.make_tables(p)
    X = np.random.default_rng(10).random((1000, 64)).astype(np.float32)
    out = lsh.hash_points(p, t, X)
    assert lsh.fingerprint_merges(out["codes"], out["keys"], 2, 8) == 0


def test_vectorised_keys_equal_scalar_fingerprint():
    g = np.random.default_rng(11)
    codes = g.integers(-300, 300, (50, 32))
    codes[0] = 0
    codes[1, :5] = [-(1 << 31), (1 << 31) - 1, -1, 1, 0]
    keys = lsh.e2lsh_keys(codes, 2, 16)
    for i in range(50):
        for t in range(2):
            assert int(keys[t, i]) == lsh.fingerprint(codes[i, t * 16:(t + 1) * 16].tolist())
