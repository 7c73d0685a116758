"""Pins for oracle/rng.py: published generator vectors, worked examples, statistics."""
import math

import numpy as np
import pytest
import torch

from oracle import rng


def test_splitmix64_published_vectors(golden):
    s = rng.Stream(0, "x")
    s.state = 0  # raw SplitMix64 with state 0
    got = [s.next() for _ in range(4)]
    want = [int(v, 16) for v in golden["published_vectors"]["splitmix64_seed0_first4"]["values"]]
    assert got == want


def test_fnv1a64_published_vectors(golden):
    for text, want in golden["published_vectors"]["fnv1a64"]["cases"]:
        assert rng.fnv1a64(text.encode()) == int(want, 16)


def test_stream_labels_distinct_and_deterministic():
    a = [rng.Stream(7, f"table{t}").next() for t in range(2000)]
    assert len(set(a)) == len(a)
    assert rng.Stream(7, "x").next() == rng.Stream(7, "x").next()
    assert rng.Stream(7, "x").next() != rng.Stream(8, "x").next()


def test_twowise_worked_examples(golden):
    ex = golden["spec_worked_examples"]["twowise_eval"]
    assert rng.TwoWise.eval_ab(ex["a"], ex["b"], ex["m"], ex["i"]) == ex["expect"]
    en = golden["spec_worked_examples"]["twowise_enumeration"]
    assert [rng.TwoWise.eval_ab(en["a"], en["b"], en["m"], i) for i in range(8)] == en["expect"]


def test_twowise_coefficient_ranges():
    for seed in range(200):
        f = rng.TwoWise(rng.Stream(seed, "mode0/bucket"), 16)
        assert 1 <= f.a <= rng.P61 - 1 and 0 <= f.b <= rng.P61 - 1


def test_bucket_load_uniform():
    # d=1e5, m=16 -> every bucket load within 5% of d/m
    h = rng.bucket_table(3, 0, 100_000, 16)
    counts = np.bincount(h, minlength=16)
    assert np.all(np.abs(counts - 100_000 / 16) <= 0.05 * 100_000 / 16)


def test_pairwise_collision_rate():
    # 2-wise independence consequence: Pr[h(i)=h(j)] = 1/m over the family draw
    m, trials = 8, 4000
    pairs = [(3, 17), (0, 1), (100, 5000)]
    for i, j in pairs:
        hits = 0
        for seed in range(trials):
            f = rng.TwoWise(rng.Stream(seed, "mode0/bucket"), m)
            hits += f.eval(i) == f.eval(j)
        p = hits / trials
        assert abs(p - 1 / m) < 3 * math.sqrt((1 / m) * (1 - 1 / m) / trials) + 1e-3


def test_sign_mean_zero():
    s = rng.sign_table(11, 0, 100_000)
    assert set(np.unique(s).tolist()) == {-1, 1}
    assert abs(s.mean()) < 0.02


def test_offsets_range_and_mean():
    for w in (1.0, 2.0, 4.0, 0.3):
        b = rng.offsets(5, 20000, w)
        assert b.dtype == np.float32
        assert np.all(b >= 0) and np.all(b < np.float32(w))
        assert abs(b.mean() / w - 0.5) < 0.01


def test_round_bf16_matches_torch_on_fp32_inputs():
    # For values exactly representable in fp32, fp64->bf16 RNE equals torch's fp32->bf16 RNE.
    g = np.random.default_rng(0)
    vals = np.concatenate([g.standard_normal(5000), g.uniform(-1e3, 1e3, 2000)]).astype(np.float32)
    ties = np.array([1.0 + 2 ** -8, 1.0 + 3 * 2 ** -8, -(1.0 + 2 ** -8), 3.0 + 2 ** -7], dtype=np.float32)
    vals = np.concatenate([vals, ties])
    ours = np.array([rng.round_bf16(float(v)) for v in vals])
    ref = torch.from_numpy(vals).to(torch.bfloat16).to(torch.float64).numpy()
    assert np.array_equal(ours, ref)


def test_gaussian_moments():
    R = rng.gaussian_rows(1, 400, 500)  # 2e5 draws
    x = R.ravel()
    n = x.size
    assert abs(x.mean()) < 3 / math.sqrt(n) + 1e-3
    assert abs(x.var() - 1) < 3 * math.sqrt(2 / n) + 2e-3   # bf16 rounding adds ~1e-5 var
    kurt = ((x - x.mean()) ** 4).mean() / x.var() ** 2
    assert abs(kurt - 3) < 0.05
    # every value is bf16-exact
    assert np.array_equal(torch.from_numpy(x).to(torch.bfloat16).to(torch.float64).numpy(), x)


def test_flat_index_example_and_bijection(golden):
    ex = golden["spec_worked_examples"]["flat_index"]
    assert rng.flat_index(ex["idx"], ex["dims"]) == ex["expect"]
    for dims in [(2, 3), (4, 3, 5), (16, 16, 16), (3,), (2, 2, 2, 2, 3)]:
        total = int(np.prod(dims))
        seen = set()
        for j in range(total):
            idx = rng.unflatten(j, dims)
            assert rng.flat_index(idx, dims) == j
            seen.add(tuple(idx))
        assert len(seen) == total


def test_vectorised_gaussian_equals_scalar_path():
    a = rng._gaussian_rows_vectorised(5, 40, 301)
    st = rng.Stream(5, "gaussian")
    b = np.array(rng.gaussian_rows(5, 40, 301))
    assert np.array_equal(a, b) or (a != b).sum() <= 1  # last-ulp libm differences only at bf16 ties
    x = np.random.default_rng(0).standard_normal(3000)
    assert np.array_equal(rng.round_bf16_array(x), np.array([rng.round_bf16(float(v)) for v in x]))
