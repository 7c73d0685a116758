"""Host-side checks of the C-ABI library (no GPU needed): it loads, exports every
symbol include/lsh.h declares, and its host parameter draw (an independent C++
implementation of DESIGN.md R1-R4) equals the oracle's bit for bit."""
import ctypes
import os
import re

import numpy as np
import pytest

import paper_2503_06737_b200 as pk
from oracle import lsh, rng

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module", autouse=True)
def built():
    from paper_2503_06737_b200 import build
    build.build()


def test_library_exports_every_declared_symbol():
    hdr = open(os.path.join(ROOT, "include", "lsh.h")).read()
    hdr = re.sub(r"/\*.*?\*/", "", hdr, flags=re.S)
    names = set(re.findall(r"\b(lsh_[a-z_]+)\s*\(", hdr))
    assert len(names) >= 19
    L = ctypes.CDLL(pk.LIB_PATH)
    for n in sorted(names):
        assert hasattr(L, n), n
    # and the binding wraps each of them under the same name
    bound = set(pk.lib().__dict__.keys())
    assert names <= bound | {n for n in names if hasattr(pk.lib(), n)}


def test_library_is_sm100a():
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", pk.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def _oracle_params(scheme, d, m, L, K, w=4.0, seed=0, mode_d=(), mode_m=()):
    return lsh.Params(scheme, d=d, m=m, L=L, K=K, w=w, seed=seed, mode_d=tuple(mode_d), mode_m=tuple(mode_m))


CASES = [
    ("CS_E2LSH", 64, 16, 2, 8, 4.0, 0, None, None),
    ("CS_SRP", 784, 160, 10, 16, 4.0, 0, None, None),
    ("CS_E2LSH", 960, 1024, 64, 16, 1.0, 0, None, None),
    ("HCS_E2LSH", 4096, 512, 32, 16, 2.0, 0, (16, 16, 16), (8, 8, 8)),
    ("HCS_SRP", 1000, 64, 4, 16, 4.0, 12345, (10, 10, 10), (4, 4, 4)),
    ("HCS_E2LSH", 50, 24, 3, 8, 0.7, 99, (4, 4, 4), (2, 3, 4)),
]


@pytest.mark.parametrize("case", CASES)
def test_host_tables_equal_oracle(case):
    scheme, d, m, L, K, w, seed, md, mm = case
    pp = pk.make_params(scheme, d, m, L, K, w, seed, md, mm)
    op = _oracle_params(scheme, d, m, L, K, w, seed, md or (), mm or ())
    ot = lsh.make_tables(op)
    for k in range(op.N):
        assert np.array_equal(pk.export_host(pp, "bucket", k), ot.h[k].astype(np.int32))
        assert np.array_equal(pk.export_host(pp, "sign", k), ot.s[k].astype(np.int32))
        co = pk.export_host(pp, "coeffs", k)
        fb = rng.TwoWise(rng.Stream(seed, f"mode{k}/bucket"), op.mode_m[k])
        fs = rng.TwoWise(rng.Stream(seed, f"mode{k}/sign"), 2)
        assert [int(x) for x in co] == [fb.a, fb.b, fs.a, fs.b]
    off = pk.export_host(pp, "offsets")
    assert off.dtype == np.float32 and np.array_equal(off.view(np.uint32), ot.b.view(np.uint32))
    coord = pk.export_host(pp, "coord")
    for j in range(0, d, max(1, d // 257)):
        l, sg = lsh.hcs_coordinate(j, op.mode_d, op.mode_m, ot.h, ot.s)
        assert coord[j] == l and coord[d + j] == sg


@pytest.mark.parametrize("m,d,seed", [(160, 784, 0), (3, 7, 5), (16, 64, 1)])
def test_host_gaussian_equals_oracle(m, d, seed):
    pp = pk.make_params("E2LSH", d, m, 1, m, 4.0, seed)
    got = pk.export_host(pp, "gaussian").astype(np.uint32) << 16
    want = lsh.make_tables(_oracle_params("E2LSH", d, m, 1, m, 4.0, seed)).R.astype(np.float32).ravel()
    assert np.array_equal(got.view(np.float32), want)


def test_invalid_parameters_rejected():
    bad = [
        pk.make_params("CS_E2LSH", 64, 16, 3, 8),       # m != L*K
        pk.make_params("CS_E2LSH", 64, 16, 2, 8, w=0.0),  # w <= 0
        pk.make_params("CS_SRP", 64, 130, 1, 130),       # SRP K > 64
        pk.make_params("HCS_SRP", 100, 16, 1, 16, mode_d=(5, 5), mode_m=(4, 4)),  # prod d_k < d
        pk.make_params("HCS_SRP", 16, 16, 1, 16, mode_d=(4, 4), mode_m=(4, 3)),   # prod m_k != m
    ]
    for p in bad:
        sz = ctypes.c_size_t(0)
        assert pk.lib().lsh_export_host(ctypes.byref(p), 2, 0, None, ctypes.byref(sz)) == 1
    assert pk.lib().lsh_strerror(1) == b"invalid parameters"


def test_no_undefined_internal_symbols():
    import subprocess
    out = subprocess.run(["nm", "-D", "--undefined-only", pk.LIB_PATH], capture_output=True, text=True).stdout
    assert "lshb" not in out, out


@pytest.mark.parametrize("scheme,d,L,K,w,seed", [("CS_E2LSH", 100, 5, 8, 2.0, 3), ("CS_SRP", 37, 3, 4, 4.0, 12345)])
def test_host_per_table_families_equal_oracle(scheme, d, L, K, w, seed):
    # NEXT-2 (reading C3): the C++ host draw of every table's family and the +-1 matrix
    pp = pk.make_params(scheme, d, L * K, L, K, w, seed, per_table=True)
    op = lsh.Params(scheme, d=d, m=L * K, L=L, K=K, w=w, seed=seed, per_table=True)
    ot = lsh.make_tables(op)
    for t in range(L):
        assert np.array_equal(pk.export_host(pp, "bucket", t), ot.h[t].astype(np.int32))
        assert np.array_equal(pk.export_host(pp, "sign", t), ot.s[t].astype(np.int32))
        co = pk.export_host(pp, "coeffs", t)
        fb = rng.TwoWise(rng.Stream(seed, f"table{t}/mode0/bucket"), K)
        fs = rng.TwoWise(rng.Stream(seed, f"table{t}/mode0/sign"), 2)
        assert [int(x) for x in co] == [fb.a, fb.b, fs.a, fs.b]
    off = pk.export_host(pp, "offsets")
    assert np.array_equal(off.view(np.uint32), ot.b.view(np.uint32))
    R = (pk.export_host(pp, "gaussian").astype(np.uint32) << 16).view(np.float32).reshape(L * K, d)
    X = np.random.default_rng(0).standard_normal((3, d)).astype(np.float32)
    np.testing.assert_allclose(X.astype(np.float64) @ R.astype(np.float64).T, lsh.project(op, ot, X), atol=1e-9)


def test_per_table_flag_validation():
    sz = ctypes.c_size_t(0)
    p = pk.make_params("HCS_SRP", 16, 16, 1, 16, mode_d=(4, 4), mode_m=(4, 4), per_table=True)
    assert pk.lib().lsh_export_host(ctypes.byref(p), 2, 0, None, ctypes.byref(sz)) == 7   # LSH_EUNSUPPORTED
    p = pk.make_params("CS_SRP", 16, 16, 2, 8)
    p.flags = 2
    assert pk.lib().lsh_export_host(ctypes.byref(p), 2, 0, None, ctypes.byref(sz)) == 1   # unknown flag bit
