"""GPU <-> oracle comparison rules (north_star tolerances).

  projections: |y_gpu - y_ref| <= 1e-4 * max(|y_ref|, 0.1 * sigma_l), sigma_l the
               dot product's natural scale sqrt(sum_i a_li^2 x_i^2); sigma_l == 0
               (empty bin) requires y_gpu == 0 exactly.
  E2LSH codes: bit-exact except entries whose quotient (scale*y+b)/w lies within
               max(1e-5, 6*2^-24*sqrt(k_l)*scale*sigma_l/w) of an integer (counted and
               reported): the north_star band, widened only where the fp32
               accumulation of k_l nonzero products cannot meet it (derived bound,
               DESIGN.md §5; CS/HCS bins keep 1e-5).  The dense tensor-core
               projection adds its rigorous accumulation bound tc_band_y().
  SRP bits:    bit-exact except entries with |y_ref| < max(1e-6, 6*2^-24*sqrt(k_l)*sigma_l)
               (counted, reported; same derivation).
  Entries with no nonzero product (an empty sum: exactly 0 in any precision) are
  never exempt: their bit / code must match exactly.
  keys:        bit-exact for every (table, point) without an exempt coordinate.
  tables:      bit-exact given identical keys.
"""

from __future__ import annotations

import numpy as np

from oracle import lsh

PROJ_RTOL = 1e-4
CODE_BAND = 1e-5
SRP_BAND = 1e-6


def on_tensor_cores(p: lsh.Params) -> bool:
    """Dense schemes and the NEXT-2 per-table families run as the tcgen05 GEMM."""
    return lsh.is_dense(p.scheme) or p.per_table


def proj_matrix(p: lsh.Params, t: lsh.Tables) -> np.ndarray:
    """[m][d] matrix the GEMM multiplies by: R, or the per-table +-1 block matrix."""
    if lsh.is_dense(p.scheme):
        return t.R.astype(np.float64)
    M = np.zeros((p.m, p.d))
    for tt in range(p.L):
        M[tt * p.K + np.asarray(t.h[tt]), np.arange(p.d)] = np.asarray(t.s[tt], np.float64)
    return M


def sigma(p: lsh.Params, t: lsh.Tables, X: np.ndarray) -> np.ndarray:
    X2 = np.asarray(X, np.float64) ** 2
    if on_tensor_cores(p):
        return np.sqrt(X2 @ (proj_matrix(p, t) ** 2).T)
    ones = [np.ones_like(s) for s in t.s]
    if lsh.is_hcs(p.scheme):
        return np.sqrt(lsh.hcs_sketch(X2, p.mode_d, p.mode_m, t.h, ones))
    return np.sqrt(lsh.cs_sketch(X2, t.h[0], ones[0], p.m))


def check_proj(y_gpu: np.ndarray, y_ref: np.ndarray, sig: np.ndarray) -> dict:
    y_gpu = np.asarray(y_gpu, np.float64)
    err = np.abs(y_gpu - y_ref)
    tol = PROJ_RTOL * np.maximum(np.abs(y_ref), 0.1 * sig)
    empty = sig == 0
    bad = (err > tol) & ~empty
    bad_empty = empty & (y_gpu != 0)
    small = (np.abs(y_ref) < 0.1 * sig) & ~empty
    return {"n": int(y_ref.size), "bad": int(bad.sum()), "bad_empty": int(bad_empty.sum()),
            "below_floor": int(small.sum()), "max_rel": float((err / np.maximum(tol, 1e-300) * PROJ_RTOL).max())
            if y_ref.size else 0.0}


FP32_U = 2.0 ** -24


def nnz_terms(p: lsh.Params, t: lsh.Tables, X: np.ndarray) -> np.ndarray:
    """Number of nonzero products in each projection entry."""
    nz = (np.asarray(X) != 0).astype(np.float64)
    if on_tensor_cores(p):
        return nz @ (proj_matrix(p, t) != 0).astype(np.float64).T
    ones = [np.ones_like(s) for s in t.s]
    if lsh.is_hcs(p.scheme):
        return lsh.hcs_sketch(nz, p.mode_d, p.mode_m, t.h, ones)
    return lsh.cs_sketch(nz, t.h[0], ones[0], p.m)


def tc_band_y(p: lsh.Params, t: lsh.Tables, X: np.ndarray) -> np.ndarray:
    """Rigorous fp32 tensor-core accumulation bound of the dense projection:
    Y = [x0|x1|x2].[R|R|R]^T accumulates in fp32 TMEM over 16-wide K steps; each step
    with a nonzero product rounds the accumulator once, by at most u * sum_i |r_li x_i|.
    """
    Xa = np.abs(np.asarray(X, np.float64))
    d = Xa.shape[1]
    chunks = (np.add.reduceat((Xa != 0).astype(np.int64), np.arange(0, d, 16), axis=1) > 0).sum(axis=1)
    abs_sum = Xa @ np.abs(proj_matrix(p, t)).T
    return 3.0 * chunks[:, None] * FP32_U * abs_sum


def code_band(p: lsh.Params, t: lsh.Tables, X: np.ndarray) -> np.ndarray:
    """Per-entry exemption half-width in quotient units (see module docstring)."""
    w = float(np.float32(p.w))
    nnz = nnz_terms(p, t, X)
    derived = 6.0 * FP32_U * np.sqrt(nnz) * lsh.e2lsh_scale(p) * sigma(p, t, X) / w
    if on_tensor_cores(p):
        derived = np.maximum(derived, tc_band_y(p, t, X) / w)
    return np.where(nnz > 0, np.maximum(CODE_BAND, derived), 0.0)


def srp_band(p: lsh.Params, t: lsh.Tables, X: np.ndarray) -> np.ndarray:
    nnz = nnz_terms(p, t, X)
    derived = 6.0 * FP32_U * np.sqrt(nnz) * sigma(p, t, X)
    if on_tensor_cores(p):
        derived = np.maximum(derived, tc_band_y(p, t, X))
    return np.where(nnz > 0, np.maximum(SRP_BAND, derived), 0.0)


def exempt_mask(p: lsh.Params, ref: dict) -> np.ndarray:
    if lsh.is_e2lsh(p.scheme):
        q = ref["quotient"]
        band = ref.get("band", CODE_BAND)
        return np.abs(q - np.round(q)) < band
    return np.abs(ref["proj"]) < ref.get("band", SRP_BAND)


def check_codes(p: lsh.Params, ref: dict, gpu_codes=None, gpu_bits=None) -> dict:
    ex = exempt_mask(p, ref)
    if lsh.is_e2lsh(p.scheme):
        mism = np.asarray(gpu_codes, np.int64) != ref["codes"]
    else:
        mism = np.asarray(gpu_bits, np.int64) != ref["bits"]
    return {"n": int(mism.size), "exempt": int(ex.sum()), "mismatch": int(mism.sum()),
            "mismatch_outside_exempt": int((mism & ~ex).sum())}


def unpack_bits(words: np.ndarray, m: int) -> np.ndarray:
    w = np.asarray(words).astype(np.uint32)
    out = np.zeros((w.shape[0], m), dtype=np.int64)
    for l in range(m):
        out[:, l] = (w[:, l >> 5] >> np.uint32(l & 31)) & 1
    return out


def check_keys(p: lsh.Params, ref: dict, gpu_keys: np.ndarray) -> dict:
    ex = exempt_mask(p, ref)  # [n][m]
    n = ex.shape[0]
    ex_t = ex.reshape(n, p.L, p.K).any(axis=2).T  # [L][n]
    mism = np.asarray(gpu_keys, np.uint64) != ref["keys"]
    return {"n": int(mism.size), "exempt": int(ex_t.sum()), "mismatch": int(mism.sum()),
            "mismatch_outside_exempt": int((mism & ~ex_t).sum())}
