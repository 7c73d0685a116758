"""GPU <-> oracle comparison rules (north_star tolerances).

  projections: |y_gpu - y_ref| <= 1e-4 * max(|y_ref|, 0.1 * sigma_l), sigma_l the
               dot product's natural scale sqrt(sum_i a_li^2 x_i^2); sigma_l == 0
               (empty bin) requires y_gpu == 0 exactly.
  E2LSH codes: bit-exact except entries whose quotient (scale*y+b)/w lies within
               1e-5 of an integer (counted and reported).
  SRP bits:    bit-exact except entries with |y_ref| < 1e-6 (counted, reported).
  keys:        bit-exact for every (table, point) without an exempt coordinate.
  tables:      bit-exact given identical keys.
"""

from __future__ import annotations

import numpy as np

from oracle import lsh

PROJ_RTOL = 1e-4
CODE_BAND = 1e-5
SRP_BAND = 1e-6


def sigma(p: lsh.Params, t: lsh.Tables, X: np.ndarray) -> np.ndarray:
    X2 = np.asarray(X, np.float64) ** 2
    if lsh.is_dense(p.scheme):
        return np.sqrt(X2 @ (t.R.astype(np.float64) ** 2).T)
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


def exempt_mask(p: lsh.Params, ref: dict) -> np.ndarray:
    if lsh.is_e2lsh(p.scheme):
        q = ref["quotient"]
        return np.abs(q - np.round(q)) < CODE_BAND
    return np.abs(ref["proj"]) < SRP_BAND


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
