"""ORACLE (test infrastructure only) — seeded randomness of the method.

The paper only says the bucket / sign hashes are "2-wise independent random hash
functions" (P:207 Def. CS, P:210 Def. HCS), that E2LSH rows r are "a sample from
the standard normal distribution" (P:167 Def. E2LSH) and that the offset b is
drawn "uniformly at random" from [0, w].  The concrete constructions
below are the DESIGN.md readings R1-R5:

  R1  stream(seed, label) = SplitMix64 seeded with seed XOR FNV-1a-64(label).
  R2  2-wise family over P = 2^61-1:  a = 1 + next() mod (P-1), b = next() mod P,
      eval(i) = ((a*(i+1) + b) mod P) mod range.
      Sign family = same construction with range 2; parity 0 -> +1, 1 -> -1.
  R3  offsets: U = (next() >> 11) * 2^-53, b = fp32(w*U), clamped below w.
  R4  Gaussian rows: Box-Muller on pairs, filled row-major, rounded to bf16 (RNE)
      so a tensor-core product with R is exact (reading B13).

Pure Python integers are used for all 64-bit / 128-bit arithmetic so that a
reader can check every step by eye.
"""

from __future__ import annotations

import math
from typing import List, Sequence

import numpy as np

MASK64 = (1 << 64) - 1
P61 = (1 << 61) - 1  # Mersenne prime 2^61 - 1

FNV64_OFFSET = 0xCBF29CE484222325  # FNV-1a 64-bit offset basis
FNV64_PRIME = 0x100000001B3        # FNV 64-bit prime
SM64_GAMMA = 0x9E3779B97F4A7C15    # SplitMix64 increment


def fnv1a64(data: bytes) -> int:
    """FNV-1a, 64 bit, over bytes (the published algorithm)."""
    h = FNV64_OFFSET
    for byte in data:
        h ^= byte
        h = (h * FNV64_PRIME) & MASK64
    return h


def fmix64(z: int) -> int:
    """SplitMix64 output finaliser (Steele et al.; the 'mix64variant13')."""
    z &= MASK64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
    return z ^ (z >> 31)


class Stream:
    """SplitMix64 generator for one labelled sub-stream (reading R1)."""

    def __init__(self, seed: int, label: str):
        self.state = (int(seed) ^ fnv1a64(label.encode("ascii"))) & MASK64

    def next(self) -> int:
        self.state = (self.state + SM64_GAMMA) & MASK64
        return fmix64(self.state)

    def unit53(self) -> float:
        """(next() >> 11) * 2^-53 in [0, 1): exact double."""
        return (self.next() >> 11) * (1.0 / (1 << 53))


class TwoWise:
    """2-wise independent family ((a(i+1)+b) mod P) mod range (reading R2)."""

    def __init__(self, stream: Stream, rng_range: int):
        if not (1 <= rng_range < P61):
            raise ValueError("range must be in [1, P-1]")
        self.a = 1 + stream.next() % (P61 - 1)
        self.b = stream.next() % P61
        self.range = rng_range

    @staticmethod
    def eval_ab(a: int, b: int, rng_range: int, i: int) -> int:
        return ((a * (i + 1) + b) % P61) % rng_range

    def eval(self, i: int) -> int:
        return self.eval_ab(self.a, self.b, self.range, i)

    def table(self, domain: int) -> List[int]:
        return [self.eval(i) for i in range(domain)]


def bucket_table(seed: int, mode: int, d_k: int, m_k: int, prefix: str = "") -> np.ndarray:
    """h_k : [d_k] -> [m_k] for mode k (k = 0 is the CS hash h), P:205 / P:212.
    `prefix` = "table{t}/" for the per-table families of NEXT-2 (reading C3)."""
    fam = TwoWise(Stream(seed, f"{prefix}mode{mode}/bucket"), m_k)
    return np.array(fam.table(d_k), dtype=np.int64)


def sign_table(seed: int, mode: int, d_k: int, prefix: str = "") -> np.ndarray:
    """s_k : [d_k] -> {+1, -1}; parity 0 -> +1, parity 1 -> -1."""
    fam = TwoWise(Stream(seed, f"{prefix}mode{mode}/sign"), 2)
    return np.array([1 if fam.eval(i) == 0 else -1 for i in range(d_k)], dtype=np.int64)


def offsets(seed: int, m: int, w: float, prefix: str = "") -> np.ndarray:
    """b_l ~ U[0, w), one per coordinate (readings B3, B4, R3); fp32 values."""
    if not w > 0:
        raise ValueError("w must be > 0")
    w32 = np.float32(w)
    st = Stream(seed, f"{prefix}offsets")
    out = np.empty(m, dtype=np.float32)
    for l in range(m):
        u = st.unit53()
        b = np.float32(float(w32) * u)
        if b >= w32:
            b = np.nextafter(w32, np.float32(0))
        out[l] = b
    return out


def round_bf16(x: float) -> float:
    """Round a double to the nearest bfloat16 (8-bit significand), ties to even.

    Operates on the IEEE-754 binary64 bit pattern: keep 1+7 significand bits,
    round the dropped 45 bits to nearest-even.  Valid for normal values in the
    fp32 exponent range (|x| < 3.38e38, which Box-Muller outputs always are).
    """
    if x == 0.0 or not math.isfinite(x):
        return x
    bits = np.array([x], dtype=np.float64).view(np.uint64)[0].item()
    drop = 52 - 7
    lsb = (bits >> drop) & 1
    rounding_bias = (1 << (drop - 1)) - 1 + lsb
    bits = ((bits + rounding_bias) >> drop) << drop
    return float(np.array([bits], dtype=np.uint64).view(np.float64)[0])


def round_bf16_array(x: np.ndarray) -> np.ndarray:
    """round_bf16 elementwise (same bit manipulation, vectorised)."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    bits = x.view(np.uint64)
    drop = np.uint64(45)
    lsb = (bits >> drop) & np.uint64(1)
    with np.errstate(over="ignore"):
        r = ((bits + (np.uint64((1 << 44) - 1) + lsb)) >> drop) << drop
    out = r.view(np.float64).copy()
    out[x == 0] = x[x == 0]
    return out


def _gaussian_rows_vectorised(seed: int, m: int, d: int) -> np.ndarray:
    """Same stream and Box-Muller as gaussian_rows, elementwise in NumPy (large m*d).

    NumPy's log/cos/sin may differ from the C library's in the last ulp; after the
    bf16 rounding this changes a value only if it sits on a rounding tie
    (probability ~2^-40 per value).  Small shapes use the scalar path, which the
    C++ draw is checked against bit for bit.
    """
    total = m * d
    pairs = (total + 1) // 2
    base = np.uint64(Stream(seed, "gaussian").state)
    k = np.arange(1, 2 * pairs + 1, dtype=np.uint64)
    with np.errstate(over="ignore"):
        st = base + k * np.uint64(SM64_GAMMA)
        z = st
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    u = (z >> np.uint64(11)).astype(np.float64) * (1.0 / (1 << 53))
    u1 = 1.0 - u[0::2]
    u2 = u[1::2]
    rho = np.sqrt(-2.0 * np.log(u1))
    vals = np.empty(2 * pairs, dtype=np.float64)
    vals[0::2] = rho * np.cos(2.0 * math.pi * u2)
    vals[1::2] = rho * np.sin(2.0 * math.pi * u2)
    return round_bf16_array(vals[:total]).reshape(m, d)


def gaussian_rows(seed: int, m: int, d: int) -> np.ndarray:
    """R in N(0,1)^{m x d}, Box-Muller, row-major fill, bf16-rounded (R4).

    Returns float64 array whose values are exactly bf16-representable.
    """
    if m * d > (1 << 20):
        return _gaussian_rows_vectorised(seed, m, d)
    st = Stream(seed, "gaussian")
    total = m * d
    vals = np.empty(total, dtype=np.float64)
    k = 0
    while k < total:
        u1 = 1.0 - st.unit53()          # in (0, 1]
        u2 = st.unit53()                # in [0, 1)
        rho = math.sqrt(-2.0 * math.log(u1))
        z0 = rho * math.cos(2.0 * math.pi * u2)
        z1 = rho * math.sin(2.0 * math.pi * u2)
        vals[k] = round_bf16(z0)
        k += 1
        if k < total:
            vals[k] = round_bf16(z1)
            k += 1
    return vals.reshape(m, d)


def flat_index(idx: Sequence[int], dims: Sequence[int]) -> int:
    """j = i_1 + sum_{k>=2} i_k prod_{t<k} d_t, 0-based column-major (reading B6)."""
    j, stride = 0, 1
    for i, dk in zip(idx, dims):
        if not 0 <= i < dk:
            raise ValueError("index out of range")
        j += i * stride
        stride *= dk
    return j


def unflatten(j: int, dims: Sequence[int]) -> List[int]:
    """Inverse of flat_index: i_k = floor(j / prod_{t<k} d_t) mod d_k."""
    out = []
    for dk in dims:
        out.append(j % dk)
        j //= dk
    return out
