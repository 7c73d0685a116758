"""ORACLE (test infrastructure only) — the paper's hashers, keys and tables.

Plain definitions in fp64 (inputs are the same fp32 arrays the GPU reads,
widened exactly).  No blocking, fusion or reordering beyond what the cited
definition states.

  * CS(p)_l = sum_{i: h(i)=l} s(i) p_i                    P:205 (eq:eq_cs, Def. CS)
  * HCS(p)_{l_1..l_N} = sum_{h_k(i_k)=l_k} prod_k s_k(i_k) p_j,
    j = i_1 + sum_{k>=2} i_k prod_{t<k} d_t               P:212-215 (eq:eqhcs, Def. HCS)
  * vec(HCS) index l = l_1 + sum_{k>=2} l_k prod_{t<k} m_t  P:613 (HCS-E2LSH proof)
  * E2LSH  h(p) = floor((<r,p> + b)/w)                    P:169 (eq:datar_lsh)
  * SRP    bit = 1 iff <r,u> > 0 else 0                   P:187-188 (Def. SRP)
  * CS-E2LSH  g(p)_l  = floor((sqrt(m) CS(p)_l + b)/w)    P:314 (Def. CS-E2LSH)
  * HCS-E2LSH g'(p)_l = floor((sqrt(m) vec(HCS(p))_l + b)/w)  P:624 (eq:eq_hca_eucl_lsh)
  * CS-SRP  xi(u)_l  = sgn(CS(u)_l), sgn(0)=0             P:918-920 (Def. CS-SRP)
  * HCS-SRP xi'(u)_l = sgn(vec(HCS(u))_l)                 P:1441-1443 (Def. HCS-SRP)
  * (m, L) index: code concatenation, store p in bucket hbar_t(p) of table t,
    query collects the bucket of hbar_t(q)                P:155 (§3.1)

Readings: B1 one sketch of total size m = L*K per point, table t
uses coordinates [tK, (t+1)K); B2 sqrt(m) with m the total size; B3 one offset
per coordinate; B6 0-based column-major; B7 logical zero padding; B9 floor
toward -inf; B10 E2LSH bucket key = 64-bit fingerprint of the K codes; B11
buckets in ascending unsigned key order, ids ascending inside a bucket.
C3 (NEXT-2, per_table=True): table t has its own CS family (h_t, s_t, b_t) of
size K drawn from streams "table{t}/...", g_t(p)_k = floor((sqrt(K) CS_t(p)_k +
b_tk)/w) -- the literal reading of "L independent hash tables".
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

from . import rng

SCHEMES = ("E2LSH", "SRP", "CS_E2LSH", "CS_SRP", "HCS_E2LSH", "HCS_SRP")
INT32_MIN, INT32_MAX = -(1 << 31), (1 << 31) - 1


def is_e2lsh(scheme: str) -> bool:
    return scheme in ("E2LSH", "CS_E2LSH", "HCS_E2LSH")


def is_dense(scheme: str) -> bool:
    return scheme in ("E2LSH", "SRP")


def is_hcs(scheme: str) -> bool:
    return scheme in ("HCS_E2LSH", "HCS_SRP")


@dataclass
class Params:
    """Problem statement of one hasher."""

    scheme: str
    d: int
    m: int
    L: int
    K: int
    w: float = 4.0
    seed: int = 0
    mode_d: Tuple[int, ...] = field(default_factory=tuple)  # HCS only
    mode_m: Tuple[int, ...] = field(default_factory=tuple)  # HCS only
    per_table: bool = False   # NEXT-2 (reading C3): L independent CS families of size K

    def __post_init__(self):
        if self.scheme not in SCHEMES:
            raise ValueError(f"unknown scheme {self.scheme}")
        if self.m < 1 or self.L * self.K != self.m:
            raise ValueError("m must equal L*K (reading B1)")
        if not self.w > 0:
            raise ValueError("w must be > 0")
        if not is_e2lsh(self.scheme) and self.K > 64:
            raise ValueError("SRP keys hold at most 64 bits")
        if self.per_table and self.scheme not in ("CS_E2LSH", "CS_SRP"):
            raise ValueError("per-table families are defined here for the CS schemes only")
        if is_hcs(self.scheme):
            if len(self.mode_d) != len(self.mode_m) or not self.mode_d:
                raise ValueError("HCS needs per-mode d_k and m_k")
            if int(np.prod(self.mode_m)) != self.m:
                raise ValueError("prod m_k must equal m")
            if int(np.prod(self.mode_d)) < self.d:
                raise ValueError("prod d_k must be >= d (zero padding, P:2003)")
        else:
            self.mode_d, self.mode_m = (self.d,), (self.m,)

    @property
    def N(self) -> int:
        return len(self.mode_d)


@dataclass
class Tables:
    """Materialised random parameters of one hasher."""

    h: List[np.ndarray]            # per mode: bucket table h_k[d_k] (per_table: per table t, h_t[d] in [K])
    s: List[np.ndarray]            # per mode: sign table s_k[d_k] in {+1,-1} (per_table: per table)
    b: np.ndarray                  # fp32 offsets, m values
    R: Optional[np.ndarray] = None  # dense only: m x d, bf16-exact values


def make_tables(p: Params) -> Tables:
    """Draw the parameters of `p` from its seed (readings R1-R4)."""
    if is_dense(p.scheme):
        R = rng.gaussian_rows(p.seed, p.m, p.d)
        return Tables(h=[], s=[], b=rng.offsets(p.seed, p.m, p.w), R=R)
    if p.per_table:
        # reading C3 ("L independent hash tables"; SURVEY 8(c) A1 "table{t}/"):
        # table t draws its own h_t : [d] -> [K], s_t and b_t[K] from streams "table{t}/..."
        pre = [f"table{t}/" for t in range(p.L)]
        h = [rng.bucket_table(p.seed, 0, p.d, p.K, pre[t]) for t in range(p.L)]
        s = [rng.sign_table(p.seed, 0, p.d, pre[t]) for t in range(p.L)]
        b = np.concatenate([rng.offsets(p.seed, p.K, p.w, pre[t]) for t in range(p.L)])
        return Tables(h=h, s=s, b=b)
    h = [rng.bucket_table(p.seed, k, dk, mk) for k, (dk, mk) in enumerate(zip(p.mode_d, p.mode_m))]
    s = [rng.sign_table(p.seed, k, dk) for k, dk in enumerate(p.mode_d)]
    return Tables(h=h, s=s, b=rng.offsets(p.seed, p.m, p.w))


# --------------------------------------------------------------------------
# Projection step (the paper's O(d) vs O(md) claim lives here)
# --------------------------------------------------------------------------

def cs_sketch(X: np.ndarray, h: np.ndarray, s: np.ndarray, m: int, ops: Optional[list] = None) -> np.ndarray:
    """CS(p)_l = sum_{h(i)=l} s(i) p_i for every row p of X.

    One multiply-add per input coordinate, independent of m ("only d
    non-zero entries, one per column").
    """
    X = np.asarray(X, dtype=np.float64)
    n, d = X.shape
    Y = np.zeros((n, m), dtype=np.float64)
    for i in range(d):
        Y[:, h[i]] += s[i] * X[:, i]
        if ops is not None:
            ops[0] += n
    return Y


def hcs_coordinate(j: int, mode_d: Sequence[int], mode_m: Sequence[int],
                   h: Sequence[np.ndarray], s: Sequence[np.ndarray]) -> Tuple[int, int]:
    """(vec index l, sign) that coordinate j of p contributes to in Def. HCS.

    (i_1..i_N) = unflatten(j) over (d_1..d_N), l_k = h_k(i_k),
    l = l_1 + sum_{k>=2} l_k prod_{t<k} m_t, sign = prod_k s_k(i_k).
    """
    idx = rng.unflatten(j, mode_d)
    l_modes = [int(h[k][idx[k]]) for k in range(len(mode_d))]
    sign = 1
    for k in range(len(mode_d)):
        sign *= int(s[k][idx[k]])
    return rng.flat_index(l_modes, mode_m), sign


def hcs_sketch(X: np.ndarray, mode_d, mode_m, h, s, ops: Optional[list] = None) -> np.ndarray:
    """vec(HCS(p)) for every row p of X, zero padding logical.

    Padding coordinates j >= d carry value 0 and are skipped (reading B7).
    """
    X = np.asarray(X, dtype=np.float64)
    n, d = X.shape
    if int(np.prod(mode_d)) < d:
        raise ValueError("prod d_k < d")
    m = int(np.prod(mode_m))
    Y = np.zeros((n, m), dtype=np.float64)
    for j in range(d):
        l, sign = hcs_coordinate(j, mode_d, mode_m, h, s)
        Y[:, l] += sign * X[:, j]
        if ops is not None:
            ops[0] += n
    return Y


def dense_project(X: np.ndarray, R: np.ndarray, ops: Optional[list] = None) -> np.ndarray:
    """<r_l, p> for every Gaussian row r_l: O(md) per point."""
    X = np.asarray(X, dtype=np.float64)
    R = np.asarray(R, dtype=np.float64)
    if ops is not None:
        ops[0] += X.shape[0] * R.shape[0] * R.shape[1]
    return X @ R.T


def project(p: Params, t: Tables, X: np.ndarray) -> np.ndarray:
    if p.per_table:
        # table t: its own count sketch of size K; coordinates [tK, (t+1)K) of the code
        return np.concatenate([cs_sketch(X, t.h[tt], t.s[tt], p.K) for tt in range(p.L)], axis=1)
    if is_dense(p.scheme):
        return dense_project(X, t.R)
    if is_hcs(p.scheme):
        return hcs_sketch(X, p.mode_d, p.mode_m, t.h, t.s)
    return cs_sketch(X, t.h[0], t.s[0], p.m)


# --------------------------------------------------------------------------
# Discretisation
# --------------------------------------------------------------------------

def e2lsh_scale(p: Params) -> float:
    """sqrt(m) for CS/HCS-E2LSH (reading B2); 1 for E2LSH;
    sqrt(K) for the per-table families, whose sketch size is K (reading C3)."""
    if p.per_table:
        return float(np.sqrt(p.K))
    return 1.0 if is_dense(p.scheme) else float(np.sqrt(p.m))


def e2lsh_quotient(Y: np.ndarray, b: np.ndarray, w: float, scale: float) -> np.ndarray:
    """(scale * y_l + b_l) / w in fp64 (the argument of the floor)."""
    return (scale * np.asarray(Y, np.float64) + np.asarray(b, np.float64)[None, :]) / float(np.float32(w))


def e2lsh_codes(Y: np.ndarray, b: np.ndarray, w: float, scale: float) -> np.ndarray:
    """z_l = floor((scale*y_l + b_l)/w), floor toward -inf (reading B9)."""
    z = np.floor(e2lsh_quotient(Y, b, w, scale))
    if z.size and (z.min() < INT32_MIN or z.max() > INT32_MAX):
        raise OverflowError("E2LSH code outside int32")
    return z.astype(np.int64)


def srp_bits(Y: np.ndarray) -> np.ndarray:
    """sgn(y) = 1 if y > 0 otherwise 0 (sgn(0) = 0, reading B8)."""
    return (np.asarray(Y) > 0).astype(np.int64)


# --------------------------------------------------------------------------
# Table keys (P:155 concatenation; reading B1, B10)
# --------------------------------------------------------------------------

def srp_keys(bits: np.ndarray, L: int, K: int) -> np.ndarray:
    """key_t = sum_{k<K} bit_{tK+k} 2^k, exact (K <= 64). Returns uint64 [L][n]."""
    n = bits.shape[0]
    out = np.zeros((L, n), dtype=np.uint64)
    for t in range(L):
        for k in range(K):
            out[t] |= bits[:, t * K + k].astype(np.uint64) << np.uint64(k)
    return out


# Reading B10: the 64-bit bucket key of one table's K codes is two
# independent 32-bit polynomial (Horner) hashes of the codes, concatenated and
# passed through the SplitMix64 finaliser.  Odd multipliers make every Horner
# step a bijection of the state; fmix64 is a bijection, so two tuples share a key
# iff both 32-bit polynomials agree.
FP_A = 0x9E3779B1   # odd 32-bit multipliers of the two lanes
FP_B = 0x85EBCA77
MASK32 = 0xFFFFFFFF


def fingerprint(words: Sequence[int]) -> int:
    """64-bit key of one table's K codes (reading B10).

    u_k = z_k as a 32-bit two's-complement word;
    a = sum_k u_k * FP_A^(K-1-k) mod 2^32, b = sum_k u_k * FP_B^(K-1-k) mod 2^32
    (evaluated by Horner: a <- a*FP_A + u_k from a = 0);
    key = fmix64(a * 2^32 + b).  Integer-only, so any two correct implementations agree.
    """
    a = b = 0
    for z in words:
        u = int(z) & MASK32
        a = (a * FP_A + u) & MASK32
        b = (b * FP_B + u) & MASK32
    return rng.fmix64((a << 32) | b)


def _fmix64_np(z: np.ndarray) -> np.ndarray:
    """rng.fmix64 applied elementwise (numpy uint64 arithmetic wraps mod 2^64)."""
    z = z.astype(np.uint64)
    z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def e2lsh_keys(codes: np.ndarray, L: int, K: int) -> np.ndarray:
    """fingerprint() of every (point, table), elementwise over points (uint64 [L][n])."""
    n = codes.shape[0]
    out = np.zeros((L, n), dtype=np.uint64)
    words = (np.asarray(codes, dtype=np.int64) & MASK32).astype(np.uint64)
    m32 = np.uint64(MASK32)
    with np.errstate(over="ignore"):
        for t in range(L):
            a = np.zeros(n, dtype=np.uint64)
            b = np.zeros(n, dtype=np.uint64)
            for k in range(K):
                a = (a * np.uint64(FP_A) + words[:, t * K + k]) & m32
                b = (b * np.uint64(FP_B) + words[:, t * K + k]) & m32
            out[t] = _fmix64_np((a << np.uint64(32)) | b)
    return out


def hash_points(p: Params, t: Tables, X: np.ndarray) -> Dict[str, np.ndarray]:
    """Projection -> discretisation -> keys for every row of X."""
    Y = project(p, t, X)
    out = {"proj": Y}
    if is_e2lsh(p.scheme):
        codes = e2lsh_codes(Y, t.b, p.w, e2lsh_scale(p))
        out["codes"] = codes
        out["quotient"] = e2lsh_quotient(Y, t.b, p.w, e2lsh_scale(p))
        out["keys"] = e2lsh_keys(codes, p.L, p.K)
    else:
        bits = srp_bits(Y)
        out["bits"] = bits
        out["keys"] = srp_keys(bits, p.L, p.K)
    return out


# --------------------------------------------------------------------------
# Grouping into buckets and lookup (reading B11)
# --------------------------------------------------------------------------

@dataclass
class TableIndex:
    ids: np.ndarray    # uint32 [n]   ids sorted by (key, id)
    ukeys: np.ndarray  # uint64 [nb]  distinct keys, ascending
    offs: np.ndarray   # uint32 [nb+1] bucket b = ids[offs[b]:offs[b+1]]


def group_table(keys_t: np.ndarray, id_base: int = 0) -> TableIndex:
    """Stable argsort of the uint64 keys (ties by ascending id), run-length."""
    keys_t = np.asarray(keys_t, dtype=np.uint64)
    n = keys_t.shape[0]
    order = np.argsort(keys_t, kind="stable")
    sk = keys_t[order]
    if n:
        head = np.ones(n, dtype=bool)
        head[1:] = sk[1:] != sk[:-1]
        starts = np.nonzero(head)[0]
    else:
        starts = np.zeros(0, dtype=np.int64)
    offs = np.concatenate([starts, [n]]).astype(np.uint32)
    return TableIndex(ids=(order + id_base).astype(np.uint32), ukeys=sk[starts].copy(), offs=offs)


def group(keys: np.ndarray, id_base: int = 0) -> List[TableIndex]:
    return [group_table(keys[t], id_base) for t in range(keys.shape[0])]


def group_by_tuple(codes_t: np.ndarray) -> Dict[tuple, List[int]]:
    """Buckets keyed by the exact K-tuple of codes (P:155 'bucket hbar_t(p)')."""
    out: Dict[tuple, List[int]] = {}
    for i, row in enumerate(np.asarray(codes_t).tolist()):
        out.setdefault(tuple(row), []).append(i)
    return out


def fingerprint_merges(codes: np.ndarray, keys: np.ndarray, L: int, K: int) -> int:
    """Rows whose exact K-tuple differs from the first tuple filed under the same (table, key)."""
    merges = 0
    for t in range(L):
        seen: Dict[int, tuple] = {}
        for i in range(codes.shape[0]):
            tup = tuple(codes[i, t * K:(t + 1) * K].tolist())
            k = int(keys[t, i])
            if k in seen and seen[k] != tup:
                merges += 1
            seen.setdefault(k, tup)
    return merges


def lookup(tix: TableIndex, qkey: int) -> Tuple[int, int]:
    """Bucket [begin, end) of qkey in one table; empty range at the insertion point."""
    pos = int(np.searchsorted(tix.ukeys, np.uint64(qkey), side="left"))
    if pos < tix.ukeys.shape[0] and int(tix.ukeys[pos]) == int(qkey):
        return int(tix.offs[pos]), int(tix.offs[pos + 1])
    at = int(tix.offs[pos]) if pos < tix.offs.shape[0] else int(tix.offs[-1])
    return at, at


def key_width(p: Params) -> int:
    """Significant bits of a key: 64 for E2LSH fingerprints, K for SRP."""
    return 64 if is_e2lsh(p.scheme) else p.K


def coarse_bin(key: int, width: int, B: int) -> int:
    """Top B bits of a `width`-bit key; the key itself if width <= B."""
    return int(key) >> (width - B) if width > B else int(key)


def coarse_counts(p: Params, keys: np.ndarray, B: int) -> np.ndarray:
    """counts[t][bin] of the per-table coarse histogram exchanged across ranks."""
    width = key_width(p)
    out = np.zeros((keys.shape[0], 1 << B), dtype=np.uint32)
    for t in range(keys.shape[0]):
        for k in keys[t].tolist():
            out[t, coarse_bin(k, width, B)] += 1
    return out


# --------------------------------------------------------------------------
# Space and time accounting (Table 1; Remark rem:hcs_space P:218-221)
# --------------------------------------------------------------------------

def param_count(p: Params) -> int:
    """Stored values of the projection structure (S:516-521 convention).

    Dense: m*d Gaussians; CS: 2d table entries (bucket + sign); HCS: 2*sum d_k;
    plus m offsets for the E2LSH variants.
    """
    if p.per_table:
        base = 2 * p.d * p.L
    elif is_dense(p.scheme):
        base = p.m * p.d
    elif is_hcs(p.scheme):
        base = 2 * sum(p.mode_d)
    else:
        base = 2 * p.d
    return base + (p.m if is_e2lsh(p.scheme) else 0)


def projection_op_count(p: Params, t: Tables, x: np.ndarray) -> int:
    """Multiply-adds the projection of one point performs (instrumented).

    Runs the projection above with its counter: one accumulation per input
    coordinate for CS/HCS (padding slots never touched), m*d for the dense one.
    """
    ops = [0]
    x = np.asarray(x, dtype=np.float64).reshape(1, -1)
    if p.per_table:
        for tt in range(p.L):
            cs_sketch(x, t.h[tt], t.s[tt], p.K, ops)
    elif is_dense(p.scheme):
        dense_project(x, t.R, ops)
    elif is_hcs(p.scheme):
        hcs_sketch(x, p.mode_d, p.mode_m, t.h, t.s, ops)
    else:
        cs_sketch(x, t.h[0], t.s[0], p.m, ops)
    return ops[0]


def global_coarse_offsets(all_counts: np.ndarray, rank: int) -> np.ndarray:
    """Global start of rank `rank`'s run of every (table, coarse bin).

    offset[t][b] = sum_{b' < b} sum_r counts[r][t][b']  +  sum_{r' < rank} counts[r'][t][b]
    i.e. the concatenation order is bin-major, rank-minor, matching the G=1 order
    of buckets (coarse bins ascend with the key) with ids ascending across ranks.
    """
    c = np.asarray(all_counts, dtype=np.int64)          # [G][L][2^B]
    totals = c.sum(axis=0)                              # [L][2^B]
    before_bins = np.concatenate([np.zeros((totals.shape[0], 1), np.int64),
                                  np.cumsum(totals, axis=1)[:, :-1]], axis=1)
    before_ranks = c[:rank].sum(axis=0) if rank > 0 else np.zeros_like(totals)
    return before_bins + before_ranks


# ---------------------------------------------------------------------------
# Query completion: candidates = the union of the query's L
# buckets ("collect the index of all the elements"), exact re-rank, top-k
# under the family's similarity (§6: Euclidean for the E2LSH family,
# cosine for the SRP family).  Reading C1: the bucket entries are taken
# in table order (t = 0..L-1, each bucket in ascending id), truncated to max_cand
# entries BEFORE removing duplicates, so the cap is deterministic.  Reading C2:
# scores are squared Euclidean distance (ascending) or cosine similarity
# (descending; 0 when a norm is 0); ties by ascending id; missing slots id -1.
# ---------------------------------------------------------------------------
def query_candidates(tables: List[TableIndex], qkeys_q: Sequence[int], max_cand: int) -> np.ndarray:
    """Distinct candidate ids of one query (ascending)."""
    lst: List[int] = []
    for t, tix in enumerate(tables):
        b, e = lookup(tix, int(qkeys_q[t]))
        lst.extend(int(v) for v in tix.ids[b:e])
    return np.unique(np.asarray(lst[:max_cand], dtype=np.int64))


def rerank(Xrows: np.ndarray, q: np.ndarray, cand: np.ndarray, k: int, metric: str) -> Tuple[np.ndarray, np.ndarray]:
    """Top-k of `cand` (global ids; Xrows[i] is the row of candidate cand[i]) by exact fp64 score."""
    Xr = np.asarray(Xrows, np.float64)
    qq = np.asarray(q, np.float64)
    if metric == "l2":
        sc = ((Xr - qq[None, :]) ** 2).sum(axis=1)
        order = np.lexsort((cand, sc))
    else:
        nx = np.sqrt((Xr ** 2).sum(axis=1))
        nq = float(np.sqrt((qq ** 2).sum()))
        dots = Xr @ qq
        sc = np.where((nx > 0) & (nq > 0), dots / np.maximum(nx * nq, 1e-300), 0.0)
        order = np.lexsort((cand, -sc))
    ids = np.full(k, -1, np.int64)
    scores = np.full(k, np.inf if metric == "l2" else -np.inf)
    top = order[:k]
    ids[: len(top)] = cand[top]
    scores[: len(top)] = sc[top]
    return ids, scores


def metric_of(p: Params) -> str:
    return "l2" if is_e2lsh(p.scheme) else "cosine"
