"""paper_2503_06737_b200 — B200-native hot path of arXiv 2503.06737.

Thin Python binding (argument marshalling only) over the C ABI in include/lsh.h,
implemented by the in-tree shared library liblsh_b200.so (CUDA, sm_100a).  Every
step of the path (projection / sketch, discretisation, key packing, grouping,
lookup) runs in that library's kernels; PyTorch only provides device memory and
streams.  There is no CPU fallback: if the library is missing this module raises.
"""

from __future__ import annotations

import ctypes
import os
from typing import Optional, Sequence, Tuple

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "liblsh_b200.so")
if os.environ.get("LSH_LIB_VARIANT"):   # e.g. "checked": device bounds-checked build (tools/gpu_checked.sh)
    LIB_PATH = os.path.join(_HERE, f"liblsh_b200_{os.environ['LSH_LIB_VARIANT']}.so")

SCHEMES = {"E2LSH": 0, "SRP": 1, "CS_E2LSH": 2, "CS_SRP": 3, "HCS_E2LSH": 4, "HCS_SRP": 5}
STATUS = {0: "LSH_OK", 1: "LSH_EINVAL", 2: "LSH_EDIM", 3: "LSH_ENOMEM", 4: "LSH_ECUDA", 5: "LSH_EOVERFLOW",
          6: "LSH_ESTATE", 7: "LSH_EUNSUPPORTED"}
EXPORT = {"bucket": 0, "sign": 1, "offsets": 2, "gaussian": 3, "coeffs": 4, "coord": 5}
MAX_MODES = 8


class LshError(RuntimeError):
    def __init__(self, status: int, where: str, detail: str = ""):
        self.status = status
        super().__init__(f"{where}: {STATUS.get(status, status)} {detail}".strip())


class lsh_params(ctypes.Structure):
    _fields_ = [("scheme", ctypes.c_int32), ("N", ctypes.c_int32), ("d", ctypes.c_int64),
                ("mode_d", ctypes.c_int32 * MAX_MODES), ("mode_m", ctypes.c_int32 * MAX_MODES),
                ("m", ctypes.c_int32), ("L", ctypes.c_int32), ("K", ctypes.c_int32), ("w", ctypes.c_float),
                ("seed", ctypes.c_uint64), ("device", ctypes.c_int32), ("flags", ctypes.c_int32)]


_lib = None


def lib() -> ctypes.CDLL:
    """Load liblsh_b200.so (raises if it was not built: no fallback path exists)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} missing: run `python -m paper_2503_06737_b200.build` "
                          "(or __graft_entry__.build()); there is no CPU fallback")
    L = ctypes.CDLL(LIB_PATH)
    vp, i32, i64, u64, sz = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64, ctypes.c_size_t
    P = ctypes.POINTER
    sig = {
        "lsh_create": (i32, [P(lsh_params), P(vp)]),
        "lsh_destroy": (None, [vp]),
        "lsh_hash": (i32, [vp, vp, i64, i64, vp, vp, vp, vp, vp]),
        "lsh_build_index": (i32, [vp, vp, i64, i64, i64, P(vp), vp]),
        "lsh_group_keys": (i32, [vp, vp, i64, i64, P(vp), vp]),
        "lsh_index_view": (i32, [vp, i32, P(vp), P(vp), P(vp), P(i64)]),
        "lsh_index_size": (i64, [vp]),
        "lsh_index_destroy": (None, [vp]),
        "lsh_query_buckets": (i32, [vp, vp, vp, i64, i64, vp, vp, vp]),
        "lsh_query_knn": (i32, [vp, vp, vp, i64, vp, i64, i64, i32, i32, vp, vp, vp, vp]),
        "lsh_index_counts": (i32, [vp, i32, vp, vp]),
        "lsh_global_offsets": (i32, [vp, i32, i32, i32, i32, vp, vp]),
        "lsh_query_global_runs": (i32, [vp, i32, i32, i64, vp, vp, vp]),
        "lsh_export_host": (i32, [P(lsh_params), i32, i32, vp, P(sz)]),
        "lsh_get_params": (i32, [vp, i32, i32, vp, P(sz)]),
        "lsh_check": (i32, [vp]),
        "lsh_group_path": (i32, [vp, P(i32)]),
        "lsh_strerror": (ctypes.c_char_p, [i32]),
        "lsh_last_cuda_error": (ctypes.c_char_p, []),
        "lsh_launch_count": (u64, []),
        "lsh_timing_enable": (None, [i32]),
        "lsh_timing_get": (i32, [ctypes.c_char_p, P(ctypes.c_double), P(i64)]),
        "lsh_timing_reset": (None, []),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    _lib = L
    return L


def _check(status: int, where: str):
    if status != 0:
        detail = ""
        if status == 4:
            detail = lib().lsh_last_cuda_error().decode(errors="replace")
        raise LshError(status, where, detail)


FLAG_PER_TABLE = 1   # include/lsh.h LSH_FLAG_PER_TABLE


def make_params(scheme: str, d: int, m: int, L: int, K: int, w: float = 4.0, seed: int = 0,
                mode_d: Optional[Sequence[int]] = None, mode_m: Optional[Sequence[int]] = None,
                device: int = 0, per_table: bool = False) -> lsh_params:
    """per_table: NEXT-2 independent families per table (LSH_FLAG_PER_TABLE, reading C3)."""
    p = lsh_params()
    p.scheme = SCHEMES[scheme]
    p.d, p.m, p.L, p.K, p.w, p.seed, p.device = d, m, L, K, w, seed, device
    p.flags = FLAG_PER_TABLE if per_table else 0
    if scheme.startswith("HCS"):
        if not mode_d or not mode_m or len(mode_d) != len(mode_m):
            raise ValueError("HCS needs mode_d and mode_m")
        p.N = len(mode_d)
        for k, (a, b) in enumerate(zip(mode_d, mode_m)):
            p.mode_d[k], p.mode_m[k] = a, b
    else:
        p.N = 1
        p.mode_d[0], p.mode_m[0] = d, m
    return p


def export_host(params: lsh_params, what: str, mode: int = 0):
    """Host-only parameter draw (lsh_export_host) as a numpy array."""
    import numpy as np
    sz = ctypes.c_size_t(0)
    st = lib().lsh_export_host(ctypes.byref(params), EXPORT[what], mode, None, ctypes.byref(sz))
    if st not in (0, 2):
        _check(st, "lsh_export_host")
    dtype = {"bucket": np.int32, "sign": np.int32, "offsets": np.float32, "gaussian": np.uint16,
             "coeffs": np.uint64, "coord": np.int32}[what]
    buf = np.zeros(sz.value // np.dtype(dtype).itemsize, dtype=dtype)
    _check(lib().lsh_export_host(ctypes.byref(params), EXPORT[what], mode, buf.ctypes.data_as(ctypes.c_void_p),
                                 ctypes.byref(sz)), "lsh_export_host")
    return buf


def launch_count() -> int:
    return int(lib().lsh_launch_count())


def timing_enable(on: bool = True):
    lib().lsh_timing_enable(1 if on else 0)


def timing_reset():
    lib().lsh_timing_reset()


def timing_get(name: str) -> Tuple[float, int]:
    ms, n = ctypes.c_double(0), ctypes.c_int64(0)
    _check(lib().lsh_timing_get(name.encode(), ctypes.byref(ms), ctypes.byref(n)), "lsh_timing_get")
    return ms.value, n.value


def global_offsets(all_counts, rank: int, stream=None):
    """lsh_global_offsets: all_counts int32/uint32 [G, L, 2^B] (CUDA) -> int64 [L, 2^B]."""
    torch = _torch()
    G, L, nb = all_counts.shape
    B = nb.bit_length() - 1
    if (1 << B) != nb:
        raise ValueError("last dimension must be 2^B")
    out = torch.empty((L, nb), dtype=torch.int64, device=all_counts.device)
    _check(lib().lsh_global_offsets(_dev_ptr(all_counts.contiguous(), name="all_counts"), G, rank, L, B,
                                    out.data_ptr(), _stream_ptr(stream)), "lsh_global_offsets")
    return out


def query_global_runs(all_ranges, rank: int, stream=None):
    """lsh_query_global_runs: all_ranges int64 [G, 2, nq, L] (CUDA; every rank's local
    begin/end) -> (gbegin, gtotal) int64 [nq, L]: where this rank's run sits inside the
    global (rank-order concatenated) bucket, and that bucket's size."""
    torch = _torch()
    if all_ranges.dtype != torch.int64 or all_ranges.dim() != 4 or all_ranges.shape[1] != 2:
        raise ValueError("all_ranges must be int64 [G, 2, nq, L]")
    G, _, nq, L = all_ranges.shape
    gbegin = torch.empty((nq, L), dtype=torch.int64, device=all_ranges.device)
    gtotal = torch.empty((nq, L), dtype=torch.int64, device=all_ranges.device)
    M = nq * L
    _check(lib().lsh_query_global_runs(_dev_ptr(all_ranges.contiguous(), name="all_ranges") if M else None, G, rank,
                                       M, gbegin.data_ptr() if M else None, gtotal.data_ptr() if M else None,
                                       _stream_ptr(stream)), "lsh_query_global_runs")
    return gbegin, gtotal


def _torch():
    import torch
    return torch


def _stream_ptr(stream) -> Optional[int]:
    torch = _torch()
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def _dev_ptr(t, dtype=None, name="tensor") -> int:
    if t is None:
        return None
    if not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    if dtype is not None and t.dtype != dtype:
        raise ValueError(f"{name} must be {dtype}")
    return t.data_ptr()


class _DevArray:
    """__cuda_array_interface__ over library-owned device memory (zero-copy view)."""

    def __init__(self, ptr: int, shape, typestr: str, owner):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr, "data": (int(ptr), False),
                                         "version": 3, "strides": None}
        self._owner = owner


class Index:
    """A built (m, L) index (lsh_index)."""

    def __init__(self, handle: "LSH", ptr: int, n: int):
        self._h = handle
        self._ptr = ctypes.c_void_p(ptr)
        self.n = n

    def view(self, t: int, copy: bool = True):
        """(ids uint32 [n], ukeys uint64 [nb], offs uint32 [nb+1]) of table t as torch tensors."""
        torch = _torch()
        ids, uk, of = ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_void_p()
        nb = ctypes.c_int64(0)
        _check(lib().lsh_index_view(self._ptr, t, ctypes.byref(ids), ctypes.byref(uk), ctypes.byref(of),
                                    ctypes.byref(nb)), "lsh_index_view")
        dev = torch.device("cuda", self._h.device)
        nbv = nb.value

        def wrap(p, count, ts, dt):
            if count == 0 or not p.value:
                return torch.zeros(count, dtype=dt, device=dev)
            x = torch.as_tensor(_DevArray(p.value, (count,), ts, self), device=dev).view(dt)
            return x.clone() if copy else x
        return (wrap(ids, self.n, "<i4", torch.uint32), wrap(uk, nbv, "<i8", torch.uint64),
                wrap(of, nbv + 1, "<i4", torch.uint32))

    def counts(self, B: int, stream=None):
        torch = _torch()
        out = torch.empty((self._h.L, 1 << B), dtype=torch.int32, device=torch.device("cuda", self._h.device))
        _check(lib().lsh_index_counts(self._ptr, B, out.data_ptr(), _stream_ptr(stream)), "lsh_index_counts")
        return out

    def close(self):
        if self._ptr is not None and self._ptr.value:
            lib().lsh_index_destroy(self._ptr)
        self._ptr = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class LSH:
    """One hasher (lsh_handle): parameters drawn from `seed`, resident on `device`."""

    def __init__(self, scheme: str, d: int, m: int, L: int, K: int, w: float = 4.0, seed: int = 0,
                 mode_d: Optional[Sequence[int]] = None, mode_m: Optional[Sequence[int]] = None, device: int = 0,
                 per_table: bool = False):
        self.scheme, self.d, self.m, self.L, self.K, self.w, self.seed = scheme, d, m, L, K, w, seed
        self.mode_d, self.mode_m, self.device, self.per_table = mode_d, mode_m, device, per_table
        self.params = make_params(scheme, d, m, L, K, w, seed, mode_d, mode_m, device, per_table)
        h = ctypes.c_void_p()
        _check(lib().lsh_create(ctypes.byref(self.params), ctypes.byref(h)), "lsh_create")
        self._h = h

    @property
    def e2lsh(self) -> bool:
        return "E2LSH" in self.scheme

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            lib().lsh_destroy(self._h)
        self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- hashing ------------------------------------------------------------
    def hash(self, X, keys: bool = True, codes: bool = False, bits: bool = False, proj: bool = False,
             stream=None, out=None):
        """Hash the rows of X (CUDA fp32 [n, ld>=d]); returns a dict of requested outputs."""
        torch = _torch()
        n, ld = self._shape(X)
        dev = X.device
        res = dict(out or {})
        if keys and "keys" not in res:
            res["keys"] = torch.empty((self.L, n), dtype=torch.uint64, device=dev)
        if codes and self.e2lsh and "codes" not in res:
            res["codes"] = torch.empty((n, self.m), dtype=torch.int32, device=dev)
        if bits and not self.e2lsh and "bits" not in res:
            res["bits"] = torch.empty((n, (self.m + 31) // 32), dtype=torch.int32, device=dev)
        if proj and "proj" not in res:
            res["proj"] = torch.empty((n, self.m), dtype=torch.float32, device=dev)
        _check(lib().lsh_hash(self._h, X.data_ptr() if n else None, n, ld,
                              _dev_ptr(res.get("keys"), name="keys"), _dev_ptr(res.get("codes"), name="codes"),
                              _dev_ptr(res.get("bits"), name="bits"), _dev_ptr(res.get("proj"), name="proj"),
                              _stream_ptr(stream)), "lsh_hash")
        return res

    def _shape(self, X):
        torch = _torch()
        if X.dtype != torch.float32 or not X.is_cuda or X.dim() != 2:
            raise ValueError("X must be a 2-D CUDA float32 tensor")
        if X.stride(1) != 1:
            raise ValueError("X rows must be contiguous")
        n = X.shape[0]
        ld = X.stride(0) if n > 1 else max(X.shape[1], self.d)
        if X.shape[1] < self.d:
            raise ValueError("X has fewer than d columns")
        return n, ld

    # -- index --------------------------------------------------------------
    def build_index(self, X, id_base: int = 0, stream=None) -> Index:
        n, ld = self._shape(X)
        ptr = ctypes.c_void_p()
        _check(lib().lsh_build_index(self._h, X.data_ptr() if n else None, n, ld, id_base, ctypes.byref(ptr),
                                     _stream_ptr(stream)), "lsh_build_index")
        return Index(self, ptr.value, n)

    def group_keys(self, keys, id_base: int = 0, stream=None) -> Index:
        torch = _torch()
        if keys.dtype != torch.uint64 or keys.dim() != 2 or keys.shape[0] != self.L:
            raise ValueError("keys must be uint64 [L, n]")
        n = keys.shape[1]
        ptr = ctypes.c_void_p()
        _check(lib().lsh_group_keys(self._h, _dev_ptr(keys.contiguous(), name="keys"), n, id_base,
                                    ctypes.byref(ptr), _stream_ptr(stream)), "lsh_group_keys")
        return Index(self, ptr.value, n)

    def query_buckets(self, index: Index, Q, stream=None):
        torch = _torch()
        nq, ld = self._shape(Q)
        begin = torch.empty((nq, self.L), dtype=torch.int64, device=Q.device)
        end = torch.empty((nq, self.L), dtype=torch.int64, device=Q.device)
        _check(lib().lsh_query_buckets(self._h, index._ptr, Q.data_ptr() if nq else None, nq, ld,
                                       begin.data_ptr() if nq else None, end.data_ptr() if nq else None,
                                       _stream_ptr(stream)), "lsh_query_buckets")
        return begin, end

    def query_knn(self, index: Index, X, Q, k: int, max_cand: int = 4096, stream=None):
        """Top-k of each query among the union of its L buckets (lsh_query_knn): ids int64
        [nq, k] (-1 when missing), scores float32 [nq, k] (squared L2 for the E2LSH family,
        cosine similarity for SRP), distinct candidates int32 [nq].  X = the indexed rows."""
        torch = _torch()
        nq, ldq = self._shape(Q)
        _, ldx = self._shape(X)
        ids = torch.empty((nq, k), dtype=torch.int64, device=Q.device)
        sc = torch.empty((nq, k), dtype=torch.float32, device=Q.device)
        nc = torch.empty((nq,), dtype=torch.int32, device=Q.device)
        _check(lib().lsh_query_knn(self._h, index._ptr, X.data_ptr(), ldx, Q.data_ptr() if nq else None, nq, ldq,
                                   k, max_cand, ids.data_ptr() if nq else None, sc.data_ptr() if nq else None,
                                   nc.data_ptr() if nq else None, _stream_ptr(stream)), "lsh_query_knn")
        return ids, sc, nc

    # -- parameters / status ------------------------------------------------
    def get_params(self, what: str, mode: int = 0):
        import numpy as np
        sz = ctypes.c_size_t(0)
        lib().lsh_get_params(self._h, EXPORT[what], mode, None, ctypes.byref(sz))
        dtype = {"bucket": np.int32, "sign": np.int32, "offsets": np.float32, "gaussian": np.uint16,
                 "coeffs": np.uint64, "coord": np.int32}[what]
        buf = np.zeros(sz.value // np.dtype(dtype).itemsize, dtype=dtype)
        _check(lib().lsh_get_params(self._h, EXPORT[what], mode, buf.ctypes.data_as(ctypes.c_void_p),
                                    ctypes.byref(sz)), "lsh_get_params")
        return buf

    def group_path(self):
        """Grouping path of the wide-key builds (lsh_group_path): 0 = fixed-capacity L1
        scatter, > 0 = histogram path after a bin overflow."""
        v = ctypes.c_int32(0)
        _check(lib().lsh_group_path(self._h, ctypes.byref(v)), "lsh_group_path")
        return int(v.value)

    def check(self):
        """Synchronise and raise LshError(LSH_EOVERFLOW) if a code left int32."""
        _check(lib().lsh_check(self._h), "lsh_check")
