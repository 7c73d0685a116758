"""Seeded synthetic inputs shaped like the paper's workloads (BASELINE.json configs).

This module holds NO arithmetic of the method: it only draws input points.  It is
the one piece both sides share (DESIGN.md §Oracle rules): the CUDA path hashes
the rows it produces and the oracle receives the identical fp32 rows.

The paper's datasets (Synthetic 50,000 x 10,000, Arcene, RNA-Seq, PEMS-SF, Gist;
P:1953-1963) are not available; the configs below stand in for them
(DESIGN.md §Inputs).  Rows are drawn in fixed 4096-row chunks, chunk c from a
generator seeded data_seed * 1_000_003 + c, so any row range - in particular a
rank's shard - is reproducible independently of how the rows are split.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Dict, Optional, Tuple

import torch

CHUNK = 4096


@dataclass(frozen=True)
class Config:
    name: str
    n: int
    d: int
    m: int
    L: int
    K: int
    w: float
    values: str                     # distribution recipe (see _draw_chunk)
    schemes: Tuple[str, ...]
    mode_d: Tuple[int, ...] = ()
    mode_m: Tuple[int, ...] = ()
    data_seed: int = 1000
    hash_seed: int = 0
    paper: str = ""


CONFIGS: Dict[str, Config] = {
    "C1": Config("C1", 1000, 64, 16, 2, 8, 4.0, "uniform01", ("CS_E2LSH", "CS_SRP"),
                 data_seed=1000, paper="toy / unit (BASELINE configs[0])"),
    "C2": Config("C2", 60000, 784, 160, 10, 16, 4.0, "sparse_u8", ("CS_E2LSH", "CS_SRP", "E2LSH", "SRP"),
                 data_seed=1001, paper="sparse 8-bit image shape (BASELINE configs[1])"),
    "C3": Config("C3", 50000, 4096, 512, 32, 16, 2.0, "gauss_unit", ("HCS_E2LSH", "HCS_SRP", "CS_E2LSH", "CS_SRP"),
                 mode_d=(16, 16, 16), mode_m=(8, 8, 8), data_seed=1002,
                 paper="paper's 'Synthetic' 50,000 points (P:1955) (BASELINE configs[2])"),
    "C4": Config("C4", 1_000_000, 960, 1024, 64, 16, 1.0, "clusters", ("CS_E2LSH", "CS_SRP"),
                 data_seed=1003, paper="Gist shape d=960 (P:1962) (BASELINE configs[3])"),
    "C5": Config("C5", 100_000, 65536, 4096, 256, 16, 4.0, "sparse_gauss", ("HCS_E2LSH", "HCS_SRP", "E2LSH"),
                 mode_d=(16, 16, 16, 16), mode_m=(8, 8, 8, 8), data_seed=1004,
                 paper="high-d sparse, PEMS-SF-like (P:1960) (BASELINE configs[4])"),
}


def _gen(device, seed: int) -> torch.Generator:
    g = torch.Generator(device=device)
    g.manual_seed(int(seed) & ((1 << 63) - 1))
    return g


def _centres(cfg: Config, device) -> torch.Tensor:
    g = _gen(device, cfg.data_seed)
    return torch.randn(1000, cfg.d, generator=g, device=device, dtype=torch.float32)


def _draw_chunk(cfg: Config, c: int, rows: int, device, centres: Optional[torch.Tensor]) -> torch.Tensor:
    g = _gen(device, cfg.data_seed * 1_000_003 + c)
    shape = (rows, cfg.d)
    if cfg.values == "uniform01":          # fp32 i.i.d. U[0,1)
        return torch.rand(shape, generator=g, device=device)
    if cfg.values == "sparse_u8":          # ~80% exact zeros, nonzeros k/255, k ~ U{1..255}
        mask = torch.rand(shape, generator=g, device=device) < 0.2
        k = torch.randint(1, 256, shape, generator=g, device=device).to(torch.float32)
        return torch.where(mask, k / 255.0, torch.zeros((), device=device))
    if cfg.values == "gauss_unit":         # N(0,1) rows, L2-normalised
        x = torch.randn(shape, generator=g, device=device)
        return x / x.norm(dim=1, keepdim=True)
    if cfg.values == "clusters":           # centre[U{0..999}] + 0.1 N(0, I)
        idx = torch.randint(0, 1000, (rows,), generator=g, device=device)
        return centres[idx] + 0.1 * torch.randn(shape, generator=g, device=device)
    if cfg.values == "sparse_gauss":       # Bernoulli(0.01) x N(0,1), dense fp32 storage
        mask = torch.rand(shape, generator=g, device=device) < 0.01
        x = torch.randn(shape, generator=g, device=device)
        return torch.where(mask, x, torch.zeros((), device=device))
    raise ValueError(cfg.values)


def rows(cfg: Config | str, r0: int, r1: int, device="cpu", out: Optional[torch.Tensor] = None) -> torch.Tensor:
    """Rows [r0, r1) of config `cfg` as a contiguous fp32 [r1-r0, d] tensor."""
    if isinstance(cfg, str):
        cfg = CONFIGS[cfg]
    r1 = min(r1, cfg.n)
    n = max(0, r1 - r0)
    if out is None:
        out = torch.empty((n, cfg.d), dtype=torch.float32, device=device)
    centres = _centres(cfg, device) if cfg.values == "clusters" else None
    c0, c1 = r0 // CHUNK, (r1 - 1) // CHUNK if n else r0 // CHUNK - 1
    for c in range(c0, c1 + 1):
        lo, hi = c * CHUNK, min((c + 1) * CHUNK, cfg.n)
        chunk = _draw_chunk(cfg, c, hi - lo, device, centres)
        a, b = max(lo, r0), min(hi, r1)
        out[a - r0:b - r0] = chunk[a - lo:b - lo]
    return out


def sample_rows(cfg: Config | str, idx, device="cpu") -> torch.Tensor:
    """Rows at arbitrary global indices (sampled parity checks at full size)."""
    if isinstance(cfg, str):
        cfg = CONFIGS[cfg]
    idx = [int(i) for i in idx]
    out = torch.empty((len(idx), cfg.d), dtype=torch.float32, device=device)
    centres = _centres(cfg, device) if cfg.values == "clusters" else None
    by_chunk: Dict[int, list] = {}
    for pos, i in enumerate(idx):
        by_chunk.setdefault(i // CHUNK, []).append((pos, i))
    for c, items in by_chunk.items():
        lo, hi = c * CHUNK, min((c + 1) * CHUNK, cfg.n)
        chunk = _draw_chunk(cfg, c, hi - lo, device, centres)
        for pos, i in items:
            out[pos] = chunk[i - lo]
    return out


def gaussian_rows_like(n: int, d: int, seed: int, device="cpu") -> torch.Tensor:
    """Generic N(0,1) fp32 rows for edge-case tests."""
    return torch.randn(n, d, generator=_gen(device, seed), device=device)
