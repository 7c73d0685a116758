"""Multi-GPU index build: one process per GPU, points sharded in
contiguous row blocks, per-shard tables built locally, and ONE collective per
build — an all-gather of the per-table coarse bucket counts over NCCL
(NVLink / NVSwitch) — followed by an on-device exclusive prefix
(`lsh_global_offsets`) that gives every rank the global position of its runs.
Points never move between GPUs.  The path partitions (independent points), so
the only exchange is the counts; the per-bucket concatenation of the ranks' runs
in rank order equals the single-GPU bucket (ids ascend across ranks).
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Optional, Tuple

from . import LSH, Index, global_offsets


def shard_range(n: int, rank: int, world: int) -> Tuple[int, int]:
    """Rows [lo, hi) owned by `rank`: contiguous blocks of ceil(n / world) rows."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank / world")
    per = (n + world - 1) // world
    lo = min(n, rank * per)
    return lo, min(n, lo + per)


@dataclass
class ShardedIndex:
    local: Index            # this rank's tables (global ids = id_base + local row)
    id_base: int
    counts: "object"        # int32 [L, 2^B]   this rank's coarse counts
    all_counts: "object"    # int32 [G, L, 2^B] everyone's (all-gathered)
    offsets: "object"       # int64 [L, 2^B]   global start of this rank's run of (t, bin)
    B: int


def build_index_sharded(h: LSH, X_shard, id_base: int, B: int = 12, group=None, stream=None) -> ShardedIndex:
    """Local build + all-gather of coarse counts + global offsets (rank, world from `group`)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    s = stream if stream is not None else torch.cuda.current_stream(X_shard.device)
    # every step below, the collective included, is ordered on `s`
    with torch.cuda.stream(s):
        idx = h.build_index(X_shard, id_base=id_base, stream=s)
        cnt = idx.counts(B, stream=s)
        all_counts = torch.empty((world,) + tuple(cnt.shape), dtype=cnt.dtype, device=cnt.device)
        if world > 1:
            dist.all_gather_into_tensor(all_counts, cnt.unsqueeze(0).contiguous(), group=group)
        else:
            all_counts.copy_(cnt.unsqueeze(0))
        off = global_offsets(all_counts, rank, stream=s)
    return ShardedIndex(idx, id_base, cnt, all_counts, off, B)
