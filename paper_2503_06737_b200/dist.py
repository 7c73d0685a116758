"""Multi-GPU index build and query: one process per GPU, points
sharded in contiguous row blocks, per-shard tables built locally, and ONE
collective per build — an all-gather of the per-table coarse bucket counts (NCCL
over NVLink / NVSwitch; through host memory under gloo) — followed by an
on-device exclusive prefix (`lsh_global_offsets`) that gives every rank the global
position of its runs.  Points never move between GPUs.  The path partitions
(independent points), so the only exchange is the counts; the per-bucket
concatenation of the ranks' runs in rank order equals the single-GPU bucket (ids
ascend across ranks).

A query is answered across shards the same way ("collect the index
of all the elements" hashed to hbar_t(q)): every rank looks the queries up in its
own tables, the (begin, end) ranges are all-gathered, and `lsh_query_global_runs`
places each rank's run inside the global bucket.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Optional, Tuple

from . import LSH, Index, global_offsets, query_global_runs


def shard_range(n: int, rank: int, world: int) -> Tuple[int, int]:
    """Rows [lo, hi) owned by `rank`: contiguous blocks of ceil(n / world) rows."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank / world")
    per = (n + world - 1) // world
    lo = min(n, rank * per)
    return lo, min(n, lo + per)


def _world(group) -> Tuple[int, int]:
    import torch.distributed as dist
    if not dist.is_initialized():
        return 1, 0
    return dist.get_world_size(group), dist.get_rank(group)


def all_gather_device(x, group=None):
    """[G, *x.shape] on x's device: NCCL gathers device memory directly; other backends
    (gloo) go through host memory.  Issued on the current stream."""
    import torch
    import torch.distributed as dist
    world, _ = _world(group)
    x = x.contiguous()
    if world == 1:
        return x.unsqueeze(0).clone()
    if dist.get_backend(group) == "nccl":
        out = torch.empty((world,) + tuple(x.shape), dtype=x.dtype, device=x.device)
        dist.all_gather_into_tensor(out, x, group=group)
        return out
    xc = x.cpu()
    parts = [torch.empty_like(xc) for _ in range(world)]
    dist.all_gather(parts, xc, group=group)
    return torch.stack(parts).to(x.device)


@dataclass
class ShardedIndex:
    local: Index            # this rank's tables (global ids = id_base + local row)
    id_base: int
    counts: "object"        # int32 [L, 2^B]   this rank's coarse counts
    all_counts: "object"    # int32 [G, L, 2^B] everyone's (all-gathered)
    offsets: "object"       # int64 [L, 2^B]   global start of this rank's run of (t, bin)
    B: int
    rank: int = 0
    world: int = 1


def build_index_sharded(h: LSH, X_shard, id_base: int, B: int = 12, group=None, stream=None) -> ShardedIndex:
    """Local build + all-gather of coarse counts + global offsets (rank, world from `group`)."""
    import torch

    world, rank = _world(group)
    s = stream if stream is not None else torch.cuda.current_stream(X_shard.device)
    # X_shard may still be in flight on the caller's current stream
    s.wait_stream(torch.cuda.current_stream(X_shard.device))
    # every step below, the collective included, is ordered on `s`
    with torch.cuda.stream(s):
        idx = h.build_index(X_shard, id_base=id_base, stream=s)
        cnt = idx.counts(B, stream=s)
        all_counts = all_gather_device(cnt, group)
        off = global_offsets(all_counts, rank, stream=s)
    return ShardedIndex(idx, id_base, cnt, all_counts, off, B, rank, world)


@dataclass
class ShardedQuery:
    begin: "object"    # int64 [nq, L] local range of this rank's run in its tables
    end: "object"
    gbegin: "object"   # int64 [nq, L] where that run starts inside the global bucket
    gtotal: "object"   # int64 [nq, L] size of the global bucket (all ranks)


def query_sharded(h: LSH, sidx: ShardedIndex, Q, group=None, stream=None) -> ShardedQuery:
    """Every rank looks the (same) queries up in its own tables; the ranges are
    all-gathered and each rank's run is placed inside the global bucket."""
    import torch

    s = stream if stream is not None else torch.cuda.current_stream(Q.device)
    s.wait_stream(torch.cuda.current_stream(Q.device))   # Q may still be in flight there
    with torch.cuda.stream(s):
        begin, end = h.query_buckets(sidx.local, Q, stream=s)
        rng = torch.stack((begin, end))                  # [2, nq, L]
        all_rng = all_gather_device(rng, group)          # [G, 2, nq, L]
        gbegin, gtotal = query_global_runs(all_rng, sidx.rank, stream=s)
    return ShardedQuery(begin, end, gbegin, gtotal)
