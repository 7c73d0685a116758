"""Multi-process (gloo, world_size 2, CPU) checks of the sharded index build's host
logic: shard ranges, the all-gather of per-table coarse counts and the global
offsets, with the per-shard tables computed by the oracle.  The GPU side of the
same path (lsh_index_counts, lsh_global_offsets, NCCL) is covered by
tests/test_gpu_parity.py::test_global_offsets_kernel and bench.py at N > 1."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import lsh
from paper_2503_06737_b200.dist import shard_range


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, scheme, n, B, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        p = lsh.Params(scheme, d=64, m=32, L=4, K=8, w=2.0, seed=3)
        t = lsh.make_tables(p)
        X = np.random.default_rng(0).standard_normal((n, 64)).astype(np.float32)
        X[100:150] = X[7]                              # a populated bucket across shards
        lo, hi = shard_range(n, rank, world)
        keys = lsh.hash_points(p, t, X[lo:hi])["keys"]
        local = lsh.group(keys, id_base=lo)
        cnt = torch.from_numpy(lsh.coarse_counts(p, keys, B).astype(np.int64))
        gathered = [torch.zeros_like(cnt) for _ in range(world)]
        dist.all_gather(gathered, cnt)
        allc = torch.stack(gathered).numpy()
        off = lsh.global_coarse_offsets(allc, rank)
        width = lsh.key_width(p)
        # place this rank's ids at their global positions, per table
        placed = []
        for tt in range(p.L):
            items = []
            for b in range(local[tt].ukeys.size):
                cb = lsh.coarse_bin(int(local[tt].ukeys[b]), width, B)
                items.append((cb, local[tt].ids[local[tt].offs[b]:local[tt].offs[b + 1]].tolist()))
            pos = {}
            cur = {}
            for cb, ids in items:
                start = off[tt, cb] + cur.get(cb, 0)
                for k, i in enumerate(ids):
                    pos[start + k] = i
                cur[cb] = cur.get(cb, 0) + len(ids)
            placed.append(pos)
        q.put((rank, placed, allc.tolist()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("scheme,B", [("CS_E2LSH", 6), ("CS_SRP", 8), ("CS_SRP", 4)])
def test_sharded_build_gloo_world2(scheme, B):
    n, world = 777, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, scheme, n, B, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    res.sort()
    # G = 1 reference
    p = lsh.Params(scheme, d=64, m=32, L=4, K=8, w=2.0, seed=3)
    t = lsh.make_tables(p)
    X = np.random.default_rng(0).standard_normal((n, 64)).astype(np.float32)
    X[100:150] = X[7]
    keys = lsh.hash_points(p, t, X)["keys"]
    glob = lsh.group(keys)
    width = lsh.key_width(p)
    allc = np.array(res[0][2])
    assert np.array_equal(allc, np.array(res[1][2]))
    assert np.array_equal(allc.sum(axis=0), lsh.coarse_counts(p, keys, B))
    for tt in range(p.L):
        merged = {}
        for r in range(world):
            for k, v in res[r][1][tt].items():
                assert k not in merged          # runs never overlap
                merged[k] = v
        assert sorted(merged) == list(range(n))  # and tile [0, n)
        order = [merged[i] for i in range(n)]
        # every coarse bin holds exactly the G=1 bin's ids; every bucket's ids keep
        # the G=1 order when the ranks' runs are concatenated in rank order
        for b in range(glob[tt].ukeys.size):
            ids = glob[tt].ids[glob[tt].offs[b]:glob[tt].offs[b + 1]].tolist()
            cb = lsh.coarse_bin(int(glob[tt].ukeys[b]), width, B)
            lo = int(lsh.global_coarse_offsets(allc, 0)[tt, cb])
            hi = lo + int(allc[:, tt, cb].sum())
            run = [i for i in order[lo:hi] if i in set(ids)]
            assert run == ids


def test_shard_range_partition():
    for n in (0, 1, 5, 777, 1_000_000):
        for world in (1, 2, 3, 4, 8):
            r = [shard_range(n, k, world) for k in range(world)]
            assert r[0][0] == 0 and r[-1][1] == n
            for a, b in zip(r, r[1:]):
                assert a[1] == b[0]


def test_global_offsets_oracle_properties():
    g = np.random.default_rng(4)
    allc = g.integers(0, 50, (3, 5, 16))
    offs = [lsh.global_coarse_offsets(allc, r) for r in range(3)]
    for t in range(5):
        spans = sorted((int(offs[r][t, b]), int(allc[r, t, b])) for r in range(3) for b in range(16))
        pos = 0
        for start, ln in spans:
            assert start == pos
            pos += ln
        assert pos == allc[:, t].sum()


def _gather_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2503_06737_b200.dist import all_gather_device
        x = torch.arange(12, dtype=torch.int64).reshape(2, 6) + 100 * rank
        out = all_gather_device(x)
        q.put((rank, out.numpy()))
    finally:
        dist.destroy_process_group()


def test_all_gather_device_gloo_world2():
    """The product's backend-agnostic gather (dist.all_gather_device) under gloo: [G, *shape]
    in rank order on every rank (the host path the GPU world-2 test uses)."""
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gather_worker, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    want = np.stack([np.arange(12).reshape(2, 6) + 100 * r for r in range(world)])
    for r in range(world):
        assert np.array_equal(res[r], want)
