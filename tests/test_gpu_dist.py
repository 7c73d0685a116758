"""The product's multi-GPU path (paper_2503_06737_b200.dist) at world size 2.

Two processes (gloo; the counts and query ranges are exchanged through host
memory) each build their shard's tables with `build_index_sharded` and answer the
same queries with `query_sharded`.  This pod has one GPU, so both ranks run on
cuda:0; their kernels never wait on one another (the only exchange is the host-side
all-gather), so this is the sharded program itself, not an emulation of peers.

Pins (SURVEY §8(c) multi-GPU; "store every point p in bucket
hbar_t(p)", "collect the index of all the elements"):
  * for every (table, key), the rank-order concatenation of the shards' buckets
    equals the single-GPU (G = 1) bucket, and no shard holds a key G = 1 lacks;
  * the all-gathered coarse counts sum to the G = 1 counts and the global offsets
    tile [0, n) per table with every coarse bin's ids in place;
  * a cross-shard query: each rank's local run sits at gbegin inside the G = 1
    bucket of the query, and gtotal equals that bucket's size.
The G = 1 index is itself bit-exact against the oracle (tests/test_gpu_fastpath.py).
"""
import os
import socket

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

N_Q = 300


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _handle(scheme, c):
    import paper_2503_06737_b200 as pk
    kw = dict(mode_d=c.mode_d, mode_m=c.mode_m) if scheme.startswith("HCS") else {}
    return pk.LSH(scheme, c.d, c.m, c.L, c.K, c.w, c.hash_seed, **kw)


def _tables(idx, L):
    out = []
    for t in range(L):
        ids, uk, of = (x.cpu().numpy() for x in idx.view(t))
        out.append((ids.astype(np.uint32), uk.astype(np.uint64), of.astype(np.uint32)))
    return out


def _worker(rank, world, port, scheme, cfg, n, B, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch.distributed as dist
    import synth
    from paper_2503_06737_b200 import dist as pdist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        c = synth.CONFIGS[cfg]
        h = _handle(scheme, c)
        lo, hi = pdist.shard_range(n, rank, world)
        X = synth.rows(c, lo, hi, device="cuda")
        s = torch.cuda.Stream()                  # not the current stream: ordering is on `s`
        sh = pdist.build_index_sharded(h, X, id_base=lo, B=B, stream=s)
        Q = synth.rows(c, 0, N_Q, device="cuda")
        qr = pdist.query_sharded(h, sh, Q, stream=s)
        s.synchronize()
        h.check()
        q.put((rank, dict(
            tables=_tables(sh.local, c.L), counts=sh.counts.cpu().numpy(), all_counts=sh.all_counts.cpu().numpy(),
            offsets=sh.offsets.cpu().numpy(), begin=qr.begin.cpu().numpy(), end=qr.end.cpu().numpy(),
            gbegin=qr.gbegin.cpu().numpy(), gtotal=qr.gtotal.cpu().numpy())))
        sh.local.close()
    except BaseException as e:  # report instead of hanging the parent
        q.put((rank, repr(e)))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("scheme,cfg,n,B", [("CS_E2LSH", "C2", 60000, 8), ("CS_SRP", "C2", 60000, 10),
                                            ("HCS_E2LSH", "C3", 20001, 12)])
def test_sharded_index_world2_equals_single_gpu(scheme, cfg, n, B):
    import torch.multiprocessing as mp
    import synth
    from oracle import lsh
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, scheme, cfg, n, B, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = dict(q.get(timeout=600) for _ in range(world))
    for pr in procs:
        pr.join(timeout=120)
    for r in range(world):
        assert isinstance(res[r], dict), res[r]
        assert procs[r].exitcode == 0

    # G = 1 run of the same program
    c = synth.CONFIGS[cfg]
    h = _handle(scheme, c)
    X = synth.rows(c, 0, n, device="cuda")
    idx = h.build_index(X)
    glob = _tables(idx, c.L)
    gcnt = idx.counts(B).cpu().numpy()
    b1, e1 = (x.cpu().numpy() for x in h.query_buckets(idx, synth.rows(c, 0, N_Q, device="cuda")))
    torch.cuda.synchronize()
    idx.close()

    # (1) per (table, key): rank-order concatenation of the shards' buckets == G = 1 bucket
    for t in range(c.L):
        gi, gu, go = glob[t]
        shard_runs = []
        for r in range(world):
            ids, uk, of = res[r]["tables"][t]
            assert np.all(np.isin(uk, gu)), (r, t)
            shard_runs.append({int(k): ids[of[b]:of[b + 1]] for b, k in enumerate(uk)})
        for b, k in enumerate(gu):
            cat = np.concatenate([sr.get(int(k), np.zeros(0, np.uint32)) for sr in shard_runs])
            assert np.array_equal(cat, gi[go[b]:go[b + 1]]), (t, b)

    # (2) coarse counts and global offsets
    allc = res[0]["all_counts"]
    for r in range(world):
        assert np.array_equal(res[r]["all_counts"], allc)
        assert np.array_equal(allc[r], res[r]["counts"])
    assert np.array_equal(allc.sum(axis=0), gcnt)
    p = lsh.Params(scheme, d=c.d, m=c.m, L=c.L, K=c.K, w=c.w, seed=c.hash_seed,
                   **(dict(mode_d=c.mode_d, mode_m=c.mode_m) if scheme.startswith("HCS") else {}))
    width = lsh.key_width(p)
    for t in range(c.L):
        gi, gu, go = glob[t]
        want = {}
        for b, k in enumerate(gu):
            want.setdefault(lsh.coarse_bin(int(k), width, B), []).extend(gi[go[b]:go[b + 1]].tolist())
        placed = np.full(n, -1, np.int64)
        for r in range(world):
            ids, uk, of = res[r]["tables"][t]
            cur = {}
            for b, k in enumerate(uk):
                cb = lsh.coarse_bin(int(k), width, B)
                start = int(res[r]["offsets"][t, cb]) + cur.get(cb, 0)
                run = ids[of[b]:of[b + 1]]
                assert np.all(placed[start:start + run.size] == -1)
                placed[start:start + run.size] = run
                cur[cb] = cur.get(cb, 0) + run.size
        assert np.all(placed >= 0)
        pos = 0
        for cb in sorted(want):
            assert sorted(placed[pos:pos + len(want[cb])].tolist()) == sorted(want[cb])
            pos += len(want[cb])

    # (3) cross-shard query runs
    assert np.array_equal(res[0]["gtotal"], e1 - b1)
    for r in range(world):
        rr = res[r]
        assert np.array_equal(rr["gtotal"], e1 - b1)
        for qi in range(N_Q):
            for t in range(c.L):
                ids = rr["tables"][t][0]
                local = ids[rr["begin"][qi, t]:rr["end"][qi, t]]
                g0 = b1[qi, t] + rr["gbegin"][qi, t]
                assert np.array_equal(glob[t][0][g0:g0 + local.size], local), (r, qi, t)
    # the queries are indexed points: every (query, table) bucket is non-empty
    assert np.all(e1 > b1)
