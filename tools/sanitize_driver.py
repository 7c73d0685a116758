"""Small workloads for compute-sanitizer (tools/gpu_sanitize.sh): every kernel family
of the library at C1/C2-sized inputs, including the rare paths (big bins on global
memory, narrow-key LSD passes, the chunked sketch, the HCS slab kernel, the dense
tcgen05 GEMM with its fused key epilogue, query lookup and query completion).

    python tools/sanitize_driver.py [--quick]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2503_06737_b200 as pk  # noqa: E402
import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--quick", action="store_true", help="C1 shapes only (racecheck is slow)")
a = ap.parse_args()


def run(name, scheme, c, n, **kw):
    X = synth.rows(c, 0, n, device="cuda")
    h = pk.LSH(scheme, c.d, c.m, c.L, c.K, c.w, c.hash_seed, **kw)
    h.hash(X, keys=True)                                  # keys-only fast path
    h.hash(X, keys=True, proj=True, codes=h.e2lsh, bits=not h.e2lsh)   # debug path
    idx = h.build_index(X)
    h.query_buckets(idx, X[:64])
    h.query_knn(idx, X, X[:16], k=8, max_cand=512)
    idx.counts(8)
    torch.cuda.synchronize()
    h.check()
    idx.close()
    h.close()
    print(f"ok {name} {scheme} n={n}", flush=True)


c1, c2, c3 = synth.CONFIGS["C1"], synth.CONFIGS["C2"], synth.CONFIGS["C3"]
for s in ("CS_E2LSH", "CS_SRP", "E2LSH", "SRP"):
    run("C1", s, c1, c1.n)
run("C1-HCS", "HCS_E2LSH", c1, c1.n, mode_d=(4, 4, 4), mode_m=(2, 2, 4))
run("C1-HCS", "HCS_SRP", c1, c1.n, mode_d=(4, 4, 4), mode_m=(2, 2, 4))

# grouping corner cases through lsh_group_keys: one dominant key (big bin on global
# memory), a long equal prefix, narrow SRP keys (LSD passes)
h = pk.LSH("CS_E2LSH", c1.d, c1.m, c1.L, c1.K, c1.w, 0)
g = torch.Generator(device="cpu").manual_seed(1)
n = 6000
k = torch.randint(0, 2**62, (c1.L, n), generator=g, dtype=torch.int64)
k[:, : n // 2] = 12345                                     # > the shared-memory bin cap
k[:, n // 2: n // 2 + 800] = (k[:, n // 2: n // 2 + 800] & 0xffff) | (7 << 40)
idx = h.group_keys(k.cuda().view(torch.uint64))
torch.cuda.synchronize()
idx.close()
hs = pk.LSH("CS_SRP", c1.d, c1.m, c1.L, c1.K, c1.w, 0)
ks = torch.randint(0, 256, (c1.L, n), generator=g, dtype=torch.int64)
idx = hs.group_keys(ks.cuda().view(torch.uint64))
torch.cuda.synchronize()
idx.close()
print("ok group corner cases", flush=True)

if not a.quick:
    for s in ("CS_E2LSH", "CS_SRP", "E2LSH"):
        run("C2", s, c2, 8192)
    run("C3", "HCS_E2LSH", c3, 2048, mode_d=c3.mode_d, mode_m=c3.mode_m)
    # chunked sketch (d > 1024)
    X = synth.gaussian_rows_like(300, 3000, 5, device="cuda")
    h = pk.LSH("CS_E2LSH", 3000, 512, 32, 16, 2.0, 1)
    idx = h.build_index(X)
    torch.cuda.synchronize()
    idx.close()
    # per-table families on the tcgen05 GEMM
    h = pk.LSH("CS_E2LSH", c2.d, c2.m, c2.L, c2.K, c2.w, 0, per_table=True)
    idx = h.build_index(synth.rows(c2, 0, 4096, device="cuda"))
    torch.cuda.synchronize()
    idx.close()
    print("ok chunked + per-table", flush=True)
print("sanitize driver done")
