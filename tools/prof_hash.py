"""Small driver for ncu captures: one warm-up call then `--reps` calls of the op.

    python tools/prof_hash.py --config C4 --scheme CS_E2LSH --op hash|build
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2503_06737_b200 as pk  # noqa: E402
import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C4")
ap.add_argument("--scheme", default="CS_E2LSH")
ap.add_argument("--op", default="hash")
ap.add_argument("--reps", type=int, default=1)
ap.add_argument("--n", type=int, default=0)
ap.add_argument("--per-table", action="store_true")
a = ap.parse_args()
c = synth.CONFIGS[a.config]
n = a.n or c.n
kw = dict(mode_d=c.mode_d, mode_m=c.mode_m) if a.scheme.startswith("HCS") else {}
h = pk.LSH(a.scheme, c.d, c.m, c.L, c.K, c.w, c.hash_seed, per_table=a.per_table, **kw)
X = synth.rows(c, 0, n, device="cuda")
keys = torch.empty((c.L, n), dtype=torch.uint64, device="cuda")
pk.timing_enable(True)
for i in range(1 + a.reps):
    if i == 1:
        torch.cuda.synchronize()
        pk.timing_reset()
        torch.cuda.nvtx.range_push("profile")   # ncu --nvtx --nvtx-include "profile/"
    if a.op == "hash":
        h.hash(X, keys=True, out={"keys": keys})
    else:
        idx = h.build_index(X)
torch.cuda.synchronize()
torch.cuda.nvtx.range_pop()
for k in ("sketch", "group_hist", "group_scan", "group_scatter", "group_sort", "dense_gemm",
          "keys_from_proj"):
    ms, cnt = pk.timing_get(k)
    if cnt:
        print(f"{k:18s} {ms / a.reps:8.3f} ms/rep  launches={cnt}")
