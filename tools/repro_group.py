"""Small grouping repro (diagnostics): python tools/repro_group.py [n] [L]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2503_06737_b200 as pk
from oracle import lsh
n = int(sys.argv[1]) if len(sys.argv) > 1 else 60000
L = int(sys.argv[2]) if len(sys.argv) > 2 else 4
g = np.random.default_rng(1)
keys = g.integers(0, 2 ** 63, (L, n), dtype=np.int64).astype(np.uint64) * np.uint64(2) + g.integers(0, 2, (L, n)).astype(np.uint64)
keys[:, : n // 3] = keys[:, :1]
h = pk.LSH("CS_E2LSH", 64, L * 16, L, 16, 4.0, 0)
idx = h.group_keys(torch.from_numpy(keys.view(np.int64)).cuda().view(torch.uint64), id_base=17)
ref = lsh.group(keys, id_base=17)
for t in range(L):
    ids, uk, of = (x.cpu().numpy() for x in idx.view(t))
    r = ref[t]
    print(t, "nb", len(uk), len(r.ukeys), "ids_eq", np.array_equal(ids.astype(np.uint32), r.ids),
          "uk_eq", len(uk) == len(r.ukeys) and np.array_equal(uk.astype(np.uint64), r.ukeys))
