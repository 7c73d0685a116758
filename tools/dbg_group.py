import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2503_06737_b200 as pk, synth
from oracle import lsh
c = synth.CONFIGS["C4"]
h = pk.LSH("CS_E2LSH", c.d, c.m, c.L, c.K, c.w, c.hash_seed)
X = synth.rows(c, 0, 100000, device="cuda")
idx = h.build_index(X); torch.cuda.synchronize()
# n=1 case
L, K = 4, 8
h2 = pk.LSH("CS_E2LSH", 64, L*K, L, K, 4.0, 0)
g = np.random.default_rng(1)
keys = g.integers(0, 2 ** 63, (L, 1), dtype=np.int64).astype(np.uint64) * np.uint64(2)
idx2 = h2.group_keys(torch.from_numpy(keys.view(np.int64)).cuda().view(torch.uint64), id_base=17)
for t in range(L):
    ids, uk, of = (x.cpu().numpy() for x in idx2.view(t))
    print(t, keys[t], uk.astype(np.uint64), of, ids)
