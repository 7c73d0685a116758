"""Key-distribution diagnostics for grouping design: per table varying bits, L1 bin sizes,
bucket-size distribution.  python tools/key_stats.py --config C4 --scheme CS_SRP"""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2503_06737_b200 as pk
import synth

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C4"); ap.add_argument("--scheme", default="CS_SRP")
ap.add_argument("--tables", type=int, default=4)
a = ap.parse_args()
c = synth.CONFIGS[a.config]
kw = dict(mode_d=c.mode_d, mode_m=c.mode_m) if a.scheme.startswith("HCS") else {}
h = pk.LSH(a.scheme, c.d, c.m, c.L, c.K, c.w, c.hash_seed, **kw)
X = synth.rows(c, 0, c.n, device="cuda")
keys = h.hash(X, keys=True)["keys"].view(torch.int64).cpu().numpy().view(np.uint64)
n = c.n
B1 = 1
while B1 < 11 and -(-n // (1 << B1)) > 2048:
    B1 += 1
print(f"{a.config} {a.scheme} n={n} L={c.L} B1={B1}")
for t in range(min(a.tables, c.L)):
    k = keys[t]
    o = np.bitwise_or.reduce(k); an = np.bitwise_and.reduce(k)
    V = int(o ^ an)
    pos = [b for b in range(63, -1, -1) if (V >> b) & 1][:B1]
    dig = np.zeros(n, np.int64)
    for p in pos:
        dig = (dig << 1) | ((k >> np.uint64(p)) & np.uint64(1)).astype(np.int64)
    bins = np.bincount(dig, minlength=1 << len(pos))
    u, cnt = np.unique(k, return_counts=True)
    print(f" t={t} varying={bin(V).count('1')} bits; L1 bins max={bins.max()} >4096: {(bins > 4096).sum()} "
          f"items in big bins={bins[bins > 4096].sum()}; distinct keys={len(u)} max bucket={cnt.max()} "
          f"buckets>64: {(cnt > 64).sum()} items in them={cnt[cnt > 64].sum()}")
