import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2503_06737_b200 as pk, synth
from oracle import lsh
from tests import parity
c = synth.CONFIGS["C5"]
p = lsh.Params("E2LSH", d=c.d, m=c.m, L=c.L, K=c.K, w=c.w, seed=c.hash_seed)
rows = np.arange(24)
Xs = synth.sample_rows(c, rows, device="cuda")
h = pk.LSH("E2LSH", c.d, c.m, c.L, c.K, c.w, 0)
out = h.hash(Xs, keys=True, codes=True, proj=True); torch.cuda.synchronize()
X = Xs.cpu().numpy(); t = lsh.make_tables(p); ref = lsh.hash_points(p, t, X)
y = out["proj"].cpu().numpy().astype(np.float64)
sig = parity.sigma(p, t, X); k = parity.nnz_terms(p, t, X)
unit = 2.0**-24 * np.sqrt(k) * sig
r = np.abs(y - ref["proj"]) / unit
print("err/(u sqrt(k) sigma): median %.3f  p99 %.3f  max %.3f" % (np.median(r), np.percentile(r, 99), r.max()))
# same for a CUDA-core fp32 sequential reference computed in numpy float32 (sequential sum)
X32 = X.astype(np.float32); R32 = t.R.astype(np.float32)
seq = np.zeros_like(y)
for i in range(4):
    acc = np.zeros(p.m, np.float32)
    for j in np.nonzero(X32[i])[0]:
        acc = acc + X32[i, j] * R32[:, j]
    seq[i] = acc
r2 = np.abs(seq[:4] - ref["proj"][:4]) / unit[:4]
print("seq fp32 err/(u sqrt(k) sigma): median %.3f  max %.3f" % (np.median(r2), r2.max()))
codes = out["codes"].cpu().numpy()
mm = codes != ref["codes"]
q = ref["quotient"]
print("mismatches", mm.sum(), "dist to boundary", np.abs(q - np.round(q))[mm][:10], "gpu-ref q err", (np.abs(y - ref["proj"]) / 4)[mm][:10])
