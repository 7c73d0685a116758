"""Quick dense tensor-core check vs the CUDA-core kernel and the oracle (small shapes)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2503_06737_b200 as pk
from oracle import lsh
for (n, d, m, L, K) in [(300, 64, 16, 2, 8), (1000, 784, 160, 10, 16), (257, 1000, 512, 32, 16), (130, 4096, 4096, 256, 16)]:
    h = pk.LSH("E2LSH", d, m, L, K, 4.0, 0)
    X = torch.randn(n, d, device="cuda")
    t0 = time.time()
    out = h.hash(X, keys=True, proj=True)
    torch.cuda.synchronize()
    y = out["proj"].cpu().numpy().astype(np.float64)
    p = lsh.Params("E2LSH", d=d, m=m, L=L, K=K, w=4.0, seed=0)
    R = lsh.make_tables(p).R
    ref = X.cpu().numpy().astype(np.float64) @ R.T
    err = np.abs(y - ref).max() / (np.abs(ref).max() + 1e-30)
    print(f"n={n} d={d} m={m}: max rel err {err:.2e}  time {time.time()-t0:.2f}s", flush=True)
