"""Recall vs L (the paper's §6 protocol):
k = 50 neighbours, K = 8 code coordinates per table, L tables (m = 8L), recall =
|S ∩ S'| / |S| averaged over the queries, S = exact top-50 (ground truth on the host,
NumPy fp64, for the query sample), S' = lsh_query_knn's top-50.  Also reports the
device time of the query batch (hash + lookup + union/re-rank).

Synthetic stand-in (the paper's datasets are not available): n points in d = 4096
(16^3 for HCS) drawn as `clusters` Gaussian centres + sigma * N(0, I), queries =
other draws from the same clusters.  Euclidean family only (E2LSH, CS-E2LSH,
HCS-E2LSH); w = 4 x the mean distance to the k-th true neighbour.

    python tools/recall.py [--n 50000] [--queries 200] [--Ls 1,2,4,8,16,32,50] [--repeats 20]

Each (scheme, L) point is averaged over `repeats` independent hash draws (seeds
0..repeats-1; the paper averages 20 repetitions); std over repeats is
reported with the mean.
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2503_06737_b200 as pk  # noqa: E402


def factor3(m):
    """m = a*b*c with a <= b <= c as balanced as possible (HCS sketch modes)."""
    best = None
    for a in range(1, int(round(m ** (1 / 3))) + 2):
        if m % a:
            continue
        r = m // a
        for b in range(a, int(r ** 0.5) + 1):
            if r % b == 0:
                c = r // b
                cand = (a, b, c)
                if best is None or max(cand) - min(cand) < max(best) - min(best):
                    best = cand
    return best


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=50000)
    ap.add_argument("--d", type=int, default=4096)
    ap.add_argument("--queries", type=int, default=200)
    ap.add_argument("--clusters", type=int, default=500)
    ap.add_argument("--sigma", type=float, default=0.35)
    ap.add_argument("--k", type=int, default=50)
    ap.add_argument("--K", type=int, default=8)
    ap.add_argument("--w", type=float, default=0.0, help="bucket width; 0 = 4 x mean distance to the k-th neighbour")
    ap.add_argument("--Ls", default="1,2,4,8,16,32,50")
    ap.add_argument("--out", default="")
    ap.add_argument("--repeats", type=int, default=1)
    ap.add_argument("--family", default="e2lsh", choices=["e2lsh", "srp"],
                    help="e2lsh: Euclidean top-k; srp: cosine top-k (CS-SRP, HCS-SRP, SRP)")
    a = ap.parse_args()
    g = torch.Generator(device="cuda").manual_seed(2025)
    C = torch.randn((a.clusters, a.d), device="cuda", generator=g)
    lab = torch.randint(0, a.clusters, (a.n + a.queries,), device="cuda", generator=g)
    P = C[lab] + a.sigma * torch.randn((a.n + a.queries, a.d), device="cuda", generator=g)
    X, Q = P[: a.n].contiguous(), P[a.n:].contiguous()
    # ground truth (host, fp64): exact top-k by squared Euclidean distance, ties by id
    Xh, Qh = X.double().cpu().numpy(), Q.double().cpu().numpy()
    xx = (Xh ** 2).sum(1)
    gt, kth = [], []
    xn = np.sqrt(xx)
    for i in range(a.queries):
        if a.family == "srp":   # cosine similarity, descending (reading C2)
            dd = -(Xh @ Qh[i]) / np.maximum(xn * np.linalg.norm(Qh[i]), 1e-300)
        else:
            dd = xx - 2.0 * (Xh @ Qh[i]) + (Qh[i] ** 2).sum()
        order = np.lexsort((np.arange(a.n), dd))
        gt.append(set(order[: a.k].tolist()))
        kth.append(float(np.sqrt(max(dd[order[a.k - 1]], 0.0))))
    if a.family == "srp":
        a.w = 1.0                          # unused by SRP (must be > 0)
    elif a.w <= 0:
        a.w = 4.0 * float(np.mean(kth))   # E2LSH width ~ a few near-neighbour radii
    rows = []
    schemes = ("CS_SRP", "HCS_SRP", "SRP") if a.family == "srp" else ("CS_E2LSH", "HCS_E2LSH", "E2LSH")
    for scheme in schemes:
        for L in [int(x) for x in a.Ls.split(",")]:
            m = a.K * L
            kw = {}
            if scheme.startswith("HCS"):
                kw = dict(mode_d=(16, 16, 16), mode_m=factor3(m))
            recs, qms, ncs = [], [], []
            for rep in range(a.repeats):
                h = pk.LSH(scheme, a.d, m, L, a.K, a.w, rep, **kw)
                idx = h.build_index(X)
                torch.cuda.synchronize()
                for _ in range(2):
                    h.query_knn(idx, X, Q, a.k, max_cand=8192)
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                ids, sc, nc = h.query_knn(idx, X, Q, a.k, max_cand=8192)
                e1.record()
                torch.cuda.synchronize()
                ids = ids.cpu().numpy()
                recs.append(float(np.mean([len(gt[i] & set(ids[i][ids[i] >= 0].tolist())) / a.k
                                           for i in range(a.queries)])))
                qms.append(e0.elapsed_time(e1))
                ncs.append(float(nc.float().mean().item()))
                idx.close()
                h.close()
            row = {"scheme": scheme, "L": L, "m": m, "recall_at_k": float(np.mean(recs)),
                   "recall_std": float(np.std(recs)), "repeats": a.repeats, "query_ms": float(np.median(qms)),
                   "mean_candidates": float(np.mean(ncs))}
            rows.append(row)
            print(json.dumps(row), flush=True)
    res = {"protocol": "PAPER.md:2000-2003 (k=50, K=8 per table, recall vs L), synthetic clustered data",
           "family": a.family,
           "n": a.n, "d": a.d, "queries": a.queries, "repeats": a.repeats, "kth_nn_distance": float(np.mean(kth)), "clusters": a.clusters, "sigma": a.sigma, "w": a.w, "rows": rows}
    if a.out:
        with open(a.out, "w") as f:
            json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
