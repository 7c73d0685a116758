"""NEXT-4: space and hashing time vs the code size m (Figs
fig:space / fig:time; Table 1) measured on B200 through the C ABI.

d = 10^4; m in {8, ..., 4096}; schemes E2LSH (dense, tcgen05 GEMM), CS-E2LSH,
CS-SRP, HCS-E2LSH / HCS-SRP with N = 2 (100 x 100) and N = 3 (22 x 22 x 21).
For each (scheme, m):
  * params      stored values of the projection structure (Table 1 convention,
                SPEC S:516): dense m*d (+m offsets), CS 2d (+m), HCS 2*sum d_k (+m)
  * single_us   one-vector hash latency (device-resident input, CUDA events,
                median of 5 means of 100 calls) -- the paper's "average running
                time for computing hashcode"
  * batch_ms    hash of a 16384-vector batch (keys only), median of 5

    python tools/time_vs_m.py [--out profiles/round1/time_vs_m.json]
"""
import argparse
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2503_06737_b200 as pk  # noqa: E402

D = 10_000
MS = (8, 16, 32, 64, 128, 256, 512, 1024, 2048, 4096)


def split(m, N):
    """m = product of N factors, as balanced as possible (powers of two here)."""
    e = m.bit_length() - 1
    parts = [e // N + (1 if i < e % N else 0) for i in range(N)]
    return tuple(1 << p for p in parts)


def params(scheme, m, mode_d):
    e2 = "E2LSH" in scheme
    if scheme in ("E2LSH", "SRP"):
        base = m * D
    elif scheme.startswith("HCS"):
        base = 2 * sum(mode_d)
    else:
        base = 2 * D
    return base + (m if e2 else 0)


def timed(fn, reps, rounds=5):
    means = []
    for _ in range(rounds):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        means.append(e0.elapsed_time(e1) / reps)
    return statistics.median(means)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="")
    ap.add_argument("--batch", type=int, default=16384)
    a = ap.parse_args()
    g = torch.Generator(device="cuda").manual_seed(0)
    X1 = torch.randn((1, D), device="cuda", generator=g)
    XB = torch.randn((a.batch, D), device="cuda", generator=g)
    rows = []
    cases = [("E2LSH", None), ("CS_E2LSH", None), ("CS_SRP", None),
             ("HCS_E2LSH", (100, 100)), ("HCS_SRP", (100, 100)), ("HCS_E2LSH", (22, 22, 21))]
    for scheme, mode_d in cases:
        for m in MS:
            K = min(m, 16)
            L = m // K
            kw = {}
            if mode_d:
                kw = dict(mode_d=mode_d, mode_m=split(m, len(mode_d)))
            h = pk.LSH(scheme, D, m, L, K, 4.0, 0, **kw)
            o1 = {"keys": torch.empty((L, 1), dtype=torch.uint64, device="cuda")}
            ob = {"keys": torch.empty((L, a.batch), dtype=torch.uint64, device="cuda")}
            for _ in range(3):
                h.hash(X1, out=o1)
                h.hash(XB, out=ob)
            torch.cuda.synchronize()
            single_ms = timed(lambda: h.hash(X1, out=o1), 100)
            batch_ms = timed(lambda: h.hash(XB, out=ob), 5)
            row = {"scheme": scheme, "N": len(mode_d) if mode_d else 1, "mode_d": mode_d, "m": m, "L": L, "K": K,
                   "params": params(scheme, m, mode_d), "single_us": single_ms * 1e3, "batch_ms": batch_ms,
                   "batch_points_per_s": a.batch / (batch_ms * 1e-3)}
            rows.append(row)
            print(json.dumps(row), flush=True)
            h.close()
    res = {"what": "NEXT-4 space/time vs m (PAPER.md:1972-1991), d = 10^4, B200, keys only", "d": D,
           "batch": a.batch, "rows": rows}
    if a.out:
        with open(a.out, "w") as f:
            json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
