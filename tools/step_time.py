"""Device time of repeated index builds (events around the loop) vs kernel-time sum."""
import argparse, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2503_06737_b200 as pk
import synth
ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C4"); ap.add_argument("--scheme", default="CS_E2LSH")
ap.add_argument("--steps", type=int, default=10); ap.add_argument("--query", action="store_true")
ap.add_argument("--keep", type=int, default=2)
a = ap.parse_args()
c = synth.CONFIGS[a.config]
kw = dict(mode_d=c.mode_d, mode_m=c.mode_m) if a.scheme.startswith("HCS") else {}
h = pk.LSH(a.scheme, c.d, c.m, c.L, c.K, c.w, c.hash_seed, **kw)
X = synth.rows(c, 0, c.n, device="cuda"); Q = X[:1000].clone()
for _ in range(3):
    idx = h.build_index(X)
torch.cuda.synchronize()
pk.timing_reset(); pk.timing_enable(True)
keep = []
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
t0 = time.perf_counter(); e0.record()
for _ in range(a.steps):
    idx = h.build_index(X)
    if a.query: h.query_buckets(idx, Q)
    keep.append(idx)
    if len(keep) > a.keep: keep.pop(0)
e1.record(); t1 = time.perf_counter(); torch.cuda.synchronize(); t2 = time.perf_counter()
tot = sum(pk.timing_get(k)[0] for k in ("sketch", "sketch_query", "group_hist", "group_scan", "group_scatter", "group_sort", "lookup"))
print(f"{a.scheme} device {e0.elapsed_time(e1)/a.steps:.3f} ms/step  kernels {tot/a.steps:.3f} ms/step  host enqueue {1e3*(t1-t0)/a.steps:.3f} ms/step  wall {1e3*(t2-t0)/a.steps:.3f}")
