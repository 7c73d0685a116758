"""Per-phase clock totals of g2w (diagnostic library built with -DLSHB_PROF).

    python -m paper_2503_06737_b200.build --variant prof
    python tools/g2w_probe.py --config C4 --scheme CS_E2LSH
"""
import argparse
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2503_06737_b200 as pk  # noqa: E402
import synth  # noqa: E402

pk.LIB_PATH = pk.LIB_PATH.replace(".so", "_prof.so")
ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C4")
ap.add_argument("--scheme", default="CS_E2LSH")
a = ap.parse_args()
c = synth.CONFIGS[a.config]
kw = dict(mode_d=c.mode_d, mode_m=c.mode_m) if a.scheme.startswith("HCS") else {}
h = pk.LSH(a.scheme, c.d, c.m, c.L, c.K, c.w, c.hash_seed, **kw)
X = synth.rows(c, 0, c.n, device="cuda")
lib = pk.lib()
buf = (ctypes.c_ulonglong * 16)()
idx = h.build_index(X)
torch.cuda.synchronize()
idx.close()
lib.lsh_debug_g2w_prof(buf, 1)
pk.timing_enable(True)
idx = h.build_index(X)
torch.cuda.synchronize()
lib.lsh_debug_g2w_prof(buf, 1)
ms, _ = pk.timing_get("group_sort")
names = ["load+wait", "emit prev", "count", "scan", "scatter", "rank", "long seg", "heads+sync", "writeback", "ids out"]
tot = sum(buf[i] for i in range(10)) or 1
print(f"group_sort {ms:.3f} ms; per-phase share of thread-0 cycles (all CTAs):")
for i, nm in enumerate(names):
    print(f"  {nm:12s} {buf[i] / tot * 100:5.1f}%  {buf[i] / 1e6:10.1f} Mcyc")
