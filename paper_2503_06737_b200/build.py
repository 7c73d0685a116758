"""Build the in-tree C-ABI shared library liblsh_b200.so for sm_100a with nvcc.

    python -m paper_2503_06737_b200.build [--verbose]

The .so is git-ignored but travels to the GPU box with the gpurun snapshot.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "liblsh_b200.so")
SOURCES = ["api.cu", "sketch.cu", "sketch_fast.cu", "sketch_chunked.cu", "sketch_hcs.cu", "group.cu", "dense_tc.cu", "knn.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
# measurement-only variants (liblsh_b200_<name>.so, loaded with LSH_LIB_VARIANT=<name>)
# (C4, measured round 2: 2048 L1 bins of ~488 keys with IPT 5 / D 11 — scatter 0.44 ->
#  0.56 ms, per-bin sort unchanged at 0.87 ms — not kept)
VARIANT_FLAGS = {"b11": ["-DLSHB_G2_IPT=5", "-DLSHB_G2_D=11", "-DLSHB_L1_AVG=512"],
                 # (C4: 4096-key tiles, 2 scatter CTAs per SM — E2LSH scatter 0.44 -> 0.92 ms
                 #  (shorter runs, more partial sectors), SRP 1.34 -> 1.22 ms — not kept)
                 "t4k": ["-DLSHB_G1_TILE=4096", "-DLSHB_SCATTER_CPS=2"],
                 # g2a CTA shape (C4 group_sort, round 2): 128 threads x 6 CTAs/SM 0.86 ms,
                 # x 7 0.88 ms; 256 x 4 0.87 ms, x 5 0.79 ms (the default), x 6 0.79 ms (spills);
                 # with the final g2a body: 256 x 5 0.683, 256 x 4 0.751, 128 x 8 0.830 ms
                 "g128": ["-DLSHB_G2_T=128", "-DLSHB_G2_CPS=6"],
                 # shared-digit segments ranked O(s^2) from the worklist up to this length,
                 # longer ones in one bitonic network (C5 / C3 HCS-E2LSH group_sort, round 2):
                 # 8: 1.88 / 0.249 ms, 32: 1.83 / 0.233, 64 (default): 1.75 / 0.229
                 "l8": ["-DLSHB_G2_LONG=8"],
                 # L1 bins of ~1950 keys (B1 = 9) at C4 (round 2): scatter 0.363 -> 0.322 ms but
                 # g2a 0.69 -> 0.76 (256 x IPT 10, 4/SM, D 12) / 0.76 (3/SM, D 13) / 0.81 (512 x 5,
                 # 2/SM, D 13); step 2.03 -> 2.06-2.12 ms: not kept
                 # K1 keys-only loop, tables per unrolled iteration (C4 E2LSH / SRP sketch,
                 # round 2): 1: 0.929 / 0.796 ms, 2 (default): 0.920 / 0.784, 4: 0.929 / 0.776
                 "tu4": ["-DLSHB_SK_TUNROLL=4"],
                 # K1 keys-only loop with one lane per point and one table per warp iteration
                 # (the round-2 kernel before the four-tables-per-warp 128-bit gathers)
                 # (C4, round 2: E2LSH sketch 0.925 lane-per-point -> 0.844 ms four tables per
                 #  warp; SRP 0.786 -> 0.810 ms, so SRP keeps the lane-per-point loop)
                 "lane1": ["-DLSHB_SK_QUAD=0"],
                 "quad1": ["-DLSHB_SK_QUAD=1"],
                 # (also measured, source reverted: the thread index pinned in a register so the
                 #  tile loop has no S2R after its barriers — C4 E2LSH sketch 0.849 vs 0.847 ms,
                 #  SRP 0.787 vs 0.787: the samples at those S2R were warps waiting at the barrier)
                 # four-table path with the first 2 / 4 pair-offset vectors read before the fold
                 # (C4 E2LSH sketch, round 2): 0 (default) 0.848, 2: 0.860, 4: 0.913 ms (spills)
                 "qpre2": ["-DLSHB_SK_QPRE=2"],
                 "qpre4": ["-DLSHB_SK_QPRE=4"],
                 # g2a digit bits below the L1 digit (C4 group_sort, round 2): 11: 0.774 ms,
                 # 12 (default): 0.660, 13: 0.914 (the 8192-counter zero + scan)
                 "d11": ["-DLSHB_G2_D=11"],
                 # g2a 512 threads x IPT 3 (cap 1536): 3/SM 0.964 ms, 2/SM 1.110 ms at C4 (not kept)
                 "g512c3": ["-DLSHB_G2_T=512", "-DLSHB_G2_IPT=3", "-DLSHB_G2_CPS=3"],
                 # L1 scatter with 1024-thread CTAs (C4, round 2): E2LSH 0.364 -> 0.353 ms,
                 # SRP LSD passes 1.28 -> 1.34 ms: not kept
                 "s1024": ["-DLSHB_SCATTER_T=1024"],
                 # K1 four-table path key stores and streamed-load L2 hints (C4 E2LSH / SRP sketch,
                 # end of round 2).  A lane's four keys as four 64-bit stores (32-byte lane stride:
                 # every store instruction touched all 32 sectors of the warp's 1 KB): 0.846 ms;
                 # two 128-bit stores: 0.784; ONE 256-bit store (the default): 0.771.  With it the
                 # four-table loop also wins for SRP (0.788 lane-per-point -> 0.712), so it is the
                 # default for both families.  X loads: L2::256B prefetch size 0.847 (no change);
                 # an L2 evict_first policy 0.846 -> 0.837 (E2LSH), 0.787 -> 0.793 (SRP lane-per-point).
                 "k1old": ["-DLSHB_SK_QUAD=1", "-DLSHB_SK_ST128=0"],
                 "st128": ["-DLSHB_SK_ST128=1"],
                 "st256cs": ["-DLSHB_SK_ST128=3"],
                 "ld256": ["-DLSHB_SK_LDHINT=1"],
                 "ef": ["-DLSHB_SK_LDHINT=2"],
                 "efe2": ["-DLSHB_SK_LDHINT=4"],
                 "b9": ["-DLSHB_L1_AVG=2048", "-DLSHB_G2_T=256", "-DLSHB_G2_IPT=10", "-DLSHB_G2_CPS=3", "-DLSHB_G2_D=13"]}

def nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _stale() -> bool:
    if not os.path.exists(OUT):
        return True
    t = os.path.getmtime(OUT)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)]
    deps.append(os.path.join(HERE, "..", "include", "lsh.h"))
    deps.append(os.path.abspath(__file__))
    return any(os.path.getmtime(p) > t for p in deps if os.path.exists(p))


def build(verbose: bool = False, force: bool = False, variant: str = "") -> str:
    """variant "checked": liblsh_b200_checked.so (-DLSHB_CHECKS: device-side bounds
    checks on every index write, reported as "LSHB_DCHECK file:line"), loaded instead of
    the product library when LSH_LIB_VARIANT=checked (tools/gpu_checked.sh)."""
    target = OUT if not variant else OUT.replace(".so", f"_{variant}.so")
    if not variant and not force and not _stale():
        return OUT
    objs = []
    tmp = os.path.join(HERE, "build" + (f"_{variant}" if variant else ""))
    os.makedirs(tmp, exist_ok=True)
    flags = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O3", "--expt-relaxed-constexpr",
                    "-I" + os.path.join(HERE, "..", "include")]
    if verbose:
        flags += ["-Xptxas", "-v"]
    if variant == "checked":
        flags += ["-DLSHB_CHECKS"]
    flags += VARIANT_FLAGS.get(variant, [])
    procs = []
    for src in SOURCES:
        obj = os.path.join(tmp, src.replace(".cu", ".o"))
        objs.append(obj)
        cmd = [nvcc()] + flags + ["-c", os.path.join(CSRC, src), "-o", obj]
        procs.append((cmd, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)))
    for cmd, pr in procs:
        out, _ = pr.communicate()
        if pr.returncode != 0 or verbose:
            sys.stderr.write(out.decode(errors="replace"))
        if pr.returncode != 0:
            raise RuntimeError("nvcc failed: " + " ".join(cmd))
    link = [nvcc()] + ARCH + ["-shared", "-cudart", "static", "-o", target + ".tmp"] + objs + ["-lpthread"]
    r = subprocess.run(link, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)
    if r.returncode != 0:
        sys.stderr.write(r.stdout.decode(errors="replace"))
        raise RuntimeError("link failed")
    os.replace(target + ".tmp", target)
    return target


if __name__ == "__main__":
    v = sys.argv[sys.argv.index("--variant") + 1] if "--variant" in sys.argv else ""
    print(build(verbose="--verbose" in sys.argv, force=True, variant=v))
