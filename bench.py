#!/usr/bin/env python
"""Benchmark of the hot path: points hashed + indexed per second.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C4] [--scheme CS_E2LSH]
    python bench.py --impl reference ...      # the oracle on host cores (reference arm)

A step = one pass of the whole hot path over the config's synthetic batch:
hash every point (sketch -> discretise -> keys, §8(a) a-2..a-4), group the points
into the buckets of all L tables (a-5), at N > 1 the NCCL all-gather of the
per-table coarse bucket counts (a-6), and a bucket lookup for a query batch
(a-7).  Weak scaling by default: every rank hashes and indexes a full config batch
(C4: 10^6 points per rank; rank r owns rows [r n, (r+1) n) of the seeded stream),
`value` = points of all ranks / max-over-ranks device time; `--scaling strong`
splits the config's n across the ranks instead.
Inputs are resident in HBM when the timed region starts; `e2e` times the same
step through the C ABI from pinned HOST buffers (H2D of X and the queries, D2H
of the per-table bucket counts and query ranges inside the timed region).
Rank 0 prints one JSON line.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "points hashed+indexed/sec"
UNIT = "points/s"
NQ = 1000          # queries looked up per step (a-7)
B_COARSE = 12      # coarse bins exchanged across ranks (§8(e))


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C4")
    ap.add_argument("--scheme", default="CS_E2LSH")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-clocks", action="store_true", help="diagnostic only: skip the nvidia-smi sampler")
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="weak: every rank hashes a full config batch (default); strong: n split across ranks")
    ap.add_argument("--per-table", action="store_true",
                    help="NEXT-2: per-table independent CS families (reading C3); not the headline workload")
    return ap.parse_args()


def dist_env():
    return int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")), \
        int(os.environ.get("LOCAL_RANK", "0"))


def shard(n, rank, world):
    per = (n + world - 1) // world
    lo = min(n, rank * per)
    return lo, min(n, lo + per)


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = "clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown," \
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown," \
             "clocks_event_reasons.sw_power_cap"

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read, daemon=True)
            self._t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            pk = json.load(f)
        return float(pk["hbm_gbs"]), "measured (copy: read + write bytes; a read-only stream can exceed it)"
    except Exception:
        return 6650.0, "fallback"


def peaks_tensor():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            pk = json.load(f)
        return float(pk["bf16_tflops_sustained"]), "measured (cuBLAS bf16 sustained)"
    except Exception:
        return 1400.0, "fallback"


# --------------------------------------------------------------------------
# reference arm: the oracle on host cores
# --------------------------------------------------------------------------

def oracle_step_sample(cfg, scheme, rows, per_table=False):
    import numpy as np
    from oracle import lsh
    import synth
    kw = dict(mode_d=cfg.mode_d, mode_m=cfg.mode_m) if scheme.startswith("HCS") else {}
    p = lsh.Params(scheme, d=cfg.d, m=cfg.m, L=cfg.L, K=cfg.K, w=cfg.w, seed=cfg.hash_seed, per_table=per_table, **kw)
    X = synth.rows(cfg, 0, rows).numpy()
    t0 = time.perf_counter()
    t = lsh.make_tables(p) if not hasattr(oracle_step_sample, "_t") else oracle_step_sample._t
    oracle_step_sample._t = t
    out = lsh.hash_points(p, t, X)
    lsh.group(out["keys"])
    return time.perf_counter() - t0


def cpu_sample_rows(cfg):
    # ~10-30 s of single-core NumPy work for the bounded sample
    return {"C1": cfg.n, "C2": 20000, "C3": 4000, "C4": 20000, "C5": 200}.get(cfg.name, 2000)


def workload_name(cfg, args):
    return f"{cfg.name}:{args.scheme}" + (":per_table" if args.per_table else "")


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    import synth
    cfg = synth.CONFIGS[args.config]
    rows = min(cfg.n, cpu_sample_rows(cfg) // (16 if args.per_table else 1))
    times = []
    for i in range(args.warmup + args.steps):
        dt = oracle_step_sample(cfg, args.scheme, rows, args.per_table)
        if i >= args.warmup:
            times.append(dt)
    tstep = statistics.median(times)
    value = rows / tstep
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": tstep * 1e3, "higher_is_better": True,
            "scaling": args.scaling, "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": workload_name(cfg, args), "n": cfg.n, "d": cfg.d, "m": cfg.m, "L": cfg.L,
                       "K": cfg.K, "w": cfg.w, "sample_rows_per_step": rows},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1,
                             "host_cores_available": len(os.sched_getaffinity(0)), "kind": "oracle",
                             "sample": f"first {rows} rows of {cfg.name} per step (hash + group), NumPy fp64"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------------
# our arm
# --------------------------------------------------------------------------

def source_hash() -> str:
    """sha256 (16 hex) of the library sources: ties an ncu capture to this build."""
    import hashlib
    h = hashlib.sha256()
    csrc = os.path.join(ROOT, "paper_2503_06737_b200", "csrc")
    for name in sorted(os.listdir(csrc)):
        with open(os.path.join(csrc, name), "rb") as f:
            h.update(name.encode() + b"\0" + f.read())
    with open(os.path.join(ROOT, "include", "lsh.h"), "rb") as f:
        h.update(f.read())
    return h.hexdigest()[:16]


def ncu_dram(workload, kernel):
    """dram bytes (read + write) per step of a kernel from the committed ncu capture of
    THIS build (profiles/round2/ncu_summary.json, keyed by source hash), else None."""
    p = os.path.join(ROOT, "profiles", "round2", "ncu_summary.json")
    try:
        with open(p) as f:
            js = json.load(f)
        if js.get("source_hash") != source_hash():
            return None
        ent = js.get("kernels", {}).get(f"{workload}/{kernel}")
        return ent.get("dram_bytes_per_step") if ent else None
    except Exception:
        return None


def ext_config(cfg, world, scaling):
    """Weak scaling: every rank hashes a full config-sized batch (rank r owns rows
    [r n, (r+1) n) of the same seeded stream extended to world * n rows)."""
    import dataclasses
    if scaling == "weak" and world > 1:
        return dataclasses.replace(cfg, n=cfg.n * world)
    return cfg


def parity_sample(h, cfg, scheme, X, rows, per_table):
    """Keys of the first `rows` rows through the keys-only hot path vs the oracle's
    (north_star tolerance rule, tests/parity.py): counts for the bench line."""
    import numpy as np
    from oracle import lsh
    from tests import parity
    kw = dict(mode_d=cfg.mode_d, mode_m=cfg.mode_m) if scheme.startswith("HCS") else {}
    p = lsh.Params(scheme, d=cfg.d, m=cfg.m, L=cfg.L, K=cfg.K, w=cfg.w, seed=cfg.hash_seed, per_table=per_table, **kw)
    t = lsh.make_tables(p)
    Xs = X[:rows]
    gk = h.hash(Xs, keys=True)["keys"].cpu().numpy()
    Xn = Xs.cpu().numpy()
    ref = lsh.hash_points(p, t, Xn)
    ref["band"] = parity.code_band(p, t, Xn) if lsh.is_e2lsh(scheme) else parity.srp_band(p, t, Xn)
    kr = parity.check_keys(p, ref, gk)
    ex = parity.exempt_mask(p, ref)
    out = {"rows": int(rows), "keys": kr["n"], "key_mismatch_outside_exempt": kr["mismatch_outside_exempt"],
           "exempt_keys": kr["exempt"], "exempt_code_entries": int(ex.sum()), "code_entries": int(ex.size),
           "rule": "keys bit-exact outside the 1e-5*w (E2LSH) / 1e-6 (SRP) bands (tests/parity.py)"}
    if lsh.is_e2lsh(scheme):
        out["fingerprint_merges"] = int(lsh.fingerprint_merges(ref["codes"], ref["keys"], p.L, p.K))
    return out


def run_ours(args):
    import torch
    import torch.distributed as dist

    rank, world, local = dist_env()
    force = os.environ.get("LSH_BENCH_FORCE_DIST") == "1"   # exercise the NCCL path at N = 1
    use_dist = world > 1 or force
    if use_dist:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    dev = torch.device("cuda", torch.cuda.current_device())

    import paper_2503_06737_b200 as pk
    import synth

    cfg = synth.CONFIGS[args.config]
    scheme = args.scheme
    kw = dict(mode_d=cfg.mode_d, mode_m=cfg.mode_m) if scheme.startswith("HCS") else {}
    h = pk.LSH(scheme, cfg.d, cfg.m, cfg.L, cfg.K, cfg.w, cfg.hash_seed, device=dev.index, per_table=args.per_table,
               **kw)
    ecfg = ext_config(cfg, world, args.scaling)
    lo, hi = (rank * cfg.n, (rank + 1) * cfg.n) if args.scaling == "weak" else shard(cfg.n, rank, world)
    n_local = hi - lo
    n_total = ecfg.n if args.scaling == "weak" else cfg.n
    X = synth.rows(ecfg, lo, hi, device=dev)
    Q = synth.rows(cfg, 0, NQ, device=dev) if rank == 0 else synth.rows(ecfg, lo, lo + min(NQ, n_local), device=dev)
    nq = Q.shape[0]
    stream = torch.cuda.current_stream()

    from paper_2503_06737_b200.dist import build_index_sharded

    def step():
        if use_dist:
            idx = build_index_sharded(h, X, id_base=lo, B=B_COARSE).local   # a-5 + a-6 (NCCL all-gather)
        else:
            idx = h.build_index(X, id_base=lo)
        b, e = h.query_buckets(idx, Q)
        return idx, b, e

    def run_steps(k, keep):
        for _ in range(k):
            keep.append(step()[0])
            if len(keep) > 2:
                keep.pop(0)

    # warm-up with the same index lifetime pattern as the timed loop (the stream-ordered
    # pool then already holds the memory of the in-flight indexes)
    keep = []
    run_steps(max(3, args.warmup), keep)
    torch.cuda.synchronize()

    # device-timed region (inputs resident in HBM; X >> L2 so no flush needed); the
    # library's per-kernel timing is OFF here
    clocks = ClockSampler(dev.index)
    if not args.no_clocks:
        clocks.start()
    if use_dist:
        dist.barrier()
    torch.cuda.synchronize()
    l0 = pk.launch_count()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    run_steps(args.steps, keep)
    ev1.record(stream)
    torch.cuda.synchronize()
    if use_dist:
        dist.barrier()
    launches = pk.launch_count() - l0
    clk = clocks.stop()
    ms_local = ev0.elapsed_time(ev1) / args.steps
    t = torch.tensor([ms_local], device=dev)
    if use_dist:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    value = n_total / (ms * 1e-3)

    # per-kernel breakdown: a separate, untimed pass with CUDA events around every launch
    # (on the launching stream)
    kb_steps = max(1, min(args.steps, 5))
    pk.timing_reset()
    pk.timing_enable(True)
    run_steps(kb_steps, keep)
    torch.cuda.synchronize()
    pk.timing_enable(False)
    names = ("sketch", "sketch_query", "group_hist", "group_scan", "group_scatter", "group_sort", "lookup", "counts",
             "global_offsets", "dense_gemm", "keys_from_proj")
    kernel_ms = {k: pk.timing_get(k)[0] / kb_steps for k in names}
    kernel_launches = {k: pk.timing_get(k)[1] for k in names}
    idx_last = keep[-1] if keep else None
    del keep[:-1]

    # end-to-end through the C ABI from pinned host buffers
    e2e = None
    if not args.no_e2e:
        Xh = X.cpu().pin_memory()
        Qh = Q.cpu().pin_memory()
        Xd = torch.empty_like(X)
        Qd = torch.empty_like(Q)
        nb_h = torch.empty((cfg.L, 1 << B_COARSE), dtype=torch.int32).pin_memory()
        be_h = torch.empty((2, nq, cfg.L), dtype=torch.int64).pin_memory()

        def e2e_step():
            Xd.copy_(Xh, non_blocking=True)
            Qd.copy_(Qh, non_blocking=True)
            if use_dist:
                shi = build_index_sharded(h, Xd, id_base=lo, B=B_COARSE)
                idx, cnt = shi.local, shi.counts
            else:
                idx = h.build_index(Xd, id_base=lo)
                cnt = idx.counts(B_COARSE)
            b, e = h.query_buckets(idx, Qd)
            nb_h.copy_(cnt, non_blocking=True)
            be_h[0].copy_(b, non_blocking=True)
            be_h[1].copy_(e, non_blocking=True)
            return idx

        ekeep = []
        for _ in range(3):
            ekeep.append(e2e_step())
            if len(ekeep) > 2:
                ekeep.pop(0)
        torch.cuda.synchronize()
        esteps = max(2, min(args.steps, 5))
        if use_dist:
            dist.barrier()
        torch.cuda.synchronize()
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a0.record(stream)
        for _ in range(esteps):
            ekeep.append(e2e_step())
            if len(ekeep) > 2:
                ekeep.pop(0)
        a1.record(stream)
        torch.cuda.synchronize()
        ekeep.clear()
        te = torch.tensor([a0.elapsed_time(a1) / esteps], device=dev)
        if use_dist:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e2e = {"value": n_total / (float(te.item()) * 1e-3), "unit": UNIT,
               "h2d_bytes_per_step": int(X.numel() * 4 + Q.numel() * 4),
               "d2h_bytes_per_step": int(nb_h.numel() * 4 + be_h.numel() * 8)}

    if rank != 0:
        if use_dist:
            dist.destroy_process_group()
        return

    hbm_peak, peak_kind = peaks()
    workload = workload_name(cfg, args)
    dense = scheme in ("E2LSH", "SRP") or args.per_table
    Ln = cfg.L * n_local
    nb_total = sum(int(idx_last.view(t, copy=False)[1].numel()) for t in range(cfg.L)) if idx_last else Ln
    # the method must read every point once (4d B) and write its index
    # payload (one u32 id per table, 4L B) plus <= 12 B of bucket metadata per bucket;
    # keys are an intermediate of the implementation (counted in ncu traffic only)
    step_alg = (4 * cfg.d + 4 * cfg.L) * n_local + 12 * nb_total
    step_roof = {"algorithmic_bytes_per_step": step_alg, "accounting": "SURVEY 8(d): 4d + 4L B/point + 12 B/bucket",
                 "achieved_gbs": step_alg / (ms * 1e-3) / 1e9}
    step_roof["frac_measured_peak"] = step_roof["achieved_gbs"] / hbm_peak
    step_roof["frac_8tbs"] = step_roof["achieved_gbs"] / 8000.0
    kinfo = None
    if dense:
        # tensor-core dense baseline: algorithmic flops 2*n*m*d (the split into 3 bf16 terms
        # triples the executed MMA work; reported separately).  Per-table families (NEXT-2)
        # run the same GEMM on the K-sparse +-1 matrix: their definitional work is only
        # 2*n*L*d flops (one signed add per coordinate and table), also reported.
        g_ms, g_n = pk.timing_get("dense_gemm")
        avg = g_ms / max(1, g_n)
        flops = 2.0 * n_local * cfg.m * cfg.d
        tf_peak, tf_kind = peaks_tensor()
        achieved = flops / (avg * 1e-3) / 1e12 if avg > 0 else None
        roof = {"kernel": "dense_gemm (tcgen05 bf16x3)", "bound": "tensor", "achieved": achieved, "peak": tf_peak,
                "peak_kind": tf_kind, "unit": "TFLOP/s", "frac": (achieved / tf_peak) if achieved else None,
                "flops_per_launch": flops, "executed_mma_flops_per_launch": 3 * flops, "traffic": None,
                "avg_launch_ms": avg}
        if args.per_table:
            roof["sparse_definitional_flops_per_launch"] = 2.0 * n_local * cfg.L * cfg.d
    else:
        # Per kernel (per step; group kernels are one launch each for wide keys, two LSD
        # scatter passes for narrow SRP keys):
        #   alg   = its share of the §8(d) algorithmic bytes (sketch: the points, 4d B;
        #           the kernel writing the ids: 4 B per (table, point) + 12 B per bucket);
        #   io    = the bytes the kernel itself must read + write given its inputs and
        #           outputs (keys 8 B, (key, id) 12 B per (table, point));
        #   dram  = ncu dram__bytes_read + dram__bytes_write of THIS build (committed
        #           capture, profiles/round2/ncu_summary.json), else null.
        narrow = (not h.e2lsh) and cfg.K <= 22
        ovf_hist = (not narrow) and h.group_path() > 0
        # group_hist: narrow keys read the keys three times (varying-bit mask, then one
        # histogram per LSD pass); wide keys take the fixed-capacity L1 scatter, which needs
        # no histogram: their hist kernels are the overflow fallback, gated off (0 bytes)
        # unless a bin overflowed (ovf_hist below, from the build's own overflow word)
        io = {
            "sketch": (4 * cfg.d + 8 * cfg.L) * n_local,
            "group_hist": 24 * Ln if narrow else (16 * Ln if ovf_hist else 0),
            "group_scatter": (20 + 24) * Ln if narrow else 20 * Ln,
            "group_sort": (8 * Ln + 12 * nb_total) if narrow else (12 * Ln + 4 * Ln + 12 * nb_total),
        }
        alg = {"sketch": 4 * cfg.d * n_local, "group_hist": 0,
               "group_scatter": 4 * Ln if narrow else 0,        # narrow keys: pass 2 writes the final ids
               "group_sort": 12 * nb_total if narrow else 4 * Ln + 12 * nb_total}
        kinfo = {}
        for k in io:
            kms = kernel_ms.get(k, 0.0)
            if kms <= 0:
                continue
            sec = kms * 1e-3
            dram = ncu_dram(workload, k)
            kinfo[k] = {"ms_per_step": kms, "launches_per_step": kernel_launches[k] / kb_steps,
                        "alg_bytes": alg[k], "alg_gbs": alg[k] / sec / 1e9, "alg_frac": alg[k] / sec / 1e9 / hbm_peak,
                        "io_bytes": io[k], "io_gbs": io[k] / sec / 1e9, "io_frac": io[k] / sec / 1e9 / hbm_peak,
                        "ncu_dram_bytes": dram, "dram_over_io": (dram / io[k]) if (dram and io[k]) else None}
        dom = max(kinfo, key=lambda k: kinfo[k]["ms_per_step"])
        d0 = kinfo[dom]
        use_alg = d0["alg_bytes"] > 0
        roof = {"kernel": dom, "bound": "hbm", "unit": "GB/s", "peak": hbm_peak, "peak_kind": peak_kind,
                "accounting": "SURVEY 8(d) algorithmic bytes" if use_alg else "kernel input + output bytes",
                "achieved": d0["alg_gbs"] if use_alg else d0["io_gbs"],
                "frac": d0["alg_frac"] if use_alg else d0["io_frac"],
                "frac_8tbs": (d0["alg_gbs"] if use_alg else d0["io_gbs"]) / 8000.0,
                "bytes_per_launch": d0["alg_bytes"] if use_alg else d0["io_bytes"],
                "io_bytes_per_launch": d0["io_bytes"], "io_frac": d0["io_frac"],
                "traffic": d0["ncu_dram_bytes"], "avg_launch_ms": d0["ms_per_step"] / max(1, d0["launches_per_step"]),
                "bytes_per_point": (4 * cfg.d) if (use_alg and dom == "sketch") else None}
    cpu = None
    par = None
    if not args.no_cpu_baseline and world == 1:
        rows = min(cfg.n, cpu_sample_rows(cfg) // (16 if args.per_table else 1))
        oracle_step_sample(cfg, scheme, min(rows, 256), args.per_table)  # warm caches / table draw
        dt = oracle_step_sample(cfg, scheme, rows, args.per_table)
        cpu = {"value": rows / dt, "unit": UNIT, "cores": 1, "host_cores_available": len(os.sched_getaffinity(0)),
               "kind": "oracle",
               "sample": f"first {rows} rows of {cfg.name}, hash + group, NumPy fp64 (single-threaded)"}
        par = parity_sample(h, cfg, scheme, X, min(rows, 4096 if cfg.d > 10000 else rows), args.per_table)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": max(3, args.warmup), "ms_per_step": ms, "higher_is_better": True, "scaling": args.scaling,
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": workload, "n": cfg.n, "n_per_rank": n_local, "n_total": n_total, "d": cfg.d,
                   "m": cfg.m, "L": cfg.L, "K": cfg.K, "w": cfg.w, "queries_per_step": NQ,
                   "parallelism": f"points sharded x{world} ({args.scaling} scaling)",
                   "l2": "inputs (%.2f GB per rank) larger than L2; no flush" % (n_local * cfg.d * 4 / 1e9)},
        "roofline": roof,
        "step_roofline": step_roof,
        "roofline_kernels": kinfo,
        "grouping_path": (None if dense else ("LSD (narrow keys)" if ((not h.e2lsh) and cfg.K <= 22) else
                          ("histogram (bin overflow)" if h.group_path() > 0 else "fixed-capacity L1 scatter"))),
        "kernel_ms_per_step": kernel_ms,
        "cpu_baseline": cpu,
        "parity": par,
        "e2e": e2e,
        "gpu_launches": int(launches),
        "clocks": clk,
        "source_hash": source_hash(),
    }
    print(json.dumps(line), flush=True)
    if use_dist:
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
