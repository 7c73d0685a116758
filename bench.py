#!/usr/bin/env python
"""Benchmark of the hot path: points hashed + indexed per second.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C4] [--scheme CS_E2LSH]
    python bench.py --impl reference ...      # the oracle on host cores (reference arm)

A step = one pass of the whole hot path over the config's synthetic batch:
hash every point (sketch -> discretise -> keys, §8(a) a-2..a-4), group the points
into the buckets of all L tables (a-5), at N > 1 the NCCL all-gather of the
per-table coarse bucket counts (a-6), and a bucket lookup for a query batch
(a-7).  Points are sharded across ranks (C4: n = 1e6 total, strong scaling).
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
        return float(pk["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def peaks_tensor():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            pk = json.load(f)
        return float(pk["bf16_tflops_sustained"]), "measured (cuBLAS bf16 sustained)"
    except Exception:
        return 1400.0, "fallback"


def ncu_traffic(config, scheme, kernel="sketch"):
    """dram bytes per launch of a kernel from the committed ncu summary (profiles/)."""
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(p) as f:
            js = json.load(f)
        ent = js.get(f"{config}/{scheme}/{kernel}")
        return ent.get("dram_bytes_per_launch") if ent else None
    except Exception:
        return None


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
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": workload_name(cfg, args), "n": cfg.n, "d": cfg.d, "m": cfg.m, "L": cfg.L,
                       "K": cfg.K, "w": cfg.w, "sample_rows_per_step": rows},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "oracle",
                             "sample": f"first {rows} rows of {cfg.name} per step (hash + group), NumPy fp64"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------------
# our arm
# --------------------------------------------------------------------------

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

    import numpy as np
    import paper_2503_06737_b200 as pk
    import synth

    cfg = synth.CONFIGS[args.config]
    scheme = args.scheme
    kw = dict(mode_d=cfg.mode_d, mode_m=cfg.mode_m) if scheme.startswith("HCS") else {}
    h = pk.LSH(scheme, cfg.d, cfg.m, cfg.L, cfg.K, cfg.w, cfg.hash_seed, device=dev.index, per_table=args.per_table,
               **kw)
    lo, hi = shard(cfg.n, rank, world)
    n_local = hi - lo
    X = synth.rows(cfg, lo, hi, device=dev)
    Q = synth.rows(cfg, 0, NQ, device=dev) if rank == 0 else synth.rows(cfg, lo, lo + min(NQ, n_local), device=dev)
    nq = Q.shape[0]
    stream = torch.cuda.current_stream()
    counts_all = torch.empty((world, cfg.L, 1 << B_COARSE), dtype=torch.int32, device=dev)
    begin = torch.empty((nq, cfg.L), dtype=torch.int64, device=dev)
    end = torch.empty((nq, cfg.L), dtype=torch.int64, device=dev)

    from paper_2503_06737_b200.dist import build_index_sharded

    def step():
        if use_dist:
            idx = build_index_sharded(h, X, id_base=lo, B=B_COARSE).local   # a-5 + a-6 (NCCL all-gather)
        else:
            idx = h.build_index(X, id_base=lo)
        b, e = h.query_buckets(idx, Q)
        return idx, b, e

    # warm-up with the same index lifetime pattern as the timed loop (the stream-ordered
    # pool then already holds the memory of the in-flight indexes)
    keep = []
    for _ in range(max(3, args.warmup)):
        keep.append(step()[0])
        if len(keep) > 2:
            keep.pop(0)
    torch.cuda.synchronize()

    # device-timed region (inputs resident in HBM; X >> L2 so no flush needed)
    pk.timing_reset()
    pk.timing_enable(True)
    clocks = ClockSampler(dev.index)
    if not args.no_clocks:
        clocks.start()
    if use_dist:
        dist.barrier()
    torch.cuda.synchronize()
    l0 = pk.launch_count()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for _ in range(args.steps):
        keep.append(step()[0])
        if len(keep) > 2:
            keep.pop(0)
    ev1.record(stream)
    torch.cuda.synchronize()
    if use_dist:
        dist.barrier()
    launches = pk.launch_count() - l0
    clk = clocks.stop()
    pk.timing_enable(False)
    ms_local = ev0.elapsed_time(ev1) / args.steps
    sketch_ms, sketch_n = pk.timing_get("sketch")
    kernel_ms = {k: pk.timing_get(k)[0] / max(1, args.steps) for k in
                 ("sketch", "sketch_query", "group_hist", "group_scan", "group_scatter", "group_sort", "lookup", "counts",
                  "global_offsets", "dense_gemm", "keys_from_proj")}
    idx_last = keep[-1] if keep else None
    del keep[:-1]
    t = torch.tensor([ms_local], device=dev)
    if use_dist:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    value = cfg.n / (ms * 1e-3)

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
        e2e = {"value": cfg.n / (float(te.item()) * 1e-3), "unit": UNIT,
               "h2d_bytes_per_step": int(X.numel() * 4 + Q.numel() * 4),
               "d2h_bytes_per_step": int(nb_h.numel() * 4 + be_h.numel() * 8)}

    if rank != 0:
        if use_dist:
            dist.destroy_process_group()
        return

    hbm_peak, peak_kind = peaks()
    dense = scheme in ("E2LSH", "SRP") or args.per_table
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
        # Algorithmic bytes per launch of each kernel of the step:
        #   sketch        read the points (4d B) + write their L keys (8 B each)
        #   group_hist    read the keys twice (varying-bit mask, L1 histogram)
        #   group_scatter wide keys: read 8 B + write key+id 12 B per (table, point);
        #                 narrow keys: two LSD passes (8 -> 12 B, then 12 -> 12 B)
        #   group_sort    wide keys: read key+id 12 B, write id 4 B + (ukey, off) 12 B per bucket;
        #                 narrow keys (RLE): read the sorted keys 8 B + 12 B per bucket
        Ln = cfg.L * n_local
        nb_total = sum(int(idx_last.view(t, copy=False)[1].numel()) for t in range(cfg.L)) if idx_last else Ln
        narrow = (not h.e2lsh) and cfg.K <= 22
        kbytes = {
            "sketch": (4 * cfg.d + 8 * cfg.L) * n_local,
            "group_hist": 16 * Ln,
            "group_scatter": (20 + 24) * Ln if narrow else 20 * Ln,
            "group_sort": (8 * Ln if narrow else 16 * Ln) + 12 * nb_total,
        }
        kinfo = {}
        for k, b in kbytes.items():
            tot_ms, cnt_l = pk.timing_get(k)
            if cnt_l == 0:
                continue
            per_step_ms = tot_ms / max(1, args.steps)
            gbs = b / (per_step_ms * 1e-3) / 1e9 if per_step_ms > 0 else None
            kinfo[k] = {"ms_per_step": per_step_ms, "algorithmic_bytes": b, "achieved_gbs": gbs,
                        "frac": (gbs / hbm_peak) if gbs else None}
        dom = max(kinfo, key=lambda k: kinfo[k]["ms_per_step"])
        roof = {"kernel": dom, "bound": "hbm", "achieved": kinfo[dom]["achieved_gbs"], "peak": hbm_peak,
                "peak_kind": peak_kind, "unit": "GB/s", "frac": kinfo[dom]["frac"],
                "algorithmic_bytes_per_launch": kinfo[dom]["algorithmic_bytes"],
                "traffic": ncu_traffic(cfg.name, scheme, dom), "avg_launch_ms": kinfo[dom]["ms_per_step"],
                "sketch_bytes_per_point": 4 * cfg.d + 8 * cfg.L}
    cpu = None
    if not args.no_cpu_baseline and world == 1:
        rows = min(cfg.n, cpu_sample_rows(cfg) // (16 if args.per_table else 1))
        oracle_step_sample(cfg, scheme, min(rows, 256), args.per_table)  # warm caches / table draw
        dt = oracle_step_sample(cfg, scheme, rows, args.per_table)
        cpu = {"value": rows / dt, "unit": UNIT, "cores": 1, "kind": "oracle",
               "sample": f"first {rows} rows of {cfg.name}, hash + group, NumPy fp64 (single-threaded)"}
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": max(3, args.warmup), "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": workload_name(cfg, args), "n": cfg.n, "d": cfg.d, "m": cfg.m, "L": cfg.L,
                   "K": cfg.K, "w": cfg.w, "queries_per_step": NQ, "parallelism": f"points sharded x{world}",
                   "l2": "inputs (%.2f GB) larger than L2; no flush" % (cfg.n * cfg.d * 4 / 1e9)},
        "roofline": roof,
        "roofline_kernels": kinfo if not dense else None,
        "kernel_ms_per_step": kernel_ms,
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": int(launches),
        "clocks": clk,
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
