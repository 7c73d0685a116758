"""Summarise ncu captures of one build into profiles/round2 (run on the GPU box:
the .ncu-rep files stay there; text + JSON come back under gpurun_out/r2/prof/).

    python tools/summarize_r2.py <out_dir> <workload>=<report.ncu-rep> ... [--launches <csv>]

Per capture: the key metrics of every kernel (<workload>_ncu_full.txt) and, per
bench timing name, the DRAM bytes (read + write) of one step of this build:
ncu_summary.json {"source_hash": ..., "kernels": {"<workload>/<timing name>": {...}}}
which bench.py reads as `traffic` / `ncu_dram_bytes` when the source hash matches.
"""
import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from bench import source_hash  # noqa: E402

TIMING = [("sketch_kernel", "sketch"), ("sketch_chunked", "sketch"), ("sketch_hcs", "sketch"),
          ("g0_mask", "group_hist"), ("g0_spec", "group_hist"), ("g1_hist", "group_hist"),
          ("g1_scan", "group_scan"), ("g1_binstart", "group_scan"), ("g1_fixscan", "group_scan"), ("g1_scatter", "group_scatter"),
          ("g2_big", "group_sort"), ("g2a", "group_sort"), ("g3_rle", "group_sort"), ("lookup", "lookup"),
          ("dense_tc", "dense_gemm"), ("split3", "dense_gemm")]
WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__inst_executed.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "lts__t_bytes.sum", "sm__cycles_elapsed.avg.per_second"]
UNIT = {"byte": 1, "kbyte": 1e3, "mbyte": 1e6, "gbyte": 1e9, "tbyte": 1e12}


def timing_name(kernel):
    for sym, name in TIMING:
        if sym in kernel:
            return name
    return None


def main():
    out_dir = sys.argv[1]
    os.makedirs(out_dir, exist_ok=True)
    summary = {"source_hash": source_hash(), "kernels": {}}
    for arg in sys.argv[2:]:
        wl, rep = arg.split("=", 1)
        if not os.path.exists(rep):
            continue
        raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        rows = list(csv.reader(raw.splitlines()))
        if len(rows) < 3:
            continue
        h, units = rows[0], rows[1]
        idx = {w: h.index(w) for w in WANT if w in h}
        ik = h.index("Kernel Name")
        per = {}
        tag = wl.replace(":", "_")
        with open(os.path.join(out_dir, f"{tag}_ncu_full.txt"), "w") as f:
            f.write(f"ncu --set full --clock-control none: {wl}, one build (tools/prof_hash.py, NVTX range 'profile')\n")
            f.write(f"source hash {summary['source_hash']}\n")
            for r in rows[2:]:
                name = r[ik].split("(")[0].replace("void ", "")
                f.write(f"== {name}\n")
                for w, i in idx.items():
                    f.write(f"   {w:62s} {r[i]} {units[i]}\n")
                tn = timing_name(name)

                def val(w):
                    return float(r[idx[w]].replace(",", "")) * UNIT.get(units[idx[w]].strip().lower(), 1)
                if tn and "dram__bytes_read.sum" in idx:
                    e = per.setdefault(tn, {"dram_read": 0.0, "dram_write": 0.0, "launches": 0, "ncu_ms": 0.0})
                    e["dram_read"] += val("dram__bytes_read.sum")
                    e["dram_write"] += val("dram__bytes_write.sum")
                    e["launches"] += 1
                    if "gpu__time_duration.sum" in idx:
                        e["ncu_ms"] += val("gpu__time_duration.sum") / 1e6 if units[idx["gpu__time_duration.sum"]].strip() == "ns" else float(r[idx["gpu__time_duration.sum"]].replace(",", "")) * {"ms": 1, "us": 1e-3, "usecond": 1e-3, "msecond": 1}.get(units[idx["gpu__time_duration.sum"]].strip(), 1)
        for tn, e in per.items():
            summary["kernels"][f"{wl}/{tn}"] = {"dram_bytes_per_step": e["dram_read"] + e["dram_write"],
                                                "dram_read": e["dram_read"], "dram_write": e["dram_write"],
                                                "launches": e["launches"], "ncu_ms_serialised": e["ncu_ms"],
                                                "source": f"profiles/round2/{tag}_ncu_full.txt"}
    with open(os.path.join(out_dir, "ncu_summary.json"), "w") as f:
        json.dump(summary, f, indent=1, sort_keys=True)
    print(json.dumps(summary, indent=1)[:4000])


if __name__ == "__main__":
    main()
