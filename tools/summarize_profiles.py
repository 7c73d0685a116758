"""Turn gpurun_out ncu captures into the committed summaries under profiles/<round>/.

    python tools/summarize_profiles.py round1

Inputs (written by tools/gpu_profile.sh on the GPU box):
  gpurun_out/bench_plain.log            the bench JSON line (no profiler)
  gpurun_out/bench_launches.csv         ncu launch list of the short bench command
  gpurun_out/<CFG>_<SCHEME>_full.ncu-rep ncu --set full captures of one build / hash
Outputs:
  profiles/<round>/bench_line.json, bench_launch_shares.txt, bench_launches.csv,
  profiles/<round>/<CFG>_<SCHEME>_ncu_full.txt (key metrics per kernel),
  profiles/ncu_summary.json (dram bytes per launch per timing name: bench `traffic`).
"""
import csv
import glob
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
rnd = sys.argv[1] if len(sys.argv) > 1 else "round1"
out_dir = os.path.join(ROOT, "profiles", rnd)
os.makedirs(out_dir, exist_ok=True)
go = os.path.join(ROOT, "gpurun_out")

# kernel symbol -> timing name used by lsh_timing_* / bench.py
TIMING = [("sketch", "sketch"), ("g0_mask", "group_hist"), ("g1_hist", "group_hist"),
          ("g1_scatter", "group_scatter"), ("g2_sort", "group_sort"), ("g3_rle", "group_sort"),
          ("lookup", "lookup"), ("g1_scan", "group_scan"), ("g1_binstart", "group_scan")]


def timing_name(kernel):
    for sym, name in TIMING:
        if sym in kernel:
            return name
    return None


# 0. bench line
bl = os.path.join(go, "bench_plain.log")
if os.path.exists(bl):
    lines = [x for x in open(bl) if x.startswith("{")]
    if lines:
        with open(os.path.join(out_dir, "bench_line.json"), "w") as f:
            f.write(lines[-1])

# 1. launch list of the bench command
src = os.path.join(go, "bench_launches.csv")
if os.path.exists(src):
    rows = [r for r in csv.reader(open(src)) if len(r) > 5]
    h = rows[0]
    ik, iv, iid = h.index("Kernel Name"), h.index("Metric Value"), h.index("ID")
    ours = [(r[iid], r[ik], float(r[iv].replace(",", ""))) for r in rows[1:] if "lshb::" in r[ik]]
    with open(os.path.join(out_dir, "bench_launches.csv"), "w") as f:
        f.write("id,kernel,gpu_time_ns\n")
        for i, k, v in ours:
            f.write(f"{i},\"{k.split('(')[0]}\",{v:.0f}\n")
    tot = {}
    for i, k, v in ours:
        kk = k.split("(")[0].replace("void ", "")
        tot[kk] = tot.get(kk, 0.0) + v
    s = sum(tot.values()) or 1.0
    with open(os.path.join(out_dir, "bench_launch_shares.txt"), "w") as f:
        f.write("ncu launch list of `python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline`\n")
        f.write("(cold-cache, serialised: compare SHARES of the step, not absolute times)\n")
        for k, v in sorted(tot.items(), key=lambda x: -x[1]):
            f.write(f"{v / s * 100:6.2f}%  {v / 1e3:10.1f} us  {k}\n")

# 2. full captures
WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__inst_executed.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "sm__cycles_elapsed.avg.per_second"]
UNIT = {"byte": 1, "kbyte": 1e3, "mbyte": 1e6, "gbyte": 1e9, "tbyte": 1e12}
pj = os.path.join(ROOT, "profiles", "ncu_summary.json")
summary = json.load(open(pj)) if os.path.exists(pj) else {}
for rep in sorted(glob.glob(os.path.join(go, "*_full.ncu-rep"))):
    tag = os.path.basename(rep)[: -len("_full.ncu-rep")]           # e.g. C4_CS_E2LSH
    if "_" not in tag:
        continue
    cfg, scheme = tag.split("_", 1)
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    if len(rows) < 3:
        continue
    h, units = rows[0], rows[1]
    idx = {w: h.index(w) for w in WANT if w in h}
    ik = h.index("Kernel Name")
    per_name = {}
    with open(os.path.join(out_dir, f"{tag}_ncu_full.txt"), "w") as f:
        f.write(f"ncu --set full --clock-control none: {cfg} {scheme} (tools/prof_hash.py, one launch per kernel)\n")
        for r in rows[2:]:
            name = r[ik].split("(")[0].replace("void ", "")
            f.write(f"== {name}\n")
            for w, i in idx.items():
                f.write(f"   {w:62s} {r[i]} {units[i]}\n")
            tn = timing_name(name)
            if tn and "dram__bytes_read.sum" in idx:
                def val(w):
                    return float(r[idx[w]].replace(",", "")) * UNIT.get(units[idx[w]].strip().lower(), 1)
                e = per_name.setdefault(tn, {"dram_read": 0.0, "dram_write": 0.0, "launches": 0})
                e["dram_read"] += val("dram__bytes_read.sum")
                e["dram_write"] += val("dram__bytes_write.sum")
                e["launches"] += 1
    for tn, e in per_name.items():
        # bench.py's traffic is per step of that timing name (all its launches of one build)
        summary[f"{cfg}/{scheme}/{tn}"] = {"dram_bytes_per_launch": e["dram_read"] + e["dram_write"],
                                           "dram_read": e["dram_read"], "dram_write": e["dram_write"],
                                           "kernels": e["launches"],
                                           "source": f"profiles/{rnd}/{tag}_ncu_full.txt"}
json.dump(summary, open(pj, "w"), indent=1, sort_keys=True)
sh = os.path.join(out_dir, "bench_launch_shares.txt")
print(open(sh).read() if os.path.exists(sh) else "no launch list")
print(json.dumps(summary, indent=1)[:3000])
