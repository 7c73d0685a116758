"""Turn gpurun_out ncu captures into the committed summaries under profiles/."""
import csv, json, os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
rnd = sys.argv[1] if len(sys.argv) > 1 else "round1"
out_dir = os.path.join(ROOT, "profiles", rnd)
os.makedirs(out_dir, exist_ok=True)
go = os.path.join(ROOT, "gpurun_out")

# 1. launch list of the bench command
src = os.path.join(go, "bench_launches.csv")
if os.path.exists(src):
    rows = [r for r in csv.reader(open(src)) if len(r) > 5]
    h = rows[0]
    ik, iv, iid = h.index("Kernel Name"), h.index("Metric Value"), h.index("ID")
    ours = [(r[iid], r[ik], float(r[iv])) for r in rows[1:] if "lshb::" in r[ik]]
    with open(os.path.join(out_dir, "bench_launches.csv"), "w") as f:
        f.write("id,kernel,gpu_time_ns\n")
        for i, k, v in ours:
            f.write(f"{i},\"{k.split('(')[0]}\",{v:.0f}\n")
    tot = {}
    for i, k, v in ours:
        kk = k.split("(")[0].replace("void ", "")
        tot[kk] = tot.get(kk, 0.0) + v
    s = sum(tot.values())
    with open(os.path.join(out_dir, "bench_launch_shares.txt"), "w") as f:
        f.write("ncu launch list of `python bench.py --steps 2 --warmup 3` (cold-cache, serialised; compare shares)\n")
        for k, v in sorted(tot.items(), key=lambda x: -x[1]):
            f.write(f"{v / s * 100:6.2f}%  {v / 1e3:10.1f} us  {k}\n")

# 2. full capture: key metrics per kernel
rep = os.path.join(go, "c4_build_full.ncu-rep")
summary = {}
if os.path.exists(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    h = rows[0]
    want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
            "smsp__inst_executed.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
            "launch__registers_per_thread", "smsp__issue_active.avg.pct_of_peak_sustained_active",
            "sm__cycles_elapsed.avg.per_second"]
    idx = {w: h.index(w) for w in want if w in h}
    ik = h.index("Kernel Name")
    lines = []
    for r in rows[2:]:
        name = r[ik].split("(")[0].replace("void ", "")
        vals = {w: r[i] for w, i in idx.items()}
        lines.append((name, vals))
    with open(os.path.join(out_dir, "c4_build_ncu_full.txt"), "w") as f:
        f.write("ncu --set full --clock-control none, C4 CS-E2LSH index build (tools/prof_hash.py)\n")
        for name, vals in lines:
            f.write(f"== {name}\n")
            for w, v in vals.items():
                f.write(f"   {w:60s} {v} {rows[1][idx[w]]}\n")
    for name, vals in lines:
        if "sketch_kernel" in name:
            try:
                mult = lambda u: {"byte": 1, "kbyte": 1e3, "mbyte": 1e6, "gbyte": 1e9}.get(u.strip().lower(), 1)
                rd = float(vals["dram__bytes_read.sum"].replace(",", "")) * mult(rows[1][idx["dram__bytes_read.sum"]])
                wr = float(vals["dram__bytes_write.sum"].replace(",", "")) * mult(rows[1][idx["dram__bytes_write.sum"]])
                summary["C4/CS_E2LSH/sketch"] = {"dram_read": rd, "dram_write": wr}
            except Exception as e:
                print("parse", e)
    prev = {}
    pj = os.path.join(ROOT, "profiles", "ncu_summary.json")
    if os.path.exists(pj):
        prev = json.load(open(pj))
    for k, v in summary.items():
        prev[k] = {"dram_bytes_per_launch": v["dram_read"] + v["dram_write"], "dram_read": v["dram_read"],
                   "dram_write": v["dram_write"], "source": f"profiles/{rnd}/c4_build_ncu_full.txt"}
    json.dump(prev, open(pj, "w"), indent=1)
print(open(os.path.join(out_dir, "bench_launch_shares.txt")).read() if os.path.exists(os.path.join(out_dir, "bench_launch_shares.txt")) else "no launches")
