"""Launch shares of the library's kernels from an ncu launch list
(`ncu --metrics gpu__time_duration.sum --csv --log-file <csv> python bench.py ...`).

    python tools/launch_shares.py <launches.csv> > launch_shares.txt
"""
import csv
import re
import sys

rows = [r for r in csv.reader(l for l in open(sys.argv[1]) if l.startswith('"'))]
h = rows[0]
ik, iv = h.index("Kernel Name"), h.index("Metric Value")
tot, cnt = {}, {}
for r in rows[1:]:
    k = r[ik]
    if "lshb::" not in k:
        continue
    name = re.sub(r"^void ", "", k.split("(")[0])
    name = name.replace("lshb::sk::", "sk::") if name.startswith("lshb::sk::") else name
    tot[name] = tot.get(name, 0.0) + float(r[iv].replace(",", "")) / 1e6
    cnt[name] = cnt.get(name, 0) + 1
s = sum(tot.values()) or 1.0
print("ncu --metrics gpu__time_duration.sum --clock-control none: python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline")
print("(C4 CS-E2LSH; 7 index builds + 7 query hashes/lookups incl. warm-up and the per-kernel timing pass; cold-cache, serialised launches)")
print("library kernels only (torch's input generation excluded); share of the library's total launch time:")
for k, v in sorted(tot.items(), key=lambda x: -x[1]):
    print(f"{k:<62} {cnt[k]:3d} launches {v:9.3f} ms total {v / cnt[k]:9.4f} ms/launch {v / s * 100:5.1f}%")
