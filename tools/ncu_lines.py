"""Aggregate an `ncu --page source --csv --print-source cuda,sass` export by CUDA source line.

    python tools/ncu_lines.py export.csv [top]
"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
hdr = None
agg = {}
for r in rows:
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or not r or not r[0].isdigit():
        continue
    try:
        s = int(r[4] or 0)
        ie = int(r[7] or 0)
    except ValueError:
        continue
    k = (int(r[0]), r[1][:100])
    a = agg.setdefault(k, [0, 0])
    a[0] += s
    a[1] += ie
tot = sum(v[0] for v in agg.values()) or 1
print("samples", tot, "warp-instr", sum(v[1] for v in agg.values()))
for (ln, src), (s, ie) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{s:7d} {100 * s / tot:5.1f}%  inst {ie:11d}  L{ln:<5d} {src}")
