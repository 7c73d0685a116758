"""Aggregate an ncu `--page source --csv` (SASS view) by barrier-delimited region:
stall samples, executed warp instructions and the top stall reasons per region.

    python tools/sass_regions.py src_<kernel>.csv [--top N]
"""
import csv
import sys


def main():
    path = sys.argv[1]
    top = int(sys.argv[3]) if len(sys.argv) > 3 and sys.argv[2] == "--top" else 12
    rows = list(csv.reader(open(path)))
    h = rows[1]
    body = [r for r in rows[2:] if len(r) == len(h) and r[0].startswith("0x")]
    # several launches may be listed: keep the first kernel block only
    seen, first = set(), []
    for r in body:
        if r[0] in seen:
            break
        seen.add(r[0])
        first.append(r)
    body = first
    ia, isrc, iss, iex = h.index("Address"), h.index("Source"), h.index("Warp Stall Sampling (All Samples)"), \
        h.index("Instructions Executed")
    stall_cols = [i for i, c in enumerate(h) if c.startswith("stall_") and "Not Issued" not in c]
    tot_s = sum(float(r[iss] or 0) for r in body)
    tot_e = sum(float(r[iex] or 0) for r in body)
    print(f"total samples {tot_s:.0f}, warp instructions {tot_e:.3e}")
    regions, cur = [], {"start": None, "s": 0.0, "e": 0.0, "n": 0, "stalls": {}, "ops": {}}
    for r in body:
        src = r[isrc].strip()
        if cur["start"] is None:
            cur["start"] = r[ia][-5:] + " " + src[:40]
        s, e = float(r[iss] or 0), float(r[iex] or 0)
        cur["s"] += s
        cur["e"] += e
        cur["n"] += 1
        op = src.split()[0] if src else "?"
        if op.startswith("@"):
            op = src.split()[1]
        cur["ops"][op.split(".")[0]] = cur["ops"].get(op.split(".")[0], 0) + e
        for i in stall_cols:
            v = float(r[i] or 0)
            if v:
                cur["stalls"][h[i]] = cur["stalls"].get(h[i], 0) + v
        if "BAR.SYNC" in src or "BAR.RED" in src or "EXIT" in src:
            regions.append(cur)
            cur = {"start": None, "s": 0.0, "e": 0.0, "n": 0, "stalls": {}, "ops": {}}
    if cur["n"]:
        regions.append(cur)
    for g in sorted(regions, key=lambda g: -g["s"])[:top]:
        st = sorted(g["stalls"].items(), key=lambda kv: -kv[1])[:4]
        ops = sorted(g["ops"].items(), key=lambda kv: -kv[1])[:6]
        print(f"{100 * g['s'] / tot_s:5.1f}% samples {100 * g['e'] / tot_e:5.1f}% inst  n={g['n']:4d}  from {g['start']}")
        print("      stalls:", ", ".join(f"{k.replace('stall_', '')}={100 * v / tot_s:.1f}%" for k, v in st))
        print("      ops:   ", ", ".join(f"{k}={100 * v / tot_e:.1f}%" for k, v in ops))


if __name__ == "__main__":
    main()
