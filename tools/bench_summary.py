"""One-line summaries of bench JSON logs: python tools/bench_summary.py gpurun_out/bench_*.log"""
import json
import sys

for f in sys.argv[1:]:
    try:
        lines = [x for x in open(f) if x.startswith("{")]
    except OSError:
        continue
    if not lines:
        print(f, "NO JSON:", open(f).read()[-1500:])
        continue
    j = json.loads(lines[-1])
    ks = {k: round(v, 3) for k, v in (j.get("kernel_ms_per_step") or {}).items() if v}
    roof = j.get("roofline") or {}
    print(f"{f}: {j['value'] / 1e6:.1f} M{j['unit']} {j['ms_per_step']:.3f} ms/step "
          f"roof={roof.get('frac')} e2e={(j.get('e2e') or {}).get('value')} {ks}")
