"""One markdown row per bench JSON line: python scripts/summarize_bench.py profiles/r02*_bench_*.json"""
import json
import sys

print("| file | workload | events/s (device) | µs/step | e2e events/s | dominant op (alone) | frac | k_prep HBM frac | clocks |")
print("|---|---|---|---|---|---|---|---|---|")
for f in sys.argv[1:]:
    try:
        d = json.load(open(f))
    except Exception as e:  # noqa: BLE001
        print(f"| {f} | unreadable: {e} |")
        continue
    r = d.get("roofline") or {}
    g = d.get("roofline_gather") or {}
    c = d.get("clocks") or {}
    e2e = (d.get("e2e") or {}).get("value")
    print(f"| {f.split('/')[-1]} | {d['config'].get('workload')} ({d['config'].get('gru')}) | {d['value'] / 1e6:.2f} M | "
          f"{d['ms_per_step'] * 1e3:.2f} | {e2e / 1e6 if e2e else float('nan'):.2f} M | "
          f"{r.get('kernel', '')[:24]} {r.get('launch_ms_mean', 0) * 1e3:.1f} µs | {r.get('frac', 0):.3f} | "
          f"{g.get('frac', float('nan')):.3f} | {c.get('sm_mhz')} MHz {c.get('reasons')} |")
