"""Markdown table of the per-config bench lines under profiles/ (tools/, documentation).

    python tools/results_table.py r02"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag = sys.argv[1] if len(sys.argv) > 1 else "r02"
print("| cfg | A-matvecs/solve (cycles) | time to p eigenpairs | matvecs/s | e2e matvecs/s | dominant kernel: algorithmic GB/s (frac) "
      "| same, device-format bytes | inner step algorithmic GB/s (frac) | inner step device-format (frac) | SM MHz (reasons) |")
print("|---|---|---|---|---|---|---|---|---|---|")
for c in ("C1", "C2", "C3", "C4", "C5"):
    f = os.path.join(ROOT, "profiles", f"{tag}_bench_{c}.json")
    if not os.path.exists(f):
        continue
    d = json.load(open(f))
    r, s = d["roofline"], d["solve"]
    df = r.get("device_format") or {}
    dfi = df.get("inner_step") or {}
    e = d.get("e2e") or {}
    kern = r["kernel"].split(": ")[-1]
    print(f"| {c} n={d['config']['n']:,} | {s['a_matvecs_per_solve']:,} ({s['cycles']}) | {d['ms_per_step']:.1f} ms | {d['value']:,.1f} | "
          f"{e.get('value', float('nan')):,.1f} | `{kern}` {r['achieved']:,.0f} ({r['frac']:.3f}) | "
          f"{df.get('achieved', float('nan')):,.0f} ({df.get('frac', float('nan')):.3f}) | "
          f"{r['inner_step']['achieved']:,.0f} ({r['inner_step']['frac']:.3f}) | "
          f"{dfi.get('achieved', float('nan')):,.0f} ({dfi.get('frac', float('nan')):.3f}) | "
          f"{d['clocks']['sm_mhz']:.0f} ({', '.join(d['clocks']['reasons']) or '-'}) |")
