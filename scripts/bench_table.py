"""Markdown table of the bench lines in profiles/<prefix>_bench_*.json
(DESIGN.md section 8).

    python scripts/bench_table.py r02
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
prefix = sys.argv[1] if len(sys.argv) > 1 else "r02"
rows = []
for name in ("c1", "c2", "c3a", "c3b", "c4", "c5"):
    path = os.path.join(ROOT, "profiles", f"{prefix}_bench_{name}.json")
    if not os.path.exists(path):
        continue
    d = json.loads(open(path).read().strip().splitlines()[-1])
    r = d["roofline"]
    e = d.get("e2e", {})
    cb = d.get("cpu_baseline", {})
    us = d["ms_per_step"] * 1e3
    rows.append(
        f"| {d['config']['workload']} | {d['config']['engine']} | {us:,.1f} | {d['value']:.3g} | {d['iterations_per_s']:.4g} | "
        f"{e.get('value', float('nan')):.3g} | {r['kernel']} {r['kernel_ms_avg'] * 1e3:,.1f} µs ({100 * r['kernel_share_of_step']:.0f}%) | "
        f"{r['bound']} {100 * r['frac']:.2f}% of {r['peak']:.4g} {r['unit']} | {cb.get('value', float('nan')):.3g} |")
print("| config | engine | µs / iteration | evals/s | iterations/s | e2e evals/s | dominant kernel (avg per launch, share of step) | roofline | CPU oracle evals/s (1 core) |")
print("|---|---|---|---|---|---|---|---|---|")
print("\n".join(rows))
