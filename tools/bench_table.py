#!/usr/bin/env python
"""Markdown table of the bench lines written by tools/bench_all.sh."""
import glob
import json
import os
import sys

rows = []
for f in sorted(glob.glob(os.path.join(sys.argv[1], "*.json"))):
    try:
        d = json.load(open(f))
    except Exception:
        continue
    name = os.path.basename(f)[:-5]
    if "ms_per_scan" in d:
        rows.append((name, f"{d['ms_per_scan']:.3f} ms / scan", f"{d['value']:.3g} entries/s", "", "", ""))
        continue
    rf = d.get("roofline") or {}
    e2e = d.get("e2e") or {}
    rows.append((name, f"{d['ms_per_step']:.4f} ms / step ({d['config']['poses']} poses)",
                 f"{d['value']:.3g} poses/s", f"{d.get('atom_evals_per_s', 0):.3g}",
                 f"{rf.get('bound', '-')} {rf.get('frac') or 0:.3f} / {rf.get('l2_literal_frac') or 0:.3f}",
                 f"{e2e.get('value', 0):.3g}" if e2e else "-"))
print("| run | time | throughput | atom-evals/s | roofline: bound, frac (serving level / L2-literal) | e2e poses/s |")
print("|---|---|---|---|---|---|")
for r in rows:
    print("| " + " | ".join(r) + " |")
