#!/usr/bin/env python3
"""Compare two measurement sets (dirs of bench JSON lines, e.g. profiles/r01_final vs
gpurun_out/final): per line and kernel, the change of frac_of_peak; flags drops > 3%."""
import glob
import json
import os
import sys

old_d, new_d = sys.argv[1], sys.argv[2]
bad = 0
for f in sorted(glob.glob(os.path.join(new_d, "*.json"))):
    name = os.path.basename(f)
    g = os.path.join(old_d, name)
    if not os.path.exists(g):
        continue
    try:
        a, b = json.load(open(g)), json.load(open(f))
    except Exception:
        continue
    ka, kb = a.get("kernels") or {}, b.get("kernels") or {}
    pairs = [(k, ka[k].get("frac_of_peak"), kb[k].get("frac_of_peak")) for k in kb if k in ka]
    if not pairs and "roofline" in a and "roofline" in b:
        pairs = [("roofline", a["roofline"].get("frac"), b["roofline"].get("frac"))]
    for k, x, y in pairs:
        if x is None or y is None:
            continue
        d = (y - x) / x
        flag = "  <-- DROP" if d < -0.03 else ("  (up)" if d > 0.03 else "")
        bad += d < -0.03
        print(f"{name[:-5]:28s} {k:16s} {x:.3f} -> {y:.3f} ({d:+.1%}){flag}")
print(f"{bad} drop(s) > 3%")
