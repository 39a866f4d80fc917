#!/usr/bin/env python3
"""Print the key numbers of gpurun_out/final/*.json (see tools/gpu_final_all.sh)."""
import glob
import json
import os
import sys

D = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/final"
for f in sorted(glob.glob(os.path.join(D, "*.json"))):
    name = os.path.basename(f)[:-5]
    try:
        d = json.loads(open(f).read())
    except Exception as e:
        print(f"{name}: unreadable ({e})")
        continue
    line = f"{name}: value={d.get('value')} {d.get('unit', '')}"
    k = d.get("kernels") or {}
    for kn, kv in k.items():
        a = kv.get("achieved_GBps", kv.get("achieved_GBps_per_gpu"))
        line += f" | {kn} {a} ({kv.get('frac_of_peak')})"
    if "roofline" in d and not k:
        r = d["roofline"]
        line += f" | roof {r.get('achieved')} ({r.get('frac')})"
    v = d.get("verified")
    if v is not None:
        line += f" | verified {v}"
    c = d.get("clocks")
    if c:
        line += f" | sm {c.get('sm_mhz')} {c.get('reasons')}"
    if d.get("e2e"):
        line += f" | e2e {d['e2e'].get('value')} frac {d['e2e'].get('roofline', {}).get('frac')}"
    if d.get("cpu_baseline"):
        line += f" | cpu {d['cpu_baseline'].get('value')} ({d['cpu_baseline'].get('cores')} cores)"
    if d.get("sweep"):
        line += " | sweep " + ", ".join(f"{p['strip_bytes'] >> 10}K:{p['frac_of_peak']}" for p in d["sweep"])
    print(line)
