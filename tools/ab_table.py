#!/usr/bin/env python3
"""Summarise A/B bench lines: python tools/ab_table.py gpurun_out/g3/*.json"""
import json
import statistics as st
import sys

for f in sys.argv[1:]:
    ls = [x for x in open(f) if x.startswith("{")]
    if not ls:
        print(f, "NO LINE")
        continue
    d = json.loads(ls[-1])
    k = d["kernels"]
    sm = d.get("step_ms", {})
    ext = {kk: (round(min(v), 4), round(st.median(v), 4), round(max(v), 4)) for kk, v in sm.items() if len(v) > 1}
    print(f.split("/")[-1], {kk: (v["avg_ms"], v["frac_of_peak"]) for kk, v in k.items()}, "min/med/max", ext,
          "clk", d["clocks"].get("sm_min_mhz"), d["clocks"].get("power_w_max"), d["clocks"]["reasons"],
          "ok", (d.get("verified") or {}).get("ok"))
