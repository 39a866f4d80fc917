#!/usr/bin/env python3
"""Markdown status tables from profiles/r01_final/*.json (README.md 'Status' section)."""
import json
import os
import sys

D = sys.argv[1] if len(sys.argv) > 1 else "profiles/r01_final"


def J(name):
    with open(os.path.join(D, name + ".json")) as f:
        return json.loads(f.read())


def f3(x):
    return f"{x:.3f}"


out = []
peak = J("bench_c2")["roofline"]["peak"]
out.append(f"Algorithmic HBM GB/s of the kernel (CUDA events, mean of 10 steps) and fraction of the measured "
           f"{peak:.0f} GB/s copy bandwidth (`MEASURED_PEAKS.json`) / of the north-star's 8 TB/s "
           f"(`profiles/r01_final/bench_c*.json`):\n")
out.append("| Config | Op | Kernel GB/s | of measured | of 8 TB/s | User-data GB/s |")
out.append("|---|---|---|---|---|---|")
names = {1: "c1 p=5 N=4 64 KiB ×4096", 2: "c2 p=13 N=12 4 MiB ×256", 3: "c3 p=257 N=64 16 MiB ×4",
         4: "c4 p=59 N=58 8 MiB ×64 (odd stripes sparse)", 5: "c5 p=61 N=60 32 MiB ×16"}
ops = {1: {"encode": "encode", "recover": "recover (all 15 pairs)"},
       2: {"encode": "encode", "recover": "recover (all 91 pairs, mixed classes)"},
       3: {"encode": "encode"}, 4: {"encode": "encode", "recover": "DD recover"},
       5: {"recover": "mixed-class recover"}}
for c in (2, 1, 3, 4, 5):
    d = J(f"bench_c{c}")
    first = True
    for k, label in ops[c].items():
        v = d["kernels"][k]
        out.append(f"| {names[c] if first else 'c%d' % c} | {label} | {v['achieved_GBps']:.0f} | {f3(v['frac_of_peak'])} | "
                   f"{f3(v['frac_of_8TBps'])} | {v['user_GBps']:.0f} |")
        first = False
b = J("bench_default")
e = b["e2e"]
cb = b["cpu_baseline"]
out.append("")
out.append(f"Bench line (c2, default, `profiles/r01_final/bench_default.json`): **{b['value']:.0f} GB/s** of user data "
           f"per step (encode + recovery), roofline frac {b['roofline']['frac']:.3f} ({b['roofline']['kernel']}); "
           f"e2e through the host-buffer API {e['value']:.1f} GB/s, PCIe-bound at {e['roofline']['frac']:.3f} of the "
           f"live-probed H2D rate ({e['roofline']['peak']} GB/s); the CPU oracle {cb['value']:.2f} GB/s on "
           f"{cb['cores']} host threads.")
out.append("")
out.append("Whole configurations (`bench.py --config K --full`: every stripe, streamed through one resident wave "
           "buffer; lost strips poisoned before recovery, every stripe proven by a scrub afterwards; 1 GPU):\n")
out.append("| Config | Stripes | Encode GB/s (of measured) | Recover GB/s (of measured) | User GB/s (all ops) | Scrub-bad words |")
out.append("|---|---|---|---|---|---|")
for c, lab in ((4, "c4 p=59 N=58 8 MiB, odd stripes sparse"), (5, "c5 p=61 N=60 32 MiB, mixed classes"),
               (2, "c2 p=13 N=12 4 MiB")):
    d = J(f"full_c{c}")
    k = d["kernels"]
    enc = f"{k['encode']['achieved_GBps_per_gpu']:.0f} ({k['encode']['frac_of_peak']:.2f})" if "encode" in k else "—"
    rec = f"{k['recover']['achieved_GBps_per_gpu']:.0f} ({k['recover']['frac_of_peak']:.2f})"
    out.append(f"| {lab} | {d['verified']['stripes']} | {enc} | {rec} | {d['value']:.0f} | "
               f"{d['verified']['scrub_bad_words_after_recovery']} |")
s = J("sweep_c3")
fr = [p["frac_of_peak"] for p in s["sweep"]]
ag = [p["achieved_GBps"] for p in s["sweep"]]
us = [p["user_GBps"] for p in s["sweep"]]
out.append("")
out.append(f"c3 strip-size sweep (`bench.py --config 3 --sweep`, p=257 N=64, encode, ≥ 4 GiB per point): every point "
           f"from 64 KiB to 16 MiB runs at {min(ag):.0f}–{max(ag):.0f} GB/s of algorithmic traffic "
           f"({min(fr):.3f}–{max(fr):.3f} of the measured copy rate), {min(us):.0f}–{max(us):.0f} GB/s of user data, "
           f"all oracle-checked.")
try:
    c1l = J("c1_literal")
    out.append("")
    out.append(f"Config 1 taken literally (`bench.py --config 1 --full`: ONE 64 KiB stripe, encode, then each of the 15 "
               f"pairs rebuilt and compared; L2-resident, so a latency figure): encode {c1l['encode_us']:.1f} µs, "
               f"recovery {c1l['value']:.1f} µs per call on average (from Python, host path included)"
               + (f", {c1l['cuda_graph']['us_per_launch']:.1f} µs per launch on the device when the 16 calls are "
                  f"replayed from a CUDA graph" if (c1l.get('cuda_graph') or {}).get('us_per_launch') else "")
               + "; every pair bit-exact, parity = oracle.")
except FileNotFoundError:
    pass
try:
    with open(os.path.join(os.path.dirname(D.rstrip("/")), "r01_primes.json")) as f:
        pr = json.load(f)
    fp = pr["fast_path"]
    enc = [v["encode"]["frac"] for v in fp.values()]
    rec = [v["recover"]["frac"] for v in fp.values()]
    gen = [v[k]["frac"] for v in pr["generic_path"].values() for k in ("encode", "recover")]
    out.append("")
    out.append(f"Other primes (`profiles/r01_primes.json`, c2 shape N = 12, 4 MiB × 256): the {len(fp)} primes added to the "
               f"fast path this round (every prime whose period lcm(p−1, 32) fits 32 lanes) encode at "
               f"{min(enc):.2f}–{max(enc):.2f} and recover at {min(rec):.2f}–{max(rec):.2f} of the copy rate; "
               f"the other {len(pr['generic_path'])} primes (generic kernel) run at {min(gen):.2f}–{max(gen):.2f}.")
except FileNotFoundError:
    pass
out.append("\n### NEXT-1 (update / scrub)\n")
out.append("| Config | Update kernel GB/s (of measured) | Scrub kernel GB/s (of measured) |")
out.append("|---|---|---|")
for c in (1, 2, 3, 4, 5):
    u, sc = J(f"next1_update_c{c}"), J(f"next1_scrub_c{c}")
    out.append(f"| c{c} | {u['roofline']['achieved']:.0f} ({f3(u['roofline']['frac'])}) | "
               f"{sc['roofline']['achieved']:.0f} ({f3(sc['roofline']['frac'])}) |")
out.append("\n### NEXT-2 (extended Q-parity)\n")
out.append("| Workload | Encode GB/s (of measured) | Recover GB/s (of measured) |")
out.append("|---|---|---|")
for n, lab in (("next2_c2_N25", "p=13 N=25, 4 MiB (all 351 pairs, mixed)"), ("next2_c2_N17", "p=13 N=17, 4 MiB"),
               ("next2_c4_N115", "p=59 N=115, 8 MiB (DD)"), ("next2_c5_N121", "p=61 N=121, 32 MiB (mixed)"),
               ("next2_c3_N300", "p=257 N=300, 16 MiB"), ("next2_c1_N9", "p=5 N=9, 64 KiB")):
    d = J(n)
    k = d["kernels"]
    enc = f"{k['encode']['achieved_GBps']:.0f} ({f3(k['encode']['frac_of_peak'])})" if "encode" in k else "—"
    rec = f"{k['recover']['achieved_GBps']:.0f} ({f3(k['recover']['frac_of_peak'])})" if "recover" in k else "—"
    out.append(f"| {lab} | {enc} | {rec} |")
out.append("\n### NEXT-3 (Z_p vs the paper's GF(256) RS comparison system, same workload and pipeline)\n")
out.append("| Workload | Z_p encode | RS encode | Z_p recover | RS recover |")
out.append("|---|---|---|---|---|")
for (a, b_, lab) in (("next3_c2_N16_zp_p17", "next3_c2_N16_rs_p17", "N=16, 4 MiB ×192 (the paper's Z_17 vs RS)"),
                     ("next3_c2_N12_zp", "next3_c2_N12_rs", "N=12, 4 MiB ×256 (c2, p=13)"),
                     ("next3_c4_N58_zp", "next3_c4_N58_rs", "N=58, 8 MiB ×64 (c4, p=59; DD)"),
                     ("next3_c5_N60_zp", "next3_c5_N60_rs", "N=60, 32 MiB ×16 (c5, p=61; mixed)")):
    z, r = J(a)["kernels"], J(b_)["kernels"]
    ze = f"{z['encode']['achieved_GBps']:.0f}" if "encode" in z else "—"
    re_ = f"{r['encode']['achieved_GBps']:.0f}" if "encode" in r else "—"
    out.append(f"| {lab} | {ze} | {re_} | {z['recover']['achieved_GBps']:.0f} | {r['recover']['achieved_GBps']:.0f} |")
out.append("\n### NEXT-4 (cross-GPU stripe layout, G ranks emulated on one GPU: HBM side only)\n")
out.append("| Workload | G | Partial GB/s enc / rec (of measured) | Combine+solve GB/s enc / rec (of measured) |")
out.append("|---|---|---|---|")
for c, g, lab in ((4, 8, "c4 p=59 N=58 8 MiB ×64 (DD)"), (5, 8, "c5 p=61 N=60 32 MiB ×16"), (2, 4, "c2 p=13 N=12 4 MiB ×256"),
                  (2, 8, "c2"), (1, 4, "c1 p=5 N=4 64 KiB ×4096"), (3, 8, "c3 p=257 N=64 16 MiB ×4")):
    k = J(f"next4_xgpu_c{c}_G{g}")["kernels"]
    out.append(f"| {lab} | {g} | {k['encode_partial']['achieved_GBps']:.0f} / {k['recover_partial']['achieved_GBps']:.0f} "
               f"({k['encode_partial']['frac_of_peak']:.2f} / {k['recover_partial']['frac_of_peak']:.2f}) | "
               f"{k['encode_combine']['achieved_GBps']:.0f} / {k['recover_combine']['achieved_GBps']:.0f} "
               f"({k['encode_combine']['frac_of_peak']:.2f} / {k['recover_combine']['frac_of_peak']:.2f}) |")
print("\n".join(out))
