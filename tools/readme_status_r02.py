#!/usr/bin/env python3
"""Markdown status tables from profiles/r02_final/*.json (README.md 'Status' section, round 2)."""
import json
import os
import sys

D = sys.argv[1] if len(sys.argv) > 1 else "profiles/r02_final"


def J(name):
    with open(os.path.join(D, name + ".json")) as f:
        t = f.read().strip()
    return json.loads(t) if t else None


def f3(x):
    return f"{x:.3f}"


out = []
peak = J("bench_c2")["roofline"]["peak"]
out.append(f"Algorithmic HBM GB/s of the kernel (CUDA events, mean of 10 steps) and fraction of the measured "
           f"{peak:.0f} GB/s copy bandwidth (`MEASURED_PEAKS.json`) / of the north-star's 8 TB/s "
           f"(`{D}/bench_c*.json`; every line verified: round trip, poisoned re-recovery, fresh encode):\n")
out.append("| Config | Op | Kernel GB/s | of measured | of 8 TB/s | User-data GB/s |")
out.append("|---|---|---|---|---|---|")
names = {1: "c1 p=5 N=4 64 KiB ×4096", 2: "c2 p=13 N=12 4 MiB ×256", 3: "c3 p=257 N=64 16 MiB ×4",
         4: "c4 p=59 N=58 8 MiB ×64 (odd stripes sparse)", 5: "c5 p=61 N=60 32 MiB ×16"}
ops = {1: {"encode": "encode", "recover": "recover (all 15 pairs)"},
       2: {"encode": "encode", "recover": "recover (pairs cycle all 91, mixed classes)"},
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
v = b["verified"]
out.append("")
out.append(f"Bench line (c2, default, `{D}/bench_default.json`): **{b['value']:.0f} GB/s** of user data "
           f"per step (encode + recovery), roofline frac {b['roofline']['frac']:.3f} ({b['roofline']['kernel']}); "
           f"e2e through the host-buffer API {e['value']:.1f} GB/s, PCIe-bound at {e['roofline']['frac']:.3f} of the "
           f"live-probed H2D rate ({e['roofline']['peak']} GB/s); verified: {v['mismatched_bytes']} bytes off after the "
           f"timed steps, {v['poisoned_recovery']['mismatched_bytes']} after re-running the last recovery over "
           f"{v['poisoned_recovery']['poisoned_bytes'] / 1e9:.1f} GB of poisoned lost strips, "
           f"{v['oracle_digest_stripes']}/{v['oracle_digest_sampled']} sampled stripes equal to the oracle at full size; "
           f"the oracle (cpu_baseline) {cb['value']:.2f} GB/s on {cb['cores']} host threads.")
d2 = J("bench_default_2")
if d2:
    out.append(f"The driver's shape (`--steps 20 --warmup 5`, `{D}/bench_default_2.json`): {d2['value']:.0f} GB/s, "
               f"recovery {d2['kernels']['recover']['frac_of_peak']:.3f} / encode {d2['kernels']['encode']['frac_of_peak']:.3f} "
               f"of the copy rate.")
fc2 = J("full_c2")
if fc2:
    out.append("")
    out.append("Config 2 as written (`bench.py --config 2 --full`: 256 stripes, encode, then each of the 91 pairs "
               "recovered in every stripe, one launch per pair; lost strips poisoned first, every launch scrub-proven, "
               "every rebuilt strip digest-checked; the oracle encodes all 256 stripes and rebuilds every pair once):\n")
    out.append("| Class | Pairs | ms per launch | Kernel GB/s | of measured | User GB/s |")
    out.append("|---|---|---|---|---|---|")
    k = fc2["kernels"]
    out.append(f"| encode | — | {k['encode']['ms']:.3f} | {k['encode']['achieved_GBps']:.0f} | {f3(k['encode']['frac_of_peak'])} | "
               f"{fc2['config']['stripes_total'] * 12 * 4194304 / (k['encode']['ms'] / 1e3) / 1e9:.0f} |")
    for cls, r in k["recover_by_class"].items():
        out.append(f"| {cls} | {r['pairs']} | {r['ms_per_launch']:.3f} | {r['achieved_GBps']:.0f} | {f3(r['frac_of_peak'])} | "
                   f"{r['user_GBps']:.0f} |")
    vv = fc2["verified"]
    out.append(f"\nWhole run {fc2['value']:.0f} GB/s of user data; scrub-bad words {vv['scrub_bad_words_after_recovery']}, "
               f"rebuilt-strip digest mismatches {vv['rebuilt_strip_digest_mismatches']} of {vv['rebuilt_strips_checked']}, "
               f"oracle encode digests {vv.get('oracle_encode_digest_stripes')}/{vv.get('oracle_encode_sampled')} stripes, "
               f"oracle pair rebuilds {vv.get('oracle_pair_digests_ok')}/{vv.get('oracle_pair_digests')} strips.")
out.append("")
out.append("Whole configurations (`bench.py --config K --full`: every stripe, streamed through one resident wave "
           "buffer; lost strips poisoned before recovery, every stripe proven by a scrub afterwards and digested; "
           "64 stripes spread over the run checked against the oracle at full size; 1 GPU):\n")
out.append("| Config | Stripes | Encode GB/s (of measured) | Recover GB/s (of measured) | User GB/s (all ops) | Scrub-bad words | Oracle digests |")
out.append("|---|---|---|---|---|---|---|")
for c, lab in ((4, "c4 p=59 N=58 8 MiB, odd stripes sparse"), (5, "c5 p=61 N=60 32 MiB, mixed classes")):
    d = J(f"full_c{c}")
    k = d["kernels"]
    enc = f"{k['encode']['achieved_GBps_per_gpu']:.0f} ({k['encode']['frac_of_peak']:.3f})" if "encode" in k else "—"
    rec = f"{k['recover']['achieved_GBps_per_gpu']:.0f} ({k['recover']['frac_of_peak']:.3f})"
    vv = d["verified"]
    cls = ", ".join(f"{kk} {x['ok']}/{x['sampled']}" for kk, x in vv.get("oracle_digest_by_class", {}).items())
    out.append(f"| {lab} | {vv['stripes']} | {enc} | {rec} | {d['value']:.0f} | {vv['scrub_bad_words_after_recovery']} | "
               f"{vv.get('oracle_digest_stripes')}/{vv.get('oracle_digest_sampled')} ({cls}) |")
s = J("sweep_c3")
if s:
    fr = [p["frac_of_peak"] for p in s["sweep"]]
    ag = [p["achieved_GBps"] for p in s["sweep"]]
    us = [p["user_GBps"] for p in s["sweep"]]
    out.append("")
    out.append(f"c3 strip-size sweep (`bench.py --config 3 --sweep`, p=257 N=64, encode, ≥ 4 GiB per point): every point "
               f"from 64 KiB to 16 MiB runs at {min(ag):.0f}–{max(ag):.0f} GB/s of algorithmic traffic "
               f"({min(fr):.3f}–{max(fr):.3f} of the measured copy rate), {min(us):.0f}–{max(us):.0f} GB/s of user data.")
c1l = J("c1_literal")
if c1l:
    out.append("")
    out.append(f"Config 1 taken literally (`bench.py --config 1 --full`: ONE 64 KiB stripe, encode, then each of the 15 "
               f"pairs rebuilt and compared; L2-resident, so a latency figure): encode {c1l['encode_us']:.1f} µs, "
               f"recovery {c1l['value']:.1f} µs per call on average (from Python, host path included)"
               + (f", {c1l['cuda_graph']['us_per_launch']:.1f} µs per launch on the device when the 16 calls are "
                  f"replayed from a CUDA graph" if (c1l.get('cuda_graph') or {}).get('us_per_launch') else "")
               + "; every pair bit-exact, parity = oracle.")
g2 = J("gpus2_gloo")
if g2:
    out.append("")
    out.append(f"Multi-rank path (`bench.py --gpus 2 --dist-backend gloo`, self-launched, both ranks on the one GPU of a "
               f"gpurun box, so not a scaling number): n_gpus {g2['n_gpus']}, {g2['ranks']['ranks_up']} ranks up, "
               f"per-rank ms {g2['per_rank_ms']}, verified {g2['verified']['ok']} "
               f"({g2['verified']['oracle_digest_stripes']}/{g2['verified']['oracle_digest_sampled']} oracle stripes).")
x2 = J("next4_xgpu_dist2_gloo")
if x2:
    vv = x2["verified"]
    out.append("")
    out.append(f"NEXT-4 over the same self-launched path (`bench.py --gpus 2 --dist-backend gloo --xgpu 2`, two ranks "
               f"sharing the gpurun box's GPU through CUDA IPC arenas, so not an NVLink number): {x2['ranks']['ranks_up']} "
               f"ranks up, every rank verified (round trip {vv['mismatched_strip_digests']} strip digests off, poisoned "
               f"recovery through the peer slots {vv['poisoned_recovery']['mismatched_strip_digests']} off over "
               f"{vv['poisoned_recovery']['poisoned_bytes'] / 1e6:.0f} MB, fresh encode "
               f"{vv['fresh_encode_mismatched_strip_digests']} off), oracle sample "
               f"{vv.get('oracle_digest_stripes')}/{vv.get('oracle_digest_sampled')}.")
pp = os.path.join(os.path.dirname(D.rstrip("/")), "r02_primes.json")
if os.path.exists(pp):
    with open(pp) as fh:
        P = json.load(fh)["primes"]
    fast = {int(p): v for p, v in P.items() if v and v["fast_path"]}
    gen = {int(p): v for p, v in P.items() if v and not v["fast_path"]}
    rng = lambda d, k: (min(v[k]["frac"] for v in d.values()), max(v[k]["frac"] for v in d.values()))  # noqa: E731
    fe, fr, ge, gr = rng(fast, "encode"), rng(fast, "recover"), rng(gen, "encode"), rng(gen, "recover")
    out.append("")
    out.append(f"Every other prime (`profiles/r02_primes.json`, c2 shape N = 12, 4 MiB × 256, oracle-sampled lines; "
               f"fraction of the measured copy rate): the {len(fast)} fast-path primes encode at {fe[0]:.2f}–{fe[1]:.2f} "
               f"and recover at {fr[0]:.2f}–{fr[1]:.2f}; the {len(gen)} large-period primes on the TMA-staged generic "
               f"kernel encode at {ge[0]:.2f}–{ge[1]:.2f} and recover at {gr[0]:.2f}–{gr[1]:.2f} (round 1: 0.27–0.40 / "
               f"0.22–0.32).")
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
