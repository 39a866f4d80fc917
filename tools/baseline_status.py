#!/usr/bin/env python3
"""Regenerate BASELINE.md section 4 ("Measured results") from profiles/r01_final/*.json."""
import json

D = "profiles/r01_final"


def J(n):
    return json.load(open(f"{D}/{n}.json"))


b = J("bench_default")
peak = b["roofline"]["peak"]
rows = []


def add(cfg, op, d, k, oracle=""):
    v = d["kernels"][k]
    rows.append(f"| {cfg} | {op} | 1 | {v['user_GBps']:.0f} | {v['achieved_GBps']:.0f} | {100 * v['frac_of_8TBps']:.1f} | "
                f"{100 * v['frac_of_peak']:.1f} | yes | {oracle} |")


add("c1 (batched 4096 stripes)", "encode", J("bench_c1"), "encode")
add("c1", "recover (15 pairs)", J("bench_c1"), "recover")
add("c2", "encode", J("bench_c2"), "encode", f"{b['cpu_baseline']['value']:.2f} ({b['cpu_baseline']['cores']})")
add("c2", "recover (91 pairs)", J("bench_c2"), "recover")
add("c3 (16 MiB)", "encode", J("bench_c3"), "encode")
add("c4 (wave of 64)", "encode", J("bench_c4"), "encode")
add("c4", "DD recover", J("bench_c4"), "recover")
add("c5 (wave of 16)", "mixed recover", J("bench_c5"), "recover")
f4, f5 = J("full_c4"), J("full_c5")
tbl = "\n".join(rows)
sec = f"""## 4. Measured results

Round 1, final build, one B200 (`profiles/r01_final/`; SM clock 1965 MHz during the timed regions,
no throttle reasons except occasional `sw_power_cap`). Algorithmic bytes per §8(d).1; "of
measured" = ÷ {peak:.1f} GB/s (`MEASURED_PEAKS.json`, rewritten per pod by the driver). ncu DRAM
bytes per launch equal the algorithmic bytes (c2: traffic/alg = 0.999 for encode and recover,
`profiles/r01_final/ncu_full_c2.txt`). Every run verified: all data and parity bytes round-trip
exactly, and sampled P/Q segments equal the CPU oracle.

| Config | Op | GPUs | User GB/s | Algorithmic GB/s | % of 8 TB/s | % of measured | Bit-exact | Oracle GB/s (threads) |
|---|---|---|---|---|---|---|---|---|
{tbl}

Default bench line (c2, encode + recovery per step): {b['value']:.0f} GB/s of user data.
Whole configurations (`--full`): c4's 4096 stripes (1.9 TB of user data) encode at
{f4['kernels']['encode']['achieved_GBps_per_gpu']:.0f} GB/s and DD-recover at {f4['kernels']['recover']['achieved_GBps_per_gpu']:.0f} GB/s;
c5's 1000 stripes recover (mixed classes) at {f5['kernels']['recover']['achieved_GBps_per_gpu']:.0f} GB/s; every stripe scrub-proven.
End to end through the host-buffer API: {b['e2e']['value']:.1f} GB/s of user data, {b['e2e']['roofline']['frac']:.3f} of this
GPU's PCIe H2D rate. The CPU oracle (the `--impl reference` arm): {b['cpu_baseline']['value']:.2f} GB/s on {b['cpu_baseline']['cores']} host threads.

2/4/8-GPU numbers: the driver's scaling run (weak scaling, stripe-sharded, no data-path
collective).
"""
s = open("BASELINE.md").read()
s = s[:s.index("## 4. Measured results")] + sec
open("BASELINE.md", "w").write(s)
