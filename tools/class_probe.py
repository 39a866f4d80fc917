#!/usr/bin/env python3
"""Per-class recovery probe (c2 shape): the same pair in every stripe, one class at a time,
under several parity layouts, CUDA events per launch (no poisoning: intact strips are rebuilt in
place, which is what the timed default bench does).  Diagnoses why DP / DQ / PQ launches of the
literal config 2 run slower than DD ones.
usage: class_probe.py [reps]"""
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_cs_0611109_b200 import raid6c as R  # noqa: E402

p, N, nbytes, S = 13, 12, 4 << 20, 256
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
pb = R.parity_bytes(p, nbytes)
ss = R.aligned_stride(nbytes)
data = torch.empty((S, N, ss), dtype=torch.uint8, device="cuda")
R.fill(data, ss, N * ss, nbytes, N, S, 0, 2, 0, 0, 0)
plan = R.Plan(p, N, nbytes)
PAIRS = {"DD": (3, 7), "DP": (3, N), "DQ": (3, N + 1), "PQ": (N, N + 1), "DD01": (0, 1)}
# parity layouts: interleaved [S, 2, ps] with ps = 256-aligned (bench) or 64 KiB-aligned, and two
# separate [S, ps] planes (P plane, Q plane)
layouts = {"inter256": (R.aligned_stride(pb), True), "inter64k": (R.aligned_stride(pb, 65536), True),
           "planes256": (R.aligned_stride(pb), False)}
alg = S * (N * nbytes + 2 * pb)
for name, (ps, inter) in layouts.items():
    if inter:
        par = torch.zeros((S, 2, ps), dtype=torch.uint8, device="cuda")
        Pp, Qp, pst = int(par.data_ptr()), int(par.data_ptr()) + ps, 2 * ps
    else:
        par = torch.zeros((2, S, ps), dtype=torch.uint8, device="cuda")
        Pp, Qp, pst = int(par[0].data_ptr()), int(par[1].data_ptr()), ps
    a = (int(data.data_ptr()), ss, N * ss, Pp, Qp, pst, S)
    plan.encode_strided(*a)
    plan.encode_strided(*a)
    res = {}
    ev = []
    for r in range(reps):
        for cls, pr in PAIRS.items():
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            plan.recover_strided(*a, [pr])
            e1.record()
            ev.append((cls, e0, e1))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        plan.encode_strided(*a)
        e1.record()
        ev.append(("encode", e0, e1))
    torch.cuda.synchronize()
    for cls, e0, e1 in ev:
        res.setdefault(cls, []).append(e0.elapsed_time(e1))
    print(name, {k: (round(statistics.median(v), 4), round(alg / (statistics.median(v) / 1e3) / 1e9, 1))
                 for k, v in res.items()}, flush=True)
    del par
    torch.cuda.empty_cache()
