#!/usr/bin/env python3
"""HBM layout probe (c2 shape): encode and the bench's mixed-pair recovery (and one same-pair DD
launch) under different strip / stripe strides -- does skewing the strips' start addresses
(so that the N rows a CTA streams at one tile offset are not all congruent modulo a large power
of two) change the DRAM rate?  CUDA events per launch, medians.
usage: layout_probe.py [reps] [config]"""
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
from paper_cs_0611109_b200 import raid6c as R  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
cfg = int(sys.argv[2]) if len(sys.argv) > 2 else 2
c = bench.CONFIGS[cfg]
p, N, nbytes, S = c["p"], c["N"], c["nbytes"], c["stripes"]
pb = R.parity_bytes(p, nbytes)
plan = R.Plan(p, N, nbytes)
alg = S * (N * nbytes + 2 * pb)
mixed = torch.tensor(bench.pair_schedule(cfg, N, S, 0, 0), dtype=torch.int32, device="cuda")
# (name, data strip stride, extra bytes per stripe, parity strip stride)
base_d, base_p = R.aligned_stride(nbytes), R.aligned_stride(pb)
LAYOUTS = [("bench", base_d, 0, base_p),
           ("d+256", base_d + 256, 0, base_p),
           ("d+1K", base_d + 1024, 0, base_p),
           ("d+4K", base_d + 4096, 0, base_p),
           ("d+16K", base_d + 16384, 0, base_p),
           ("d+1K,s+32K", base_d + 1024, 32768, base_p + 1024),
           ("bench", base_d, 0, base_p)]
for name, ss, sx, ps in LAYOUTS:
    dst = N * ss + sx
    data = torch.empty(S * dst, dtype=torch.uint8, device="cuda")
    par = torch.zeros((S, 2, ps), dtype=torch.uint8, device="cuda")
    R.fill(data, ss, dst, nbytes, N, S, 0, cfg, 0, 0, c["sparse"])
    a = (int(data.data_ptr()), ss, dst, int(par.data_ptr()), int(par.data_ptr()) + ps, 2 * ps, S)
    plan.encode_strided(*a)
    ev = []
    for r in range(reps):
        for what in ("encode", "mixed", "DD"):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            if what == "encode":
                plan.encode_strided(*a)
            elif c["ops"] != "enc":
                plan.recover_strided(*a, mixed if what == "mixed" else [(3, 7)])
            e1.record()
            ev.append((what, e0, e1))
    torch.cuda.synchronize()
    res = {}
    for what, e0, e1 in ev:
        res.setdefault(what, []).append(e0.elapsed_time(e1))
    print(f"c{cfg} {name:12s} ss={ss} stripe={dst} ps={ps}",
          {k: (round(statistics.median(v), 4), round(alg / (statistics.median(v) / 1e3) / 1e9, 1))
           for k, v in res.items() if statistics.median(v) > 0.01}, flush=True)
    del data, par
    torch.cuda.empty_cache()
