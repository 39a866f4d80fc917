#!/usr/bin/env python3
"""Profiling driver: for each requested config, one untimed warm-up pass then one encode and
one recovery launch (bench.py's pair schedules) -- small enough to run under ncu --set full.
usage: prof_configs.py 1 3 4 5"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
from paper_cs_0611109_b200 import raid6c as R  # noqa: E402

SIZES = {1: 4096, 2: 64, 3: 4, 4: 16, 5: 4}
for cfg in [int(x) for x in sys.argv[1:]]:
    c = bench.CONFIGS[cfg]
    p, N, nbytes, S = c["p"], c["N"], c["nbytes"], SIZES[cfg]
    pb = R.parity_bytes(p, nbytes)
    ss, ps = R.aligned_stride(nbytes), R.aligned_stride(pb)
    data = torch.empty((S, N, ss), dtype=torch.uint8, device="cuda")
    par = torch.zeros((S, 2, ps), dtype=torch.uint8, device="cuda")
    R.fill(data, ss, N * ss, nbytes, N, S, 0, cfg, 0, 0, c["sparse"])
    plan = R.Plan(p, N, nbytes)
    a = (int(data.data_ptr()), ss, N * ss, int(par.data_ptr()), int(par.data_ptr()) + ps, 2 * ps, S)
    pairs = torch.tensor(bench.pair_schedule(cfg, N, S, 0, 0), dtype=torch.int32, device="cuda")
    for rep in range(2):
        plan.encode_strided(*a)
        if c["ops"] != "enc":
            plan.recover_strided(*a, pairs)
    plan.sync()
    print(f"c{cfg} done", flush=True)
    del data, par, plan
    torch.cuda.empty_cache()
