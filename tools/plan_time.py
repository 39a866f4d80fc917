#!/usr/bin/env python3
"""Plan-creation time (the extended code builds its per-pair multiplier table) for a few (p, N)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_cs_0611109_b200 import raid6c as R  # noqa: E402

R.Plan(13, 12, 4096).close()
for p, N in [(13, 12), (13, 25), (59, 115), (61, 121), (257, 300), (257, 513), (11, 21)]:
    t0 = time.perf_counter()
    pl = R.Plan(p, N, 1 << 20)
    t = time.perf_counter() - t0
    pl.close()
    print(f"p={p} N={N}: plan_create {t * 1e3:.1f} ms")
