#!/usr/bin/env python3
"""Debug: config-5-like waves with poisoned lost strips; per stripe compare the rebuilt strips
with the pre-recovery snapshot and the scrub count.  usage: debug_full_c5.py [waves] [wave] [nbytes]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synthetic  # noqa: E402
from paper_cs_0611109_b200 import raid6c as R  # noqa: E402

waves = int(sys.argv[1]) if len(sys.argv) > 1 else 4
wave = int(sys.argv[2]) if len(sys.argv) > 2 else 16
nbytes = int(sys.argv[3]) if len(sys.argv) > 3 else 32 << 20
p, N = 61, 60
pb = R.parity_bytes(p, nbytes)
ss, ps = R.aligned_stride(nbytes), R.aligned_stride(pb)
data = torch.empty((wave, N, ss), dtype=torch.uint8, device="cuda")
par = torch.zeros((wave, 2, ps), dtype=torch.uint8, device="cuda")
counts = torch.zeros(wave, dtype=torch.int32, device="cuda")
plan = R.Plan(p, N, nbytes)
a = (int(data.data_ptr()), ss, N * ss, int(par.data_ptr()), int(par.data_ptr()) + ps, 2 * ps, wave)
tot_bad = 0
for w in range(waves):
    w0 = w * wave
    R.fill(data, ss, N * ss, nbytes, N, wave, 0, 5, w0, 0, 0)
    plan.encode_strided(*a)
    plan.sync()
    A_d, A_p = data.clone(), par.clone()
    pairs = [synthetic.erasure_pair(0, 5, w0 + s, N) for s in range(wave)]
    for s, (i, j) in enumerate(pairs):
        for k in (i, j):
            (data[s, k] if k < N else par[s, k - N]).fill_(0xA5)
    torch.cuda.synchronize()
    plan.recover_strided(*a, pairs)
    plan.scrub_strided(*a, counts)
    plan.sync()
    for s, (i, j) in enumerate(pairs):
        bad = int(counts[s])
        msgs = []
        for k in (i, j):
            got = data[s, k, :nbytes] if k < N else par[s, k - N, :pb]
            ref = A_d[s, k, :nbytes] if k < N else A_p[s, k - N, :pb]
            d = (got != ref).nonzero().flatten()
            if d.numel():
                msgs.append(f"strip {k}: {d.numel()} bytes differ, range [{int(d.min())},{int(d.max())}] "
                            f"first {d[:6].tolist()}")
        if bad or msgs:
            tot_bad += bad
            print(f"wave {w} stripe {w0 + s} pair ({i},{j}) {synthetic.pair_class(N, i, j)} scrub {bad}; " + "; ".join(msgs),
                  flush=True)
print("total scrub bad", tot_bad)
