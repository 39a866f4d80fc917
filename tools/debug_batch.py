#!/usr/bin/env python3
"""Debug helper: run a bench-like batch (encode + in-place recover with per-stripe pairs) and
report where results differ from the first encode.  usage: debug_batch.py p N nbytes S"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synthetic  # noqa: E402
from paper_cs_0611109_b200 import raid6c as R  # noqa: E402

p, N, nbytes, S = (int(x) for x in sys.argv[1:5])
pb = R.parity_bytes(p, nbytes)
ss, ps = R.aligned_stride(nbytes), R.aligned_stride(pb)
data = torch.empty((S, N, ss), dtype=torch.uint8, device="cuda")
par = torch.zeros((S, 2, ps), dtype=torch.uint8, device="cuda")
R.fill(data, ss, N * ss, nbytes, N, S, 0, 1, 0, 0, 0)
plan = R.Plan(p, N, nbytes)
a = (int(data.data_ptr()), ss, N * ss, int(par.data_ptr()), int(par.data_ptr()) + ps, 2 * ps, S)
plan.encode_strided(*a)
plan.sync()
A_d, A_p = data.clone(), par.clone()


def diff(tag):
    torch.cuda.synchronize()
    dd = (data[:, :, :nbytes] != A_d[:, :, :nbytes])
    dp = (par[:, :, :pb] != A_p[:, :, :pb])
    nd, np_ = int(dd.sum()), int(dp.sum())
    msg = f"{tag}: data mismatches {nd}, parity mismatches {np_}"
    if nd:
        idx = dd.nonzero()[:8].tolist()
        msg += f" first data (stripe,strip,byte) {idx}"
        strips = sorted(set((s, k) for s, k, _ in dd.nonzero().tolist()))
        msg += f" #strips {len(strips)} e.g. {strips[:6]}"
        offs = dd.nonzero()[:, 2]
        msg += f" byte range [{int(offs.min())},{int(offs.max())}]"
    if np_:
        idx = dp.nonzero()[:8].tolist()
        msg += f" first parity {idx}"
    print(msg, flush=True)
    data.copy_(A_d)
    par.copy_(A_p)
    torch.cuda.synchronize()


for rep in range(3):
    plan.encode_strided(*a)
    plan.sync()
    diff(f"re-encode {rep}")
allp = synthetic.all_pairs(N)
for i, j in allp:
    plan.recover_strided(*a, [(i, j)])
    plan.sync()
    diff(f"uniform pair ({i},{j}) [{synthetic.pair_class(N, i, j)}]")
for step in range(4):
    pairs = [allp[(s + 37 * step) % len(allp)] for s in range(S)]
    plan.recover_strided(*a, torch.tensor(pairs, dtype=torch.int32, device="cuda"))
    plan.sync()
    diff(f"mixed step {step}")
# repeated encode+recover sequence like the bench
for step in range(6):
    pairs = [allp[(s + 37 * step) % len(allp)] for s in range(S)]
    plan.encode_strided(*a)
    plan.recover_strided(*a, torch.tensor(pairs, dtype=torch.int32, device="cuda"))
plan.sync()
diff("bench-like 6 steps")
