#!/usr/bin/env python3
"""Debug: extended-code small-write update vs re-encode.  usage: debug_update_ext.py p N nbytes S [host]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_cs_0611109_b200 import raid6c as R  # noqa: E402
from tests.gpu_util import Batch  # noqa: E402

p, N, nbytes, S = (int(x) for x in sys.argv[1:5])
host = len(sys.argv) > 5
b = Batch(p, N, nbytes, S)
b.fill_synthetic(seed=3, cfg=2)
plan = R.Plan(p, N, nbytes)
plan.encode_strided(*b.args())
cnt = torch.zeros(S, dtype=torch.int32, device="cuda")
plan.scrub_strided(*b.args(), cnt)
plan.sync()
print("scrub after encode", cnt.tolist())
ns = R.aligned_stride(nbytes)
new = torch.empty((S, ns), dtype=torch.uint8, device="cuda")
R.fill(new, ns, ns, nbytes, 1, S, 9, 2, 0, 0, 0)
dl = [(7 * s) % N for s in range(S)]
disks = dl if host else torch.tensor(dl, dtype=torch.int32, device="cuda")
plan.update_strided(*b.args(), new, ns, disks)
plan.scrub_strided(*b.args(), cnt)
plan.sync()
print("disks", dl)
print("scrub after update", cnt.tolist())
par_upd = b.par.clone()
plan.encode_strided(*b.args())
plan.sync()
pb = b.pb
for s in range(S):
    for w in range(2):
        d = (par_upd[s, w, :pb] != b.par[s, w, :pb]).nonzero().flatten()
        if d.numel():
            print(f"stripe {s} disk {dl[s]} {'PQ'[w]}: {d.numel()} bytes differ, range [{int(d.min())},{int(d.max())}] first {d[:8].tolist()}")
for s in range(S):
    dd = (b.data[s, dl[s], :nbytes] != new[s, :nbytes]).nonzero().flatten()
    if dd.numel():
        print(f"stripe {s}: data strip not replaced at {dd.numel()} bytes, first {dd[:8].tolist()}")
