#!/usr/bin/env python3
"""Per-launch overhead probe: the c1 batch (p=5, N=4, 64 KiB x 4096) timed as (a) K encodes
back to back under one event pair, (b) K encodes each bracketed by events, (c) alternating
encode / recover as bench.py does.  usage: launch_gap.py [cfg] [K]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
from paper_cs_0611109_b200 import raid6c as R  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 1
K = int(sys.argv[2]) if len(sys.argv) > 2 else 20
c = bench.CONFIGS[cfg]
p, N, nbytes, S = c["p"], c["N"], c["nbytes"], c["stripes"]
pb = R.parity_bytes(p, nbytes)
ss, ps = R.aligned_stride(nbytes), R.aligned_stride(pb)
data = torch.empty((S, N, ss), dtype=torch.uint8, device="cuda")
par = torch.zeros((S, 2, ps), dtype=torch.uint8, device="cuda")
R.fill(data, ss, N * ss, nbytes, N, S, 0, cfg, 0, 0, c["sparse"])
st = torch.cuda.Stream()
plan = R.Plan(p, N, nbytes, 0, st)
a = (int(data.data_ptr()), ss, N * ss, int(par.data_ptr()), int(par.data_ptr()) + ps, 2 * ps, S)
pairs = torch.tensor(bench.pair_schedule(cfg, N, S, 0, 0), dtype=torch.int32, device="cuda")
alg = S * (N * nbytes + 2 * pb)
torch.cuda.synchronize()


def ev():
    return torch.cuda.Event(enable_timing=True)


for _ in range(5):
    plan.encode_strided(*a)
    plan.recover_strided(*a, pairs)
st.synchronize()
with torch.cuda.stream(st):
    e0, e1 = ev(), ev()
    e0.record(st)
    for _ in range(K):
        plan.encode_strided(*a)
    e1.record(st)
    st.synchronize()
    t = e0.elapsed_time(e1) / K
    print(f"(a) {K} encodes back to back: {t*1e3:.1f} us/launch  {alg/t/1e6:.0f} GB/s")
    es = [(ev(), ev()) for _ in range(K)]
    for i in range(K):
        es[i][0].record(st)
        plan.encode_strided(*a)
        es[i][1].record(st)
    st.synchronize()
    ts = [x.elapsed_time(y) for x, y in es]
    print(f"(b) bracketed encodes: mean {sum(ts)/K*1e3:.1f} us  min {min(ts)*1e3:.1f}  max {max(ts)*1e3:.1f}")
    es = [(ev(), ev(), ev()) for _ in range(K)]
    for i in range(K):
        es[i][0].record(st)
        plan.encode_strided(*a)
        es[i][1].record(st)
        plan.recover_strided(*a, pairs)
        es[i][2].record(st)
    st.synchronize()
    te = [x.elapsed_time(y) for x, y, _ in es]
    tr = [y.elapsed_time(z) for _, y, z in es]
    print(f"(c) alternating: encode mean {sum(te)/K*1e3:.1f} us, recover mean {sum(tr)/K*1e3:.1f} us")
    e0.record(st)
    for _ in range(K):
        plan.recover_strided(*a, pairs)
    e1.record(st)
    st.synchronize()
    t = e0.elapsed_time(e1) / K
    print(f"(d) {K} recovers back to back: {t*1e3:.1f} us/launch  {alg/t/1e6:.0f} GB/s")
    import time
    st.synchronize()
    t0 = time.perf_counter()
    for _ in range(K):
        plan.encode_strided(*a)
    t1 = time.perf_counter()
    st.synchronize()
    print(f"(e) host enqueue: {(t1 - t0) / K * 1e6:.1f} us per encode call")
    # CUDA graph of K encodes (host overhead removed)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        for _ in range(K):
            plan.encode_strided(*a)
    st.synchronize()
    g.replay()
    st.synchronize()
    e0.record(st)
    g.replay()
    e1.record(st)
    st.synchronize()
    t = e0.elapsed_time(e1) / K
    print(f"(f) graph of {K} encodes: {t*1e3:.1f} us/launch  {alg/t/1e6:.0f} GB/s")
