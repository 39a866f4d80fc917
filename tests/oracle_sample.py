"""Full-size oracle results for sampled stripes, as per-strip digests (test / bench harness).

The oracle (oracle/oracle.c) is single-threaded per call and slow (one byte per bit), and the
configs' stripes are 48 MB (c2) to 2 GB (c5).  Every output word of encode and recovery
depends only on the input words at the same position (Eq. (znparity): P_w and
Q_w are sums over disks of word w; the recovery solves each word position on its own,
PAPER.md:1124-1160), so a stripe is cut into word-aligned segments -- byte offsets that are
multiples of lcm(p-1, 8), i.e. whole groups of 8 words that also start on 8-byte digest words --
the oracle is run on each segment in a thread pool over the host cores, and the segments'
outputs are reduced to digests (synthetic.digest word terms, which add across pieces).
tests/test_oracle_sample.py checks that the segmented results equal the oracle on whole strips.

Only tests/ and bench.py's cpu_baseline leg use this module (it calls the oracle).
"""
from __future__ import annotations

import concurrent.futures as cf
import math
import os
import time

import numpy as np

import oracle
import synthetic

_M64 = (1 << 64) - 1


def segment_bytes(p: int, target: int = 1 << 20) -> int:
    """Segment length: a multiple of lcm(p-1, 8) bytes (whole 8-word groups on digest words)."""
    unit = (p - 1) * 8 // math.gcd(p - 1, 8)
    return max(unit, (target // unit) * unit)


def segments(p: int, nbytes: int, target: int = 1 << 20):
    L = segment_bytes(p, target)
    return [(b0, min(nbytes, b0 + L)) for b0 in range(0, nbytes, L)]


def host_threads(cap: int = 64) -> int:
    return max(1, min(cap, len(os.sched_getaffinity(0))))


def _segment_task(p, N, nbytes, cfg, sparse, seed, stripe, pairs, b0, b1, keep=False):
    """Oracle encode (and one recovery per pair) of bytes [b0, b1) of every strip of one stripe.
    Returns (oracle seconds, {strip key: word terms}, {strip key: bytes} if keep) with keys
    'P', 'Q', (x, y, k)."""
    data = [synthetic.strip_bytes(seed, cfg, stripe, k, nbytes, sparse, lo=b0, hi=b1) for k in range(N)]
    w0 = b0 // 8
    t0 = time.perf_counter()
    P, Q = oracle.encode(p, data, b1 - b0)
    secs = time.perf_counter() - t0
    out = {"P": synthetic.word_terms(P, w0), "Q": synthetic.word_terms(Q, w0)}
    raw = {"P": P, "Q": Q} if keep else None
    for (x, y) in pairs:
        strips = [d.copy() for d in data] + [P.copy(), Q.copy()]
        strips[x][:] = 0
        strips[y][:] = 0
        t0 = time.perf_counter()
        oracle.recover(p, N, x, y, strips, b1 - b0)
        secs += time.perf_counter() - t0
        out[(x, y, x)] = synthetic.word_terms(strips[x], w0)
        out[(x, y, y)] = synthetic.word_terms(strips[y], w0)
        if keep:
            raw[(x, y, x)], raw[(x, y, y)] = strips[x], strips[y]
    return secs, out, raw


def stripe_digests(p, N, nbytes, cfg, items, seed=0, sparse_of=lambda s: False, threads=None,
                   seg_target=1 << 20, keep=False):
    """Oracle digests of sampled stripes at full size.

    items: list of (global stripe index, list of erasure pairs (x, y), x < y).
    Returns (digests, info): digests[s] = {'P': d, 'Q': d, (x, y, k): d for each pair and k in
    (x, y)} (d = synthetic.digest of the oracle's full-length strip); info = {'oracle_s': summed
    seconds inside oracle calls, 'wall_s', 'threads', 'user_bytes': user data the oracle
    processed (N*bytes per encode and per recovery)}; with keep=True also info['strips'][s][key] =
    the oracle's full-length output strip (uint8 array) for every digest key."""
    pb = oracle.parity_bytes(p, nbytes)
    threads = threads or host_threads()
    segs = segments(p, nbytes, seg_target)
    tasks = [(s, pairs, b0, b1) for (s, pairs) in items for (b0, b1) in segs]
    acc = {s: {} for s, _ in items}
    raws = {s: {} for s, _ in items}
    osecs = 0.0
    t0 = time.perf_counter()
    with cf.ThreadPoolExecutor(max_workers=threads) as ex:
        futs = [ex.submit(_segment_task, p, N, nbytes, cfg, sparse_of(s), seed, s, pairs, b0, b1, keep)
                for (s, pairs, b0, b1) in tasks]
        for (s, _, _, _), f in zip(tasks, futs):
            secs, out, raw = f.result()
            osecs += secs
            a = acc[s]
            for k, v in out.items():
                a[k] = (a.get(k, 0) + v) & _M64
            if keep:
                for k, v in raw.items():
                    raws[s].setdefault(k, []).append(v)
    wall = time.perf_counter() - t0
    lt_p, lt_d = synthetic.length_term(pb), synthetic.length_term(nbytes)
    dig = {}
    for s, pairs in items:
        a = acc[s]
        d = {"P": (a["P"] + lt_p) & _M64, "Q": (a["Q"] + lt_p) & _M64}
        for (x, y) in pairs:
            for k in (x, y):
                d[(x, y, k)] = (a[(x, y, k)] + (lt_d if k < N else lt_p)) & _M64
        dig[s] = d
    user = sum((1 + len(pairs)) * N * nbytes for _, pairs in items)
    info = {"oracle_s": osecs, "wall_s": wall, "threads": threads, "user_bytes": user,
            "segment_bytes": segs[0][1] - segs[0][0] if segs else 0}
    if keep:  # segments were submitted in order, so concatenation restores each strip
        info["strips"] = {s: {k: np.concatenate(v) for k, v in r.items()} for s, r in raws.items()}
    return dig, info


def data_digests(N, nbytes, cfg, stripes, seed=0, sparse_of=lambda s: False, threads=None):
    """Digests of the generator's data strips (the expected content of rebuilt data strips):
    {s: [digest of strip k for k < N]}."""
    threads = threads or host_threads()

    def one(sk):
        s, k = sk
        return synthetic.digest(synthetic.strip_bytes(seed, cfg, s, k, nbytes, sparse_of(s)))

    keys = [(s, k) for s in stripes for k in range(N)]
    with cf.ThreadPoolExecutor(max_workers=threads) as ex:
        vals = list(ex.map(one, keys))
    out = {s: [0] * N for s in stripes}
    for (s, k), v in zip(keys, vals):
        out[s][k] = v
    return out


def sample_stripes(total: int, k: int):
    """k stripe indices spread evenly over [0, total) (so every block shard of any G <= k is hit)."""
    k = max(1, min(k, total))
    return sorted({(2 * i + 1) * total // (2 * k) for i in range(k)})
