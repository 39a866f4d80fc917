"""NEXT-4 host logic on CPU: the cross-GPU stripe layout's strip blocks and word ranges, and a
world-size-2 gloo rehearsal of the split itself with the oracle doing the arithmetic: every
rank computes the partial syndromes of the strips it holds (Eq. (PQxy), with
the other ranks' strips zeroed), the word-range owners exchange and add them, and solving from
the summed syndromes (Lemma 23.2) gives the lost strips."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def test_strip_blocks_partition_every_stripe():
    from paper_cs_0611109_b200 import xgpu
    for N in [1, 2, 4, 12, 58, 60, 64, 300]:
        for G in [1, 2, 3, 4, 8, 16]:
            if G > N + 2:
                continue
            blocks = [xgpu.strip_block(r, G, N) for r in range(G)]
            assert blocks[0][0] == 0 and blocks[-1][1] == N + 2
            assert all(a[1] == b[0] for a, b in zip(blocks, blocks[1:]))
            assert max(h - l for l, h in blocks) - min(h - l for l, h in blocks) <= 1
            for k in range(N + 2):
                lo, hi = blocks[xgpu.strip_owner(k, G, N)]
                assert lo <= k < hi
    with pytest.raises(ValueError):
        xgpu.strip_block(2, 2, 5)


def test_word_ranges_are_word_aligned_and_cover():
    """Range boundaries must fall on word boundaries (a word never straddles two owners) and
    on 16-byte multiples (TMA stores into the slots); G ranges cover the parity strip."""
    from paper_cs_0611109_b200 import raid6c as R
    from paper_cs_0611109_b200 import xgpu
    for p in [3, 5, 7, 11, 13, 17, 19, 59, 61, 127, 257]:
        n = p - 1
        for nbytes in [1, 100, 4096, 65536, 4 << 20, 8 << 20, (8 << 20) + 3]:
            pb = R.parity_bytes(p, nbytes)
            for G in [1, 2, 3, 4, 8]:
                rb = R.xgpu_range_bytes(p, nbytes, G)
                assert rb % 16 == 0 and (8 * rb) % n == 0, (p, nbytes, G, rb)
                rs = xgpu.word_ranges(pb, rb, G)
                assert rs[0][0] == 0 and rs[-1][1] == pb
                assert all(a[1] == b[0] for a, b in zip(rs, rs[1:]))
                assert (G - 1) * rb < pb + rb * G  # no range is wasted beyond rounding
                assert xgpu.slot_stride(rb) >= rb and xgpu.slot_stride(rb) % 16 == 0
    with pytest.raises(R.Raid6Error):
        R.xgpu_range_bytes(4, 100, 2)
    with pytest.raises(R.Raid6Error):
        R.xgpu_range_bytes(13, 100, 0)


def test_alg_bytes_accounting():
    from paper_cs_0611109_b200 import xgpu
    N, nb, pb, G, rb = 12, 1000, 1001, 4, 256
    tot_p = sum(xgpu.alg_bytes(N, nb, pb, G, r, rb)["partial"] for r in range(G))
    assert tot_p == N * nb + 2 * G * pb  # every data strip once + G partial pairs
    tot_c = sum(xgpu.alg_bytes(N, nb, pb, G, r, rb)["combine"] for r in range(G))
    assert tot_c == 2 * G * pb + 2 * pb  # every partial once + P and Q once


def _partials(p, N, strips, lost, block, nbytes):
    """Oracle partial syndromes of the strips in `block` that survive: (dP_r, dQ_r) as the
    oracle parity of the stripe with every other data strip zeroed, plus P / Q if held."""
    import oracle
    lo, hi = block
    sub = [strips[k] if (lo <= k < hi and k not in lost) else np.zeros(nbytes, np.uint8) for k in range(N)]
    dP, dQ = oracle.encode(p, sub, nbytes)
    if lo <= N < hi and N not in lost:
        dP = dP ^ strips[N]
    if lo <= N + 1 < hi and N + 1 not in lost:
        dQ = dQ ^ strips[N + 1]
    return dP, dQ


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist
    import oracle
    import synthetic
    from paper_cs_0611109_b200 import xgpu
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    p, N, nbytes = 13, 12, 300
    pb = oracle.parity_bytes(p, nbytes)
    unit = 3 * (p - 1)  # 16-byte-free toy granule: 24 bytes = 16 whole 12-bit words
    rb = ((pb + world - 1) // world + unit - 1) // unit * unit
    ranges = xgpu.word_ranges(pb, rb, world)
    data = synthetic.stripe_strips(0, 16, 0, N, nbytes)
    P, Q = oracle.encode(p, data, nbytes)
    strips = data + [P, Q]
    ok = []
    for lost in [(N, N + 1), (1, 10), (3, N), (5, N + 1), (0, 11)]:
        dP, dQ = _partials(p, N, strips, lost, xgpu.strip_block(rank, world, N), nbytes)
        # exchange: owner g receives range g of every rank's partials (all_gather stands in for
        # the peer stores of the partial kernel)
        got = [torch.zeros(2 * pb, dtype=torch.uint8) for _ in range(world)]
        dist.all_gather(got, torch.from_numpy(np.concatenate([dP, dQ])))
        lo, hi = ranges[rank]
        sP = np.bitwise_xor.reduce([g.numpy()[:pb][lo:hi] for g in got])
        sQ = np.bitwise_xor.reduce([g.numpy()[pb:][lo:hi] for g in got])
        # solve on the owner from the summed syndromes: the syndromes of a stripe whose
        # surviving strips are all zero and whose P, Q are (sP, sQ) (linearity)
        full_P = np.zeros(pb, np.uint8)
        full_Q = np.zeros(pb, np.uint8)
        full_P[lo:hi], full_Q[lo:hi] = sP, sQ
        # the recovery is linear: solving a stripe whose surviving strips are zero and whose
        # P, Q are the summed syndromes gives the lost data strips (Lemma 23.2 proof); a lost
        # parity strip is that solution plus its own syndrome (e.g. DP: P = dP + d_x)
        x, y = lost
        zs = [np.zeros(nbytes, np.uint8) for _ in range(N)] + [full_P.copy(), full_Q.copy()]
        zs[x][:] = 0
        zs[y][:] = 0
        oracle.recover(p, N, x, y, zs, nbytes)
        rec = {x: zs[x], y: zs[y]}
        if N in lost:
            rec[N] = rec[N] ^ full_P
        if N + 1 in lost:
            rec[N + 1] = rec[N + 1] ^ full_Q
        for k in (x, y):
            ln = nbytes if k < N else pb
            a, b = min(lo, ln), min(hi, ln)
            ok.append(bool(np.array_equal(rec[k][a:b], strips[k][a:b])))
    dist.barrier()
    dist.destroy_process_group()
    q.put((rank, ok))


def test_gloo_world2_partial_syndromes_sum_and_solve():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    for rank, ok in res:
        assert ok and all(ok), (rank, ok)


def test_arena_layouts_hold_every_strip_once_and_slots_do_not_overlap():
    """xgpu.Distributed's IPC arenas: every global strip lives in exactly one rank's arena, all
    regions are 16-byte aligned (TMA), and strips and slots never overlap."""
    from paper_cs_0611109_b200 import xgpu
    for N, G, S in [(12, 4, 3), (58, 8, 2), (4, 3, 5), (300, 8, 1), (2, 4, 2)]:
        ss, ps, pst = 4096, 4352, xgpu.slot_stride(1000)
        held = {}
        for r in range(G):
            lay = xgpu.arena_layout(r, G, N, S, ss, ps, pst)
            regions = []
            for k, off in lay["strip_off"].items():
                assert k not in held
                held[k] = r
                regions.append((off, off + S * (ss if k < N else ps)))
            for src in range(G):
                for which in (0, 1):
                    o = lay["slot_off"] + (2 * src + which) * S * pst
                    regions.append((o, o + S * pst))
            regions.sort()
            assert all(a % 16 == 0 for a, _ in regions)
            assert all(b <= c for (_, b), (c, _) in zip(regions, regions[1:]))
            assert regions[-1][1] <= lay["size"]
        assert sorted(held) == list(range(N + 2))
