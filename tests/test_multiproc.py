"""N>1 host logic on CPU: world-size-2 gloo process group.  Checks the stripe partitions
(disjoint, covering), the max/sum reductions bench.py uses, and that per-stripe results are
invariant to the number of ranks (sharding invariance: every rank derives its data from the
global stripe index, so the union of the shards' oracle parities equals the 1-rank result)."""
import hashlib
import os
import socket

import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _digest_stripes(lo, hi, p=13, N=4, nbytes=300):
    import oracle
    import synthetic
    out = {}
    for s in range(lo, hi):
        data = synthetic.stripe_strips(0, 2, s, N, nbytes)
        P, Q = oracle.encode(p, data, nbytes)
        out[s] = hashlib.sha256(P.tobytes() + Q.tobytes()).hexdigest()
    return out


def _worker(rank, world, port, total, q):
    import sys
    sys.path.insert(0, ROOT)
    import torch.distributed as dist
    from paper_cs_0611109_b200 import shard
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    lo, hi = shard.block_range(rank, world, total)
    dig = _digest_stripes(lo, hi)
    mx = shard.max_over_ranks(10.0 + rank)
    sm = shard.sum_over_ranks([hi - lo, rank + 1])
    assert shard.gather_over_ranks(10.0 + rank) == [10.0 + r for r in range(world)]
    dist.barrier()
    dist.destroy_process_group()
    q.put((rank, lo, hi, dig, mx, sm))


@pytest.mark.parametrize("world,total", [(2, 7), (2, 10)])
def test_gloo_world2_sharding_and_reductions(world, total):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, total, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    res.sort()
    covered = []
    merged = {}
    for rank, lo, hi, dig, mx, sm in res:
        covered += list(range(lo, hi))
        merged.update(dig)
        assert mx == 10.0 + world - 1
        assert sm == [total, sum(range(1, world + 1))]
    assert covered == list(range(total))
    assert merged == _digest_stripes(0, total)  # invariant to the number of ranks


def test_block_and_weak_ranges():
    from paper_cs_0611109_b200 import shard
    for G in [1, 2, 4, 8]:
        for S in [0, 1, 7, 1000, 4096]:
            rs = [shard.block_range(r, G, S) for r in range(G)]
            assert rs[0][0] == 0 and rs[-1][1] == S
            assert all(a[1] == b[0] for a, b in zip(rs, rs[1:]))
            assert max(h - l for l, h in rs) - min(h - l for l, h in rs) <= 1
    assert shard.block_range(3, 8, 4096) == (1536, 2048)
    assert shard.weak_range(3, 256) == (768, 1024)
    with pytest.raises(ValueError):
        shard.block_range(2, 2, 5)
    assert shard.max_over_ranks(3.5) == 3.5 and shard.sum_over_ranks([1, 2]) == [1, 2]
