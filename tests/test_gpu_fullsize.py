"""Full-size parity: whole strips of the BASELINE configs against the oracle.

Each config runs in bench.py's launch configuration (a persistent grid with more work items than
CTAs, so every CTA loops over several items -- the path where the TMA stage-release race once
lived), and for at least two stripes per config the WHOLE P/Q strips and the WHOLE rebuilt strips
are compared byte for byte with the oracle's (tests/oracle_sample.py: the oracle run on
word-aligned segments in a host thread pool, pinned to whole-strip oracle calls by
tests/test_oracle_sample.py).  Also: the per-strip digest kernel equals its host twin."""
import numpy as np
import pytest
import torch

import synthetic
from paper_cs_0611109_b200 import raid6c as R
from tests import oracle_sample as OS
from tests.gpu_util import Batch

pytestmark = pytest.mark.gpu


def _np(t):
    return t.cpu().numpy()


def _poison(b, s, ks):
    for k in ks:
        b.strip(s, k).fill_(0xA5)


@pytest.mark.parametrize("nbytes,offset", [(1, 0), (7, 3), (8, 0), (4097, 1), (65536, 0), (4194305, 0),
                                           (33554438, 5)])
def test_digest_kernel_matches_host(nbytes, offset):
    S, K = 2, 3
    stride = nbytes + 40
    g = torch.Generator().manual_seed(nbytes)
    host = torch.randint(0, 256, (S * K * stride + offset,), dtype=torch.uint8, generator=g)
    dev = host.cuda()
    out = torch.zeros(S * K, dtype=torch.int64, device="cuda")
    R.digest(int(dev.data_ptr()) + offset, stride, K * stride, nbytes, K, S, out)
    torch.cuda.synchronize()
    got = [int(v) & ((1 << 64) - 1) for v in out.cpu().tolist()]
    hb = host.numpy()
    for s in range(S):
        for t in range(K):
            o = offset + s * K * stride + t * stride
            assert got[s * K + t] == synthetic.digest(hb[o:o + nbytes]), (s, t)


def test_digest_of_device_fill_matches_generator():
    p, N, nbytes, S = 59, 58, 8 << 20, 2
    b = Batch(p, N, nbytes, S)
    b.fill_synthetic(seed=0, cfg=4, stripe0=10, sparse_mode=2)
    out = torch.zeros(S * N, dtype=torch.int64, device="cuda")
    R.digest(b.data, b.ss, N * b.ss, nbytes, N, S, out)
    got = [int(v) & ((1 << 64) - 1) for v in out.cpu().tolist()]
    exp = OS.data_digests(N, nbytes, 4, [10, 11], sparse_of=lambda s: s % 2 == 1)
    assert got == exp[10] + exp[11]


def _full_check(p, N, nbytes, cfg, S, check, pairs_of, sparse_mode=0, encode_only=False):
    """S stripes in one persistent launch; the stripes in `check` are compared whole with the
    oracle: P, Q after encode and, unless encode_only, both rebuilt strips of pairs_of(s)."""
    b = Batch(p, N, nbytes, S)
    b.fill_synthetic(seed=0, cfg=cfg, sparse_mode=sparse_mode)
    plan = R.Plan(p, N, nbytes)
    # every fast kernel's tile is at most 15360 B and its grid at most 3 CTAs per SM: more items
    # than CTAs means every CTA loops over several items
    grid_cap = torch.cuda.get_device_properties(0).multi_processor_count * 3
    assert (nbytes // 15360) * S > grid_cap, "the launch must be persistent (several items per CTA)"
    plan.encode_strided(*b.args())
    plan.sync()
    sparse_of = (lambda s: s % 2 == 1) if sparse_mode == 2 else (lambda s: False)
    items = [(s, [] if encode_only else [pairs_of(s)]) for s in check]
    _, info = OS.stripe_digests(p, N, nbytes, cfg, items, sparse_of=sparse_of, keep=True)
    ref = info["strips"]
    for s in check:
        assert np.array_equal(_np(b.strip(s, N)), ref[s]["P"]), ("P", s)
        assert np.array_equal(_np(b.strip(s, N + 1)), ref[s]["Q"]), ("Q", s)
    if encode_only:
        return
    pairs = [pairs_of(s) for s in range(S)]
    for s, pr in enumerate(pairs):
        _poison(b, s, pr)
    plan.recover_strided(*b.args(), torch.tensor(pairs, dtype=torch.int32, device="cuda"))
    plan.sync()
    for s in check:
        x, y = pairs[s]
        for k in (x, y):
            assert np.array_equal(_np(b.strip(s, k)), ref[s][(x, y, k)]), ("rebuilt", s, (x, y), k)


def test_c2_whole_strips_every_class():
    N = 12
    cls = [(2, 9), (5, N), (7, N + 1), (N, N + 1)]  # DD, DP, DQ, PQ
    _full_check(13, N, 4 << 20, 2, 4, [0, 1, 2, 3], lambda s: cls[s % 4])


def test_c3_whole_strips_encode():
    _full_check(257, 64, 16 << 20, 3, 2, [0, 1], None, encode_only=True)


def test_c4_whole_strips_dd_uniform_and_sparse():
    N = 58
    dd = [(i, j) for i in range(N) for j in range(i + 1, N)]
    _full_check(59, N, 8 << 20, 4, 4, [0, 1], lambda s: dd[(s * 411) % len(dd)], sparse_mode=2)


def test_c5_whole_strips_dd_and_dp():
    N = 60
    pairs = [(3, 40), (17, N)]
    _full_check(61, N, 32 << 20, 5, 2, [0, 1], lambda s: pairs[s])


def test_c1_whole_strips_persistent_batch():
    N = 4
    allp = synthetic.all_pairs(N)
    _full_check(5, N, 64 << 10, 1, 1024, [0, 1, 2, 3, 1021, 1022, 1023], lambda s: allp[s % 15])
