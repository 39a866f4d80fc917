"""Edge cases of the C ABI on the GPU: empty batches, the maximum strip count (p = 257 with the
extended code's 2p-1 = 513 data strips), and a strip longer than 4 GiB (64-bit offsets in the
kernels), each against the CPU oracle."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import oracle  # noqa: E402
from paper_cs_0611109_b200 import raid6c as R  # noqa: E402
from tests.gpu_util import Batch, segment_bounds  # noqa: E402


def test_zero_stripes_is_a_no_op():
    p, N, nbytes = 13, 12, 5000
    b = Batch(p, N, nbytes, 2)
    b.dbuf.fill_(0x11)
    b.pbuf.fill_(0x22)
    plan = R.Plan(p, N, nbytes)
    args = list(b.args())
    args[-1] = 0
    plan.encode_strided(*args)
    plan.recover_strided(*args, [(0, 1)])
    cnt = torch.zeros(2, dtype=torch.int32, device="cuda")
    plan.scrub_strided(*args, cnt)
    plan.sync()
    assert bool((b.dbuf == 0x11).all()) and bool((b.pbuf == 0x22).all())


def test_maximum_strip_count_extended_code():
    """p = 257, N = 513 data strips + P + Q = 515 strips per stripe (RAID6C_MAX_STRIPS)."""
    p, N, nbytes = 257, 513, 96
    assert R.ext_supported(p)
    rng = np.random.default_rng(7)
    data = [rng.integers(0, 256, nbytes, dtype=np.uint8) for _ in range(N)]
    P, Q = oracle.encode_ext(p, data, nbytes)
    b = Batch(p, N, nbytes, 1)
    b.set_data_numpy(0, data)
    plan = R.Plan(p, N, nbytes)
    plan.encode_strided(*b.args())
    plan.sync()
    assert np.array_equal(b.numpy_strip(0, N), P) and np.array_equal(b.numpy_strip(0, N + 1), Q)
    orig = data + [P, Q]
    for i, j in [(0, 512), (256, 257), (300, 511), (5, N), (400, N), (511, N + 1), (N, N + 1)]:
        for k in (i, j):
            b.strip(0, k).fill_(0xA5)
        plan.recover_strided(*b.args(), [(i, j)])
        plan.sync()
        for k in (i, j):
            assert np.array_equal(b.numpy_strip(0, k), orig[k]), (i, j, k)


def test_strip_longer_than_4_gib():
    """One stripe whose strips are 4 GiB + 4 KiB + 5 bytes long: byte offsets past 2^32 in the TMA
    tiles, the ragged tail and the recovery, checked on word-aligned segments at the start,
    across the 2^32 boundary and at the end against the oracle, and by a full round trip."""
    p, N = 13, 2
    nbytes = (4 << 30) + 4096 + 5
    pb = R.parity_bytes(p, nbytes)
    ss, ps = R.aligned_stride(nbytes), R.aligned_stride(pb)  # 16-byte aligned strides: the TMA path
    gen = torch.Generator(device="cuda").manual_seed(99)
    buf = torch.randint(0, 256, (N, ss), dtype=torch.uint8, device="cuda", generator=gen)
    data = buf[:, :nbytes]
    par = torch.zeros((2, ps), dtype=torch.uint8, device="cuda")
    plan = R.Plan(p, N, nbytes)
    a = (int(buf.data_ptr()), ss, N * ss, int(par.data_ptr()), int(par.data_ptr()) + ps, 2 * ps, 1)
    plan.encode_strided(*a)
    plan.sync()
    n = p - 1
    g32 = ((1 << 32) // n - 4) * n  # a word-group boundary just below 2^32 (8 words = n bytes)
    for b0, b1 in [segment_bounds(p, nbytes, "head"), (g32, g32 + 8 * n), segment_bounds(p, nbytes, "tail")]:
        segs = [data[k, b0:b1].cpu().numpy() for k in range(N)]
        P, Q = oracle.encode(p, segs, b1 - b0)
        e = b0 + P.size
        assert np.array_equal(par[0, b0:e].cpu().numpy(), P), (b0, "P")
        assert np.array_equal(par[1, b0:e].cpu().numpy(), Q), (b0, "Q")
    ref = data[1].clone()
    refq = par[1, :pb].clone()
    data[1].fill_(0)
    par[1, :pb].fill_(0)
    plan.recover_strided(*a, [(1, N + 1)])  # DQ: d_1 from P, then Q re-encoded
    plan.sync()
    assert torch.equal(data[1], ref) and torch.equal(par[1, :pb], refq)
    del buf, data, par, ref, refq
    torch.cuda.empty_cache()
