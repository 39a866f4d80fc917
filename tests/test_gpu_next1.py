"""NEXT-1: small-write parity update and scrub, on the GPU through the C ABI,
against the oracle: an updated stripe must equal the oracle's encode of the stripe with the
strip replaced (definition; Eq. (znparity)), and scrub counts must equal the
oracle's per-word check of both parity equations (oracle.count_bad_words)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import oracle  # noqa: E402
import synthetic  # noqa: E402
from paper_cs_0611109_b200 import raid6c as R  # noqa: E402
from tests.gpu_util import Batch  # noqa: E402

CASES = [(13, 12, 3 * 12288 + 777, 3, 0), (5, 4, 65536, 3, 0), (59, 58, 2 * 14848 + 50, 2, 0),
         (61, 60, 2 * 15360 + 9, 2, 0), (257, 64, 2 * 8192 + 33, 2, 0), (17, 16, 12000, 2, 0),
         (11, 10, 2000, 2, 0), (23, 22, 2000, 2, 0), (13, 12, 5000, 2, 3), (3, 3, 1000, 2, 0), (7, 7, 777, 3, 1),
         (67, 30, 3000, 2, 0)] + [(p, min(p - 1, 30), 2 * 16384 + 77, 2, 0) for p in (23, 31, 41, 47, 73, 97, 113, 233, 241)]


def _np(t):
    return t.cpu().numpy()


@pytest.mark.parametrize("p,N,nbytes,S,offset", CASES)
def test_update_matches_reencode(p, N, nbytes, S, offset):
    b = Batch(p, N, nbytes, S, offset=offset, align=256 if offset == 0 else 0)
    b.fill_synthetic(seed=11, cfg=6)
    plan = R.Plan(p, N, nbytes)
    plan.encode_strided(*b.args())
    ns = R.aligned_stride(nbytes) if offset == 0 else nbytes + 5
    newbuf = torch.zeros(S * ns + offset + 16, dtype=torch.uint8, device="cuda")
    new = newbuf[offset:offset + S * ns].view(S, ns)
    R.fill(new, ns, ns, nbytes, 1, S, 11, 8, 0, 0, 0)
    disks = [(3 * s + 1) % N for s in range(S)]
    for trial, dk in enumerate([disks, torch.tensor(disks, dtype=torch.int32, device="cuda")]):
        if trial == 1:  # second update back to the original bytes, disks passed on the device
            for s in range(S):
                new[s, :nbytes].copy_(torch.from_numpy(synthetic.strip_bytes(11, 6, s, disks[s], nbytes)))
        plan.update_strided(*b.args(), int(new.data_ptr()), ns, dk)
        plan.sync()
        for s in range(S):
            data = synthetic.stripe_strips(11, 6, s, N, nbytes)
            if trial == 0:
                data[disks[s]] = _np(new[s, :nbytes])
            P, Q = oracle.encode(p, data, nbytes)
            for k in range(N):
                assert np.array_equal(_np(b.strip(s, k)), data[k]), (trial, s, k)
            assert np.array_equal(_np(b.strip(s, N)), P), (trial, s)
            assert np.array_equal(_np(b.strip(s, N + 1)), Q), (trial, s)


def test_update_uniform_disk_and_errors():
    p, N, nbytes, S = 13, 12, 4096, 2
    b = Batch(p, N, nbytes, S)
    b.fill_synthetic(seed=12, cfg=6)
    plan = R.Plan(p, N, nbytes)
    plan.encode_strided(*b.args())
    new = torch.full((S, nbytes), 0x3C, dtype=torch.uint8, device="cuda")
    plan.update_strided(*b.args(), new, nbytes, [N - 1])
    plan.sync()
    for s in range(S):
        data = synthetic.stripe_strips(12, 6, s, N, nbytes)
        data[N - 1] = np.full(nbytes, 0x3C, np.uint8)
        P, Q = oracle.encode(p, data, nbytes)
        assert np.array_equal(_np(b.strip(s, N)), P) and np.array_equal(_np(b.strip(s, N + 1)), Q)
    with pytest.raises(R.Raid6Error, match="INVALID_INDEX"):
        plan.update_strided(*b.args(), new, nbytes, [N])  # parity strips cannot be "updated"
    with pytest.raises(R.Raid6Error, match="SIZE"):
        plan.update_strided(*b.args(), new, nbytes, [0, 1, 2])


@pytest.mark.parametrize("p,N,nbytes,S,offset", CASES)
def test_scrub_counts_match_oracle(p, N, nbytes, S, offset):
    b = Batch(p, N, nbytes, S, offset=offset, align=256 if offset == 0 else 0)
    b.fill_synthetic(seed=13, cfg=6)
    plan = R.Plan(p, N, nbytes)
    plan.encode_strided(*b.args())
    cnt = torch.full((S,), 777, dtype=torch.int32, device="cuda")
    plan.scrub_strided(*b.args(), cnt)
    plan.sync()
    assert cnt.cpu().tolist() == [0] * S
    rng = np.random.default_rng(p * 100 + N)
    pb = R.parity_bytes(p, nbytes)
    for s in range(S):  # corrupt a few bytes in data, P and Q (none in stripe 0 of odd cases)
        if s == 0 and S > 2:
            continue
        for _ in range(3 + s):
            k = int(rng.integers(N + 2))
            ln = nbytes if k < N else pb
            pos = int(rng.integers(ln))
            t = b.strip(s, k)
            t[pos] ^= int(rng.integers(1, 256))
    plan.scrub_strided(*b.args(), cnt)
    plan.sync()
    got = cnt.cpu().tolist()
    for s in range(S):
        strips = [_np(b.strip(s, k)).copy() for k in range(N + 2)]
        assert got[s] == oracle.count_bad_words(p, N, strips, nbytes), s


@pytest.mark.parametrize("p,N,nbytes", [(13, 12, 5000), (13, 16, 4 * 12288 + 1000), (61, 60, 15360 + 9)])
def test_update_new_data_read_only_to_strip_length(p, N, nbytes):
    """The new-data row is `bytes` long even when parity strips are longer (R5): with the new rows
    packed back to back (new_stride == bytes) and 0xFF around them, bytes past each row must not
    leak into P, Q (a regression: the row was once read to parity length)."""
    S = 3
    b = Batch(p, N, nbytes, S)
    b.fill_synthetic(seed=13, cfg=6)
    plan = R.Plan(p, N, nbytes)
    plan.encode_strided(*b.args())
    assert R.parity_bytes(p, nbytes) > nbytes
    newbuf = torch.full((S * nbytes + 64,), 0xFF, dtype=torch.uint8, device="cuda")
    new = newbuf[:S * nbytes].view(S, nbytes)
    R.fill(new, nbytes, nbytes, nbytes, 1, S, 14, 8, 0, 0, 0)
    disks = [(5 * s + 2) % N for s in range(S)]
    plan.update_strided(*b.args(), int(new.data_ptr()), nbytes, torch.tensor(disks, dtype=torch.int32, device="cuda"))
    plan.sync()
    for s in range(S):
        data = synthetic.stripe_strips(13, 6, s, N, nbytes)
        data[disks[s]] = _np(new[s])
        P, Q = (oracle.encode_ext if N > p else oracle.encode)(p, data, nbytes)
        assert np.array_equal(_np(b.strip(s, N)), P), s
        assert np.array_equal(_np(b.strip(s, N + 1)), Q), s
