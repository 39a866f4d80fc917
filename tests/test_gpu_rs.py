"""NEXT-3: the GF(256) Reed-Solomon comparison system on the GPU (raid6c_rs_*), bit-exact vs the
RS oracle (oracle.rs_encode / rs_recover, written from Sec. 4.1-4.4 of the paper)."""
import itertools

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import oracle  # noqa: E402
import synthetic  # noqa: E402
from paper_cs_0611109_b200 import raid6c as R  # noqa: E402


def _batch(N, nbytes, S, offset=0, align=True):
    ss = R.aligned_stride(nbytes) if align else nbytes
    buf = torch.zeros(S * (N + 2) * ss + offset + 64, dtype=torch.uint8, device="cuda")
    v = buf[offset:offset + S * (N + 2) * ss].view(S, N + 2, ss)
    R.fill(v, ss, (N + 2) * ss, nbytes, N, S, 31, 11, 0, 0, 0)
    base = int(v.data_ptr())
    # data strips 0..N-1, P = N, Q = N+1 inside each stripe row
    args = (base, ss, (N + 2) * ss, base + N * ss, base + (N + 1) * ss, (N + 2) * ss, S)
    return v, args


@pytest.mark.parametrize("N,nbytes,S,offset", [(1, 1000, 2, 0), (4, 3 * 12288 + 77, 2, 0), (12, 12288 * 2 + 5, 3, 0),
                                               (16, 20000, 2, 0), (64, 12288 + 300, 1, 0), (255, 777, 1, 0),
                                               (12, 5000, 2, 3)])
def test_rs_encode_recover(N, nbytes, S, offset):
    v, a = _batch(N, nbytes, S, offset, offset == 0)
    R.rs_encode_strided(N, nbytes, *a)
    torch.cuda.synchronize()
    refs = []
    for s in range(S):
        data = synthetic.stripe_strips(31, 11, s, N, nbytes)
        P, Q = oracle.rs_encode(data, nbytes)
        assert np.array_equal(v[s, N, :nbytes].cpu().numpy(), P)
        assert np.array_equal(v[s, N + 1, :nbytes].cpu().numpy(), Q)
        refs.append(data + [P, Q])
    allp = list(itertools.combinations(range(N + 2), 2))
    rng = np.random.default_rng(N)
    picks = allp if len(allp) <= 40 else [allp[int(t)] for t in rng.choice(len(allp), 40, replace=False)]
    for t, (i, j) in enumerate(picks):
        pairs = [(i, j)] + [allp[int(rng.integers(len(allp)))] for _ in range(S - 1)]
        for s, (x, y) in enumerate(pairs):
            v[s, x, :nbytes] = 0xA5
            v[s, y, :nbytes] = 0x5A
        er = torch.tensor(pairs, dtype=torch.int32, device="cuda") if t % 2 else pairs
        R.rs_recover_strided(N, nbytes, *a, er)
        torch.cuda.synchronize()
        for s, (x, y) in enumerate(pairs):
            for k in (x, y):
                assert np.array_equal(v[s, k, :nbytes].cpu().numpy(), refs[s][k]), (N, s, x, y, k)


def test_rs_argument_errors():
    t = torch.zeros(64, dtype=torch.uint8, device="cuda")
    with pytest.raises(R.Raid6Error, match="INVALID_N"):
        R.rs_encode_strided(256, 16, t, 16, 64, t, t, 64, 1)
    with pytest.raises(R.Raid6Error, match="INVALID_INDEX"):
        R.rs_recover_strided(2, 16, t, 16, 64, t, t, 64, 1, [(1, 1)])
