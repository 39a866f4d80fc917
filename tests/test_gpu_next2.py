"""NEXT-2: the extended Q-parity of Eq. (qext), up to
2p-1 data strips, on the GPU through the C ABI vs the oracle (oracle.encode_ext /
oracle.recover_ext, which follow Eq. (qext) and the Lemma 23.2 proof literally)."""
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
from tests.gpu_util import Batch  # noqa: E402

# (p, N, bytes, stripes); fast-path primes and a generic one (67)
CASES = [(5, 9, 3 * 10752 + 517, 2), (13, 25, 2 * 12288 + 99, 2), (13, 17, 5000, 2), (17, 33, 11000, 2),
         (59, 90, 14848 + 333, 2), (61, 121, 15360 + 17, 2), (257, 300, 8192 + 64, 1), (11, 21, 3000, 2),
         (19, 37, 1500, 2), (23, 45, 1500, 2), (43, 60, 1200, 2), (23, 30, 3 * 16384 + 99, 2),
         (41, 51, 3 * 16384 + 5, 2), (47, 60, 2 * 16384 + 1, 2), (89, 100, 16384 + 77, 1), (101, 120, 4000, 1),
         (233, 240, 3000, 1), (241, 300, 2000, 1), (67, 80, 1000, 1)]


def _np(t):
    return t.cpu().numpy()


def _stripes(b, p, N, nbytes, S, seed, cfg):
    b.fill_synthetic(seed=seed, cfg=cfg)
    refs = []
    for s in range(S):
        data = synthetic.stripe_strips(seed, cfg, s, N, nbytes)
        P, Q = oracle.encode_ext(p, data, nbytes)
        refs.append(data + [P, Q])
    return refs


@pytest.mark.parametrize("p,N,nbytes,S", CASES)
def test_ext_encode_and_recover(p, N, nbytes, S):
    assert R.ext_supported(p)
    b = Batch(p, N, nbytes, S)
    refs = _stripes(b, p, N, nbytes, S, 21, 10)
    plan = R.Plan(p, N, nbytes)
    plan.encode_strided(*b.args())
    plan.sync()
    for s in range(S):
        assert np.array_equal(_np(b.strip(s, N)), refs[s][N]), s
        assert np.array_equal(_np(b.strip(s, N + 1)), refs[s][N + 1]), s
    allp = list(itertools.combinations(range(N + 2), 2))
    rng = np.random.default_rng(p + N)
    # every class, basic/extended/mixed data pairs, both pair orders
    pick = [(0, 1), (0, p), (p - 1, p), (1, N - 1), (N - 2, N - 1), (0, N), (N - 1, N), (p, N + 1), (N, N + 1),
            (2, N + 1)]
    pick = [(i, j) for i, j in pick if i < j < N + 2]
    pick += [allp[int(t)] for t in rng.choice(len(allp), 12, replace=False)]
    for t, (i, j) in enumerate(pick):
        pairs = [(i, j)] + [allp[int(rng.integers(len(allp)))] for _ in range(S - 1)]
        for s, (x, y) in enumerate(pairs):
            b.strip(s, x).fill_(0xA5)
            b.strip(s, y).fill_(0x5A)
        if t % 3 == 2:
            plan.recover_strided(*b.args(), torch.tensor(pairs, dtype=torch.int32, device="cuda"))
        else:
            plan.recover_strided(*b.args(), pairs if t % 3 == 0 else [(j, i)] if S == 1 else pairs)
        plan.sync()
        for s, (x, y) in enumerate(pairs):
            for k in (x, y):
                assert np.array_equal(_np(b.strip(s, k)), refs[s][k]), (p, N, s, x, y, k)


def test_ext_all_pairs_small():
    """p = 5 with the maximum 2p-1 = 9 data strips: every one of the C(11,2) = 55 pairs."""
    p, N, nbytes = 5, 9, 4 * 10752 + 300
    b = Batch(p, N, nbytes, 1)
    refs = _stripes(b, p, N, nbytes, 1, 22, 10)
    plan = R.Plan(p, N, nbytes)
    plan.encode_strided(*b.args())
    for i, j in itertools.combinations(range(N + 2), 2):
        b.strip(0, i).fill_(0xA5)
        b.strip(0, j).fill_(0x5A)
        plan.recover_strided(*b.args(), [(i, j)])
        plan.sync()
        for k in range(N + 2):
            assert np.array_equal(_np(b.strip(0, k)), refs[0][k]), (i, j, k)


def test_ext_single_stripe_api():
    p, N, nbytes = 13, 25, 777
    rng = np.random.default_rng(5)
    data = [rng.integers(0, 256, nbytes, dtype=np.uint8) for _ in range(N)]
    P, Q = oracle.encode_ext(p, data, nbytes)
    pb = R.parity_bytes(p, nbytes)
    strips = [torch.from_numpy(d).cuda() for d in data] + [torch.zeros(pb, dtype=torch.uint8, device="cuda")
                                                            for _ in range(2)]
    R.encode(p, N, strips[:N], strips[N], strips[N + 1], nbytes)
    assert np.array_equal(_np(strips[N]), P) and np.array_equal(_np(strips[N + 1]), Q)
    orig = data + [P, Q]
    for i, j in [(3, 20), (14, 22), (0, N), (24, N + 1)]:
        strips[i].fill_(0)
        strips[j].fill_(0)
        R.recover(p, N, i, j, strips, nbytes)
        assert np.array_equal(_np(strips[i]), orig[i]) and np.array_equal(_np(strips[j]), orig[j])


@pytest.mark.parametrize("p,N,nbytes,S", [(13, 25, 2 * 12288 + 99, 2), (61, 100, 15360 + 17, 2), (11, 21, 3000, 2)])
def test_ext_update_and_scrub(p, N, nbytes, S):
    b = Batch(p, N, nbytes, S)
    b.fill_synthetic(seed=23, cfg=10)
    plan = R.Plan(p, N, nbytes)
    plan.encode_strided(*b.args())
    cnt = torch.zeros(S, dtype=torch.int32, device="cuda")
    plan.scrub_strided(*b.args(), cnt)
    plan.sync()
    assert cnt.cpu().tolist() == [0] * S
    ns = R.aligned_stride(nbytes)
    new = torch.empty((S, ns), dtype=torch.uint8, device="cuda")
    R.fill(new, ns, ns, nbytes, 1, S, 24, 10, 0, 0, 0)
    disks = [N - 1 - s for s in range(S)]  # extended-part strips (k >= p)
    plan.update_strided(*b.args(), new, ns, disks)
    plan.sync()
    for s in range(S):
        data = synthetic.stripe_strips(23, 10, s, N, nbytes)
        data[disks[s]] = _np(new[s, :nbytes])
        P, Q = oracle.encode_ext(p, data, nbytes)
        assert np.array_equal(_np(b.strip(s, N)), P) and np.array_equal(_np(b.strip(s, N + 1)), Q)
    b.strip(0, p + 1)[5] ^= 0x10
    b.strip(S - 1, N + 1)[7] ^= 0x01
    plan.scrub_strided(*b.args(), cnt)
    plan.sync()
    got = cnt.cpu().tolist()
    for s in range(S):
        strips = [_np(b.strip(s, k)).copy() for k in range(N + 2)]
        assert got[s] == oracle.count_bad_words(p, N, strips, nbytes) and got[s] >= 1
