"""Randomised differential test (fixed seeds): random odd prime p <= 257 (fast and generic
kernels), random N (basic code, and the extended code of Eq. (qext) when p satisfies
Theorem 25.3), random strip length (ragged tails, lengths below one word group), random stripe
count, pointer offset and per-stripe erasure pairs -- GPU encode and recovery through the C ABI
against the CPU oracle, byte for byte.  Each case is small enough for the oracle."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import oracle  # noqa: E402
from paper_cs_0611109_b200 import raid6c as R  # noqa: E402
from tests.gpu_util import Batch  # noqa: E402

PRIMES = [p for p in range(3, 258) if all(p % q for q in range(2, int(p ** 0.5) + 1))]

FAST = [3, 5, 7, 11, 13, 17, 19, 29, 37, 53, 59, 61, 257,
        23, 31, 41, 43, 47, 73, 89, 97, 101, 109, 113, 137, 193, 233, 241]


def _case(seed):
    rng = np.random.default_rng(1000 + seed)
    p = int(rng.choice(FAST if rng.random() < 0.5 else PRIMES))
    if R.ext_supported(p) and rng.random() < 0.35:
        N = min(2 * p - 1, p + int(rng.integers(1, 24)))  # extended code (Eq. (qext))
    else:
        N = int(rng.integers(1, min(p, 40) + 1))
    nbytes = int(rng.choice([1, 2, 7, 31, 100, 999, 4096, 12345, 40000]))
    if N > 64:
        nbytes = min(nbytes, 4096)  # keep the oracle fast
    S = int(rng.integers(1, 4))
    offset = int(rng.choice([0, 0, 0, 4, 9]))
    return rng, p, N, nbytes, S, offset


@pytest.mark.parametrize("seed", range(40))
def test_fuzz_encode_recover_vs_oracle(seed):
    rng, p, N, nbytes, S, offset = _case(seed)
    b = Batch(p, N, nbytes, S, offset=offset, align=256 if offset == 0 else 0)
    refs = []
    for s in range(S):
        data = [rng.integers(0, 256, nbytes, dtype=np.uint8) for _ in range(N)]
        if rng.random() < 0.2:  # sparse stripe
            for d in data:
                d[rng.random(nbytes) < 0.9] = 0
        b.set_data_numpy(s, data)
        P, Q = (oracle.encode_ext if N > p else oracle.encode)(p, data, nbytes)
        refs.append(data + [P, Q])
    plan = R.Plan(p, N, nbytes)
    b.par.fill_(0x3C)
    plan.encode_strided(*b.args())
    plan.sync()
    for s in range(S):
        assert np.array_equal(b.numpy_strip(s, N), refs[s][N]), (p, N, nbytes, s, "P")
        assert np.array_equal(b.numpy_strip(s, N + 1), refs[s][N + 1]), (p, N, nbytes, s, "Q")
    for rnd in range(3):
        pairs = []
        for s in range(S):
            i, j = (int(v) for v in rng.choice(N + 2, 2, replace=False))
            pairs.append((i, j))
            for k in (i, j):
                b.strip(s, k).fill_(int(rng.integers(0, 256)))
        er = torch.tensor(pairs, dtype=torch.int32, device="cuda") if rnd == 1 else pairs
        plan.recover_strided(*b.args(), er)
        plan.sync()
        for s, (i, j) in enumerate(pairs):
            for k in (i, j):
                assert np.array_equal(b.numpy_strip(s, k), refs[s][k]), (p, N, nbytes, S, offset, s, (i, j), k)
    plan.close()
