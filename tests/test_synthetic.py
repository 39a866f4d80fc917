"""The seeded input generator (synthetic/): determinism, sub-range consistency, the
sparse-byte distribution of config 4, and the erasure-pair draw of config 5."""
import numpy as np

import synthetic


def test_deterministic_and_subranges():
    a = synthetic.strip_bytes(0, 2, 5, 3, 1000)
    b = synthetic.strip_bytes(0, 2, 5, 3, 1000)
    assert np.array_equal(a, b) and a.dtype == np.uint8 and a.size == 1000
    for lo, hi in [(0, 7), (3, 11), (8, 16), (999, 1000), (123, 877)]:
        assert np.array_equal(synthetic.strip_bytes(0, 2, 5, 3, 1000, lo=lo, hi=hi), a[lo:hi])
    assert not np.array_equal(a, synthetic.strip_bytes(0, 2, 5, 4, 1000))
    assert not np.array_equal(a, synthetic.strip_bytes(0, 2, 6, 3, 1000))
    assert not np.array_equal(a, synthetic.strip_bytes(1, 2, 5, 3, 1000))


def test_known_first_word():
    # SplitMix64 finalizer of key 0 (seed 0, cfg 0, stripe 0, strip 0, k 0) is 0.
    assert int(synthetic.mix64(np.array([0], np.uint64))[0]) == 0
    # and of 1 (standard SplitMix64 finalizer value)
    assert int(synthetic.mix64(np.array([1], np.uint64))[0]) == 0x5692161D100B05E5


def test_uniform_and_sparse_distribution():
    u = synthetic.strip_bytes(0, 4, 0, 0, 1 << 20)
    assert abs(u.mean() - 127.5) < 1.0
    s = synthetic.strip_bytes(0, 4, 1, 0, 1 << 20, sparse=True)
    z = (s == 0).mean()
    assert 0.895 < z < 0.905
    nz = s[s != 0]
    assert nz.min() >= 1 and nz.max() == 255


def test_pairs_and_classes():
    N = 12
    pairs = synthetic.all_pairs(N)
    assert len(pairs) == 91
    cls = [synthetic.pair_class(N, i, j) for i, j in pairs]
    assert cls.count("DD") == 66 and cls.count("DP") == 12 and cls.count("DQ") == 12 and cls.count("PQ") == 1
    seen = set()
    for s in range(2000):
        i, j = synthetic.erasure_pair(0, 5, s, 60)
        assert 0 <= i < j < 62
        seen.add(synthetic.pair_class(60, i, j))
    assert seen == {"DD", "DP", "DQ", "PQ"}
