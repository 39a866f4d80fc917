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


def _digest_loop(b):
    """The digest definition written out with Python integers (tiny inputs only)."""
    M = (1 << 64) - 1

    def mix(z):
        z &= M
        z ^= z >> 30
        z = (z * 0xBF58476D1CE4E5B9) & M
        z ^= z >> 27
        z = (z * 0x94D049BB133111EB) & M
        return z ^ (z >> 31)

    h = mix(len(b) ^ 0xBB67AE8584CAA73B)
    for k in range(0, (len(b) + 7) // 8):
        w = int.from_bytes(bytes(b[8 * k:8 * k + 8]).ljust(8, b"\0"), "little")
        h = (h + mix(w + k * 0x9E3779B97F4A7C15 + 0x6A09E667F3BCC909)) & M
    return h


def test_digest_definition_and_sensitivity():
    rng = np.random.default_rng(7)
    for n in [0, 1, 7, 8, 9, 63, 64, 100, 1001]:
        b = rng.integers(0, 256, n, dtype=np.uint8)
        d = synthetic.digest(b)
        assert d == _digest_loop(b), n
        if n:
            c = b.copy()
            c[rng.integers(0, n)] ^= np.uint8(1 << int(rng.integers(0, 8)))
            assert synthetic.digest(c) != d  # one flipped bit always changes it
            c = np.roll(b, 8)
            if not np.array_equal(c, b):
                assert synthetic.digest(c) != d  # position-sensitive
    # zero padding past len is not the same as a longer strip of zeros
    assert synthetic.digest(np.zeros(9, np.uint8)) != synthetic.digest(np.zeros(16, np.uint8))
    # chunked evaluation (> 4 Mi words) equals the single-pass definition
    big = np.random.default_rng(3).integers(0, 256, (1 << 25) + 13, dtype=np.uint8)
    w = np.zeros(((big.size + 7) // 8) * 8, np.uint8)
    w[:big.size] = big
    k = np.arange(w.size // 8, dtype=np.uint64)
    with np.errstate(over="ignore"):
        t = synthetic.mix64(w.view("<u8") + k * np.uint64(0x9E3779B97F4A7C15) + np.uint64(0x6A09E667F3BCC909))
        h0 = int(synthetic.mix64(np.array([big.size ^ 0xBB67AE8584CAA73B], np.uint64))[0])
    assert synthetic.digest(big) == (h0 + int(t.sum(dtype=np.uint64))) % (1 << 64)
    assert synthetic.combine_digests([1, 2]) != synthetic.combine_digests([2, 1])
    # pieces split at 8-byte boundaries add up to the whole
    b = big[:100001]
    parts = (synthetic.word_terms(b[:24000]) + synthetic.word_terms(b[24000:80000], 3000)
             + synthetic.word_terms(b[80000:], 10000))
    assert (synthetic.length_term(b.size) + parts) % (1 << 64) == synthetic.digest(b)
