"""Pins for the NEXT-2 oracle (extended Q-parity, Sec. 3.3 of the paper): Theorem 25.3's
condition against the paper's printed list of failing primes and Corollary 25.4, the cone
property (condition (1)) by explicit inversion, Eq. (qext) against the independent polynomial
definition, reduction to the basic code, brute-force uniqueness and all-pairs round trips."""
import itertools
import random

import numpy as np
import pytest

import oracle
from tests import polyref

PRIMES = [q for q in range(3, 258) if all(q % d for d in range(2, int(q ** 0.5) + 1))]


def test_theorem_25_3_failing_primes():
    """'In the first 500 primes, the only primes that fail are Mersenne and 73'
    -> below 258: the Mersenne primes 3, 7, 31, 127 and 73.  Corollary 25.4:
    Fermat primes N > 3 pass (5, 17, 257), Mersenne primes fail."""
    fails = [p for p in PRIMES if not oracle.ext_condition(p)]
    assert fails == [3, 7, 31, 73, 127]
    for fermat in (5, 17, 257):
        assert oracle.ext_condition(fermat)


@pytest.mark.parametrize("p,passes", [(5, True), (11, True), (13, True), (7, False)])
def test_theorem_25_3_cone_property(p, passes):
    """Condition (1) for g = S_p: every sum of two distinct elements of
    S = {Id, g, ..., g^{p-1}, Id+g, ..., Id+g^{p-1}} is invertible iff p passes."""
    n = p - 1
    S = [oracle.ext_coeff(p, k) for k in range(2 * p - 1)]
    singular = 0
    for a, b in itertools.combinations(range(2 * p - 1), 2):
        if oracle.gf2_inverse(S[a] ^ S[b]) is None:
            singular += 1
    assert (singular == 0) == passes
    for k in range(2 * p - 1):
        assert oracle.gf2_inverse(S[k]) is not None  # every coefficient itself invertible


def _ext_poly(p, k):
    return polyref.xk(p, k) if k < p else polyref.polymod(1 ^ (1 << (k - p + 1)), polyref.phi(p))


@pytest.mark.parametrize("p,D,nbytes", [(5, 9, 7), (13, 25, 11), (17, 33, 6), (11, 21, 9), (59, 70, 30)])
def test_encode_ext_matches_polynomial_definition(p, D, nbytes):
    """Eq. (qext): Q = sum_{k<p} x^k d_k + sum_{k>=p} (1 + x^{k-p+1}) d_k."""
    rng = np.random.default_rng(p + D)
    data = [rng.integers(0, 256, nbytes, dtype=np.uint8) for _ in range(D)]
    P, Q = oracle.encode_ext(p, data, nbytes)
    n = p - 1
    W = oracle.word_count(p, nbytes)
    pb = oracle.parity_bytes(p, nbytes)
    ws = [polyref.words_of(d.tobytes(), nbytes, n, W) for d in data]
    qw = [0] * W
    pw = [0] * W
    for k in range(D):
        c = _ext_poly(p, k)
        for w in range(W):
            pw[w] ^= ws[k][w]
            qw[w] ^= polyref.ring_mul(p, c, ws[k][w])
    assert P.tobytes() == polyref.bytes_of(pw, n, pb) and Q.tobytes() == polyref.bytes_of(qw, n, pb)


@pytest.mark.parametrize("p,D", [(5, 5), (13, 7), (17, 17), (61, 9)])
def test_encode_ext_reduces_to_basic(p, D):
    rng = np.random.default_rng(D)
    data = [rng.integers(0, 256, 13, dtype=np.uint8) for _ in range(D)]
    a, b = oracle.encode_ext(p, data), oracle.encode(p, data)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


def test_encode_ext_rejects():
    with pytest.raises(ValueError):
        oracle.encode_ext(7, [np.zeros(3, np.uint8)] * 8)   # 7 fails Theorem 25.3
    with pytest.raises(ValueError):
        oracle.encode_ext(5, [np.zeros(3, np.uint8)] * 10)  # D > 2p - 1


@pytest.mark.parametrize("p,D", [(5, 9), (5, 7)])
def test_ext_bruteforce_unique_recovery(p, D):
    """Lemma 23.2 with the cone of Theorem 25.3: every pair has exactly one solution (all
    2^{2n} candidates enumerated, parity equations evaluated with tests/polyref.py)."""
    n = p - 1
    rng = random.Random(D)
    words = [rng.randrange(1 << n) for _ in range(D)]
    P, Q = oracle.encode_ext(p, [np.array([w], np.uint8) for w in words], 1)
    full = words + [int(P[0]) & ((1 << n) - 1), int(Q[0]) & ((1 << n) - 1)]
    cs = [_ext_poly(p, k) for k in range(D)]

    def holds(v):
        ps = qs = 0
        for k in range(D):
            ps ^= v[k]
            qs ^= polyref.ring_mul(p, cs[k], v[k])
        return ps == v[D] and qs == v[D + 1]

    for i, j in itertools.combinations(range(D + 2), 2):
        sols = [(a, b) for a in range(1 << n) for b in range(1 << n)
                if holds(full[:i] + [a] + full[i + 1:j] + [b] + full[j + 1:])]
        assert sols == [(full[i], full[j])]
        strips = [np.array([w], np.uint8) for w in full[:D]] + [P.copy(), Q.copy()]
        strips[i][:] = 0
        strips[j][:] = 0
        oracle.recover_ext(p, D, i, j, strips, 1)
        assert (int(strips[i][0]) & ((1 << n) - 1), int(strips[j][0]) & ((1 << n) - 1)) == sols[0]


@pytest.mark.parametrize("p,D,nbytes", [(5, 9, 9), (13, 25, 10), (17, 33, 8), (11, 15, 7)])
def test_ext_roundtrip_pairs(p, D, nbytes):
    rng = np.random.default_rng(p * D)
    data = [rng.integers(0, 256, nbytes, dtype=np.uint8) for _ in range(D)]
    P, Q = oracle.encode_ext(p, data, nbytes)
    orig = data + [P, Q]
    pairs = list(itertools.combinations(range(D + 2), 2))
    if len(pairs) > 120:
        pairs = [pairs[i] for i in rng.choice(len(pairs), 120, replace=False)]
        pairs += [(0, D + 1), (D - 1, D), (p, p + 1), (0, p), (p - 1, D - 1), (D, D + 1)]
    for i, j in pairs:
        strips = [s.copy() for s in orig]
        strips[i][:] = 0xA5
        strips[j][:] = 0x5A
        oracle.recover_ext(p, D, j, i, strips, nbytes)
        for k in range(D + 2):
            assert np.array_equal(strips[k], orig[k]), (i, j, k)


def test_ext_recover_basic_agrees_with_section_4():
    """For D <= p the Lemma 23.2 formulas (recover_ext) and the Sec. 4.3/4.6 formulas (recover)
    are two derivations of the same unique solution."""
    p, D, nbytes = 13, 12, 20
    rng = np.random.default_rng(3)
    data = [rng.integers(0, 256, nbytes, dtype=np.uint8) for _ in range(D)]
    P, Q = oracle.encode(p, data, nbytes)
    for i, j in [(0, 1), (3, 9), (2, D), (5, D + 1), (D, D + 1)]:
        a = [s.copy() for s in data + [P, Q]]
        b = [s.copy() for s in data + [P, Q]]
        oracle.recover(p, D, i, j, a, nbytes)
        oracle.recover_ext(p, D, i, j, b, nbytes)
        assert all(np.array_equal(x, y) for x, y in zip(a, b))


@pytest.mark.parametrize("p", [5, 13, 17])
def test_ext_coeff_matrices(p):
    """g_k of Eq. (qext) equals S^k (k < p) and Id + S^{k-p+1} (k >= p), with S^k built by
    repeated matrix multiplication (oracle_sylvester_power) -- two constructions agree."""
    n = p - 1
    I = np.eye(n, dtype=np.uint8)
    for k in range(2 * p - 1):
        expect = oracle.sylvester_power(p, k) if k < p else oracle.sylvester_power(p, k - p + 1) ^ I
        np.testing.assert_array_equal(oracle.ext_coeff(p, k), expect)
