"""Pins for the NEXT-3 oracle: GF(2^8) Reed-Solomon RAID-6 exactly as the paper's Sec. 4.1-4.4
describe it (the comparison system), against the printed matrix Eq. (g02), the paper's two
byte formulas, textbook polynomial arithmetic mod 0x11D, field axioms, the §4.4 identities and
brute force."""
import itertools
import os

import numpy as np
import pytest

import oracle
from tests import polyref

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
POLY = 0x11D  # x^8 + x^4 + x^3 + x^2 + 1


def _g02():
    rows = [l.strip() for l in open(os.path.join(GOLD, "rs_g02.txt")) if l.strip() and not l.startswith("#")]
    return np.array([[int(c) for c in r] for r in rows], dtype=np.uint8)


def test_mul2_equals_printed_matrix():
    """Eq. (g02): y = G x for every byte x."""
    G = _g02()
    assert G.shape == (8, 8)
    for x in range(256):
        v = np.array([(x >> i) & 1 for i in range(8)], dtype=np.uint8)
        y = (G.astype(int) @ v) % 2
        assert oracle.rs_mul2(x) == sum(int(b) << i for i, b in enumerate(y))


def test_mul2_signed_formula():
    """int8 y = (x + x) ^ (((x < 0) ? 0xff : 0x00) & 0x1d)."""
    for x in range(256):
        sx = x - 256 if x & 0x80 else x
        y = ((x + x) & 0xFF) ^ ((0xFF if sx < 0 else 0) & 0x1D)
        assert oracle.rs_mul2(x) == y


def test_mul_is_polynomial_product_mod_0x11d():
    for a in range(256):
        for b in range(0, 256, 7):
            assert oracle.rs_mul(a, b) == polyref.polymod(polyref.clmul(a, b), POLY)
    assert oracle.rs_mul(0x80, 0x02) == 0x1D  # SPEC.md:402, from the Sec. 4.2 formula


def test_generator_order_and_inverses():
    """g = {02} generates the multiplicative group: order 255."""
    seen = {oracle.rs_exp(k) for k in range(255)}
    assert len(seen) == 255 and oracle.rs_exp(255) == 1
    for a in range(1, 256):
        assert oracle.rs_mul(a, oracle.rs_inv(a)) == 1
    assert oracle.rs_inv(0) == 0


def test_section_4_4_identities():
    """A = (1 + g^{y-x})^{-1};  B = g^{-x}(1 + g^{y-x})^{-1} = (g^x + g^y)^{-1}."""
    for x, y in [(0, 1), (0, 254), (3, 17), (100, 200), (250, 254)]:
        A = oracle.rs_inv(1 ^ oracle.rs_exp(y - x))
        B = oracle.rs_mul(oracle.rs_inv(oracle.rs_exp(x)), A)
        assert B == oracle.rs_inv(oracle.rs_exp(x) ^ oracle.rs_exp(y))


@pytest.mark.parametrize("N,nbytes", [(1, 5), (4, 33), (12, 100), (64, 17), (255, 3)])
def test_rs_encode_definition(N, nbytes):
    """Eq. (rsparity): Q = sum g^i D_i with products by textbook polynomial arithmetic."""
    rng = np.random.default_rng(N)
    data = [rng.integers(0, 256, nbytes, dtype=np.uint8) for _ in range(N)]
    P, Q = oracle.rs_encode(data)
    for b in range(nbytes):
        q = p = 0
        for i in range(N):
            gi = polyref.polymod(1 << 0, POLY)
            for _ in range(i):
                gi = polyref.polymod(gi << 1, POLY)
            q ^= polyref.polymod(polyref.clmul(gi, int(data[i][b])), POLY)
            p ^= int(data[i][b])
        assert (P[b], Q[b]) == (p, q)


@pytest.mark.parametrize("N,nbytes", [(1, 9), (3, 20), (12, 31), (40, 7)])
def test_rs_roundtrip_all_pairs(N, nbytes):
    rng = np.random.default_rng(N + 1)
    data = [rng.integers(0, 256, nbytes, dtype=np.uint8) for _ in range(N)]
    P, Q = oracle.rs_encode(data)
    orig = data + [P, Q]
    pairs = list(itertools.combinations(range(N + 2), 2))
    if len(pairs) > 200:
        pairs = pairs[::7]
    for i, j in pairs:
        strips = [s.copy() for s in orig]
        strips[i][:] = 0xA5
        strips[j][:] = 0x5A
        oracle.rs_recover(N, j, i, strips, nbytes)
        for k in range(N + 2):
            assert np.array_equal(strips[k], orig[k]), (i, j, k)


def test_rs_bruteforce_unique():
    N = 3
    data = [np.array([v], np.uint8) for v in (0x12, 0xC3, 0x7E)]
    P, Q = oracle.rs_encode(data)
    full = [0x12, 0xC3, 0x7E, int(P[0]), int(Q[0])]

    def holds(v):
        q = 0
        for i in range(N):
            q ^= oracle.rs_mul(oracle.rs_exp(i), v[i])
        return v[0] ^ v[1] ^ v[2] == v[3] and q == v[4]

    for i, j in itertools.combinations(range(N + 2), 2):
        sols = []
        for a in range(256):
            for b in range(256):
                v = list(full)
                v[i], v[j] = a, b
                if holds(v):
                    sols.append((a, b))
        assert sols == [(full[i], full[j])]
