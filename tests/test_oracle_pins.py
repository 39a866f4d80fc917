"""Pins the CPU oracle (oracle/) to things other than itself: values printed in the
paper (tests/golden/, each with its citation), closed forms, invariants, special
cases, an independent polynomial-arithmetic definition (tests/polyref.py) and brute
force on tiny inputs.  CPU only."""
import itertools
import os
import random

import numpy as np
import pytest

import oracle
from tests import polyref

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = os.path.join(HERE, "golden")
PRIMES_SMALL = [3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37, 41, 43, 47, 53, 59, 61]


def _lines(name):
    with open(os.path.join(GOLD, name)) as f:
        return [l.rstrip("\n") for l in f if l.strip() and not l.startswith("#")]


def _bitmat(rows):
    return np.array([[int(c) for c in r] for r in rows], dtype=np.uint8)


def _sections(name):
    out, cur = {}, None
    for l in _lines(name):
        if l.startswith("["):
            cur = l[1:l.index("]")]
            out[cur] = []
        else:
            out[cur].append(l)
    return out


# ------------------------------------------------------------ multiplication by x
def test_sylvester_equals_z17_display():
    """the printed 16x16 matrix is S_17."""
    G = _bitmat(_lines("z17_multiply_by_g.txt"))
    assert G.shape == (16, 16)
    np.testing.assert_array_equal(oracle.sylvester(17), G)


def test_mul_x_unit_vectors_z17():
    """y = (x15, x0^x15, ..., x14^x15)."""
    for j in range(16):
        expect = (1 << (j + 1)) if j < 15 else 0xFFFF
        assert oracle.mul_x(17, 1 << j) == expect


def test_sylvester_small_instances():
    """Lemma 26.1 pattern: S_5 and S_3 = G."""
    np.testing.assert_array_equal(oracle.sylvester(5), _bitmat(_lines("sylvester_S5.txt")))
    g = _sections("gf4_p3.txt")
    np.testing.assert_array_equal(oracle.sylvester(3), _bitmat(g["G"]))
    I = np.eye(2, dtype=np.uint8)
    np.testing.assert_array_equal(oracle.sylvester(3) ^ I, _bitmat(g["Id+G"]))
    order = int(g["order"][0])
    np.testing.assert_array_equal(oracle.sylvester_power(3, order), I)
    assert not np.array_equal(oracle.sylvester_power(3, 1), I)
    assert not np.array_equal(oracle.sylvester_power(3, 2), I)


def _int16(v):
    v &= 0xFFFF
    return v - 0x10000 if v & 0x8000 else v


def test_mul_x_int16_formula():
    """int16 y = (x + x) ^ ((x < 0) ? 0xffff : 0x0000)."""
    rng = random.Random(1)
    xs = [0, 1, 0x7FFF, 0x8000, 0xFFFF] + [rng.randrange(1 << 16) for _ in range(300)]
    for x in xs:
        y = ((x + x) & 0xFFFF) ^ (0xFFFF if _int16(x) < 0 else 0)
        assert oracle.mul_x(17, x) == y


def test_mul_xk_formula_16bit_logical():
    """y = (x << k) ^ (x >> (17-k)) ^ (((x << (k-1)) < 0) ? 0xffff : 0),
    read with 16-bit logical shifts and a bit-15 test (R9)."""
    rng = random.Random(2)
    for k in range(1, 17):
        for x in [0x0001, 0x8000, 0xFFFF] + [rng.randrange(1 << 16) for _ in range(40)]:
            sh = (x << (k - 1)) & 0xFFFF
            y = ((x << k) & 0xFFFF) ^ (x >> (17 - k)) ^ (0xFFFF if sh & 0x8000 else 0)
            assert oracle.mul_xk(17, k, x) == y, (k, hex(x))


@pytest.mark.parametrize("p", [3, 5, 7, 13, 17, 59, 61])
def test_powers_closed_form(p):
    """Eq. (powers): with the paper's labels X_m = component m of the
    vector written (x_{N-1}, ..., x_1) top to bottom (so X_m = bit n-m),
    S^k X = (X_k, ..., X_k) + (X_{k-1}, ..., X_1, 0, X_{N-1}, ..., X_{k+1})."""
    n = p - 1
    rng = random.Random(p)
    for k in range(1, p + 1):
        for _ in range(6):
            v = rng.randrange(1 << n)
            X = lambda m: ((v >> (n - m)) & 1) if 1 <= m <= n else 0
            second = []
            for r in range(n):
                if r < k - 1:
                    second.append(X(k - 1 - r))
                elif r == k - 1:
                    second.append(0)
                else:
                    second.append(X(p - 1 - (r - k)))
            expect = sum(((X(k) ^ second[r]) << r) for r in range(n))
            assert oracle.mul_xk(p, k, v) == expect


@pytest.mark.parametrize("p", PRIMES_SMALL + [97, 257])
def test_mul_xk_matches_polynomial_definition(p):
    """x^k a in F2[x]/(Phi_p) by carry-less multiply + long division (tests/polyref.py)."""
    n = p - 1
    rng = random.Random(100 + p)
    for _ in range(8):
        k = rng.randrange(0, p + 2)
        a = rng.randrange(1 << n)
        assert oracle.mul_xk(p, k, a) == polyref.ring_mul(p, polyref.xk(p, k), a)


# ------------------------------------------------------------ group structure
@pytest.mark.parametrize("p", [3, 5, 7, 11, 13, 17])
def test_lemma_26_1_order_and_invertibility(p):
    """Lemma 26.1(i)-(ii), and Lemma 24.3 (Id + g^m invertible,
    PAPER.md:478-511): S^p = Id, S^k != Id (0<k<p), Id + S^m invertible (0<m<p),
    and the char. polynomial relation sum_k S^k = 0 (Lemma 24.2, Eq. (rootsum))."""
    n = p - 1
    I = np.eye(n, dtype=np.uint8)
    np.testing.assert_array_equal(oracle.sylvester_power(p, p), I)
    acc = np.zeros((n, n), np.uint8)
    for k in range(p):
        Sk = oracle.sylvester_power(p, k)
        acc ^= Sk
        if 0 < k:
            assert not np.array_equal(Sk, I)
            assert oracle.gf2_inverse(Sk ^ I) is not None
    np.testing.assert_array_equal(acc, np.zeros((n, n), np.uint8))


def test_even_order_degenerate():
    """Lemma 26.1(ii): Id + S_N is degenerate for even N (inverse(Id+S_4))."""
    S4 = oracle.sylvester(4)
    assert oracle.gf2_inverse(S4 ^ np.eye(3, dtype=np.uint8)) is None
    S6 = oracle.sylvester(6)
    assert oracle.gf2_inverse(S6 ^ np.eye(5, dtype=np.uint8)) is None


def test_gauss_jordan_inverse_is_inverse():
    rng = np.random.default_rng(5)
    for n in [2, 4, 12, 16, 40]:
        for _ in range(4):
            M = rng.integers(0, 2, (n, n), dtype=np.uint8)
            R = oracle.gf2_inverse(M)
            if R is not None:
                np.testing.assert_array_equal(oracle.gf2_matmul(M, R), np.eye(n, dtype=np.uint8))


# ------------------------------------------------------------ inverse of 1 + x^z
def test_inverse_series_z17():
    """g^{-k} = g^{17-k}; (1+g)^{-1} = 1 + g^2 + ... + g^16;
    (1+g^z)^{-1} = 1 + g^{2z} + ... + g^{16z}."""
    p, n = 17, 16
    I = np.eye(n, dtype=np.uint8)
    for k in range(1, 17):
        np.testing.assert_array_equal(oracle.gf2_matmul(oracle.sylvester_power(p, k),
                                                        oracle.sylvester_power(p, 17 - k)), I)
    for z in range(1, 17):
        series = np.zeros((n, n), np.uint8)
        for m in range(9):
            series ^= oracle.sylvester_power(p, (2 * z * m) % p)
        inv = oracle.gf2_inverse(oracle.sylvester_power(p, z) ^ I)
        np.testing.assert_array_equal(inv, series)
    # derived value (Appendix A): (1+x)^{-1} = x + x^3 + ... + x^15 = 0xAAAA
    inv1 = oracle.gf2_inverse(oracle.sylvester(17) ^ I)
    col0 = oracle.gf2_matvec(inv1, np.array([1] + [0] * 15, np.uint8))
    assert sum(int(b) << j for j, b in enumerate(col0)) == 0xAAAA


@pytest.mark.parametrize("p", [3, 5, 7, 13, 59, 61])
def test_inverse_series_general_p(p):
    """Reading R11: (1+x^z)^{-1} = sum_{m=0}^{(p-1)/2} x^{2zm} for every odd prime p."""
    n = p - 1
    I = np.eye(n, dtype=np.uint8)
    for z in ([1, 2, p - 1] if p > 13 else range(1, p)):
        series = np.zeros((n, n), np.uint8)
        for m in range((p + 1) // 2):
            series ^= oracle.sylvester_power(p, (2 * z * m) % p)
        np.testing.assert_array_equal(oracle.gf2_inverse(oracle.sylvester_power(p, z) ^ I), series)


@pytest.mark.parametrize("p", [3, 5, 7, 11, 13])
def test_inverse_bruteforce_ring(p):
    """Brute-force ring inversion on tiny p: the unique c in R_p with (1 + x^z) c = 1
    (polynomial arithmetic, tests/polyref.py) equals the oracle's Gauss-Jordan inverse."""
    n = p - 1
    I = np.eye(n, dtype=np.uint8)
    for z in range(1, p):
        a = polyref.polymod(1 ^ (1 << z), polyref.phi(p))
        sols = [c for c in range(1 << n) if polyref.ring_mul(p, a, c) == 1]
        assert len(sols) == 1
        inv = oracle.gf2_inverse(oracle.sylvester_power(p, z) ^ I)
        col0 = oracle.gf2_matvec(inv, np.array([1] + [0] * (n - 1), np.uint8))
        assert sum(int(b) << j for j, b in enumerate(col0)) == sols[0]


# ------------------------------------------------------------ Appendix A (derived)
def test_appendix_a_vectors():
    s = _sections("appendix_a.txt")
    h = lambda sec: [int(t, 16) for t in s[sec][0].split()]
    assert [oracle.mul_xk(5, k, 0x8) for k in range(6)] == h("mul_xk p=5 a=0x8")
    assert [oracle.mul_xk(5, k, 0x1) for k in range(6)] == h("mul_xk p=5 a=0x1")
    I = np.eye(4, dtype=np.uint8)
    got = []
    for z in range(1, 5):
        inv = oracle.gf2_inverse(oracle.sylvester_power(5, z) ^ I)
        col0 = oracle.gf2_matvec(inv, np.array([1, 0, 0, 0], np.uint8))
        got.append(sum(int(b) << j for j, b in enumerate(col0)))
    assert got == h("inv_one_plus_xz p=5")
    # one word per disk: strips of 1 byte hold 2 nibble-words; use the low nibble
    d = [np.array([v], np.uint8) for v in (1, 2, 4, 8)]
    P, Q = oracle.encode(5, d)
    assert [P[0] & 0xF, Q[0] & 0xF] == h("encode_words p=5 N=4")
    d = [np.array([v], np.uint8) for v in (0x21, 0x43, 0x65, 0x97)]
    P, Q = oracle.encode(5, d)
    assert [int(P[0]), int(Q[0])] == h("encode_bytes p=5 N=4")
    e = h("p=17")
    assert oracle.mul_x(17, 0x8000) == e[0]
    assert oracle.mul_xk(17, 16, 0x0001) == e[1]
    # layout pins
    rows = s["layout p=13 N=2"]
    P, Q = oracle.encode(13, [np.zeros(3, np.uint8), np.array([0xAB, 0xCD, 0xEF], np.uint8)])
    assert list(P) == [int(t, 16) for t in rows[0].split()]
    assert list(Q) == [int(t, 16) for t in rows[1].split()]
    P, Q = oracle.encode(17, [np.zeros(2, np.uint8), np.array([0x01, 0x80], np.uint8)])
    assert list(Q) == [int(t, 16) for t in s["layout p=17 N=2"][0].split()]


# ------------------------------------------------------------ the small codes of Sec. 2
def _parse_eqs(rows):
    eqs = []
    for r in rows:
        lhs, rhs = r.split("=")
        eqs.append((lhs.strip(), [t.strip() for t in rhs.split("+")]))
    return eqs


def test_hordiag_exhaustive():
    """Eq. (hordiag), over all 16 inputs (p = 3, N = 2)."""
    s = _sections("hordiag_p3.txt")
    eqs = _parse_eqs(s[[k for k in s if k.startswith("hordiag")][0]])
    for d11, d12, d21, d22 in itertools.product([0, 1], repeat=4):
        env = dict(d11=d11, d12=d12, d21=d21, d22=d22)
        s1 = np.array([d11 | (d12 << 1)], np.uint8)
        s2 = np.array([d21 | (d22 << 1)], np.uint8)
        P, Q = oracle.encode(3, [s1, s2])
        got = dict(pi11=P[0] & 1, pi12=(P[0] >> 1) & 1, pi21=Q[0] & 1, pi22=(Q[0] >> 1) & 1)
        for lhs, terms in eqs:
            assert got[lhs] == sum(env[t] for t in terms) % 2, (lhs, env)


def test_hordiag_recovery_display_exhaustive():
    """Recovery display: both data disks lost, rebuilt from the parities."""
    s = _sections("hordiag_p3.txt")
    eqs = _parse_eqs(s[[k for k in s if k.startswith("recovery")][0]])
    for d11, d12, d21, d22 in itertools.product([0, 1], repeat=4):
        s1 = np.array([d11 | (d12 << 1)], np.uint8)
        s2 = np.array([d21 | (d22 << 1)], np.uint8)
        P, Q = oracle.encode(3, [s1, s2])
        pi = dict(pi11=P[0] & 1, pi12=(P[0] >> 1) & 1, pi21=Q[0] & 1, pi22=(Q[0] >> 1) & 1)
        strips = [np.array([0xFF], np.uint8), np.array([0x5A], np.uint8), P.copy(), Q.copy()]
        oracle.recover(3, 2, 0, 1, strips, 1)
        got = dict(d11=strips[0][0] & 1, d12=(strips[0][0] >> 1) & 1,
                   d21=strips[1][0] & 1, d22=(strips[1][0] >> 1) & 1)
        for lhs, terms in eqs:
            assert got[lhs] == sum(pi[t] for t in terms) % 2


def test_gf4_five_disk_code():
    """Eq. (gf4)/(p52): pi_2 = d1 + G d2 + G^2 d3 (p = 3, N = 3)."""
    G = _bitmat(_sections("gf4_p3.txt")["G"])
    G2 = (G.astype(int) @ G.astype(int) % 2).astype(np.uint8)
    for vals in itertools.product(range(4), repeat=3):
        strips = [np.array([v], np.uint8) for v in vals]
        P, Q = oracle.encode(3, strips)
        bits = [np.array([v & 1, v >> 1], np.uint8) for v in vals]
        q = bits[0] ^ (G.astype(int) @ bits[1] % 2).astype(np.uint8) ^ (G2.astype(int) @ bits[2] % 2).astype(np.uint8)
        assert (Q[0] & 3) == int(q[0]) | (int(q[1]) << 1)
        assert (P[0] & 3) == vals[0] ^ vals[1] ^ vals[2]


# ------------------------------------------------------------ encode invariants
def _rand_strips(rng, N, nbytes):
    return [rng.integers(0, 256, nbytes, dtype=np.uint8) for _ in range(N)]


@pytest.mark.parametrize("p,N,nbytes", [(3, 3, 7), (5, 4, 9), (7, 6, 13), (13, 12, 31),
                                        (17, 17, 10), (59, 58, 29), (61, 60, 23), (257, 5, 70),
                                        (11, 1, 5), (13, 13, 3)])
def test_encode_matches_polynomial_definition(p, N, nbytes):
    """Q = sum x^i d_i in F2[x]/(Phi_p), per word, via tests/polyref.py (independent of the
    Sylvester-step Horner the oracle uses); ragged lengths exercise the zero-extended tail."""
    rng = np.random.default_rng(p * 1000 + N)
    data = _rand_strips(rng, N, nbytes)
    P, Q = oracle.encode(p, data)
    Pr, Qr = polyref.encode_ref(p, [d.tobytes() for d in data], nbytes)
    assert P.tobytes() == Pr and Q.tobytes() == Qr


@pytest.mark.parametrize("p,N", [(3, 3), (5, 4), (7, 7), (13, 12), (17, 5)])
def test_encode_matrix_tier_equals_horner(p, N):
    """Tier A (S^i mat-vec, Corollary 24.4 matrix) == Horner."""
    rng = np.random.default_rng(7 + p)
    data = _rand_strips(rng, N, 11)
    assert all(np.array_equal(a, b) for a, b in zip(oracle.encode(p, data), oracle.encode(p, data, matrix=True)))


@pytest.mark.parametrize("p", [3, 5, 13, 17, 59, 61])
def test_rootsum_identical_strips(p):
    """Lemma 24.2 (Eq. (rootsum)): N = p identical strips -> Q = 0, P = d."""
    rng = np.random.default_rng(p)
    d = rng.integers(0, 256, 17, dtype=np.uint8)
    P, Q = oracle.encode(p, [d] * p)
    assert not Q.any()
    W = oracle.word_count(p, 17)
    assert P[:17].tobytes() == d.tobytes()
    assert P.size == oracle.parity_bytes(p, 17) and W * (p - 1) <= 8 * P.size


def test_zero_linearity_impulse():
    """All-zero -> 0; linearity; impulse: only disk i nonzero -> P = d, Q = x^i d."""
    p, N, nb = 13, 6, 9
    rng = np.random.default_rng(3)
    Z = [np.zeros(nb, np.uint8)] * N
    P, Q = oracle.encode(p, Z)
    assert not P.any() and not Q.any()
    a, b = _rand_strips(rng, N, nb), _rand_strips(rng, N, nb)
    Pa, Qa = oracle.encode(p, a)
    Pb, Qb = oracle.encode(p, b)
    Pab, Qab = oracle.encode(p, [x ^ y for x, y in zip(a, b)])
    assert np.array_equal(Pab, Pa ^ Pb) and np.array_equal(Qab, Qa ^ Qb)
    for i in range(N):
        d = [np.zeros(nb, np.uint8) for _ in range(N)]
        d[i] = a[i]
        P, Q = oracle.encode(p, d)
        W = oracle.word_count(p, nb)
        words = polyref.words_of(a[i].tobytes(), nb, p - 1, W)
        qw = polyref.words_of(Q.tobytes(), P.size, p - 1, W)
        assert all(qw[w] == oracle.mul_xk(p, i, words[w]) for w in range(W))


def test_sizes_at_configs():
    """W and parity_bytes at BASELINE.json configs."""
    assert (oracle.word_count(5, 65536), oracle.parity_bytes(5, 65536)) == (131072, 65536)
    assert (oracle.word_count(13, 4 << 20), oracle.parity_bytes(13, 4 << 20)) == (2796203, 4194305)
    assert (oracle.word_count(257, 16 << 20), oracle.parity_bytes(257, 16 << 20)) == (524288, 16 << 20)
    assert (oracle.word_count(59, 8 << 20), oracle.parity_bytes(59, 8 << 20)) == (1157050, 8388613)
    assert (oracle.word_count(61, 32 << 20), oracle.parity_bytes(61, 32 << 20)) == (4473925, 33554438)


def test_invalid_arguments():
    with pytest.raises(ValueError):
        oracle.encode(9, [np.zeros(3, np.uint8)] * 2)      # not prime
    with pytest.raises(ValueError):
        oracle.encode(5, [np.zeros(3, np.uint8)] * 6)      # N > p
    strips = [np.zeros(3, np.uint8)] * 2 + [np.zeros(oracle.parity_bytes(5, 3), np.uint8)] * 2
    with pytest.raises(ValueError):
        oracle.recover(5, 2, 1, 1, [s.copy() for s in strips], 3)


# ------------------------------------------------------------ recovery
def _stripe(p, N, nbytes, rng):
    data = _rand_strips(rng, N, nbytes)
    P, Q = oracle.encode(p, data)
    return data + [P, Q]


@pytest.mark.parametrize("p,N,nbytes", [(3, 1, 4), (3, 3, 5), (5, 4, 7), (7, 2, 6), (13, 12, 10),
                                        (13, 13, 4), (17, 16, 9), (59, 5, 30), (61, 7, 33)])
def test_recover_roundtrip_all_pairs(p, N, nbytes):
    """Encode -> erase every pair (poisoned) -> recover == original (Lemma 23.2,
    PAPER.md:370-406)."""
    rng = np.random.default_rng(p * 31 + N)
    orig = _stripe(p, N, nbytes, rng)
    for i, j in itertools.combinations(range(N + 2), 2):
        strips = [s.copy() for s in orig]
        strips[i][:] = 0xA5
        strips[j][:] = 0x5A
        oracle.recover(p, N, j, i, strips, nbytes)  # reversed order on purpose
        for k in range(N + 2):
            assert np.array_equal(strips[k], orig[k]), (i, j, k)


@pytest.mark.parametrize("p,N", [(3, 2), (3, 3), (5, 3), (5, 5)])
def test_bruteforce_unique_recovery(p, N):
    """Uniqueness (Lemma 23.2, Corollary 24.4): enumerating all 2^{2n} candidates for the two
    lost words, exactly one satisfies both parity equations (checked with the independent
    polynomial definition), and it is what the oracle recovers."""
    n = p - 1
    rng = random.Random(p * 10 + N)
    nbytes = 1
    words = [rng.randrange(1 << n) for _ in range(N)]
    data = [np.array([w], np.uint8) for w in words]  # word 0 = low n bits of the byte
    P, Q = oracle.encode(p, data)
    pw, qw = int(P[0]) & ((1 << n) - 1), int(Q[0]) & ((1 << n) - 1)
    full = words + [pw, qw]

    def holds(v):
        ps = 0
        qs = 0
        for i in range(N):
            ps ^= v[i]
            qs ^= polyref.ring_mul(p, polyref.xk(p, i), v[i])
        return ps == v[N] and qs == v[N + 1]

    for i, j in itertools.combinations(range(N + 2), 2):
        sols = []
        for a in range(1 << n):
            for b in range(1 << n):
                v = list(full)
                v[i], v[j] = a, b
                if holds(v):
                    sols.append((a, b))
        assert sols == [(full[i], full[j])]
        strips = [np.array([v], np.uint8) for v in full[:N]] + [P.copy(), Q.copy()]
        strips[i][:] = 0
        strips[j][:] = 0
        oracle.recover(p, N, i, j, strips, nbytes)
        assert (int(strips[i][0]) & ((1 << n) - 1), int(strips[j][0]) & ((1 << n) - 1)) == sols[0]


def _gf2_solve(A, b):
    """Plain Gaussian elimination over GF(2) (test-local, independent of oracle.c)."""
    A = A.copy() % 2
    b = b.copy() % 2
    m, n = A.shape
    row = 0
    piv = []
    for c in range(n):
        r = next((r for r in range(row, m) if A[r, c]), None)
        if r is None:
            continue
        A[[row, r]] = A[[r, row]]
        b[[row, r]] = b[[r, row]]
        for rr in range(m):
            if rr != row and A[rr, c]:
                A[rr] ^= A[row]
                b[rr] ^= b[row]
        piv.append(c)
        row += 1
    assert row == n, "singular"
    x = np.zeros(n, np.uint8)
    for k, c in enumerate(piv):
        x[c] = b[k]
    return x


@pytest.mark.parametrize("p,N", [(5, 4), (7, 5), (13, 4)])
def test_recover_matches_parity_check_solve(p, N):
    """Tier A: for each pair, solve the 2n x 2n system given by the parity
    check matrix of Corollary 24.4 for the lost words of word 0."""
    n = p - 1
    rng = np.random.default_rng(p + N)
    nbytes = (n + 7) // 8 * 2
    orig = _stripe(p, N, nbytes, rng)
    W = oracle.word_count(p, nbytes)
    words = [polyref.words_of(s.tobytes(), s.size, n, W)[0] for s in orig]
    Spow = [polyref_matrix(p, i) for i in range(N)]
    I = np.eye(n, dtype=np.uint8)
    Z = np.zeros((n, n), np.uint8)
    blocks_top = [I] * N + [I, Z]
    blocks_bot = Spow + [Z, I]
    for i, j in itertools.combinations(range(N + 2), 2):
        vec = lambda w: np.array([(w >> t) & 1 for t in range(n)], np.uint8)
        rhs = np.zeros(2 * n, np.uint8)
        for k in range(N + 2):
            if k in (i, j):
                continue
            rhs[:n] ^= (blocks_top[k].astype(int) @ vec(words[k]) % 2).astype(np.uint8)
            rhs[n:] ^= (blocks_bot[k].astype(int) @ vec(words[k]) % 2).astype(np.uint8)
        A = np.block([[blocks_top[i], blocks_top[j]], [blocks_bot[i], blocks_bot[j]]]).astype(np.uint8)
        sol = _gf2_solve(A, rhs)
        strips = [s.copy() for s in orig]
        strips[i][:] = 0
        strips[j][:] = 0
        oracle.recover(p, N, i, j, strips, nbytes)
        gi = polyref.words_of(strips[i].tobytes(), strips[i].size, n, W)[0]
        gj = polyref.words_of(strips[j].tobytes(), strips[j].size, n, W)[0]
        assert gi == sum(int(b) << t for t, b in enumerate(sol[:n]))
        assert gj == sum(int(b) << t for t, b in enumerate(sol[n:]))


def polyref_matrix(p, k):
    """Matrix of multiplication by x^k, columns from the polynomial definition."""
    n = p - 1
    M = np.zeros((n, n), np.uint8)
    for c in range(n):
        v = polyref.ring_mul(p, polyref.xk(p, k), 1 << c)
        for r in range(n):
            M[r, c] = (v >> r) & 1
    return M


def test_syndrome_checker():
    p, N, nb = 13, 5, 20
    rng = np.random.default_rng(9)
    st = _stripe(p, N, nb, rng)
    assert oracle.count_bad_words(p, N, st, nb) == 0
    st[2][3] ^= 0x10
    assert oracle.count_bad_words(p, N, st, nb) == 1
