"""Independent textbook polynomial arithmetic over F2, used ONLY by tests to pin the
oracle.  It shares no code with oracle.c: ring elements are Python ints, products are
carry-less multiplications, and reduction is generic long division by
Phi_p = 1 + x + ... + x^{p-1} (the definition of R_p in the north star / PAPER.md:764-768).
"""


def clmul(a: int, b: int) -> int:
    r = 0
    while b:
        if b & 1:
            r ^= a
        a <<= 1
        b >>= 1
    return r


def polymod(a: int, m: int) -> int:
    dm = m.bit_length() - 1
    while a.bit_length() - 1 >= dm:
        a ^= m << (a.bit_length() - 1 - dm)
    return a


def phi(p: int) -> int:
    return (1 << p) - 1  # 1 + x + ... + x^{p-1}


def ring_mul(p: int, a: int, b: int) -> int:
    return polymod(clmul(a, b), phi(p))


def xk(p: int, k: int) -> int:
    return polymod(1 << k, phi(p))


def words_of(strip: bytes, nbytes: int, n: int, W: int):
    """LSB-first bit stream -> W words of n bits (the layout convention R2, written
    independently of oracle.c with a little-endian big integer)."""
    v = int.from_bytes(bytes(strip[:nbytes]), "little")
    mask = (1 << n) - 1
    return [(v >> (w * n)) & mask for w in range(W)]


def bytes_of(words, n: int, nbytes: int) -> bytes:
    v = 0
    for w, x in enumerate(words):
        v |= x << (w * n)
    return v.to_bytes(nbytes, "little")


def encode_ref(p: int, data, nbytes: int):
    """P = sum d_i, Q = sum x^i d_i in R_p, word by word (Eq. (znparity) / (rsparity))."""
    n = p - 1
    W = (8 * nbytes + n - 1) // n
    pb = (W * n + 7) // 8
    ws = [words_of(d, nbytes, n, W) for d in data]
    P = [0] * W
    Q = [0] * W
    for i, dw in enumerate(ws):
        c = xk(p, i)
        for w in range(W):
            P[w] ^= dw[w]
            Q[w] ^= ring_mul(p, c, dw[w])
    return bytes_of(P, n, pb), bytes_of(Q, n, pb)
