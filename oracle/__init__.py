"""CPU oracle for Z_p-RAID (arxiv cs/0611109) -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` leg may import this package.  The product path
(``paper_cs_0611109_b200``) never imports it, and the two share no code.

This module is a thin ctypes binding over ``oracle.c`` (plain C, one byte per bit,
Horner with single Sylvester steps, Gauss-Jordan for the DD inverse).  Every C
function cites the paper passage it follows; see oracle.c.

Parity pins: every function here is pinned by tests/test_oracle_pins.py against
values printed in the paper, closed forms, invariants and brute force.  The byte
layout of non-16-bit words is a convention (R2/R5): pinned by
hand-derived vectors only.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_SO = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib_handle = None


def build(force: bool = False) -> str:
    """Compile oracle.c into liboracle.so with gcc (plain -O2, no vectorisation tricks)."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        tmp = _SO + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c99", "-fPIC", "-shared", "-Wall", "-o", tmp, _SRC])
        os.replace(tmp, _SO)
    return _SO


def _lib():
    global _lib_handle
    with _lock:
        if _lib_handle is None:
            lib = ctypes.CDLL(build())
            u8p = ctypes.POINTER(ctypes.c_uint8)
            pp = ctypes.POINTER(u8p)
            sz = ctypes.c_size_t
            i = ctypes.c_int
            lib.oracle_n.argtypes = [i]
            lib.oracle_word_count.argtypes = [i, sz]
            lib.oracle_word_count.restype = sz
            lib.oracle_parity_bytes.argtypes = [i, sz]
            lib.oracle_parity_bytes.restype = sz
            lib.oracle_valid_p.argtypes = [i]
            lib.oracle_mul_x.argtypes = [i, u8p, u8p]
            lib.oracle_mul_xk.argtypes = [i, i, u8p, u8p]
            lib.oracle_sylvester.argtypes = [i, u8p]
            lib.oracle_gf2_matmul.argtypes = [i, u8p, u8p, u8p]
            lib.oracle_gf2_matvec.argtypes = [i, u8p, u8p, u8p]
            lib.oracle_sylvester_power.argtypes = [i, i, u8p]
            lib.oracle_gf2_inverse.argtypes = [i, u8p, u8p]
            lib.oracle_encode.argtypes = [i, i, pp, sz, u8p, u8p]
            lib.oracle_encode_matrix.argtypes = [i, i, pp, sz, u8p, u8p]
            lib.oracle_recover.argtypes = [i, i, i, i, pp, sz]
            lib.oracle_count_bad_words.argtypes = [i, i, pp, sz]
            lib.oracle_count_bad_words.restype = sz
            lib.oracle_ext_condition.argtypes = [i]
            lib.oracle_ext_coeff.argtypes = [i, i, u8p]
            lib.oracle_encode_ext.argtypes = [i, i, pp, sz, u8p, u8p]
            lib.oracle_recover_ext.argtypes = [i, i, i, i, pp, sz]
            u8 = ctypes.c_uint8
            for nm, res, args in [("oracle_rs_mul2", u8, [u8]), ("oracle_rs_mul", u8, [u8, u8]),
                                  ("oracle_rs_exp", u8, [i]), ("oracle_rs_inv", u8, [u8])]:
                f = getattr(lib, nm)
                f.restype = res
                f.argtypes = args
            lib.oracle_rs_encode.argtypes = [i, pp, sz, u8p, u8p]
            lib.oracle_rs_recover.argtypes = [i, i, i, pp, sz]
            _lib_handle = lib
    return _lib_handle


def _p(a: np.ndarray):
    assert a.dtype == np.uint8 and a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8))


def _ptr_array(arrs):
    u8p = ctypes.POINTER(ctypes.c_uint8)
    return (u8p * len(arrs))(*[_p(a) for a in arrs])


# ------------------------------------------------------------------ sizes
def word_count(p: int, nbytes: int) -> int:
    return int(_lib().oracle_word_count(p, nbytes))


def parity_bytes(p: int, nbytes: int) -> int:
    return int(_lib().oracle_parity_bytes(p, nbytes))


def valid_p(p: int) -> bool:
    return bool(_lib().oracle_valid_p(p))


# ------------------------------------------------------- word-level (bits)
def _bits(v, n):
    """int -> bit array (bit j = coefficient of x^j)."""
    return np.array([(int(v) >> j) & 1 for j in range(n)], dtype=np.uint8)


def _int(bits) -> int:
    return sum(int(b) << j for j, b in enumerate(bits))


def mul_x(p: int, a: int) -> int:
    n = p - 1
    x = _bits(a, n)
    y = np.zeros(n, np.uint8)
    _lib().oracle_mul_x(p, _p(x), _p(y))
    return _int(y)


def mul_xk(p: int, k: int, a: int) -> int:
    n = p - 1
    x = _bits(a, n)
    y = np.zeros(n, np.uint8)
    _lib().oracle_mul_xk(p, k, _p(x), _p(y))
    return _int(y)


# ------------------------------------------------------------- matrices
def sylvester(p: int) -> np.ndarray:
    n = p - 1
    S = np.zeros((n, n), np.uint8)
    _lib().oracle_sylvester(p, _p(S))
    return S


def sylvester_power(p: int, k: int) -> np.ndarray:
    n = p - 1
    S = np.zeros((n, n), np.uint8)
    _lib().oracle_sylvester_power(p, k, _p(S))
    return S


def gf2_matmul(A: np.ndarray, B: np.ndarray) -> np.ndarray:
    n = A.shape[0]
    A = np.ascontiguousarray(A, np.uint8)
    B = np.ascontiguousarray(B, np.uint8)
    C = np.zeros((n, n), np.uint8)
    _lib().oracle_gf2_matmul(n, _p(A), _p(B), _p(C))
    return C


def gf2_matvec(M: np.ndarray, v: np.ndarray) -> np.ndarray:
    n = M.shape[0]
    M = np.ascontiguousarray(M, np.uint8)
    v = np.ascontiguousarray(v, np.uint8)
    y = np.zeros(n, np.uint8)
    _lib().oracle_gf2_matvec(n, _p(M), _p(v), _p(y))
    return y


def gf2_inverse(M: np.ndarray):
    """Gauss-Jordan inverse over GF(2); None if singular."""
    n = M.shape[0]
    M = np.ascontiguousarray(M, np.uint8)
    R = np.zeros((n, n), np.uint8)
    ok = _lib().oracle_gf2_inverse(n, _p(M), _p(R))
    return R if ok else None


# --------------------------------------------------------- stripe level
def _as_strips(data, nbytes):
    data = [np.ascontiguousarray(d, np.uint8) for d in data]
    for d in data:
        assert d.size == nbytes
    return data


def encode(p: int, data, nbytes: int | None = None, matrix: bool = False):
    """Encode one stripe.  data: sequence of N uint8 arrays (``nbytes`` each).
    Returns (P, Q) as uint8 arrays of parity_bytes(p, nbytes)."""
    if nbytes is None:
        nbytes = int(np.asarray(data[0]).size)
    data = _as_strips(data, nbytes)
    N = len(data)
    pb = parity_bytes(p, nbytes)
    P = np.zeros(pb, np.uint8)
    Q = np.zeros(pb, np.uint8)
    fn = _lib().oracle_encode_matrix if matrix else _lib().oracle_encode
    rc = fn(p, N, _ptr_array(data), nbytes, _p(P), _p(Q))
    if rc != 0:
        raise ValueError(f"oracle_encode: invalid arguments p={p} N={N}")
    return P, Q


def recover(p: int, N: int, lost_i: int, lost_j: int, strips, nbytes: int):
    """Double-erasure recovery in place.  strips: list of N+2 uint8 arrays
    (0..N-1 data of ``nbytes``, N = P, N+1 = Q of parity_bytes); the two lost
    entries are overwritten.  Returns the list."""
    assert len(strips) == N + 2
    for s in strips:
        assert s.dtype == np.uint8 and s.flags["C_CONTIGUOUS"]
    rc = _lib().oracle_recover(p, N, lost_i, lost_j, _ptr_array(strips), nbytes)
    if rc != 0:
        raise ValueError(f"oracle_recover failed rc={rc} (p={p} N={N} lost=({lost_i},{lost_j}))")
    return strips


def count_bad_words(p: int, N: int, strips, nbytes: int) -> int:
    return int(_lib().oracle_count_bad_words(p, N, _ptr_array(strips), nbytes))


# ------------------------------------------------------ extended Q-parity (NEXT-2)
def ext_condition(p: int) -> bool:
    """Theorem 25.3(3): gcd(X^p + 1, X^m + X + 1) = 1 for all 0 < m < p."""
    return bool(_lib().oracle_ext_condition(p))


def ext_coeff(p: int, k: int) -> np.ndarray:
    n = p - 1
    G = np.zeros((n, n), np.uint8)
    _lib().oracle_ext_coeff(p, k, _p(G))
    return G


def encode_ext(p: int, data, nbytes: int | None = None):
    """Eq. (qext): D = len(data) data strips, 1 <= D <= 2p-1."""
    if nbytes is None:
        nbytes = int(np.asarray(data[0]).size)
    data = _as_strips(data, nbytes)
    pb = parity_bytes(p, nbytes)
    P = np.zeros(pb, np.uint8)
    Q = np.zeros(pb, np.uint8)
    rc = _lib().oracle_encode_ext(p, len(data), _ptr_array(data), nbytes, _p(P), _p(Q))
    if rc != 0:
        raise ValueError(f"oracle_encode_ext: invalid arguments p={p} D={len(data)}")
    return P, Q


def recover_ext(p: int, D: int, lost_i: int, lost_j: int, strips, nbytes: int):
    assert len(strips) == D + 2
    rc = _lib().oracle_recover_ext(p, D, lost_i, lost_j, _ptr_array(strips), nbytes)
    if rc != 0:
        raise ValueError(f"oracle_recover_ext failed rc={rc} (p={p} D={D} lost=({lost_i},{lost_j}))")
    return strips


# ------------------------------------------------------ GF(256) Reed-Solomon (NEXT-3)
def rs_mul2(x: int) -> int:
    return int(_lib().oracle_rs_mul2(x))


def rs_mul(a: int, b: int) -> int:
    return int(_lib().oracle_rs_mul(a, b))


def rs_exp(k: int) -> int:
    return int(_lib().oracle_rs_exp(k))


def rs_inv(a: int) -> int:
    return int(_lib().oracle_rs_inv(a))


def rs_encode(data, nbytes: int | None = None):
    """Eq. (rsparity): returns (P, Q), each ``nbytes`` long."""
    if nbytes is None:
        nbytes = int(np.asarray(data[0]).size)
    data = _as_strips(data, nbytes)
    P = np.zeros(nbytes, np.uint8)
    Q = np.zeros(nbytes, np.uint8)
    if _lib().oracle_rs_encode(len(data), _ptr_array(data), nbytes, _p(P), _p(Q)) != 0:
        raise ValueError("oracle_rs_encode: invalid arguments")
    return P, Q


def rs_recover(N: int, lost_i: int, lost_j: int, strips, nbytes: int):
    assert len(strips) == N + 2
    if _lib().oracle_rs_recover(N, lost_i, lost_j, _ptr_array(strips), nbytes) != 0:
        raise ValueError("oracle_rs_recover failed")
    return strips
