"""Counter-based synthetic strip generator (numpy).  See synthetic/__init__.py."""
from __future__ import annotations

import numpy as np

GOLDEN = 0x9E3779B97F4A7C15
SPARSE_A = 0xA5A5A5A55A5A5A5A
SPARSE_B = 0x3C3C3C3CC3C3C3C3
ERASE_DOMAIN = 0xD1B54A32D192ED03
SPARSE_ZERO_BELOW = 58982  # 0.9 * 65536 = 58982.4
_M64 = (1 << 64) - 1


def mix64(z: np.ndarray) -> np.ndarray:
    """SplitMix64 finalizer on a uint64 array (wrapping arithmetic)."""
    z = np.asarray(z, dtype=np.uint64).copy()
    with np.errstate(over="ignore"):
        z ^= z >> np.uint64(30)
        z *= np.uint64(0xBF58476D1CE4E5B9)
        z ^= z >> np.uint64(27)
        z *= np.uint64(0x94D049BB133111EB)
        z ^= z >> np.uint64(31)
    return z


def _keys(seed: int, cfg: int, stripe: int, strip: int, k0: int, k1: int) -> np.ndarray:
    assert 0 <= stripe < 8192 and 0 <= strip < 512 and k1 <= (1 << 22)
    hi = ((((cfg * 8192 + stripe) * 512 + strip) << 22) + (seed * GOLDEN)) & _M64
    ks = np.arange(k0, k1, dtype=np.uint64)
    with np.errstate(over="ignore"):
        return ks + np.uint64(hi)  # k < 2^22 occupies the zero low bits: + == |


def strip_bytes(seed: int, cfg: int, stripe: int, strip: int, nbytes: int,
                sparse: bool = False, lo: int = 0, hi: int | None = None) -> np.ndarray:
    """Bytes [lo, hi) of strip ``strip`` of stripe ``stripe`` (``nbytes`` long)."""
    if hi is None:
        hi = nbytes
    assert 0 <= lo <= hi <= nbytes
    if hi == lo:
        return np.zeros(0, np.uint8)
    k0, k1 = lo // 8, (hi + 7) // 8
    keys = _keys(seed, cfg, stripe, strip, k0, k1)
    base = mix64(keys)
    b = base.view(np.uint8).copy()  # little-endian host (x86)
    if sparse:
        with np.errstate(over="ignore"):
            da = mix64(keys ^ np.uint64(SPARSE_A))
            db = mix64(keys ^ np.uint64(SPARSE_B))
        draws = np.stack([da, db], axis=1).view(np.uint16).reshape(-1)  # 8 draws per word
        nz = 1 + (b % np.uint8(255))
        b = np.where(draws < SPARSE_ZERO_BELOW, np.uint8(0), nz).astype(np.uint8)
    off = lo - k0 * 8
    return np.ascontiguousarray(b[off:off + (hi - lo)])


def stripe_strips(seed: int, cfg: int, stripe: int, N: int, nbytes: int, sparse: bool = False):
    return [strip_bytes(seed, cfg, stripe, t, nbytes, sparse) for t in range(N)]


def all_pairs(N: int):
    """All C(N+2, 2) erasure pairs (i < j) over indices 0..N+1 (N = P, N+1 = Q),
    lexicographic."""
    return [(i, j) for i in range(N + 2) for j in range(i + 1, N + 2)]


def pair_class(N: int, i: int, j: int) -> str:
    i, j = min(i, j), max(i, j)
    if i == N and j == N + 1:
        return "PQ"
    if j == N + 1:
        return "DQ"
    if j == N:
        return "DP"
    return "DD"


def erasure_pair(seed: int, cfg: int, stripe: int, N: int):
    """Degraded-stream draw (config 5): class ~ U{DD, DP, DQ, PQ}, then indices uniform
    within the class.  Returns (i, j) with i < j."""
    h = int(mix64(np.array([(seed * GOLDEN + ERASE_DOMAIN + cfg * 8192 + stripe) & _M64],
                           dtype=np.uint64))[0])
    cls = h & 3
    r1 = (h >> 8) & 0xFFFFFF
    r2 = (h >> 32) & 0xFFFFFF
    if cls == 0 and N >= 2:  # DD
        x = r1 % N
        y = r2 % (N - 1)
        if y >= x:
            y += 1
        return (min(x, y), max(x, y))
    if cls == 1 or (cls == 0 and N < 2):  # DP
        return (r1 % N, N)
    if cls == 2:  # DQ
        return (r1 % N, N + 1)
    return (N, N + 1)
