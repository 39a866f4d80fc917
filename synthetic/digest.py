"""Per-strip 64-bit digest (numpy), the host twin of the harness kernel ``raid6c_digest``.

Not the RAID method: a comparison tool.  Full-size GPU outputs (GiB per stripe) are reduced to
one u64 per strip on the device, the oracle's outputs for the same seeded stripes are reduced
the same way on the host cores, and the two are compared (bench.py ``--full`` oracle sample,
tests/test_gpu_digest.py).  Definition (include/raid6c.h, raid6c_digest):

    digest(b) = mix64(len ^ DIGEST_LEN) + sum_k mix64(w_k + k*GOLDEN + DIGEST_DOMAIN)   (mod 2^64)

w_k = little-endian u64 of bytes [8k, 8k+8) of b, zero past len; mix64 = SplitMix64 finalizer.
mix64 is a bijection, so changing one word always changes its term, hence the digest.
"""
from __future__ import annotations

import numpy as np

from .gen import GOLDEN, mix64

DIGEST_DOMAIN = 0x6A09E667F3BCC909
DIGEST_LEN = 0xBB67AE8584CAA73B
_CHUNK = 1 << 22  # words per numpy pass (bounded temporaries)


_M64 = (1 << 64) - 1


def length_term(nbytes: int) -> int:
    """The length term mix64(len ^ DIGEST_LEN) of a strip of ``nbytes`` bytes."""
    return int(mix64(np.array([nbytes ^ DIGEST_LEN], dtype=np.uint64))[0])


def word_terms(b: np.ndarray, word0: int = 0) -> int:
    """sum_k mix64(w_k + (word0 + k)*GOLDEN + DIGEST_DOMAIN) mod 2^64 over the words of ``b``,
    which starts at word ``word0`` (byte 8*word0) of its strip; a ragged end is zero-padded.
    A strip's digest is length_term(len) plus the word terms of its pieces (any split at
    8-byte boundaries), so pieces can be digested in parallel."""
    b = np.ascontiguousarray(b, dtype=np.uint8).reshape(-1)
    n = b.size
    nw = (n + 7) // 8
    if n % 8:
        pad = np.zeros(nw * 8, np.uint8)
        pad[:n] = b
        b = pad
    w = b.view("<u8")
    h = 0
    with np.errstate(over="ignore"):
        for k0 in range(0, nw, _CHUNK):
            k = np.arange(word0 + k0, word0 + min(nw, k0 + _CHUNK), dtype=np.uint64)
            t = w[k0:k0 + k.size] + k * np.uint64(GOLDEN) + np.uint64(DIGEST_DOMAIN)
            h = (h + int(mix64(t).sum(dtype=np.uint64))) & _M64
    return h


def digest(b: np.ndarray) -> int:
    """Digest of a uint8 array (any length)."""
    b = np.ascontiguousarray(b, dtype=np.uint8).reshape(-1)
    return (length_term(b.size) + word_terms(b)) & _M64


def combine(digests) -> int:
    """Order-sensitive digest of a sequence of u64 digests (e.g. every strip of a run, in global
    stripe order): the same definition applied to their little-endian bytes."""
    return digest(np.asarray(list(digests), dtype=np.uint64).view(np.uint8))
