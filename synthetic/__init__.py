"""Seeded synthetic inputs shared by tests, smoke() and bench.py.

This module holds NO arithmetic of the RAID method: it only produces bytes
(and erasure pairs) from a counter-based hash.  The GPU fill kernel
``raid6c_fill`` (paper_cs_0611109_b200/csrc/fill.cu) implements the same
generator independently; tests/test_gpu_parity.py checks the two agree
bit-for-bit.

Generator spec:
  key(seed, cfg, stripe, strip, k) = seed*GOLDEN + ((((cfg*8192 + stripe)*512 + strip) << 22) | k)
  u64 word k of a strip = mix64(key)                      (uniform bytes, little-endian)
  sparse: byte b of word k is 0 when its 16-bit draw < 58982 (p ~= 0.9),
          else 1 + (uniform byte b % 255).  Draws: bytes 0-3 from mix64(key ^ SPARSE_A),
          bytes 4-7 from mix64(key ^ SPARSE_B), 16 bits each, little-endian.
mix64 is the SplitMix64 finalizer.

``synthetic.digest`` (a harness comparison tool, also not the method) reduces a strip to a u64;
the device twin is ``raid6c_digest``.
"""
from .gen import (GOLDEN, SPARSE_A, SPARSE_B, ERASE_DOMAIN, mix64, strip_bytes,
                  stripe_strips, erasure_pair, all_pairs, pair_class)
from .digest import digest, combine as combine_digests, length_term, word_terms

__all__ = ["GOLDEN", "SPARSE_A", "SPARSE_B", "ERASE_DOMAIN", "mix64", "strip_bytes",
           "stripe_strips", "erasure_pair", "all_pairs", "pair_class", "digest", "combine_digests", "length_term", "word_terms"]
