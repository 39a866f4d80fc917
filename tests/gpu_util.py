"""Helpers for the GPU parity tests: stripe batches in device memory, oracle segments."""
from __future__ import annotations

import numpy as np
import torch

import oracle
import synthetic
from paper_cs_0611109_b200 import raid6c as R


class Batch:
    """S stripes laid out as data [S, N, ss] and parity [S, 2, ps] inside one uint8 buffer,
    optionally shifted by `offset` bytes (to exercise unaligned pointers)."""

    def __init__(self, p, N, nbytes, S, offset=0, align=256, device="cuda"):
        self.p, self.N, self.nbytes, self.S = p, N, nbytes, S
        self.pb = R.parity_bytes(p, nbytes)
        self.ss = R.aligned_stride(nbytes, align) if align else nbytes
        self.ps = R.aligned_stride(self.pb, align) if align else self.pb
        self.dbuf = torch.zeros(S * N * self.ss + offset + 64, dtype=torch.uint8, device=device)
        self.pbuf = torch.zeros(S * 2 * self.ps + offset + 64, dtype=torch.uint8, device=device)
        self.off = offset
        self.data = self.dbuf[offset:offset + S * N * self.ss].view(S, N, self.ss)
        self.par = self.pbuf[offset:offset + S * 2 * self.ps].view(S, 2, self.ps)

    # raw addresses for the strided calls
    def args(self):
        return (int(self.data.data_ptr()), self.ss, self.N * self.ss, int(self.par.data_ptr()),
                int(self.par.data_ptr()) + self.ps, 2 * self.ps, self.S)

    def strip(self, s, k):
        """Tensor view of strip k of stripe s (data: nbytes, P/Q: parity bytes)."""
        if k < self.N:
            return self.data[s, k, :self.nbytes]
        return self.par[s, k - self.N, :self.pb]

    def set_data_numpy(self, s, strips):
        for k, a in enumerate(strips):
            self.data[s, k, :self.nbytes].copy_(torch.from_numpy(np.ascontiguousarray(a)))

    def fill_synthetic(self, seed=0, cfg=0, stripe0=0, sparse_mode=0):
        R.fill(self.data, self.ss, self.N * self.ss, self.nbytes, self.N, self.S, seed, cfg, stripe0, 0, sparse_mode)

    def numpy_strip(self, s, k):
        return self.strip(s, k).cpu().numpy()


def oracle_stripe(p, N, nbytes, seed, cfg, stripe, sparse=False):
    data = synthetic.stripe_strips(seed, cfg, stripe, N, nbytes, sparse)
    P, Q = oracle.encode(p, data, nbytes)
    return data, P, Q


def segment_bounds(p, nbytes, which, nwords8=4):
    """A byte segment [b0, b1) of a strip that starts on a word boundary (w0 multiple of 8):
    which='head' | 'mid' | 'tail' (tail runs to the end of the strip)."""
    n = p - 1
    unit = n  # 8 words = n bytes
    W = (8 * nbytes + n - 1) // n
    groups = W // 8
    if which == "head":
        g0 = 0
    elif which == "mid":
        g0 = max(0, groups // 2 - nwords8 // 2)
    else:
        g0 = max(0, groups - nwords8)
    b0 = g0 * unit
    b1 = nbytes if which == "tail" else min(nbytes, b0 + nwords8 * unit)
    return b0, b1


def oracle_segment_parity(p, data_segments, seg_len):
    """Oracle P, Q of a word-aligned segment (a stripe of `seg_len`-byte strips)."""
    return oracle.encode(p, data_segments, seg_len)
