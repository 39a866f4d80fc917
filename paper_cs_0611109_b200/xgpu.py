"""Cross-GPU stripe layout: the strips of ONE stripe spread over G ranks.

The parity equations of Eq. (znparity) and the recovery syndromes of
Eq. (PQxy) are sums over disks, and the reduction pi: R' -> R_p is a ring
homomorphism (Eq. (powers)), so each rank folds only the strips it holds
into reduced partial syndromes, and the owner of each word range sums the G partials and runs
the class solve (Lemma 23.2; Sec. 4.6):

    step = raid6c_partial_strided (every rank, its strips; outputs go to the range owners' slots)
           -> cross-rank barrier ->
           raid6c_combine_strided (every rank, its word range; rebuilt strips go to their owners)

Layout (host logic, tested on CPU):
  * rank r holds the global strip indices ``strip_block(r)`` = [floor(r(N+2)/G), floor((r+1)(N+2)/G))
    of every stripe (data 0..N-1, then P = N and Q = N+1 on the last rank(s));
  * rank g owns word range g: bytes [g*R, min((g+1)*R, parity_bytes)) of the parity-format
    strips, R = raid6c_xgpu_range_bytes(p, bytes, G) (whole kernel tiles);
  * rank g keeps one slot per source rank for its range: slot[src] holds (dP_src, dQ_src).

Two drivers share that logic:
  * ``Emulated``: G virtual ranks inside one process on one GPU (every pointer local).  Its
    kernels never wait on one another -- each phase is a set of independent launches, the
    phases are stream-ordered -- which is how the path is parity-tested and its kernels timed
    on a single B200 (B200_PROFILING.md: emulate ranks as launches over all ranks' data).
  * ``Distributed``: one process per GPU; each rank allocates one arena (raid6c_dev_alloc), the
    arenas are exchanged as CUDA IPC handles over torch.distributed, and the partial kernel
    stores straight into peer slots (NVLink) while the combine kernel writes rebuilt strips
    into their owners' arenas.  The barrier between phases is a stream-ordered collective
    (NCCL all-reduce of one element) or, under gloo, a stream sync + host barrier.
"""
from __future__ import annotations


# ------------------------------------------------------------------ host logic (no GPU needed)
def strip_block(rank: int, world: int, N: int) -> tuple[int, int]:
    """Global strip indices [k_lo, k_hi) held by `rank` (block partition of the N+2 strips)."""
    if world < 1 or not (0 <= rank < world) or N < 1:
        raise ValueError("bad rank/world/N")
    return (rank * (N + 2)) // world, ((rank + 1) * (N + 2)) // world


def strip_owner(k: int, world: int, N: int) -> int:
    """Rank holding global strip k."""
    for r in range(world):
        lo, hi = strip_block(r, world, N)
        if lo <= k < hi:
            return r
    raise ValueError(f"strip {k} out of range")


def word_ranges(pbytes: int, range_bytes: int, world: int) -> list[tuple[int, int]]:
    """Byte range [lo, hi) of the parity-format strip owned by each rank (possibly empty)."""
    if range_bytes <= 0 or range_bytes * world < pbytes:
        raise ValueError("ranges do not cover the strip")
    return [(min(g * range_bytes, pbytes), min((g + 1) * range_bytes, pbytes)) for g in range(world)]


def slot_stride(range_bytes: int, align: int = 256) -> int:
    """Per-stripe stride of one partial slot (>= range_bytes, 16-B aligned for the TMA stores)."""
    return (range_bytes + align - 1) // align * align


def arena_layout(rank: int, world: int, N: int, S: int, strip_stride: int, parity_stride: int,
                 slot_pstride: int) -> dict:
    """Byte layout of rank's IPC arena (xgpu.Distributed): its strips [k_lo, k_hi) for S stripes
    (strip k of stripe s at strip_off[k] + s * stride(k)), then its 2 * world partial slots
    (source r's dP / dQ slot at slot_off + (2r + which) * S * slot_pstride)."""
    k_lo, k_hi = strip_block(rank, world, N)
    off, strip_off = 0, {}
    for k in range(k_lo, k_hi):
        strip_off[k] = off
        off += S * (strip_stride if k < N else parity_stride)
    slot_off = off
    off += world * 2 * S * slot_pstride
    return {"strip_off": strip_off, "slot_off": slot_off, "size": max(off, 256)}


def alg_bytes(N: int, nbytes: int, pbytes: int, world: int, rank: int, range_bytes: int,
              pairs=None) -> dict:
    """Algorithmic bytes per stripe of one rank's two launches (DESIGN.md NEXT-4):
    partial = its surviving strips read + 2 partial strips written (to the owners);
    combine = world partial pairs of its range read + the rebuilt bytes of its range written."""
    k_lo, k_hi = strip_block(rank, world, N)
    lo, hi = word_ranges(pbytes, range_bytes, world)[rank]
    x, y = (N, N + 1) if pairs is None else (min(pairs), max(pairs))
    rd = sum((nbytes if k < N else pbytes) for k in range(k_lo, k_hi) if k not in (x, y))
    part = rd + 2 * pbytes
    wr = sum(max(0, min(hi, nbytes if k < N else pbytes) - lo) for k in (x, y))
    comb = 2 * world * (hi - lo) + wr
    return {"partial": part, "combine": comb}


# ------------------------------------------------------------------ drivers (CUDA)
class Emulated:
    """G virtual ranks of the cross-GPU layout on one GPU (all buffers local).

    data [S, N, ss] / par [S, 2, ps]: the stripes by global strip index (as in the batched
    calls); slots [G_owner, G_src, 2, S, slot_stride] hold the partial syndromes."""

    def __init__(self, plan, world: int, data, par, S: int):
        import torch
        from . import raid6c as R  # noqa: F401  (fails loudly without libraid6c.so)
        self.plan, self.G, self.S = plan, world, S
        self.N, self.nbytes, self.pbytes = plan.N, plan.nbytes, plan.pbytes
        self.ss, self.ps = data.shape[2], par.shape[2]
        self.range = plan.xgpu_range_bytes(world)
        self.pstride = slot_stride(self.range)
        self.ranges = word_ranges(self.pbytes, self.range, world)
        self.slots = torch.empty((world, world, 2, S, self.pstride), dtype=torch.uint8, device=data.device)
        d0, p0 = int(data.data_ptr()), int(par.data_ptr())
        self.strips = [d0 + k * self.ss for k in range(self.N)] + [p0, p0 + self.ps]
        self.data_stride, self.parity_stride = self.N * self.ss, 2 * self.ps

    def _slot(self, owner, src, which):
        return int(self.slots[owner, src, which].data_ptr())

    def partial(self, rank: int, erasures=None):
        k_lo, k_hi = strip_block(rank, self.G, self.N)
        held = [a if k_lo <= k < k_hi else None for k, a in enumerate(self.strips)]
        self.plan.partial_strided(held, self.data_stride, self.parity_stride, self.S, erasures, k_lo, k_hi,
                                  [self._slot(g, rank, 0) for g in range(self.G)],
                                  [self._slot(g, rank, 1) for g in range(self.G)], self.pstride, self.range)

    def combine(self, rank: int, erasures=None):
        lo, hi = self.ranges[rank]
        if hi <= lo:
            return
        self.plan.combine_strided(self.strips, self.data_stride, self.parity_stride, self.S, erasures,
                                  [self._slot(rank, r, 0) for r in range(self.G)],
                                  [self._slot(rank, r, 1) for r in range(self.G)], self.pstride, lo, hi)

    def step(self, erasures=None):
        """One encode (erasures None) or recovery step of all G virtual ranks, stream-ordered."""
        for r in range(self.G):
            self.partial(r, erasures)
        for g in range(self.G):
            self.combine(g, erasures)


class _DevBytes:
    """A device byte range seen by torch through __cuda_array_interface__ (no copy, no ownership)."""

    def __init__(self, ptr: int, nbytes: int):
        self.__cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1", "data": (int(ptr), False),
                                         "version": 3, "strides": None}


class Distributed:
    """One process per GPU.  Rank r's arena = its strips [k_lo, k_hi) for S stripes, then its G
    slots (one per source rank) of its word range.  Peer arenas are mapped with CUDA IPC."""

    def __init__(self, plan, S: int, device: int, backend: str = "nccl"):
        import torch
        import torch.distributed as dist
        from . import raid6c as R
        self.R, self.dist, self.torch = R, dist, torch
        self.plan, self.S, self.dev = plan, S, device
        self.G, self.rank = dist.get_world_size(), dist.get_rank()
        self.N, self.nbytes, self.pbytes = plan.N, plan.nbytes, plan.pbytes
        self.backend = backend
        self.ss = slot_stride(self.nbytes)
        self.ps = slot_stride(self.pbytes)
        self.range = plan.xgpu_range_bytes(self.G)
        self.pstride = slot_stride(self.range)
        self.ranges = word_ranges(self.pbytes, self.range, self.G)
        self.blocks = [strip_block(r, self.G, self.N) for r in range(self.G)]
        # arena layout (identical offsets on every rank for a given owner)
        self.layout = [self._arena_layout(r) for r in range(self.G)]
        size = self.layout[self.rank]["size"]
        self.base = R.dev_alloc(size, device)
        handle = R.ipc_export(self.base)
        handles = [None] * self.G
        dist.all_gather_object(handles, handle)
        self.peer = [self.base if r == self.rank else R.ipc_open(handles[r], device) for r in range(self.G)]
        self.strips = [None] * (self.N + 2)  # global strip k -> address in its owner's arena
        for r in range(self.G):
            for k, off in self.layout[r]["strip_off"].items():
                self.strips[k] = self.peer[r] + off
        self._flag = torch.zeros(1, dtype=torch.int32, device=torch.device("cuda", device))

    def _arena_layout(self, r):
        return arena_layout(r, self.G, self.N, self.S, self.ss, self.ps, self.pstride)

    def slot(self, owner, src, which):
        """Address of owner's slot for source rank `src` (which: 0 = dP, 1 = dQ)."""
        return self.peer[owner] + self.layout[owner]["slot_off"] + (2 * src + which) * self.S * self.pstride

    def strip_addr(self, k):
        return self.strips[k]

    def stride(self, k):
        return self.ss if k < self.N else self.ps

    def held_strip(self, k):
        """Zero-copy uint8 tensor [S, stride(k)] over held strip k in this rank's arena (for
        verification: poisoning and digests; the path itself takes raw addresses)."""
        k_lo, k_hi = self.blocks[self.rank]
        if not (k_lo <= k < k_hi):
            raise ValueError(f"strip {k} is not held by rank {self.rank}")
        n = self.S * self.stride(k)
        buf = _DevBytes(self.strips[k], n)
        t = self.torch.as_tensor(buf, device=self.torch.device("cuda", self.dev))
        return t.view(self.S, self.stride(k))

    def barrier(self, stream):
        """Every rank's previous launches complete before any rank's next launch starts."""
        if self.backend == "nccl":
            with self.torch.cuda.stream(stream):
                self.dist.all_reduce(self._flag)  # stream-ordered: completes only when all ranks arrive
        else:
            stream.synchronize()
            self.dist.barrier()

    def step(self, stream, erasures=None):
        k_lo, k_hi = self.blocks[self.rank]
        held = [a if k_lo <= k < k_hi else None for k, a in enumerate(self.strips)]
        self.plan.partial_strided(held, self.ss, self.ps, self.S, erasures, k_lo, k_hi,
                                  [self.slot(g, self.rank, 0) for g in range(self.G)],
                                  [self.slot(g, self.rank, 1) for g in range(self.G)], self.pstride, self.range)
        self.barrier(stream)
        lo, hi = self.ranges[self.rank]
        if hi > lo:
            self.plan.combine_strided(self.strips, self.ss, self.ps, self.S, erasures,
                                      [self.slot(self.rank, r, 0) for r in range(self.G)],
                                      [self.slot(self.rank, r, 1) for r in range(self.G)], self.pstride, lo, hi)
        self.barrier(stream)

    def close(self):
        for r in range(self.G):
            if r != self.rank and self.peer[r]:
                self.R.ipc_close(self.peer[r])
        if self.base:
            self.R.dev_free(self.base)
            self.base = 0
