"""NEXT-4: the cross-GPU stripe layout -- partial syndromes per rank
(raid6c_partial_strided) + combine-and-solve per word-range owner (raid6c_combine_strided) --
against the CPU oracle (oracle.encode / recover / encode_ext / recover_ext).

On one GPU the G ranks are emulated as independent launches over all ranks' data
(xgpu.Emulated: no kernel waits on another); the real one-process-per-GPU path with CUDA IPC
peer pointers runs as two processes sharing cuda:0 (test_distributed_ipc_two_processes)."""
import os
import subprocess
import sys

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import oracle  # noqa: E402
import synthetic  # noqa: E402
from paper_cs_0611109_b200 import raid6c as R  # noqa: E402
from paper_cs_0611109_b200 import xgpu  # noqa: E402
from tests.gpu_util import Batch  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

# (p, N, bytes, stripes, G): fast-path primes (several tiles + ragged tail), generic primes,
# the extended code (N > p), G = 1 .. 8 incl. ranks that hold only parity or nothing of a range
CASES = [(13, 12, 3 * 12288 + 1001, 3, 4), (13, 12, 3 * 12288 + 1001, 3, 1), (5, 4, 4 * 10752 + 77, 3, 3),
         (59, 58, 2 * 14848 + 333, 2, 8), (61, 60, 2 * 15360 + 17, 2, 5), (257, 64, 3 * 4096 + 64, 2, 8),
         (17, 16, 2 * 10752 + 9, 2, 2), (3, 2, 5000, 3, 4), (7, 6, 4000, 2, 3), (11, 10, 3000, 2, 3),
         (19, 18, 2500, 2, 4), (13, 25, 2 * 12288 + 99, 2, 4), (59, 90, 14848 + 333, 1, 6),
         (23, 22, 3000, 2, 3), (67, 40, 2000, 2, 4), (43, 60, 1500, 1, 5), (41, 40, 2 * 16384 + 33, 2, 3),
         (47, 46, 2 * 16384 + 5, 2, 5), (89, 60, 16384 + 77, 2, 4), (233, 100, 16384 + 77, 1, 4), (71, 30, 2000, 2, 3)]


def _np(t):
    return t.cpu().numpy()


def _refs(b, p, N, nbytes, S, seed, cfg):
    b.fill_synthetic(seed=seed, cfg=cfg)
    refs = []
    for s in range(S):
        data = synthetic.stripe_strips(seed, cfg, s, N, nbytes)
        P, Q = (oracle.encode_ext if N > p else oracle.encode)(p, data, nbytes)
        refs.append(data + [P, Q])
    return refs


def _pairs(p, N, G):
    """Every class, lost strips on the same rank and on different ranks."""
    blocks = [xgpu.strip_block(r, G, N) for r in range(G)]
    cand = [(0, 1), (0, N - 1), (N - 2, N - 1), (0, N), (N - 1, N), (1, N + 1), (N, N + 1)]
    for lo, hi in blocks:
        if hi - lo >= 2:
            cand.append((lo, lo + 1))
    if N > p:
        cand += [(0, p), (p - 1, p), (p, N - 1)]
    return sorted({(i, j) for i, j in cand if 0 <= i < j < N + 2})


@pytest.mark.parametrize("p,N,nbytes,S,G", CASES)
def test_xgpu_encode_and_recover(p, N, nbytes, S, G):
    b = Batch(p, N, nbytes, S)
    refs = _refs(b, p, N, nbytes, S, 31, 12)
    plan = R.Plan(p, N, nbytes)
    emu = xgpu.Emulated(plan, G, b.data, b.par, S)
    b.par.fill_(0x5A)  # parity is an output of the encode
    emu.step(None)
    plan.sync()
    for s in range(S):
        assert np.array_equal(_np(b.strip(s, N)), refs[s][N]), (s, "P")
        assert np.array_equal(_np(b.strip(s, N + 1)), refs[s][N + 1]), (s, "Q")
    pairs = _pairs(p, N, G)
    for t, (i, j) in enumerate(pairs):
        per = [(i, j) if s == 0 else pairs[(t + 3 * s) % len(pairs)] for s in range(S)]  # mixed classes
        for s, (x, y) in enumerate(per):
            for k in (x, y):
                b.strip(s, k).fill_(0xA5)  # lost strips are never read
        er = torch.tensor(per, dtype=torch.int32, device="cuda") if t % 2 else per
        emu.step(er)
        plan.sync()
        for s, (x, y) in enumerate(per):
            for k in (x, y):
                assert np.array_equal(_np(b.strip(s, k)), refs[s][k]), (p, N, G, s, (x, y), k)


@pytest.mark.parametrize("p,N,G", [(13, 12, 4), (59, 58, 3), (11, 10, 2), (23, 22, 3)])
def test_xgpu_partials_are_oracle_subset_parity(p, N, G):
    """Encode partial of rank r = the oracle parity of the stripe with every strip outside the
    rank's block zeroed (linearity of Eq. (znparity)); unaligned slots take the direct path."""
    nbytes, S = 2 * 12288 + 515, 2
    b = Batch(p, N, nbytes, S)
    refs = _refs(b, p, N, nbytes, S, 5, 13)
    plan = R.Plan(p, N, nbytes)
    emu = xgpu.Emulated(plan, G, b.data, b.par, S)
    for r in range(G):
        emu.partial(r, None)
    plan.sync()
    for r in range(G):
        lo, hi = xgpu.strip_block(r, G, N)
        for s in range(S):
            sub = [refs[s][k] if lo <= k < hi else np.zeros(nbytes, np.uint8) for k in range(N)]
            P, Q = oracle.encode(p, sub, nbytes)
            for g, (a0, a1) in enumerate(emu.ranges):
                if a1 <= a0:
                    continue
                gp = _np(emu.slots[g, r, 0, s, :a1 - a0])
                gq = _np(emu.slots[g, r, 1, s, :a1 - a0])
                assert np.array_equal(gp, P[a0:a1]), (r, s, g)
                assert np.array_equal(gq, Q[a0:a1]), (r, s, g)


def test_xgpu_unaligned_strips():
    """Strip bases off the 16-byte grid: the partial kernel's direct (non-TMA) path."""
    p, N, nbytes, S, G = 13, 12, 2 * 12288 + 77, 2, 3
    b = Batch(p, N, nbytes, S, offset=4, align=0)
    refs = _refs(b, p, N, nbytes, S, 8, 14)
    plan = R.Plan(p, N, nbytes)
    emu = xgpu.Emulated(plan, G, b.data, b.par, S)
    emu.step(None)
    for s, (x, y) in enumerate([(2, 9), (4, N)]):
        for k in (x, y):
            b.strip(s, k).fill_(0)
    emu.step([(2, 9), (4, N)])
    plan.sync()
    for s in range(S):
        for k in range(N + 2):
            assert np.array_equal(_np(b.strip(s, k)), refs[s][k]), (s, k)


def test_xgpu_argument_errors():
    p, N, nbytes = 13, 12, 4096
    plan = R.Plan(p, N, nbytes)
    rb = plan.xgpu_range_bytes(2)
    d = torch.zeros(N * nbytes, dtype=torch.uint8, device="cuda")
    strips = [int(d.data_ptr()) + k * nbytes for k in range(N)] + [None, None]
    slot = torch.zeros(4 * rb, dtype=torch.uint8, device="cuda")
    sp = [int(slot.data_ptr()), int(slot.data_ptr()) + rb]
    with pytest.raises(R.Raid6Error):  # k_hi beyond N+2
        plan.partial_strided(strips, nbytes, nbytes, 1, None, 0, N + 3, sp, sp, rb, rb)
    with pytest.raises(R.Raid6Error):  # a held strip is NULL (P is in [0, N+1))
        plan.partial_strided(strips, nbytes, nbytes, 1, None, 0, N + 1, sp, sp, rb, rb)
    with pytest.raises(R.Raid6Error):  # range not a multiple of the tile
        plan.partial_strided(strips, nbytes, nbytes, 1, None, 0, N, sp, sp, rb, rb + 1)
    with pytest.raises(R.Raid6Error):  # output strips (P, Q) missing in the combine
        plan.combine_strided(strips, nbytes, nbytes, 1, None, sp, sp, rb, 0, rb)
    with pytest.raises(R.Raid6Error):  # bad erasure index
        plan.combine_strided(strips, nbytes, nbytes, 1, [(0, N + 2)], sp, sp, rb, 0, rb)
    full = [int(d.data_ptr()) + k * nbytes for k in range(N + 2)]
    with pytest.raises(R.Raid6Error):  # range end off the granule grid (and not the strip end)
        plan.combine_strided(full, nbytes, nbytes, 1, None, sp, sp, rb, 0, rb - 16)


def test_distributed_ipc_two_processes():
    """The one-process-per-GPU driver (CUDA IPC arenas, peer stores into owner slots) with two
    ranks sharing cuda:0 under gloo.  The ranks' kernels never wait on each other: the barrier
    between phases is a stream sync + host barrier."""
    env = dict(os.environ, MASTER_ADDR="127.0.0.1", MASTER_PORT=str(29500 + os.getpid() % 1000))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", f"--master-port={env['MASTER_PORT']}",
           os.path.join(ROOT, "tests", "xgpu_ipc_worker.py")]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert r.stdout.count("xgpu-ipc ok") == 2, r.stdout[-3000:]
