"""GPU parity tests: libraid6c (through its C ABI) vs the CPU oracle, bit-exact.

Sizes the oracle finishes in seconds (spanning several TMA tiles plus a ragged tail),
every erasure pair for small N, unaligned pointers, the generic (runtime-p) kernel, and at
BASELINE.json's full sizes -- in bench.py's launch configuration -- sampled word-aligned
segments checked against the oracle plus whole-strip round-trip equality with the
generator's bytes.  All inputs are seeded (synthetic/)."""
import itertools

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # collected on CPU boxes but never run there
    pytest.skip("needs a CUDA device", allow_module_level=True)

import oracle  # noqa: E402
import synthetic  # noqa: E402
from paper_cs_0611109_b200 import raid6c as R  # noqa: E402
from tests.gpu_util import Batch, segment_bounds  # noqa: E402

FAST = [3, 5, 7, 11, 13, 17, 19, 29, 37, 53, 59, 61, 257,
        23, 31, 41, 43, 47, 73, 89, 97, 101, 109, 113, 137, 193, 233, 241]
GENERIC = [67, 71, 79, 83, 103, 127, 131, 251]  # period lcm(n, 32) above 32 lanes


def _poison(b, s, ks):
    for k in ks:
        b.strip(s, k).fill_(0xA5)


def _np(t):
    return t.cpu().numpy()


# ------------------------------------------------------------------ generator
def test_fill_matches_numpy_generator():
    for mode, nbytes, S in [(0, 1000, 3), (1, 4099, 2), (2, 777, 4)]:
        b = Batch(13, 5, nbytes, S)
        b.fill_synthetic(seed=7, cfg=3, stripe0=11, sparse_mode=mode)
        torch.cuda.synchronize()
        for s in range(S):
            sparse = mode == 1 or (mode == 2 and (11 + s) % 2 == 1)
            for k in range(5):
                ref = synthetic.strip_bytes(7, 3, 11 + s, k, nbytes, sparse)
                assert np.array_equal(_np(b.strip(s, k)), ref), (mode, s, k)


# ------------------------------------------------------------------ north-star single-stripe API
@pytest.mark.parametrize("p", FAST + GENERIC)
def test_encode_single_matches_oracle(p):
    assert R.has_fast_path(p) == (p in FAST)
    rng = np.random.default_rng(p)
    for N, nbytes in [(1, 1), (min(p, 3), 37), (p - 1, 5000), (p, 1024 + 7)]:
        if p == 257 and N > 70:
            N = 64
        data = [rng.integers(0, 256, nbytes, dtype=np.uint8) for _ in range(N)]
        P, Q = oracle.encode(p, data, nbytes)
        pb = R.parity_bytes(p, nbytes)
        dd = [torch.from_numpy(d).cuda() for d in data]
        gP = torch.full((pb,), 0x5A, dtype=torch.uint8, device="cuda")
        gQ = torch.full((pb,), 0x5A, dtype=torch.uint8, device="cuda")
        R.encode(p, N, dd, gP, gQ, nbytes)
        assert np.array_equal(_np(gP), P), (p, N, nbytes)
        assert np.array_equal(_np(gQ), Q), (p, N, nbytes)


@pytest.mark.parametrize("p,N,nbytes", [(3, 3, 100), (5, 4, 65536), (7, 7, 999), (13, 12, 3 * 12288 + 4097),
                                        (17, 17, 2000), (59, 9, 30000), (61, 11, 16000), (257, 6, 20000),
                                        (11, 10, 1500), (29, 5, 777)])
def test_recover_single_all_pairs(p, N, nbytes):
    rng = np.random.default_rng(p * 7 + N)
    data = [rng.integers(0, 256, nbytes, dtype=np.uint8) for _ in range(N)]
    P, Q = oracle.encode(p, data, nbytes)
    orig = data + [P, Q]
    pairs = list(itertools.combinations(range(N + 2), 2))
    if len(pairs) > 40:
        pairs = pairs[:10] + [pairs[i] for i in rng.choice(len(pairs), 30, replace=False)]
    for i, j in pairs:
        strips = [torch.from_numpy(a.copy()).cuda() for a in orig]
        strips[i].fill_(0xA5)
        strips[j].fill_(0x5A)
        R.recover(p, N, j, i, strips, nbytes)
        for k in (i, j):
            assert np.array_equal(_np(strips[k]), orig[k]), (p, N, i, j, k)


# ------------------------------------------------------------------ batched / strided API (TMA path)
@pytest.mark.parametrize("p,N,nbytes,S", [(13, 12, 5 * 12288 + 1234, 3), (5, 4, 4 * 12288 + 4096, 2),
                                          (59, 58, 3 * 14848 + 99, 2), (61, 60, 2 * 15360 + 7, 2),
                                          (257, 64, 3 * 8192 + 5000, 2), (3, 3, 12288 * 3 + 1, 2),
                                          (17, 16, 12288 * 2 + 30, 2), (7, 6, 12288 * 2 + 13, 2),
                                          (19, 18, 9000, 2)] +
                         [(p, min(p - 1, 40), 3 * 16384 + 1001, 2) for p in FAST[13:]])
def test_batch_encode_and_mixed_recover(p, N, nbytes, S):
    b = Batch(p, N, nbytes, S)
    b.fill_synthetic(seed=1, cfg=9, stripe0=0)
    b.par.fill_(0x77)
    plan = R.Plan(p, N, nbytes)
    plan.encode_strided(*b.args())
    plan.sync()
    refs = []
    for s in range(S):
        data = synthetic.stripe_strips(1, 9, s, N, nbytes)
        P, Q = oracle.encode(p, data, nbytes)
        assert np.array_equal(_np(b.strip(s, N)), P), (p, s)
        assert np.array_equal(_np(b.strip(s, N + 1)), Q), (p, s)
        refs.append(data + [P, Q])
    # mixed classes across stripes, host pairs then device pairs
    allp = synthetic.all_pairs(N)
    rng = np.random.default_rng(p)
    for trial in range(3):
        pairs = [allp[int(rng.integers(len(allp)))] for _ in range(S)]
        if trial == 0:
            pairs[0] = (0, 1) if N >= 2 else (0, N)
        for s, (i, j) in enumerate(pairs):
            _poison(b, s, (i, j))
        if trial == 2:
            dev = torch.tensor(pairs, dtype=torch.int32, device="cuda")
            plan.recover_strided(*b.args(), dev)
        else:
            plan.recover_strided(*b.args(), pairs)
        plan.sync()
        for s, (i, j) in enumerate(pairs):
            for k in (i, j):
                assert np.array_equal(_np(b.strip(s, k)), refs[s][k]), (p, trial, s, i, j, k)
    plan.close()


@pytest.mark.parametrize("offset", [1, 3, 8, 15])
def test_unaligned_pointers(offset):
    p, N, nbytes, S = 13, 12, 3 * 12288 + 5, 2
    b = Batch(p, N, nbytes, S, offset=offset, align=0)
    b.fill_synthetic(seed=2, cfg=1)
    plan = R.Plan(p, N, nbytes)
    plan.encode_strided(*b.args())
    plan.sync()
    for s in range(S):
        data = synthetic.stripe_strips(2, 1, s, N, nbytes)
        P, Q = oracle.encode(p, data, nbytes)
        assert np.array_equal(_np(b.strip(s, N)), P)
        assert np.array_equal(_np(b.strip(s, N + 1)), Q)
        orig = data + [P, Q]
        for (i, j) in [(0, 5), (3, N), (7, N + 1), (N, N + 1)]:
            _poison(b, s, (i, j))
            plan.recover_strided(*b.args(), [(i, j)] * 1)
            plan.sync()
            assert np.array_equal(_np(b.strip(s, i)), orig[i])
            assert np.array_equal(_np(b.strip(s, j)), orig[j])


@pytest.mark.parametrize("p,N", [(5, 4), (13, 12), (13, 17), (59, 20), (127, 9)])
def test_pq_only_recovery_runs_as_encode(p, N):
    """Launches whose every pair is {P, Q} (host list, either order; the single-stripe call) are
    dispatched to the encode kernel: poisoned P and Q must come back equal to the oracle's."""
    nbytes, S = 3 * 15360 + 333, 3
    b = Batch(p, N, nbytes, S)
    b.fill_synthetic(seed=12, cfg=2)
    plan = R.Plan(p, N, nbytes)
    ref = []
    for s in range(S):
        data = synthetic.stripe_strips(12, 2, s, N, nbytes)
        ref.append(oracle.encode_ext(p, data, nbytes) if N > p else oracle.encode(p, data, nbytes))
    for pairs in ([(N, N + 1)], [(N + 1, N), (N, N + 1), (N + 1, N)]):
        for s in range(S):
            _poison(b, s, (N, N + 1))
        plan.recover_strided(*b.args(), pairs)
        plan.sync()
        for s in range(S):
            assert np.array_equal(_np(b.strip(s, N)), ref[s][0]), (p, N, pairs, s)
            assert np.array_equal(_np(b.strip(s, N + 1)), ref[s][1]), (p, N, pairs, s)
    _poison(b, 1, (N, N + 1))
    R.recover(p, N, N + 1, N, [int(b.strip(1, k).data_ptr()) for k in range(N + 2)], nbytes)
    assert np.array_equal(_np(b.strip(1, N)), ref[1][0]) and np.array_equal(_np(b.strip(1, N + 1)), ref[1][1])


@pytest.mark.parametrize("p,N,nbytes", [(3, 2, 65536), (5, 4, 65536), (5, 4, 3 * 10752 + 77), (13, 12, 4 * 15360 + 333),
                                        (17, 16, 2 * 13440 + 1008), (59, 58, 2 * 14848 + 5), (61, 60, 15360 + 1),
                                        (257, 64, 3 * 8192 + 96), (233, 30, 14848 + 700)])
def test_light_recovery_dp_dq_batches(p, N, nbytes):
    """Launches with no DD stripe (host pair lists of DP / DQ / PQ) run on the light recovery
    kernel: every rebuilt strip must equal the generator's / the oracle's bytes."""
    S = 5
    b = Batch(p, N, nbytes, S)
    b.fill_synthetic(seed=21, cfg=4)
    plan = R.Plan(p, N, nbytes)
    plan.encode_strided(*b.args())
    plan.sync()
    orig = []
    for s in range(S):
        data = synthetic.stripe_strips(21, 4, s, N, nbytes)
        P, Q = oracle.encode(p, data, nbytes)
        assert np.array_equal(_np(b.strip(s, N)), P) and np.array_equal(_np(b.strip(s, N + 1)), Q)
        orig.append(data + [P, Q])
    mixes = [[(N - 1, N)] * S, [(0, N + 1)] * S,
             [(s % N, N + (s % 2)) for s in range(S)], [(N, N + 1), (N + 1, 1), (2 % N, N), (N, N + 1), (N + 1, 0)]]
    for pairs in mixes:
        for s, (i, j) in enumerate(pairs):
            _poison(b, s, (i, j))
        plan.recover_strided(*b.args(), pairs if len(set(pairs)) > 1 else pairs[:1])
        plan.sync()
        for s, (i, j) in enumerate(pairs):
            for k in (i, j):
                assert np.array_equal(_np(b.strip(s, k)), orig[s][k]), (p, N, pairs, s, k)
    for (i, j) in [(1, N), (N + 1, N - 1)]:  # the single-stripe call
        _poison(b, 2, (i, j))
        R.recover(p, N, i, j, [int(b.strip(2, k).data_ptr()) for k in range(N + 2)], nbytes)
        for k in (i, j):
            assert np.array_equal(_np(b.strip(2, k)), orig[2][k]), (p, N, i, j, k)


@pytest.mark.parametrize("p,N,nbytes,S,dd_every", [(5, 4, 65536, 400, 0), (13, 12, 4 * 15360 + 333, 480, 3),
                                                   (61, 60, 3 * 15360 + 16, 640, 3)])
def test_large_mixed_host_table_batches(p, N, nbytes, S, dd_every):
    """Mixed-class batches from HOST pair tables, large enough that every CTA of the persistent
    launch walks several items of different classes (a raw list, then a prebuilt raid6c_erasure
    array; pairs in either index order).  Every lost strip is poisoned first; afterwards every
    byte of the batch must equal the pre-erasure snapshot (untouched neighbours included), and on
    stripes spread over the batch the data the generator's bytes and the parity the oracle's."""
    b = Batch(p, N, nbytes, S)
    b.fill_synthetic(seed=33, cfg=1)
    plan = R.Plan(p, N, nbytes)
    plan.encode_strided(*b.args())
    plan.sync()
    snap_d, snap_p = b.data.clone(), b.par.clone()
    allp = synthetic.all_pairs(N)
    dd = [pr for pr in allp if pr[1] < N]
    li = [pr for pr in allp if pr[1] >= N]
    if dd_every == 0:   # the bench's c1 schedule: cycle through every pair (6 of 15 are data-data)
        pairs = [allp[(s + 37) % len(allp)] for s in range(S)]
    else:               # every dd_every-th stripe data-data
        pairs = [dd[(7 * s) % len(dd)] if s % dd_every == 0 else li[(5 * s) % len(li)] for s in range(S)]
        pairs = [(j, i) if s % 2 else (i, j) for s, (i, j) in enumerate(pairs)]
    for rep in range(2):  # twice: the second call rewrites the plan's device table behind the first
        for s, (i, j) in enumerate(pairs):
            _poison(b, s, (i, j))
        n0 = R.launch_count()
        plan.recover_strided(*b.args(), pairs if rep == 0 else R.erasure_array(pairs))
        plan.sync()
        assert R.launch_count() - n0 == 1
        assert torch.equal(b.data, snap_d) and torch.equal(b.par, snap_p)
    sample = sorted(set(list(range(0, S, max(1, S // 10))) + [S - 1, S - 2, 1]))
    for s in sample:
        data = synthetic.stripe_strips(33, 1, s, N, nbytes)
        P, Q = oracle.encode(p, data, nbytes)
        ref = data + [P, Q]
        for k in range(N + 2):
            assert np.array_equal(_np(b.strip(s, k)), ref[k]), (p, s, k, pairs[s])
    plan.close()


def test_lost_strips_never_read_and_neighbours_untouched():
    """Poisoned lost strips do not change the result; bytes outside the strips are untouched."""
    p, N, nbytes, S = 13, 12, 2 * 12288 + 77, 2
    b = Batch(p, N, nbytes, S)
    b.fill_synthetic(seed=3, cfg=2)
    plan = R.Plan(p, N, nbytes)
    plan.encode_strided(*b.args())
    plan.sync()
    # guard bytes between strips (stride padding) must stay as they are
    b.data[:, :, nbytes:].fill_(0xEE)
    b.par[:, :, b.pb:].fill_(0xEE)
    snap = b.data.clone(), b.par.clone()
    for fillv in (0x00, 0xFF, 0xA5):
        for s in range(S):
            b.strip(s, 2).fill_(fillv)
            b.strip(s, 9).fill_(fillv)
        plan.recover_strided(*b.args(), [(2, 9)])
        plan.sync()
        assert torch.equal(b.data, snap[0]) and torch.equal(b.par, snap[1])


# ------------------------------------------------------------------ host-buffer API (e2e path)
def test_host_buffer_api_matches_device_path():
    p, N, nbytes, S = 13, 12, 2 * 12288 + 901, 5
    b = Batch(p, N, nbytes, S)
    b.fill_synthetic(seed=4, cfg=2)
    plan = R.Plan(p, N, nbytes)
    plan.encode_strided(*b.args())
    plan.sync()
    hd = b.data.cpu().pin_memory()
    hp = torch.zeros_like(b.par, device="cpu").pin_memory()
    plan.encode_batch(hd, hp)
    assert torch.equal(hp[:, :, :b.pb], b.par[:, :, :b.pb].cpu())
    h2d, d2h = plan.host_traffic()
    assert h2d == S * N * nbytes and d2h == S * 2 * b.pb
    pairs = [(0, 1), (4, N), (5, N + 1), (N, N + 1), (10, 11)]
    ref_d, ref_p = hd.clone(), hp.clone()
    for s, (i, j) in enumerate(pairs):
        for k in (i, j):
            if k < N:
                hd[s, k, :nbytes] = 0xA5
            else:
                hp[s, k - N, :b.pb] = 0xA5
    plan.recover_batch(hd, hp, pairs)
    assert torch.equal(hd, ref_d) and torch.equal(hp[:, :, :b.pb], ref_p[:, :, :b.pb])


@pytest.mark.parametrize("p,N,nbytes", [(5, 4, 2 * 10752 + 1024), (13, 12, 2 * 15360 + 333), (257, 20, 8192 + 96),
                                        (67, 9, 5000), (5, 9, 4096 + 7)])
def test_single_erasure(p, N, nbytes):
    """lost_j = RAID6C_NONE (optional): strip lost_i alone is rebuilt -- as the pair
    (lost_i, Q), or (P, Q) for lost_i = Q -- through the single-stripe call, a host pair table and
    the host-buffer call; every strip of the stripe must then hold the generator's data and the
    oracle's parity (fast, generic and extended-code plans)."""
    S = 3
    b = Batch(p, N, nbytes, S)
    b.fill_synthetic(seed=44, cfg=2)
    plan = R.Plan(p, N, nbytes)
    plan.encode_strided(*b.args())
    plan.sync()
    enc = oracle.encode_ext if N > p else oracle.encode
    ref = []
    for s in range(S):
        data = synthetic.stripe_strips(44, 2, s, N, nbytes)
        P, Q = enc(p, data, nbytes)
        ref.append(data + [P, Q])

    def check(tag):
        for s in range(S):
            for k in range(N + 2):
                assert np.array_equal(_np(b.strip(s, k)), ref[s][k]), (p, N, tag, s, k)

    check("encode")
    for i in range(N + 2):  # the single-stripe call, every strip of stripe 1
        _poison(b, 1, (i,))
        R.recover(p, N, i, R.NONE, [int(b.strip(1, k).data_ptr()) for k in range(N + 2)], nbytes)
        check(("single", i))
    tables = [[(s % (N + 2), R.NONE) for s in range(S)],                      # singles only
              [(N + 1, R.NONE), (0, N - 1) if N > 1 else (0, N), (N, R.NONE)],  # mixed with a pair
              [(N - 1, R.NONE)]]                                              # one entry for every stripe
    for t in tables:
        full = t if len(t) == S else t * S
        for s, (i, j) in enumerate(full):
            _poison(b, s, (i,) if j == R.NONE else (i, j))
        plan.recover_strided(*b.args(), t)
        plan.sync()
        check(("table", t))
    # the host-buffer call
    hd = b.data.cpu().pin_memory()
    hp = b.par.cpu().pin_memory()
    hd[0, 0, :nbytes] = 0xA5
    hp[1, 1, :b.pb] = 0xA5
    hd[2, N - 1, :nbytes] = 0xA5
    plan.recover_host(hd, b.ss, N * b.ss, hp, int(hp.data_ptr()) + b.ps, 2 * b.ps, S,
                      [(0, R.NONE), (N + 1, R.NONE), (N - 1, R.NONE)])
    plan.sync()
    for s in range(S):
        for k in range(N + 2):
            got = hd[s, k, :nbytes].numpy() if k < N else hp[s, k - N, :b.pb].numpy()
            assert np.array_equal(got, ref[s][k]), (p, N, "host", s, k)
    with pytest.raises(R.Raid6Error, match="INVALID_INDEX"):
        plan.recover_strided(*b.args(), [(R.NONE, 0)])   # lost_i must name a strip
    with pytest.raises(R.Raid6Error, match="INVALID_INDEX"):
        plan.recover_strided(*b.args(), [(0, -2)])
    plan.close()


# ------------------------------------------------------------------ argument errors (T1)
def test_argument_errors_are_synchronous():
    t = torch.zeros(64, dtype=torch.uint8, device="cuda")
    with pytest.raises(R.Raid6Error, match="INVALID_P"):
        R.Plan(9, 3, 100)
    with pytest.raises(R.Raid6Error, match="INVALID_N"):
        R.Plan(5, 10, 100)  # N > 2p - 1
    with pytest.raises(R.Raid6Error, match="INVALID_N"):
        R.Plan(7, 8, 100)  # N > p but 7 fails Theorem 25.3
    with pytest.raises(R.Raid6Error, match="SIZE"):
        R.Plan(5, 2, 0)
    plan = R.Plan(5, 2, 16)
    with pytest.raises(R.Raid6Error, match="INVALID_INDEX"):
        plan.recover_strided(t, 16, 32, t, int(t.data_ptr()) + 16, 32, 1, [(1, 1)])
    with pytest.raises(R.Raid6Error, match="INVALID_INDEX"):
        plan.recover_strided(t, 16, 32, t, int(t.data_ptr()) + 16, 32, 1, [(0, 4)])
    with pytest.raises(R.Raid6Error, match="NULL"):
        plan.encode_strided(0, 16, 32, t, t, 32, 1)
    with pytest.raises(R.Raid6Error, match="INVALID_INDEX"):
        R.recover(5, 2, 0, 0, [t, t, t, t], 16)
    plan.sync()


# ------------------------------------------------------------------ full BASELINE sizes (sampled)
def _check_segments(b, p, N, nbytes, seed, cfg, stripes, sparse_of=lambda s: False):
    for s in stripes:
        for which in ("head", "mid", "tail"):
            b0, b1 = segment_bounds(p, nbytes, which)
            segs = [synthetic.strip_bytes(seed, cfg, s, k, nbytes, sparse_of(s), lo=b0, hi=b1) for k in range(N)]
            P, Q = oracle.encode(p, segs, b1 - b0)
            e = b0 + P.size
            assert np.array_equal(_np(b.par[s, 0, b0:e]), P), (s, which)
            assert np.array_equal(_np(b.par[s, 1, b0:e]), Q), (s, which)


def _roundtrip_full(b, plan, pairs):
    S = b.S
    ref_d, ref_p = b.data.clone(), b.par.clone()
    for s, (i, j) in enumerate(pairs):
        _poison(b, s, (i, j))
    plan.recover_strided(*b.args(), torch.tensor(pairs, dtype=torch.int32, device="cuda"))
    plan.sync()
    cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
    R.count_mismatch(b.data, ref_d, b.data.numel(), cnt)
    R.count_mismatch(b.par, ref_p, b.par.numel(), cnt)
    torch.cuda.synchronize()
    assert int(cnt.item()) == 0


def test_config1_full():
    """c1: p=5, N=4, 64 KiB, seed 0: full oracle encode + all 15 pairs."""
    p, N, nbytes = 5, 4, 65536
    b = Batch(p, N, nbytes, 1)
    b.fill_synthetic(seed=0, cfg=1)
    plan = R.Plan(p, N, nbytes)
    plan.encode_strided(*b.args())
    plan.sync()
    data = synthetic.stripe_strips(0, 1, 0, N, nbytes)
    P, Q = oracle.encode(p, data, nbytes)
    assert np.array_equal(_np(b.strip(0, N)), P) and np.array_equal(_np(b.strip(0, N + 1)), Q)
    orig = data + [P, Q]
    for i, j in synthetic.all_pairs(N):
        _poison(b, 0, (i, j))
        plan.recover_strided(*b.args(), [(i, j)])
        plan.sync()
        for k in range(N + 2):
            assert np.array_equal(_np(b.strip(0, k)), orig[k]), (i, j, k)


def test_config2_full_size_all_91_pairs():
    """c2: p=13, N=12, 4 MiB strips; 8 stripes in bench.py's launch configuration; all 91 pairs
    (stripe s takes pair (s + 8r) mod 91 in round r) round-trip exactly; sampled oracle segments."""
    p, N, nbytes, S = 13, 12, 4 << 20, 8
    b = Batch(p, N, nbytes, S)
    b.fill_synthetic(seed=0, cfg=2)
    plan = R.Plan(p, N, nbytes)
    plan.encode_strided(*b.args())
    plan.sync()
    _check_segments(b, p, N, nbytes, 0, 2, [0, 5])
    allp = synthetic.all_pairs(N)
    for r in range(12):
        _roundtrip_full(b, plan, [allp[(s + 8 * r) % 91] for s in range(S)])


def test_config3_p257_sweep_points():
    """c3: p=257, N=64, encode at 64 KiB (full oracle) and 16 MiB (sampled)."""
    p, N = 257, 64
    for nbytes, S, full in [(64 << 10, 2, True), (16 << 20, 1, False)]:
        b = Batch(p, N, nbytes, S)
        b.fill_synthetic(seed=0, cfg=3)
        plan = R.Plan(p, N, nbytes)
        plan.encode_strided(*b.args())
        plan.sync()
        if full:
            for s in range(S):
                data = synthetic.stripe_strips(0, 3, s, N, nbytes)
                P, Q = oracle.encode(p, data, nbytes)
                assert np.array_equal(_np(b.strip(s, N)), P) and np.array_equal(_np(b.strip(s, N + 1)), Q)
        else:
            _check_segments(b, p, N, nbytes, 0, 3, [0])
        _roundtrip_full(b, plan, [(3, 60)] * S)


def test_config4_full_size_dd():
    """c4: p=59, N=58, 8 MiB; even stripes uniform, odd sparse; DD pairs (s mod 1653)."""
    p, N, nbytes, S = 59, 58, 8 << 20, 4
    b = Batch(p, N, nbytes, S)
    b.fill_synthetic(seed=0, cfg=4, sparse_mode=2)
    plan = R.Plan(p, N, nbytes)
    plan.encode_strided(*b.args())
    plan.sync()
    _check_segments(b, p, N, nbytes, 0, 4, [0, 1], sparse_of=lambda s: s % 2 == 1)
    dd = [(i, j) for i in range(N) for j in range(i + 1, N)]
    assert len(dd) == 1653
    _roundtrip_full(b, plan, [dd[s * 411 % 1653] for s in range(S)])


def test_config5_full_size_degraded_stream():
    """c5: p=61, N=60, 32 MiB; per-stripe seeded erasure pairs over all classes."""
    p, N, nbytes, S = 61, 60, 32 << 20, 4
    b = Batch(p, N, nbytes, S)
    b.fill_synthetic(seed=0, cfg=5)
    plan = R.Plan(p, N, nbytes)
    plan.encode_strided(*b.args())
    plan.sync()
    _check_segments(b, p, N, nbytes, 0, 5, [1])
    pairs = [(3, 40), (7, N), (11, N + 1), (N, N + 1)]
    _roundtrip_full(b, plan, pairs)
    _roundtrip_full(b, plan, [synthetic.erasure_pair(0, 5, s, N) for s in range(S)])


# ------------------------------------------------------------------ pipeline race stress
@pytest.mark.parametrize("p,N,nbytes,S", [(5, 4, 65536, 4096), (13, 12, 4 << 20, 48), (257, 64, 1 << 20, 24),
                                          (61, 60, 2 << 20, 16), (59, 58, 2 << 20, 16)])
def test_pipeline_race_stress(p, N, nbytes, S):
    """Many items per persistent CTA (warp 0 lags behind while it drives the bulk stores):
    repeated encodes must be bit-identical and in-place mixed recoveries must leave every
    byte unchanged.  Guards the TMA stage-release ordering."""
    b = Batch(p, N, nbytes, S)
    b.fill_synthetic(seed=5, cfg=7)
    plan = R.Plan(p, N, nbytes)
    plan.encode_strided(*b.args())
    plan.sync()
    ref_d, ref_p = b.data.clone(), b.par.clone()
    allp = synthetic.all_pairs(N)
    cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
    for step in range(4):
        plan.encode_strided(*b.args())
        pairs = torch.tensor([allp[(s * 7 + 37 * step) % len(allp)] for s in range(S)], dtype=torch.int32,
                             device="cuda")
        plan.recover_strided(*b.args(), pairs)
    plan.sync()
    R.count_mismatch(b.data, ref_d, b.data.numel(), cnt)
    R.count_mismatch(b.par, ref_p, b.par.numel(), cnt)
    torch.cuda.synchronize()
    assert int(cnt.item()) == 0
    # and the parity itself is the oracle's (sampled segments of the first and last stripe)
    for s in (0, S - 1):
        for which in ("head", "tail"):
            b0, b1 = segment_bounds(p, nbytes, which)
            segs = [synthetic.strip_bytes(5, 7, s, k, nbytes, lo=b0, hi=b1) for k in range(N)]
            P, Q = oracle.encode(p, segs, b1 - b0)
            assert np.array_equal(_np(b.par[s, 0, b0:b0 + P.size]), P)
            assert np.array_equal(_np(b.par[s, 1, b0:b0 + Q.size]), Q)


@pytest.mark.parametrize("p", [5, 13, 17, 59, 61, 257, 11, 67] + FAST[13:])
def test_dd_solve_every_z(p):
    """The DD solve (1 + x^z)^{-1} (reading R11) for every z = y - x in
    1..N-1 with N = p - 1 data strips, at varying x (the rotation origin): one stripe per z,
    batched, through the TMA path with a ragged tail.  The encode of the batch is checked
    against the oracle first; the rebuilt strips must equal the originals."""
    N = p - 1
    nbytes = {5: 10752 + 333, 13: 12288 + 333, 17: 10752 + 77, 59: 14848 + 333, 61: 15360 + 333,
              257: 8192 + 96, 11: 3000, 67: 2000}.get(p, 16384 + 333)
    zs = list(range(1, N))
    S = len(zs)
    b = Batch(p, N, nbytes, S)
    b.fill_synthetic(seed=41, cfg=17)
    plan = R.Plan(p, N, nbytes)
    plan.encode_strided(*b.args())
    plan.sync()
    for s in (0, S - 1):
        data = synthetic.stripe_strips(41, 17, s, N, nbytes)
        P, Q = oracle.encode(p, data, nbytes)
        assert np.array_equal(_np(b.strip(s, N)), P) and np.array_equal(_np(b.strip(s, N + 1)), Q)
    orig = b.data.clone()
    pairs = []
    for s, z in enumerate(zs):
        x = (7 * z + s) % (N - z)
        pairs.append((x + z, x))  # reversed order: the library canonicalises
        _poison(b, s, (x, x + z))
    plan.recover_strided(*b.args(), torch.tensor(pairs, dtype=torch.int32, device="cuda"))
    plan.sync()
    bad = (b.data[:, :, :nbytes] != orig[:, :, :nbytes]).nonzero()
    assert bad.numel() == 0, (p, bad[:5].tolist(), [pairs[int(i)] for i in bad[:5, 0].tolist()])


def test_erasure_table_reuse_across_streams():
    """A plan's device erasure table is rewritten by the next call with host pairs; when that
    call runs on another stream (plan_set_stream), it must not overwrite the table under the
    previous, still-running recovery (event-ordered rewrite)."""
    p, N, nbytes = 13, 12, 4 << 20
    big = Batch(p, N, nbytes, 48)
    small = Batch(p, N, nbytes, 2)
    big.fill_synthetic(seed=51, cfg=18)
    small.fill_synthetic(seed=52, cfg=18)
    sa, sb = torch.cuda.Stream(), torch.cuda.Stream()
    plan = R.Plan(p, N, nbytes, 0, sa)
    plan.encode_strided(*big.args())
    plan.set_stream(sb)
    plan.encode_strided(*small.args())
    plan.sync()
    plan.set_stream(sa)
    plan.sync()
    ref_big, ref_small = (big.data.clone(), big.par.clone()), (small.data.clone(), small.par.clone())
    allp = list(itertools.combinations(range(N + 2), 2))
    pairs_big = [allp[(5 * s) % len(allp)] for s in range(big.S)]
    pairs_small = [(0, 1), (2, 3)]
    for s, pr in enumerate(pairs_big):
        _poison(big, s, pr)
    for s, pr in enumerate(pairs_small):
        _poison(small, s, pr)
    torch.cuda.synchronize()
    plan.set_stream(sa)
    plan.recover_strided(*big.args(), pairs_big)      # host pairs -> the plan's table
    plan.set_stream(sb)
    plan.recover_strided(*small.args(), pairs_small)  # rewrites the table on another stream
    torch.cuda.synchronize()
    plan.set_stream(sa)
    plan.sync()
    for b, (rd, rp) in ((big, ref_big), (small, ref_small)):
        assert torch.equal(b.data, rd) and torch.equal(b.par, rp)


@pytest.mark.parametrize("args", [("13", "12", "1000003", "8"), ("59", "58", "300001", "4"), ("11", "10", "5000", "4"),
                                  ("13", "25", "100000", "4"), ("5", "1", "777", "4")])
def test_c_example_roundtrip(tmp_path, args):
    """examples/c_api_roundtrip.c: encode + recovery of every class through the C ABI from C."""
    import os
    import subprocess
    from tests.test_abi import _build_c_example
    if os.path.basename(R.LIB_PATH) != "libraid6c.so":
        pytest.skip("variant library (RAID6C_LIB)")
    exe = str(tmp_path / "c_api_roundtrip")
    r = _build_c_example(exe)
    assert r.returncode == 0, r.stderr
    r = subprocess.run([exe, *args], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert " 0 strips differ" in r.stdout


def _pack_words(words, n, nbytes):
    """LSB-first bit stream of n-bit words (reading R2) -> nbytes bytes (test-local packing)."""
    v = 0
    for w, x in enumerate(words):
        v |= int(x) << (w * n)
    return np.frombuffer(v.to_bytes(nbytes, "little"), dtype=np.uint8).copy()


def _unpack_words(buf, n, count):
    v = int.from_bytes(bytes(buf), "little")
    return [(v >> (w * n)) & ((1 << n) - 1) for w in range(count)]


@pytest.mark.parametrize("p", FAST + [67, 127, 251])
def test_rotation_unit_vectors(p):
    """Multiplication by x^a (Eq. (powers)) on every unit vector e_b, for every
    amount a < min(p, 64): stripe a holds only data strip a, whose word b is e_b (b < n), so the
    encoded Q word b must equal the oracle's x^a e_b (one Sylvester step at a time) and P word b
    must be e_b.  Checks each rotation amount and bit position (incl. the wrap into the slot
    overflow and its reduction) in isolation."""
    n = p - 1
    N = min(p, 64)
    nbytes = (n * n + 7) // 8
    b = Batch(p, N, nbytes, N)
    b.data.zero_()
    unit = _pack_words([1 << w for w in range(n)], n, nbytes)
    for a in range(N):
        b.data[a, a, :nbytes].copy_(torch.from_numpy(unit))
    plan = R.Plan(p, N, nbytes)
    plan.encode_strided(*b.args())
    plan.sync()
    for a in range(N):
        Pw = _unpack_words(b.numpy_strip(a, N), n, n)
        Qw = _unpack_words(b.numpy_strip(a, N + 1), n, n)
        assert Pw == [1 << w for w in range(n)], a
        for w in range(n):
            assert Qw[w] == oracle.mul_xk(p, a, 1 << w), (p, a, w)


# every prime instantiated in the p-templated generic kernel (zp_generic.cuh), each its own code
GENERIC_ALL = [67, 71, 79, 83, 103, 107, 127, 131, 139, 149, 151, 157, 163, 167, 173, 179, 181, 191, 197,
               199, 211, 223, 227, 229, 239, 251]


@pytest.mark.parametrize("p", GENERIC_ALL)
def test_generic_prime_encode_recover_scrub(p):
    """Each generic-kernel prime (its own template instantiation: group geometry g = 2 or 4,
    NL = 3..8 limbs): batched encode vs the oracle, every recovery class vs the originals on an
    unaligned batch with a ragged tail, and a zero scrub count after encode."""
    assert not R.has_fast_path(p)
    N, nbytes, S = 9, 4 * 1024 + 77, 3
    b = Batch(p, N, nbytes, S, offset=3, align=0)
    b.fill_synthetic(seed=p, cfg=21)
    b.par.fill_(0x6B)
    plan = R.Plan(p, N, nbytes)
    plan.encode_strided(*b.args())
    plan.sync()
    refs = []
    for s in range(S):
        data = synthetic.stripe_strips(p, 21, s, N, nbytes)
        P, Q = oracle.encode(p, data, nbytes)
        assert np.array_equal(b.numpy_strip(s, N), P) and np.array_equal(b.numpy_strip(s, N + 1), Q), (p, s)
        refs.append(data + [P, Q])
    cnt = torch.full((S,), 99, dtype=torch.int32, device="cuda")
    plan.scrub_strided(*b.args(), cnt)
    plan.sync()
    assert cnt.cpu().tolist() == [0] * S
    for pairs in ([(0, 8), (3, N), (5, N + 1)], [(N, N + 1), (1, 2), (7, N)]):
        for s, (i, j) in enumerate(pairs):
            _poison(b, s, (i, j))
        plan.recover_strided(*b.args(), pairs)
        plan.sync()
        for s, (i, j) in enumerate(pairs):
            for k in (i, j):
                assert np.array_equal(b.numpy_strip(s, k), refs[s][k]), (p, s, i, j, k)
    # small-write update of one strip per stripe (unaligned new rows) vs the oracle's re-encode
    ns = nbytes + 5
    newbuf = torch.zeros(S * ns + 16, dtype=torch.uint8, device="cuda")
    new = newbuf[1:1 + S * ns].view(S, ns)
    R.fill(new, ns, ns, nbytes, 1, S, p, 8, 0, 0, 0)
    disks = [(4 * s + 2) % N for s in range(S)]
    plan.update_strided(*b.args(), int(new.data_ptr()), ns, disks)
    plan.sync()
    for s in range(S):
        data = refs[s][:N]
        data[disks[s]] = new[s, :nbytes].cpu().numpy()
        P, Q = oracle.encode(p, data, nbytes)
        for k in range(N):
            assert np.array_equal(b.numpy_strip(s, k), data[k]), (p, s, k)
        assert np.array_equal(b.numpy_strip(s, N), P) and np.array_equal(b.numpy_strip(s, N + 1), Q), (p, s)


# ------------------------------------------------------------------ long-run pipeline check
@pytest.mark.parametrize("p,N,nbytes,S,launches", [(13, 12, 4 << 20, 256, 400), (61, 60, 32 << 20, 8, 200)])
def test_long_run_round_trip(p, N, nbytes, S, launches):
    """bench.py's resident batch driven for hundreds of back-to-back launches (encode, then a
    recovery of a different pair in every stripe, repeated), the round trip checked every 20
    launches: a stage released before its reads completed (a TMA refill racing the consumers)
    shows up here as bytes that stop matching.  c2 at full size; c5 strips, 8 stripes."""
    b = Batch(p, N, nbytes, S)
    b.fill_synthetic(seed=0, cfg=2 if p == 13 else 5)
    plan = R.Plan(p, N, nbytes)
    plan.encode_strided(*b.args())
    plan.sync()
    ref_d, ref_p = b.data.clone(), b.par.clone()
    allp = synthetic.all_pairs(N)
    cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
    pairs = [torch.tensor([allp[(s + 37 * t) % len(allp)] for s in range(S)], dtype=torch.int32, device="cuda")
             for t in range(launches // 2)]
    for t in range(launches // 2):
        plan.encode_strided(*b.args())
        plan.recover_strided(*b.args(), pairs[t])
        if t % 10 == 9:
            plan.sync()
            R.count_mismatch(b.data, ref_d, b.data.numel(), cnt)
            R.count_mismatch(b.par, ref_p, b.par.numel(), cnt)
            torch.cuda.synchronize()
            assert int(cnt.item()) == 0, f"mismatch after {2 * (t + 1)} launches"


# ------------------------------------------------------------------ partial last TMA tile
@pytest.mark.parametrize("p,N", [(3, 2), (5, 4), (17, 16)])
@pytest.mark.parametrize("rest", [16, 1024, 7152])
@pytest.mark.parametrize("S", [2, 600])
def test_partial_last_tile(p, N, rest, S):
    """Lane-aligned words (n | 32) finish a strip whose length leaves `rest` bytes after the
    last whole tile with one partial TMA tile (encode / recovery kernels, ZpArgs::last_tile).
    Strips of 3 whole tiles + rest bytes (rest a multiple of 16) in a persistent launch: every
    stripe's P/Q equal the oracle, and every erasure class rebuilds the whole strips, with the
    guard bytes past each strip untouched.  S = 600: a persistent launch (recovery then keeps the
    direct tail path); S = 2: a small launch (recovery takes the partial tile too)."""
    nbytes = 3 * 10752 + rest if rest < 10752 else rest
    b = Batch(p, N, nbytes, S, align=0)
    assert b.pb == nbytes
    b.fill_synthetic(seed=0, cfg=1)
    plan = R.Plan(p, N, nbytes)
    plan.encode_strided(*b.args())
    plan.sync()
    for s in sorted({0, 1, S - 1}):
        data = synthetic.stripe_strips(0, 1, s, N, nbytes)
        P, Q = oracle.encode(p, data, nbytes)
        assert np.array_equal(_np(b.strip(s, N)), P) and np.array_equal(_np(b.strip(s, N + 1)), Q), s
    allp = synthetic.all_pairs(N)
    ref_d, ref_p = b.data.clone(), b.par.clone()
    guard_d, guard_p = b.dbuf[-64:].clone(), b.pbuf[-64:].clone()
    for r in range(len(allp) if S == 2 else 1):  # small launches: every pair
        pairs = [allp[(s + r) % len(allp)] for s in range(S)]
        for s, pr in enumerate(pairs):
            _poison(b, s, pr)
        plan.recover_strided(*b.args(), torch.tensor(pairs, dtype=torch.int32, device="cuda"))
        plan.sync()
        assert torch.equal(b.data, ref_d) and torch.equal(b.par, ref_p), pairs
        assert torch.equal(b.dbuf[-64:], guard_d) and torch.equal(b.pbuf[-64:], guard_p)
