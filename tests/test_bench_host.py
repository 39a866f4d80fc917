"""CPU checks of bench.py's workload definitions against BASELINE.json (the five configs), and of
its erasure schedules (every pair / class is exercised as the configs require)."""
import json
import os
import re

import pytest

import bench
import synthetic

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _baseline_configs():
    with open(os.path.join(ROOT, "BASELINE.json")) as f:
        return json.load(f)["configs"]


def test_configs_match_baseline_json():
    cfgs = _baseline_configs()
    assert len(cfgs) == 5
    for i, text in enumerate(cfgs, start=1):
        c = bench.CONFIGS[i]
        p = int(re.search(r"p=(\d+)", text).group(1))
        N = int(re.search(r"N=(\d+)", text).group(1))
        assert (c["p"], c["N"]) == (p, N), (i, text)
    assert bench.CONFIGS[1]["nbytes"] == 64 << 10 and "64 KiB" in cfgs[0]
    assert bench.CONFIGS[2]["nbytes"] == 4 << 20 and bench.CONFIGS[2]["stripes"] == 256 and "256 stripes" in cfgs[1]
    assert bench.CONFIGS[3]["nbytes"] == 16 << 20 and "16 MiB" in cfgs[2]
    assert bench.CONFIGS[4]["nbytes"] == 8 << 20 and bench.FULL_STRIPES[4] == 4096 and "4096 stripes" in cfgs[3]
    assert bench.CONFIGS[5]["nbytes"] == 32 << 20 and bench.FULL_STRIPES[5] == 1000 and "1,000 stripes" in cfgs[4]
    assert bench.CONFIGS[4]["sparse"] == 2 and "sparse" in cfgs[3]  # odd stripes sparse (50 / 50)
    assert bench.CONFIGS[3]["ops"] == "enc" and "encode-only" in cfgs[2]
    assert bench.CONFIGS[5]["ops"] == "rec"


def test_c2_schedule_cycles_all_91_pairs():
    N = 12
    seen = set()
    for step in range(3):
        seen |= set(bench.pair_schedule(2, N, 256, 0, step))
    assert seen == set(synthetic.all_pairs(N)) and len(seen) == 91


def test_c4_schedule_covers_every_dd_pair_twice():
    N = 58
    pairs = bench.pair_schedule(4, N, 4096, 0, 0)
    dd = [(i, j) for i in range(N) for j in range(i + 1, N)]
    assert len(dd) == 1653
    counts = {}
    for pr in pairs:
        assert pr[1] < N  # double-data-disk recovery only
        counts[pr] = counts.get(pr, 0) + 1
    assert set(counts) == set(dd) and min(counts.values()) >= 2


def test_c5_degraded_stream_mixes_classes_uniformly():
    N = 60
    pairs = bench.pair_schedule(5, N, 1000, 0, 0)
    classes = [synthetic.pair_class(N, i, j) for i, j in pairs]
    for cls in ("DD", "DP", "DQ", "PQ"):
        share = classes.count(cls) / len(classes)
        assert 0.2 < share < 0.3, (cls, share)
    # the stream is a function of the global stripe index only (identical for any sharding)
    assert bench.pair_schedule(5, N, 500, 500, 0) == pairs[500:]


@pytest.mark.parametrize("cfg,N,nbytes", [(2, 12, 4 << 20), (4, 58, 8 << 20)])
def test_alg_bytes_recover_reads_n_writes_two(cfg, N, nbytes):
    pb = nbytes + 5  # any parity length: the formula is N strips read + 2 strips written per stripe
    pairs = bench.pair_schedule(cfg, N, 10, 0, 0)
    assert bench.alg_bytes_recover(N, nbytes, pb, pairs) == 10 * (N * nbytes + 2 * pb)


def test_gpus_n_without_enough_gpus_fails_loudly():
    """--gpus 2 over NCCL on a box with fewer GPUs must exit non-zero (never run one rank)."""
    import subprocess
    import sys
    import torch
    if torch.cuda.device_count() >= 2:
        pytest.skip("this check needs a box with fewer than 2 GPUs")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "1"],
                       capture_output=True, text=True, timeout=300,
                       env={k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")})
    assert r.returncode == 2 and "needs 2 visible GPUs" in r.stderr
    assert not [ln for ln in r.stdout.splitlines() if ln.startswith("{")]


def test_world_size_must_match_gpus():
    import subprocess
    import sys
    env = dict(os.environ, WORLD_SIZE="3", RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "1"],
                       capture_output=True, text=True, timeout=300, env=env)
    assert r.returncode == 2 and "3 rank(s) running but --gpus 2" in r.stderr
