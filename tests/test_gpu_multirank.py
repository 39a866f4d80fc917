"""bench.py's multi-rank path on the GPU box (one GPU per gpurun call, so the ranks share cuda:0
under gloo; the kernels of different ranks never wait on each other).

* `bench.py --gpus N` with no torchrun environment brings up N ranks itself and reports
  n_gpus = N, N per-rank times and N ranks in its line (never one rank silently).
* Sharding invariance on the GPU: the whole c4 configuration cut into
  G = 1, 2, 4 block shards gives the same per-strip digests of every strip of the run
  (verified.digest_all), and each run's oracle digest sample (spread over all shards) matches.
  Stripes are independent (Eq. (znparity)), so the results cannot depend on G."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _bench(*args, timeout=900):
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), *args]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=timeout)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-5000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-3000:]
    return json.loads(lines[0]), r.stderr


def test_nccl_plumbing_on_one_rank():
    """The NCCL path itself (never reached by the gloo rehearsals): a ONE-rank process group forced
    with RAID6C_FORCE_DIST=1 runs init_process_group("nccl", device_id=...), the object gathers, the
    barriers around the timed region and the device-tensor collectives of shard.py on the box's
    GPU, for the bench step and for a whole-config (--full) run."""
    import socket
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    env = dict(os.environ, RAID6C_FORCE_DIST="1", RANK="0", WORLD_SIZE="1", LOCAL_RANK="0",
               MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    for extra in (["--stripes", "16", "--steps", "2", "--e2e-steps", "1"], ["--full", "--config", "4", "--stripes", "8"]):
        cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "1", "--warmup", "3", "--oracle-stripes", "2",
               *extra]
        r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=900, env=env)
        assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-5000:]
        lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
        assert len(lines) == 1, r.stdout[-3000:]
        d = json.loads(lines[0])
        assert d["n_gpus"] == 1 and d["ranks"]["backend"] == "nccl" and d["ranks"]["ranks_up"] == 1
        assert d["verified"]["ok"] and ("--full" in extra or len(d["per_rank_ms"]) == 1)


def test_self_launch_two_ranks():
    d, err = _bench("--gpus", "2", "--dist-backend", "gloo", "--config", "2", "--stripes", "8", "--steps", "2",
                    "--warmup", "3", "--no-e2e", "--oracle-stripes", "4")
    assert d["n_gpus"] == 2 and len(d["per_rank_ms"]) == 2
    assert d["ranks"]["ranks_up"] == 2 and [r["rank"] for r in d["ranks"]["ranks"]] == [0, 1]
    v = d["verified"]
    assert v["ok"] and v["mismatched_bytes"] == 0 and v["poisoned_recovery"]["mismatched_bytes"] == 0
    assert v["poisoned_recovery"]["poisoned_bytes"] > 0
    assert v["oracle_digest_stripes"] == v["oracle_digest_sampled"] == 4
    assert d["cpu_baseline"]["kind"] == "oracle"


@pytest.mark.parametrize("cfg,stripes", [(4, 8)])
def test_full_config_digests_invariant_to_sharding(cfg, stripes):
    out = {}
    for G in (1, 2, 4):
        d, _ = _bench("--gpus", str(G), "--dist-backend", "gloo", "--full", "--config", str(cfg), "--stripes",
                      str(stripes), "--warmup", "3", "--oracle-stripes", "4")
        v = d["verified"]
        assert d["n_gpus"] == G and v["ok"] and v["scrub_bad_words_after_recovery"] == 0
        assert v["digested_stripes"] == stripes
        assert v["oracle_digest_stripes"] == v["oracle_digest_sampled"] == 4
        out[G] = v["digest_all"]
    assert out[1] == out[2] == out[4], out


def test_xgpu_distributed_two_ranks_matches_single_gpu():
    """NEXT-4 over the self-launched multi-rank path: `--xgpu 2 --gpus 2` brings up two ranks (here
    sharing cuda:0 under gloo), each holding half of every stripe's strips in an IPC arena; the
    partial kernel stores into the peer's slots and the combine writes rebuilt strips into their
    holders.  The line must verify on every rank (round trip, poisoned recovery, fresh encode), the
    oracle sample must match, and the digests of every strip must equal those of the one-GPU
    emulation and of the single-GPU bench path on the same stripes (Eq. (PQxy) as sums over disks,
    PAPER.md:971-979; uniqueness, Lemma 23.2)."""
    common = ["--config", "2", "--stripes", "4", "--steps", "2", "--warmup", "3", "--oracle-stripes", "2"]
    d, err = _bench("--gpus", "2", "--dist-backend", "gloo", "--xgpu", "2", *common)
    v = d["verified"]
    assert d["n_gpus"] == 2 and len(d["per_rank_ms"]) == 2 and d["ranks"]["ranks_up"] == 2
    assert not d["config"]["emulated"]
    assert v["ok"] and v["mismatched_strip_digests"] == 0
    assert v["poisoned_recovery"]["poisoned_bytes"] > 0 and v["poisoned_recovery"]["mismatched_strip_digests"] == 0
    assert v["fresh_encode_mismatched_strip_digests"] == 0
    assert v["oracle_digest_stripes"] == v["oracle_digest_sampled"] == 2
    e, _ = _bench("--gpus", "1", "--xgpu", "2", *common)
    assert e["config"]["emulated"] and e["verified"]["ok"]
    s, _ = _bench("--gpus", "1", "--no-e2e", *common)
    assert v["digest_all"] == e["verified"]["digest_all"] == s["verified"]["digest_all"]
