#!/usr/bin/env python3
"""Benchmark: Z_p-RAID encode + 2-erasure recovery on B200 (libraid6c, sm_100a kernels).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 2] [--impl ours|reference]

A "step" is one pass of the whole hot path over one batch of synthetic stripes already
resident in HBM: encode every stripe (P, Q), then rebuild an erasure pair in every stripe
(per-stripe pairs cycling over all C(N+2,2) pairs, i.e. every class DD/DP/DQ/PQ), in place.
Default workload = BASELINE.json configs[1] (c2): p=13, N=12, 4 MiB strips, 256 stripes
per GPU (weak scaling: every rank owns its own 256 stripes; no data-path collective).

metric value = user-data GB/s of the whole job = G * 2 * N * bytes * stripes / max-rank time
(encode and recovery each process the stripe's N user strips once).  Inputs (14 GiB) are
> 100x L2, so no L2 flush is needed between steps.  See DESIGN.md "Measurement".
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # cfg: p, N, strip bytes, stripes per GPU per step, sparse_mode, ops
    1: dict(p=5, N=4, nbytes=64 << 10, stripes=4096, sparse=0, ops="enc+rec",
            desc="c1 batched: p=5 N=4 64KiB x 4096 stripes (1 GiB user data), pairs cycle all 15"),
    2: dict(p=13, N=12, nbytes=4 << 20, stripes=256, sparse=0, ops="enc+rec",
            desc="c2: p=13 N=12 (12-bit words) 4MiB x 256 stripes, encode + recover, pairs cycle all 91"),
    3: dict(p=257, N=64, nbytes=16 << 20, stripes=4, sparse=0, ops="enc",
            desc="c3: p=257 N=64 (256-bit words) 16MiB x 4 stripes (4 GiB user data), encode only"),
    4: dict(p=59, N=58, nbytes=8 << 20, stripes=64, sparse=2, ops="enc+dd",
            desc="c4 wave: p=59 N=58 8MiB x 64 stripes (odd stripes sparse 0.9), encode + DD recovery"),
    5: dict(p=61, N=60, nbytes=32 << 20, stripes=16, sparse=0, ops="rec",
            desc="c5 wave: p=61 N=60 32MiB x 16 stripes, degraded-stream recovery (mixed classes)"),
}
METRIC = "encode and 2-erasure recover GB/s of user data per GPU and at 8 GPUs; % HBM roofline"


def _env_rank():
    return int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("LOCAL_RANK", "0"))


def measured_peak():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md: 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi clocks/throttle sampling during the timed region (B200_PROFILING.md)."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for l in self.lines:
            f = [x.strip() for x in l.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx.append(float(f[2]))
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def pair_schedule(cfg, N, stripes, stripe0, step):
    """Erasure pair of each stripe for a given step (host list of (i, j))."""
    import synthetic
    allp = synthetic.all_pairs(N)
    if cfg == 4:  # double-data-disk recovery: (s mod 1653)-th data pair
        dd = [(i, j) for i in range(N) for j in range(i + 1, N)]
        return [dd[(stripe0 + s) % len(dd)] for s in range(stripes)]
    if cfg == 5:  # degraded stream: seeded class + indices per stripe
        return [synthetic.erasure_pair(0, 5, stripe0 + s + step * stripes, N) for s in range(stripes)]
    return [allp[(stripe0 + s + 37 * step) % len(allp)] for s in range(stripes)]


def alg_bytes_recover(N, nbytes, pb, pairs):
    """N surviving strips read + 2 rebuilt strips written = every strip of the stripe once."""
    return len(pairs) * (N * nbytes + 2 * pb)


def traffic_from_profile(cfg):
    """dram bytes (read+write) per launch from the committed `ncu --set full` summary, or None."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return d.get(f"c{cfg}")
    except Exception:
        return None


# ====================================================================== our arm
def run_ours(args):
    import torch
    import torch.distributed as dist
    from paper_cs_0611109_b200 import raid6c as R
    from paper_cs_0611109_b200 import shard

    rank, world, local = _env_rank()
    local = local % torch.cuda.device_count()  # (only differs in the 1-GPU multi-rank rehearsal)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:  # gloo: rehearse the multi-rank path with several ranks on one GPU (host-side collectives only)
            dist.init_process_group("gloo")
    c = CONFIGS[args.config]
    p, N, S = args.prime or c["p"], args.data_strips or c["N"], args.stripes or c["stripes"]
    nbytes = args.strip_bytes or c["nbytes"]
    if args.strip_bytes and not args.stripes and args.config == 3:  # c3 sweep: >= 4 GiB per point
        S = max(1, -(-(4 << 30) // (N * nbytes)))
    if args.data_strips and not args.stripes:  # keep the batch's user data about the config's
        S = max(1, (c["stripes"] * c["N"]) // N)
    if args.strip_bytes or args.data_strips or args.prime:
        c = dict(c, desc=f"{c['desc']} [p={p} N={N}{' (extended code, Eq. qext)' if N > p else ''}, strip {nbytes} B, "
                         f"{S} stripes]")
    rs = args.code == "rs"  # NEXT-3: the paper's GF(256) Reed-Solomon comparison system, same workload
    pb = nbytes if rs else R.parity_bytes(p, nbytes)
    ss, ps = R.aligned_stride(nbytes), R.aligned_stride(pb)
    if rs:
        c = dict(c, desc=f"RS GF(256) baseline (Eq. rsparity) on {c['desc']}")
    stripe0 = shard.weak_range(rank, S)[0]  # weak scaling: each rank owns distinct global stripes
    stream = torch.cuda.Stream(device=dev)
    data = torch.empty((S, N, ss), dtype=torch.uint8, device=dev)
    par = torch.zeros((S, 2, ps), dtype=torch.uint8, device=dev)
    R.fill(data, ss, N * ss, nbytes, N, S, 0, args.config, stripe0, 0, c["sparse"], stream)
    a_data, a_par = int(data.data_ptr()), int(par.data_ptr())
    enc_args = (a_data, ss, N * ss, a_par, a_par + ps, 2 * ps, S)
    if rs:
        class _RSPlan:  # same call shape as Plan for the timed loop
            def encode_strided(self, *a):
                R.rs_encode_strided(N, nbytes, *a, stream=stream)

            def recover_strided(self, *a):
                R.rs_recover_strided(N, nbytes, *a[:-1], a[-1], stream=stream)

            def sync(self):
                stream.synchronize()

            def close(self):
                pass

            def encode_host(self, *a):
                raise NotImplementedError

        plan = _RSPlan()
    else:
        plan = R.Plan(p, N, nbytes, local, stream)
    ops = c["ops"]
    do_enc = ops.startswith("enc")
    do_rec = ops != "enc"
    if not do_enc:  # recovery-only stream still needs valid parity: encode once (untimed)
        plan.encode_strided(*enc_args)
    total_steps = args.warmup + args.steps
    pair_lists = [pair_schedule(args.config, N, S, stripe0, t) for t in range(total_steps)]
    pair_dev = [torch.tensor(pl, dtype=torch.int32, device=dev) for pl in pair_lists]
    torch.cuda.synchronize(dev)

    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(total_steps)]

    def step(t):
        with torch.cuda.stream(stream):
            ev[t][0].record(stream)
            if do_enc:
                plan.encode_strided(*enc_args)
            ev[t][1].record(stream)
            if do_rec:
                plan.recover_strided(*enc_args, pair_dev[t])
            ev[t][2].record(stream)

    for t in range(args.warmup):
        step(t)
    stream.synchronize()
    # snapshot for verification after the timed region (recovery rewrites lost strips in place)
    ref_data, ref_par = (data.clone(), par.clone()) if args.verify else (None, None)
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    launches0 = R.launch_count()
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    t_start.record(stream)
    for t in range(args.warmup, total_steps):
        step(t)
    t_end.record(stream)
    stream.synchronize()
    torch.cuda.synchronize(dev)
    launches = R.launch_count() - launches0
    clk = clocks.stop()
    plan.sync()
    elapsed_ms = t_start.elapsed_time(t_end)
    enc_ms = [ev[t][0].elapsed_time(ev[t][1]) for t in range(args.warmup, total_steps)]
    rec_ms = [ev[t][1].elapsed_time(ev[t][2]) for t in range(args.warmup, total_steps)]
    per_rank = shard.gather_over_ranks(elapsed_ms, dev)
    per_rank_ms = [round(x, 3) for x in per_rank]
    elapsed_ms = max(per_rank)

    # ---------------------------------------------------------------- verification
    verified = None
    if args.verify:
        cnt = torch.zeros(1, dtype=torch.int64, device=dev)
        torch.cuda.synchronize(dev)  # cnt is zeroed on torch's stream; the compare runs on `stream`
        if do_rec:
            # ref snapshot was taken after warm-up steps; data/parity must be bit-identical
            R.count_mismatch(data, ref_data, data.numel(), cnt, stream)
            R.count_mismatch(par, ref_par, par.numel(), cnt, stream)
        stream.synchronize()
        mism = int(cnt.item())
        checked = 2 * data.numel() if do_rec else 0
        oracle_ok = None
        if rank == 0 and args.oracle_check:
            oracle_ok = (rs_sample_check if rs else oracle_sample_check)(p, N, nbytes, args.config, c["sparse"],
                                                                        stripe0, par)
        tot = shard.sum_over_ranks([mism, checked], dev)
        verified = {"mismatched_bytes": tot[0], "checked_bytes": tot[1], "oracle_segments_match": oracle_ok}
        del ref_data, ref_par

    # ---------------------------------------------------------------- e2e (host buffers, public API)
    e2e = None
    if args.e2e and do_enc and not rs:
        try:
            e2e = run_e2e(args, R, torch, plan, data, par, S, N, nbytes, pb, ss, ps, pair_lists, do_rec, world, dev)
        except (RuntimeError, MemoryError) as exc:  # e.g. pinned host memory exhausted at large N
            e2e = {"value": None, "unit": "GB/s", "error": f"{type(exc).__name__}: {exc}"[:300]}

    user_bytes_step = (int(do_enc) + int(do_rec)) * N * nbytes * S
    value = world * user_bytes_step * args.steps / (elapsed_ms / 1e3) / 1e9
    peak, peak_src = measured_peak()
    enc_alg = S * (N * nbytes + 2 * pb)
    rec_alg = alg_bytes_recover(N, nbytes, pb, pair_lists[-1]) if do_rec else 0
    kern = []
    if do_enc:
        d = statistics.mean(enc_ms)
        kern.append(("encode", enc_alg, d))
    if do_rec:
        d = statistics.mean(rec_ms)
        kern.append(("recover", rec_alg, d))
    dom = max(kern, key=lambda k: k[2])
    # the committed ncu traffic belongs to the config's default launch only
    overridden = bool(args.prime or args.data_strips or args.strip_bytes or args.stripes or rs)
    traffic = None if overridden else traffic_from_profile(args.config)
    roof = {
        "kernel": (f"rs_kernel<{'true' if dom[0] == 'recover' else 'false'}> ({dom[0]})" if rs else
                   f"zp_kernel<{p},{1 if dom[0] == 'recover' else 0}> ({dom[0]})"),
        "bound": "hbm", "achieved": round(dom[1] / (dom[2] / 1e3) / 1e9, 1), "peak": peak, "unit": "GB/s",
        "frac": round(dom[1] / (dom[2] / 1e3) / 1e9 / peak, 4), "peak_source": peak_src,
        "traffic": traffic.get(dom[0]) if isinstance(traffic, dict) else None,
        "alg_bytes_per_launch": dom[1], "avg_launch_ms": round(dom[2], 4),
    }
    launch_ms = {"encode": enc_ms, "recover": rec_ms}  # per timed step, this rank
    per_kernel = {k[0]: {"alg_bytes": k[1], "avg_ms": round(k[2], 4),
                         "median_ms": round(statistics.median(launch_ms[k[0]]), 4),
                         "best_ms": round(min(launch_ms[k[0]]), 4),
                         "achieved_GBps": round(k[1] / (k[2] / 1e3) / 1e9, 1),
                         "frac_of_peak": round(k[1] / (k[2] / 1e3) / 1e9 / peak, 4),
                         "frac_of_8TBps": round(k[1] / (k[2] / 1e3) / 1e9 / 8000.0, 4),
                         "user_GBps": round(S * N * nbytes / (k[2] / 1e3) / 1e9, 1)} for k in kern}
    line = {
        "metric": METRIC, "value": round(value, 2), "unit": "GB/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(elapsed_ms / args.steps, 4), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u32 (bitwise GF(2) words)",
        "data": "synthetic (seeded SplitMix64 counter generator, generated on device)",
        "config": {"workload": c["desc"], "p": p, "N": N, "strip_bytes": nbytes, "parity_bytes": pb,
                   "stripes_per_gpu": S, "ops": ops, "parallelism": f"stripe-sharded x{world} (no data-path collective)",
                   "l2": "working set >= 1 GiB >> 126 MB L2 (no flush needed)"},
        "roofline": roof, "kernels": per_kernel, "gpu_launches": launches, "clocks": clk,
        "per_rank_ms": per_rank_ms,
        "verified": verified, "e2e": e2e,
        "fast_path": R.has_fast_path(p), "code": args.code,
    }
    if rank == 0 and world == 1 and args.cpu_baseline and not rs:  # the oracle baseline: rank 0 at N=1 only
        line["cpu_baseline"] = cpu_baseline(args, p, N, nbytes, args.config, c["sparse"])
    if rank == 0:
        print(json.dumps(line), flush=True)
    plan.close()
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


FULL_STRIPES = {2: 256, 4: 4096, 5: 1000}  # BASELINE.json configs[1], [3], [4]: whole-config stripe counts


def run_c1_literal(args):
    """--config 1 --full: BASELINE.json configs[0] literally -- ONE stripe (p=5, N=4, 64 KiB, seed 0):
    encode, then recover each of the C(6,2) = 15 erasure pairs (lost strips poisoned first) and
    compare with the original.  The whole stripe (384 KiB) is L2-resident, so this is a latency
    measurement (CUDA events per launch, mean over --steps repetitions), not an HBM number."""
    import torch
    import numpy as np
    import synthetic
    from paper_cs_0611109_b200 import raid6c as R
    torch.cuda.set_device(0)
    p, N, nbytes = 5, 4, 64 << 10
    pb = R.parity_bytes(p, nbytes)
    ss, ps = R.aligned_stride(nbytes), R.aligned_stride(pb)
    stream = torch.cuda.Stream()
    data = torch.empty((1, N, ss), dtype=torch.uint8, device="cuda")
    par = torch.zeros((1, 2, ps), dtype=torch.uint8, device="cuda")
    R.fill(data, ss, N * ss, nbytes, N, 1, 0, 1, 0, 0, 0, stream)
    plan = R.Plan(p, N, nbytes, 0, stream)
    a = (int(data.data_ptr()), ss, N * ss, int(par.data_ptr()), int(par.data_ptr()) + ps, 2 * ps, 1)
    pairs = synthetic.all_pairs(N)
    pair_dev = [torch.tensor([pr], dtype=torch.int32, device="cuda") for pr in pairs]
    flat = lambda k: data[0, k, :nbytes] if k < N else par[0, k - N, :pb]  # noqa: E731
    for _ in range(args.warmup):
        plan.encode_strided(*a)
    stream.synchronize()
    ref = [flat(k).clone() for k in range(N + 2)]
    reps = max(1, args.steps)
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    t_enc, t_rec, bad = [], {}, 0
    with torch.cuda.stream(stream):
        for _ in range(reps):
            e0, e1 = ev(), ev()
            e0.record(stream)
            plan.encode_strided(*a)
            e1.record(stream)
            stream.synchronize()
            t_enc.append(e0.elapsed_time(e1))
            for i, pr in enumerate(pairs):
                for k in pr:
                    flat(k).fill_(0xA5)
                e0, e1 = ev(), ev()
                e0.record(stream)
                plan.recover_strided(*a, pair_dev[i])
                e1.record(stream)
                stream.synchronize()
                t_rec.setdefault(pr, []).append(e0.elapsed_time(e1))
                bad += sum(int((flat(k) != ref[k]).sum().item()) for k in pr)
    # the same 16 launches (encode + 15 recoveries) captured once in a CUDA graph and replayed:
    # the device-side time per launch, without the per-call host path (Python, ctypes, ABI checks)
    graph = {"us_per_launch": None}
    try:
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=stream):
            plan.encode_strided(*a)
            for i in range(len(pairs)):
                plan.recover_strided(*a, pair_dev[i])
        with torch.cuda.stream(stream):  # replays run on the current stream
            flat(N).fill_(0xA5)
            flat(N + 1).fill_(0xA5)
            g.replay()  # the captured encode must rewrite P and Q
            stream.synchronize()
            graph["parity_rewritten_by_replay"] = bool(torch.equal(flat(N), ref[N]) and torch.equal(flat(N + 1), ref[N + 1]))
            for _ in range(3):
                g.replay()
            greps = 50
            e0, e1 = ev(), ev()
            e0.record(stream)
            for _ in range(greps):
                g.replay()
            e1.record(stream)
            stream.synchronize()
        graph["us_per_launch"] = round(1e3 * e0.elapsed_time(e1) / (greps * (1 + len(pairs))), 2)
        graph["launches_per_replay"] = 1 + len(pairs)
        graph["bytes_differing_after_replays"] = sum(int((flat(k) != ref[k]).sum().item()) for k in range(N + 2))
    except Exception as ex:  # noqa: BLE001 -- reported, not fatal: the per-call numbers stand
        graph["error"] = str(ex).splitlines()[0][:200]
    import oracle
    P, Q = oracle.encode(p, synthetic.stripe_strips(0, 1, 0, N, nbytes), nbytes)
    oracle_ok = bool(np.array_equal(ref[N].cpu().numpy(), P) and np.array_equal(ref[N + 1].cpu().numpy(), Q))
    alg = N * nbytes + 2 * pb
    enc_us = 1e3 * sum(t_enc) / len(t_enc)
    rec_us = {f"{i}-{j}": round(1e3 * sum(v) / len(v), 2) for (i, j), v in t_rec.items()}
    mean_rec = sum(rec_us.values()) / len(rec_us)
    line = {"metric": "config 1 literal: single-stripe encode + 15 recoveries, launch latency (L2-resident)",
            "value": round(mean_rec, 2), "unit": "us per recovery launch", "higher_is_better": False,
            "n_gpus": 1, "steps": reps, "warmup": args.warmup, "dtype": "u32 (bitwise GF(2) words)",
            "data": "synthetic (seed 0)", "config": {"workload": "c1 literal: p=5 N=4 64 KiB, 1 stripe, all 15 pairs",
                                                     "l2": "384 KiB stripe: L2-resident, not an HBM number"},
            "encode_us": round(enc_us, 2), "recover_us_per_pair": rec_us,
            "effective_GBps": {"encode": round(alg / (enc_us * 1e-6) / 1e9, 1),
                               "recover_mean": round(alg / (mean_rec * 1e-6) / 1e9, 1)},
            "verified": {"bytes_differing_after_recovery": bad, "parity_matches_oracle": oracle_ok},
            "cuda_graph": graph,
            "gpu_launches": reps * (1 + len(pairs))}
    print(json.dumps(line), flush=True)
    plan.close()


def run_full(args):
    """--full: the whole configuration, not one resident batch.

    The config's S stripes (c4: 4096, c5: 1000, c2: 256) are block-partitioned over the ranks
    (strong scaling: rank r owns [floor(r*S/G), floor((r+1)*S/G))), and each rank streams its
    block through one resident wave buffer (c4: 64 x 58 x 8 MiB, c5: 16 x 60 x 32 MiB), allocated
    once.  Per wave: generate on device (untimed), encode (timed, except c5 where parity is only
    the recovery's input), poison the wave's lost strips (untimed), recover them in place (timed),
    scrub the wave (untimed).  The scrub proves every recovery: with the N surviving strips given,
    the lost pair is the unique solution of both parity equations (Lemma 23.2),
    so a stripe with zero violating words after recovery was rebuilt exactly.  Sampled P/Q
    segments are compared with the CPU oracle.  value = user bytes of all ranks / max-rank sum of
    the timed kernel intervals (CUDA events on the plan's stream)."""
    import torch
    import torch.distributed as dist
    import synthetic
    from paper_cs_0611109_b200 import raid6c as R
    from paper_cs_0611109_b200 import shard

    rank, world, local = _env_rank()
    local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group("gloo")
    if args.config not in FULL_STRIPES:
        raise SystemExit(f"--full applies to configs {sorted(FULL_STRIPES)}")
    c = CONFIGS[args.config]
    p, N, nbytes = c["p"], c["N"], c["nbytes"]
    total = args.stripes or FULL_STRIPES[args.config]
    lo, hi = shard.block_range(rank, world, total)
    wave = min(c["stripes"], max(1, hi - lo))
    pb = R.parity_bytes(p, nbytes)
    ss, ps = R.aligned_stride(nbytes), R.aligned_stride(pb)
    stream = torch.cuda.Stream(device=dev)
    data = torch.empty((wave, N, ss), dtype=torch.uint8, device=dev)
    par = torch.zeros((wave, 2, ps), dtype=torch.uint8, device=dev)
    counts = torch.zeros(wave, dtype=torch.int32, device=dev)
    bad_total = torch.zeros(1, dtype=torch.int64, device=dev)
    plan = R.Plan(p, N, nbytes, local, stream)
    a_data, a_par = int(data.data_ptr()), int(par.data_ptr())
    do_enc = c["ops"] != "rec"
    flat_d, flat_p = data.view(wave * N, ss), par.view(wave * 2, ps)

    def wave_tables(w0, n):
        """Erasure pairs and poison row indices of one wave, uploaded once before timing and kept
        alive for the whole run (they are read on `stream` long after the host moves on)."""
        pairs = pair_schedule(args.config, N, n, w0, 0)
        dl = [s * N + k for s, pr in enumerate(pairs) for k in pr if k < N]
        pl = [s * 2 + (k - N) for s, pr in enumerate(pairs) for k in pr if k >= N]
        return (w0, n, pairs, torch.tensor(pairs, dtype=torch.int32, device=dev),
                torch.tensor(dl, dtype=torch.int64, device=dev), torch.tensor(pl, dtype=torch.int64, device=dev))

    tables = [wave_tables(w0, min(wave, hi - w0)) for w0 in range(lo, hi, wave)]
    torch.cuda.synchronize(dev)

    def run_wave(tab):
        """One wave (fill, encode, poison, recover, scrub) on `stream`; returns its events."""
        w0, n, pairs, pair_dev, dl, pl = tab
        args_ = (a_data, ss, N * ss, a_par, a_par + ps, 2 * ps, n)
        e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        with torch.cuda.stream(stream):
            R.fill(data, ss, N * ss, nbytes, N, n, 0, args.config, w0, 0, c["sparse"], stream)
            e[0].record(stream)
            plan.encode_strided(*args_)
            e[1].record(stream)
            if dl.numel():
                flat_d.index_fill_(0, dl, 0xA5)  # lost strips: never read by recovery
            if pl.numel():
                flat_p.index_fill_(0, pl, 0xA5)
            e[2].record(stream)
            plan.recover_strided(*args_, pair_dev)
            e[3].record(stream)
            plan.scrub_strided(*args_, counts)
            bad_total.add_(counts[:n].sum())
        return e

    for _ in range(args.warmup):  # warm-up on the first wave (not counted)
        run_wave(tables[0])
    stream.synchronize()
    bad_total.zero_()
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    launches0 = R.launch_count()
    wall0 = time.perf_counter()
    evs, classes, nst = [], {}, 0
    for tab in tables:
        evs.append(run_wave(tab))
        nst += tab[1]
        for (i, j) in tab[2]:
            k = synthetic.pair_class(N, i, j)
            classes[k] = classes.get(k, 0) + 1
    stream.synchronize()
    wall = time.perf_counter() - wall0
    launches = R.launch_count() - launches0
    clk = clocks.stop()
    enc_ms = sum(e[0].elapsed_time(e[1]) for e in evs) if do_enc else 0.0
    rec_ms = sum(e[2].elapsed_time(e[3]) for e in evs)
    timed_ms = enc_ms + rec_ms
    oracle_ok = None
    if rank == 0 and args.oracle_check:
        last_w0 = lo + ((hi - lo - 1) // wave) * wave
        oracle_ok = oracle_sample_check(p, N, nbytes, args.config, c["sparse"], last_w0,
                                        par[:min(wave, hi - last_w0)])
    bad = int(bad_total.item())
    t_max = shard.max_over_ranks(timed_ms, dev)
    enc_max = shard.max_over_ranks(enc_ms, dev)
    rec_max = shard.max_over_ranks(rec_ms, dev)
    tot = shard.sum_over_ranks([nst, bad] + [classes.get(k, 0) for k in ("DD", "DP", "DQ", "PQ")], dev)
    nst_all, bad_all = tot[0], tot[1]
    ops_n = int(do_enc) + 1
    user = ops_n * N * nbytes * nst_all
    value = user / (t_max / 1e3) / 1e9
    peak, peak_src = measured_peak()
    per = {}
    if do_enc:
        per["encode"] = enc_max
    per["recover"] = rec_max
    kern = {k: {"alg_bytes_per_rank": nst * (N * nbytes + 2 * pb), "sum_ms_max_rank": round(v, 3),
                "achieved_GBps_per_gpu": round(nst * (N * nbytes + 2 * pb) / (v / 1e3) / 1e9, 1),
                "frac_of_peak": round(nst * (N * nbytes + 2 * pb) / (v / 1e3) / 1e9 / peak, 4),
                "user_GBps_all_gpus": round(N * nbytes * nst_all / (v / 1e3) / 1e9, 1)} for k, v in per.items()}
    dom = max(per, key=per.get)
    ach = nst * (N * nbytes + 2 * pb) / (per[dom] / 1e3) / 1e9
    line = {
        "metric": METRIC, "value": round(value, 2), "unit": "GB/s", "n_gpus": world, "steps": 1,
        "warmup": args.warmup, "ms_per_step": round(t_max, 3), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "u32 (bitwise GF(2) words)",
        "data": "synthetic (seeded SplitMix64 counter generator, generated on device per wave, untimed)",
        "config": {"workload": f"c{args.config} full: {total} stripes of p={p} N={N} {nbytes} B strips, "
                               f"block-sharded over {world} GPU(s), waves of {wave} ({c['ops']})",
                   "p": p, "N": N, "strip_bytes": nbytes, "parity_bytes": pb, "stripes_total": total,
                   "stripes_this_rank0": hi - lo if rank == 0 else None, "wave": wave, "ops": c["ops"],
                   "parallelism": f"stripe-sharded x{world} (no data-path collective)",
                   "l2": "each wave >= 30 GiB >> 126 MB L2 (no flush needed)",
                   "timed": "sum of per-wave encode + recover kernel intervals; generation, poisoning, scrub untimed"},
        "roofline": {"kernel": f"zp_kernel<{p},{1 if dom == 'recover' else 0}> ({dom})", "bound": "hbm",
                     "achieved": round(ach, 1), "peak": peak, "unit": "GB/s", "frac": round(ach / peak, 4),
                     "peak_source": peak_src},
        "kernels": kern, "gpu_launches": launches, "clocks": clk, "wall_s_rank0": round(wall, 2),
        "classes": dict(zip(("DD", "DP", "DQ", "PQ"), tot[2:])),
        "verified": {"stripes": nst_all, "scrub_bad_words_after_recovery": bad_all,
                     "oracle_segments_match": oracle_ok},
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    plan.close()
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def run_xgpu(args):
    """--xgpu G (NEXT-4): the cross-GPU stripe layout, the strips of each stripe
    spread over G ranks (xgpu.py).  One step = encode (partial + combine) then one recovery
    (partial + combine) of every stripe.  At --gpus 1 the G ranks are emulated on the one GPU
    (xgpu.Emulated: each phase is G independent launches over all ranks' data), so the numbers
    are HBM-only: the NVLink transfer of the partial syndromes (peer stores) is not exercised.
    Under torchrun (world > 1) each rank is a GPU (xgpu.Distributed, CUDA IPC + NCCL barrier)."""
    import torch
    import torch.distributed as dist
    from paper_cs_0611109_b200 import raid6c as R
    from paper_cs_0611109_b200 import shard, xgpu

    rank, world, local = _env_rank()
    local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group(args.dist_backend, device_id=dev if args.dist_backend == "nccl" else None)
    c = CONFIGS[args.config]
    p, N = args.prime or c["p"], args.data_strips or c["N"]
    nbytes = args.strip_bytes or c["nbytes"]
    S = args.stripes or c["stripes"]
    G = world if world > 1 else args.xgpu
    pb = R.parity_bytes(p, nbytes)
    stream = torch.cuda.Stream(device=dev)
    plan = R.Plan(p, N, nbytes, local, stream)
    pairs = pair_schedule(4 if args.config == 4 else 2, N, S, 0, 0)
    pair_dev = torch.tensor(pairs, dtype=torch.int32, device=dev)
    if world == 1:
        ss, ps = R.aligned_stride(nbytes), R.aligned_stride(pb)
        data = torch.empty((S, N, ss), dtype=torch.uint8, device=dev)
        par = torch.zeros((S, 2, ps), dtype=torch.uint8, device=dev)
        R.fill(data, ss, N * ss, nbytes, N, S, 0, args.config, 0, 0, c["sparse"], stream)
        X = xgpu.Emulated(plan, G, data, par, S)

        def phase(which, er):
            for r in range(G):
                (X.partial if which == 0 else X.combine)(r, er)
    else:
        X = xgpu.Distributed(plan, S, local, backend=args.dist_backend)
        k_lo, k_hi = X.blocks[rank]
        for k in range(k_lo, min(k_hi, N)):
            R.fill(X.strip_addr(k), 0, X.ss, nbytes, 1, S, 0, args.config, 0, k, c["sparse"], stream)

        def phase(which, er):
            if which == 0:
                X.plan.partial_strided([a if k_lo <= k < k_hi else None for k, a in enumerate(X.strips)], X.ss, X.ps,
                                       S, er, k_lo, k_hi, [X.slot(g, rank, 0) for g in range(G)],
                                       [X.slot(g, rank, 1) for g in range(G)], X.pstride, X.range)
            else:
                lo, hi = X.ranges[rank]
                if hi > lo:
                    X.plan.combine_strided(X.strips, X.ss, X.ps, S, er, [X.slot(rank, r, 0) for r in range(G)],
                                           [X.slot(rank, r, 1) for r in range(G)], X.pstride, lo, hi)
            X.barrier(stream)
    torch.cuda.synchronize(dev)
    total = args.warmup + args.steps
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(5)] for _ in range(total)]

    def step(t):
        with torch.cuda.stream(stream):
            ev[t][0].record(stream)
            phase(0, None)
            ev[t][1].record(stream)
            phase(1, None)
            ev[t][2].record(stream)
            phase(0, pair_dev)
            ev[t][3].record(stream)
            phase(1, pair_dev)
            ev[t][4].record(stream)

    for t in range(args.warmup):
        step(t)
    stream.synchronize()
    if world > 1:
        dist.barrier()
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    launches0 = R.launch_count()
    for t in range(args.warmup, total):
        step(t)
    stream.synchronize()
    launches = R.launch_count() - launches0
    clk = clocks.stop()
    ms = [[ev[t][i].elapsed_time(ev[t][i + 1]) for i in range(4)] for t in range(args.warmup, total)]
    mean = [statistics.mean(m[i] for m in ms) for i in range(4)]
    mean = [shard.max_over_ranks(v, dev) for v in mean]
    step_ms = sum(mean)
    # verification (emulation): the layout's P, Q equal the single-GPU encode's, and the recovered
    # strips equal the stripes before the step (recovery in place of intact strips)
    verified = None
    if world == 1:
        ref = par.clone()
        plan.encode_strided(int(data.data_ptr()), X.ss, N * X.ss, int(par.data_ptr()), int(par.data_ptr()) + X.ps,
                            2 * X.ps, S)
        cnt = torch.zeros(1, dtype=torch.int64, device=dev)
        torch.cuda.synchronize(dev)
        R.count_mismatch(par, ref, par.numel(), cnt, stream)
        dref = data.clone()
        torch.cuda.synchronize(dev)
        for s, (x, y) in enumerate(pairs):
            for k in (x, y):
                (data[s, k, :nbytes] if k < N else par[s, k - N, :pb]).fill_(0xA5)
        torch.cuda.synchronize(dev)
        with torch.cuda.stream(stream):
            phase(0, pair_dev)
            phase(1, pair_dev)
        R.count_mismatch(data, dref, data.numel(), cnt, stream)
        R.count_mismatch(par, ref, par.numel(), cnt, stream)
        stream.synchronize()
        verified = {"mismatched_bytes_vs_single_gpu_path": int(cnt.item())}
    # algorithmic bytes per phase (all G ranks): partial = every surviving strip read once + G
    # partial pairs written; combine = G partial pairs read + 2 rebuilt strips written
    enc_part = S * (N * nbytes + 2 * G * pb)
    comb = S * (2 * G * pb + 2 * pb)
    rec_part = sum(N * nbytes + 2 * pb - ((nbytes if x < N else pb) + (nbytes if y < N else pb)) + 2 * G * pb
                   for (x, y) in pairs)
    rec_comb = sum(2 * G * pb + (nbytes if x < N else pb) + (nbytes if y < N else pb) for (x, y) in pairs)
    alg = [enc_part, comb, rec_part, rec_comb]
    peak, peak_src = measured_peak()
    names = ["encode_partial", "encode_combine", "recover_partial", "recover_combine"]
    kern = {nm: {"alg_bytes_all_ranks": a, "avg_ms": round(m, 4),
                 "achieved_GBps": round(a / (m / 1e3) / 1e9 / (1 if world == 1 else world), 1),
                 "frac_of_peak": round(a / (m / 1e3) / 1e9 / (1 if world == 1 else world) / peak, 4)}
            for nm, a, m in zip(names, alg, mean)}
    dom = max(range(4), key=lambda i: mean[i])
    user = 2 * S * N * nbytes
    line = {"metric": "cross-GPU stripe layout (NEXT-4): encode + recover GB/s of user data", "value":
            round(user / (step_ms / 1e3) / 1e9, 2), "unit": "GB/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(step_ms, 4), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "u32 (bitwise GF(2) words)",
            "data": "synthetic (device generator)",
            "config": {"workload": f"{c['desc']} with each stripe's strips spread over {G} ranks"
                                   + (" (emulated on one GPU: HBM only, no NVLink)" if world == 1 else ""),
                       "p": p, "N": N, "strip_bytes": nbytes, "stripes": S, "ranks": G,
                       "range_bytes": X.range, "emulated": world == 1},
            "roofline": {"kernel": names[dom], "bound": "hbm", "achieved": kern[names[dom]]["achieved_GBps"],
                         "peak": peak, "unit": "GB/s", "frac": kern[names[dom]]["frac_of_peak"],
                         "peak_source": peak_src},
            "kernels": kern, "gpu_launches": launches, "clocks": clk, "verified": verified}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        X.close()
        dist.barrier()
        dist.destroy_process_group()
    plan.close()


def run_sweep(args):
    """--sweep (config 3, BASELINE.json configs[2]): encode-only write-throughput sweep over strip
    sizes 64 KiB -> 16 MiB (x2 steps, 9 points), each point >= 4 GiB of user data
    (ceil(4 GiB / (64 * strip)) stripes).  Each point is a separate `bench.py --strip-bytes B`
    process (so every point gets a fresh allocator); one JSON line collects them."""
    rank, world, _ = _env_rank()
    if world > 1:
        raise SystemExit("--sweep is a 1-GPU measurement")
    pts = []
    for k in range(9):
        b = (64 << 10) << k
        cmd = [sys.executable, os.path.abspath(__file__), "--config", "3", "--strip-bytes", str(b),
               "--steps", str(args.steps), "--warmup", str(args.warmup), "--no-e2e", "--no-cpu-baseline"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise SystemExit(f"sweep point {b} failed:\n{r.stderr[-2000:]}")
        d = json.loads(r.stdout.strip().splitlines()[-1])
        kk = d["kernels"]["encode"]
        pts.append({"strip_bytes": b, "stripes": d["config"]["stripes_per_gpu"], "user_GBps": kk["user_GBps"],
                    "achieved_GBps": kk["achieved_GBps"], "frac_of_peak": kk["frac_of_peak"],
                    "avg_ms": kk["avg_ms"], "verified_oracle": d["verified"]["oracle_segments_match"],
                    "clocks": d["clocks"]})
    peak, peak_src = measured_peak()
    best = max(pts, key=lambda q: q["achieved_GBps"])
    worst = min(pts, key=lambda q: q["achieved_GBps"])
    line = {"metric": METRIC + " (c3 encode write-throughput sweep)", "value": worst["user_GBps"], "unit": "GB/s",
            "n_gpus": 1, "steps": args.steps, "warmup": args.warmup, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "u32 (bitwise GF(2) words)", "data": "synthetic (device generator)",
            "config": {"workload": "c3 sweep: p=257 N=64, strip 64 KiB -> 16 MiB, >= 4 GiB user data per point",
                       "value_is": "the minimum user GB/s over the sweep points"},
            "roofline": {"bound": "hbm", "achieved": worst["achieved_GBps"], "peak": peak, "unit": "GB/s",
                         "frac": round(worst["achieved_GBps"] / peak, 4), "peak_source": peak_src,
                         "best_frac": round(best["achieved_GBps"] / peak, 4)},
            "sweep": pts}
    print(json.dumps(line), flush=True)


def run_next1(args):
    """--op update | scrub (NEXT-1): small-write parity update and scrub of the
    config's stripes, one launch per step, CUDA events on the plan's stream."""
    import torch
    from paper_cs_0611109_b200 import raid6c as R

    rank, world, local = _env_rank()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    c = CONFIGS[args.config]
    p, N, S = c["p"], args.data_strips or c["N"], args.stripes or c["stripes"]
    if args.data_strips and not args.stripes:
        S = max(1, (c["stripes"] * c["N"]) // N)
    nbytes = args.strip_bytes or c["nbytes"]
    pb = R.parity_bytes(p, nbytes)
    ss, ps = R.aligned_stride(nbytes), R.aligned_stride(pb)
    stream = torch.cuda.Stream(device=dev)
    data = torch.empty((S, N, ss), dtype=torch.uint8, device=dev)
    par = torch.zeros((S, 2, ps), dtype=torch.uint8, device=dev)
    R.fill(data, ss, N * ss, nbytes, N, S, 0, args.config, 0, 0, c["sparse"], stream)
    news = [torch.empty((S, ss), dtype=torch.uint8, device=dev) for _ in range(2)]
    for i, nb in enumerate(news):
        R.fill(nb, ss, ss, nbytes, 1, S, 1 + i, args.config, 0, 0, 0, stream)
    plan = R.Plan(p, N, nbytes, local, stream)
    a = (int(data.data_ptr()), ss, N * ss, int(par.data_ptr()), int(par.data_ptr()) + ps, 2 * ps, S)
    plan.encode_strided(*a)
    disks = torch.tensor([(7 * s) % N for s in range(S)], dtype=torch.int32, device=dev)
    counts = torch.zeros(S, dtype=torch.int32, device=dev)

    def launch(t):
        if args.op == "update":
            plan.update_strided(*a, int(news[t % 2].data_ptr()), ss, disks)
        else:
            plan.scrub_strided(*a, counts)

    total = args.warmup + args.steps
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(total)]
    torch.cuda.synchronize(dev)
    launches0 = R.launch_count()
    for t in range(total):
        with torch.cuda.stream(stream):
            evs[t][0].record(stream)
            launch(t)
            evs[t][1].record(stream)
    stream.synchronize()
    launches = R.launch_count() - launches0 - args.warmup
    ms = statistics.mean(evs[t][0].elapsed_time(evs[t][1]) for t in range(args.warmup, total))
    plan.scrub_strided(*a, counts)  # verification: every stripe consistent after the updates
    stream.synchronize()
    bad = int(counts.sum().item())
    if args.op == "update":
        alg = S * (3 * nbytes + 4 * pb)
        user = S * nbytes
        metric = "small-write parity update (NEXT-1) GB/s of rewritten user data"
    else:
        alg = S * (N * nbytes + 2 * pb)
        user = S * N * nbytes
        metric = "scrub (NEXT-1) GB/s of user data checked"
    peak, peak_src = measured_peak()
    ach = alg / (ms / 1e3) / 1e9
    line = {"metric": metric, "value": round(user / (ms / 1e3) / 1e9, 2), "unit": "GB/s", "n_gpus": 1,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 4), "higher_is_better": True,
            "op": args.op, "dtype": "u32 (bitwise GF(2) words)", "data": "synthetic (device generator)",
            "config": {"workload": c["desc"], "p": p, "N": N, "strip_bytes": nbytes, "stripes": S},
            "roofline": {"bound": "hbm", "achieved": round(ach, 1), "peak": peak, "unit": "GB/s",
                         "frac": round(ach / peak, 4), "peak_source": peak_src, "alg_bytes_per_launch": alg},
            "gpu_launches": launches, "verified": {"scrub_bad_words_after": bad}}
    if rank == 0:
        print(json.dumps(line), flush=True)
    plan.close()


def run_e2e(args, R, torch, plan, data, par, S, N, nbytes, pb, ss, ps, pair_lists, do_rec, world, dev):
    """Same workload through the host-buffer public API (raid6c_encode_host/recover_host):
    H2D of inputs and D2H of results inside the timed region, pinned host memory."""
    from paper_cs_0611109_b200 import shard
    err = None
    try:
        hd = torch.empty((S, N, ss), dtype=torch.uint8).pin_memory()
        hp = torch.zeros((S, 2, ps), dtype=torch.uint8).pin_memory()
    except (RuntimeError, MemoryError) as exc:
        err = f"{type(exc).__name__}: {exc}"[:300]
    if shard.sum_over_ranks([int(err is not None)], dev)[0]:  # every rank skips if any rank failed
        raise RuntimeError(err or "pinned host allocation failed on another rank")
    hd.copy_(data)  # device -> pinned host, no pageable temporary
    hd_ptr, hp_ptr = int(hd.data_ptr()), int(hp.data_ptr())
    a = (hd_ptr, ss, N * ss, hp_ptr, hp_ptr + ps, 2 * ps, S)
    steps = max(1, args.e2e_steps)
    times, h2d, d2h = [], 0, 0
    for t in range(1 + steps):
        if world > 1:
            import torch.distributed as dist
            dist.barrier()
        t0 = time.perf_counter()
        plan.encode_host(*a)
        b1 = plan.host_traffic()
        if do_rec:
            plan.recover_host(*a, pair_lists[t % len(pair_lists)])
            b2 = plan.host_traffic()
        else:
            b2 = (0, 0)
        t1 = time.perf_counter()
        if t >= 1:
            times.append(t1 - t0)
            h2d, d2h = b1[0] + b2[0], b1[1] + b2[1]
    # correctness of the host path vs the device path (parity of the same stripes)
    same = bool(torch.equal(hp[:, :, :pb], par[:, :, :pb].cpu()))
    tm = shard.max_over_ranks(statistics.mean(times), dev)
    user = (1 + int(do_rec)) * N * nbytes * S * world
    # the e2e roofline: this GPU's pinned H2D copy rate with a concurrent D2H (the host path moves
    # inputs in and results out at the same time), probed here on 1 GiB + 256 MiB buffers
    probe = None
    try:
        n1 = 1 << 30
        src = hd.view(-1)[:n1]
        dst = data.view(-1)[:n1].clone()
        back = torch.empty(n1 // 4, dtype=torch.uint8).pin_memory()
        s_in, s_out = torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev)
        for _ in range(2):
            torch.cuda.synchronize(dev)
            t0 = time.perf_counter()
            with torch.cuda.stream(s_in):
                dst.copy_(src, non_blocking=True)
            with torch.cuda.stream(s_out):
                back.copy_(dst[:n1 // 4], non_blocking=True)
            torch.cuda.synchronize(dev)
            probe = n1 / (time.perf_counter() - t0) / 1e9
        del dst, back
    except (RuntimeError, MemoryError):
        probe = None
    h2d_rate = h2d / tm / 1e9
    return {"value": round(user / tm / 1e9, 2), "unit": "GB/s", "h2d_bytes_per_step": h2d,
            "d2h_bytes_per_step": d2h, "steps": steps, "s_per_step": round(tm, 4),
            "api": "raid6c_encode_host + raid6c_recover_host (pinned host buffers)",
            "matches_device_path": same,
            "roofline": {"bound": "pcie", "achieved": round(h2d_rate, 1), "unit": "GB/s (H2D)",
                         "peak": round(probe, 1) if probe else None,
                         "frac": round(h2d_rate / probe, 4) if probe else None,
                         "peak_source": "live probe: pinned 1 GiB H2D with a concurrent 256 MiB D2H"}}


def rs_sample_check(p, N, nbytes, cfg, sparse_mode, stripe0, par):
    """RS baseline: sampled byte segments of P/Q of two stripes against oracle.rs_encode."""
    import numpy as np
    import oracle
    import synthetic
    ok = True
    for s in (0, par.shape[0] - 1):
        gs = stripe0 + s
        sparse = sparse_mode == 1 or (sparse_mode == 2 and gs % 2 == 1)
        for b0 in (0, nbytes // 2, max(0, nbytes - 4096)):
            b1 = min(nbytes, b0 + 4096)
            segs = [synthetic.strip_bytes(0, cfg, gs, k, nbytes, sparse, lo=b0, hi=b1) for k in range(N)]
            P, Q = oracle.rs_encode(segs, b1 - b0)
            ok &= bool(np.array_equal(par[s, 0, b0:b1].cpu().numpy(), P))
            ok &= bool(np.array_equal(par[s, 1, b0:b1].cpu().numpy(), Q))
    return ok


def oracle_sample_check(p, N, nbytes, cfg, sparse_mode, stripe0, par):
    """Sampled word-aligned P/Q segments of two stripes against the CPU oracle."""
    import numpy as np
    import oracle
    import synthetic
    n = p - 1
    ok = True
    for s in (0, par.shape[0] - 1):
        gs = stripe0 + s
        sparse = sparse_mode == 1 or (sparse_mode == 2 and gs % 2 == 1)
        W = (8 * nbytes + n - 1) // n
        for g0 in (0, (W // 8) // 2, max(0, W // 8 - 2)):
            b0 = g0 * n
            b1 = min(nbytes, b0 + 2 * n)
            if g0 == max(0, W // 8 - 2):
                b1 = nbytes
            segs = [synthetic.strip_bytes(0, cfg, gs, k, nbytes, sparse, lo=b0, hi=b1) for k in range(N)]
            P, Q = (oracle.encode_ext if N > p else oracle.encode)(p, segs, b1 - b0)
            e = b0 + P.size
            ok &= bool(np.array_equal(par[s, 0, b0:e].cpu().numpy(), P))
            ok &= bool(np.array_equal(par[s, 1, b0:e].cpu().numpy(), Q))
    return ok


# ====================================================================== oracle (CPU) arm
def _oracle_work(p, N, nbytes, cfg, sparse_mode, budget_s, max_threads):
    """Time the oracle as it stands on a bounded sample of the same workload: per stripe,
    encode + one recovery (pair from the same schedule).  Returns (user_bytes, seconds, threads, sample)."""
    import concurrent.futures as cf
    import numpy as np
    import oracle
    import synthetic
    oracle.build()
    ncores = len(os.sched_getaffinity(0))
    threads = max(1, min(ncores, max_threads))
    ops = CONFIGS[cfg]["ops"]
    # bounded strip length so one task is ~1-3 s of CPU work
    sample_bytes = min(nbytes, 1 << 20)
    pb = oracle.parity_bytes(p, sample_bytes)

    def task(s):
        sparse = sparse_mode == 1 or (sparse_mode == 2 and s % 2 == 1)
        data = [synthetic.strip_bytes(0, cfg, s, k, nbytes, sparse, lo=0, hi=sample_bytes) for k in range(N)]
        t0 = time.perf_counter()
        user = 0
        ext = N > p
        P, Q = (oracle.encode_ext if ext else oracle.encode)(p, data, sample_bytes)
        if ops != "rec":
            user += N * sample_bytes
        if ops != "enc":
            i, j = pair_schedule(cfg, N, 1, s, 0)[0]
            strips = [d.copy() for d in data] + [P.copy(), Q.copy()]
            strips[i][:] = 0
            strips[j][:] = 0
            (oracle.recover_ext if ext else oracle.recover)(p, N, i, j, strips, sample_bytes)
            user += N * sample_bytes
        return user, time.perf_counter() - t0

    # calibrate one task, then size the sample to the budget
    u0, t0 = task(0)
    per = max(t0, 1e-3)
    ntasks = max(threads, int(budget_s * threads / per))
    ntasks = min(ntasks, 16 * threads)  # ~budget_s of wall time on the host cores
    t_start = time.perf_counter()
    users = 0
    with cf.ThreadPoolExecutor(max_workers=threads) as ex:
        for u, _ in ex.map(task, range(1, 1 + ntasks)):
            users += u
    wall = time.perf_counter() - t_start
    sample = (f"{ntasks} stripes x {N} strips truncated to {sample_bytes} B "
              f"({'encode' if ops != 'rec' else ''}{' + ' if ops == 'enc+rec' or ops == 'enc+dd' else ''}"
              f"{'one recovery' if ops != 'enc' else ''} each), bit-array oracle, {threads} threads")
    return users, wall, threads, sample


def cpu_baseline(args, p, N, nbytes, cfg, sparse_mode):
    users, wall, threads, sample = _oracle_work(p, N, nbytes, cfg, sparse_mode, args.cpu_budget, args.cpu_threads)
    return {"value": round(users / wall / 1e9, 6), "unit": "GB/s", "cores": threads, "kind": "oracle",
            "sample": sample, "seconds": round(wall, 2)}


def run_reference(args):
    rank, world, _ = _env_rank()
    if rank != 0:
        return  # under torchrun only rank 0 runs the CPU arm
    c = CONFIGS[args.config]
    p, N, nbytes = c["p"], c["N"], c["nbytes"]
    vals, cores, sample, secs = [], 0, "", []
    budget = max(2.0, args.cpu_budget / max(1, args.steps + args.warmup))
    for t in range(args.warmup + args.steps):
        users, wall, threads, sample = _oracle_work(p, N, nbytes, args.config, c["sparse"], budget, args.cpu_threads)
        if t >= args.warmup:
            vals.append(users / wall / 1e9)
            secs.append(wall)
        cores = threads
    v = statistics.mean(vals)
    line = {
        "impl": "reference", "metric": METRIC, "value": round(v, 6), "unit": "GB/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(1e3 * statistics.mean(secs), 2),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bit arrays (uint8 per bit)",
        "data": "synthetic (seeded SplitMix64 counter generator)",
        "config": {"workload": c["desc"], "p": p, "N": N, "strip_bytes": nbytes, "ops": c["ops"]},
        "cpu_baseline": {"value": round(v, 6), "unit": "GB/s", "cores": cores, "kind": "oracle", "sample": sample},
        "e2e": {"value": round(v, 6), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=2, choices=sorted(CONFIGS))
    ap.add_argument("--stripes", type=int, default=0, help="override stripes per GPU per step")
    ap.add_argument("--strip-bytes", type=int, default=0, help="override strip length (c3 sweep)")
    ap.add_argument("--prime", type=int, default=0, help="override p (e.g. 17 for the paper's Z_17)")
    ap.add_argument("--data-strips", type=int, default=0,
                    help="override N (p < N <= 2p-1 selects the extended code of Eq. (qext), NEXT-2)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--code", default="zp", choices=["zp", "rs"],
                    help="zp = the paper's Z_p code (default); rs = its GF(256) RS comparison system (NEXT-3)")
    ap.add_argument("--op", default="step", choices=["step", "update", "scrub"],
                    help="step = encode + recover (the metric); update / scrub = NEXT-1 kernels")
    ap.add_argument("--full", action="store_true",
                    help="whole config (c4: 4096, c5: 1000, c2: 256 stripes) block-sharded over the ranks, "
                         "c1: the literal single stripe with all 15 pairs (latency); "
                         "streamed in waves (strong scaling); --stripes overrides the total")
    ap.add_argument("--xgpu", type=int, default=0,
                    help="NEXT-4: spread each stripe's strips over G ranks (emulated on one GPU at --gpus 1)")
    ap.add_argument("--sweep", action="store_true", help="config 3 strip-size sweep 64 KiB -> 16 MiB")
    ap.add_argument("--no-verify", dest="verify", action="store_false")
    ap.add_argument("--no-oracle-check", dest="oracle_check", action="store_false")
    ap.add_argument("--no-e2e", dest="e2e", action="store_false")
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--no-cpu-baseline", dest="cpu_baseline", action="store_false")
    ap.add_argument("--cpu-budget", type=float, default=15.0, help="seconds of oracle work for cpu_baseline")
    ap.add_argument("--cpu-threads", type=int, default=64)
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="gloo: rehearse N>1 on fewer GPUs (ranks share devices; timing not meaningful)")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        print("note: warm-up raised to 3 (timing rule)", file=sys.stderr)
        args.warmup = 3
    if args.gpus > 1 and _env_rank()[1] == 1:
        print(f"note: --gpus {args.gpus} without a torchrun launch runs one rank (launch with "
              f"python -m torch.distributed.run --nproc-per-node {args.gpus} ...)", file=sys.stderr)
    if args.impl == "reference":
        run_reference(args)
    elif args.op != "step":
        run_next1(args)
    elif args.full and args.config == 1:
        run_c1_literal(args)
    elif args.full:
        run_full(args)
    elif args.xgpu:
        run_xgpu(args)
    elif args.sweep:
        run_sweep(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
