#!/usr/bin/env python3
"""Summarise an ncu --set full report: key throughput / traffic / stall metrics per kernel.
usage: ncu_summary.py report.ncu-rep [alg_bytes_per_launch ...]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
alg = [float(x) for x in sys.argv[2:]]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, data = rows[0], rows[1], rows[2:]
WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__grid_size", "launch__block_size",
        "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic", "launch__occupancy_limit_registers",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
        "smsp__pcsamp_warps_issue_stalled_long_scoreboard", "smsp__pcsamp_warps_issue_stalled_wait",
        "smsp__pcsamp_warps_issue_stalled_barrier", "smsp__pcsamp_warps_issue_stalled_math_pipe_throttle",
        "smsp__pcsamp_warps_issue_stalled_selected", "smsp__pcsamp_warps_issue_stalled_not_selected",
        "smsp__pcsamp_warps_issue_stalled_branch_resolving", "smsp__pcsamp_warps_issue_stalled_short_scoreboard",
        "smsp__pcsamp_sample_count"]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3,
         "ns": 1e-9, "us": 1e-6, "ms": 1e-3}
for i, d in enumerate(data):
    name = d[hdr.index("Kernel Name")]
    print(f"== {name}")
    vals = {}
    for w in WANT:
        if w in hdr:
            j = hdr.index(w)
            print(f"   {w:70s} {d[j]:>16s} {units[j]}")
            try:
                vals[w] = float(d[j].replace(",", "")) * SCALE.get(units[j], 1)
            except ValueError:
                pass
    t = vals.get("gpu__time_duration.sum")
    rd, wr = vals.get("dram__bytes_read.sum"), vals.get("dram__bytes_write.sum")
    if t and rd is not None and wr is not None:
        print(f"   dram traffic {rd + wr:.4e} B in {t * 1e6:.1f} us = {(rd + wr) / t / 1e9:.1f} GB/s")
        if i < len(alg):
            print(f"   algorithmic {alg[i]:.4e} B -> {alg[i] / t / 1e9:.1f} GB/s; traffic/alg = {(rd + wr) / alg[i]:.3f}")
