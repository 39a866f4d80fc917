#!/usr/bin/env python3
"""Per-instruction stall hotspots of one kernel from an ncu source-page export.
usage: ncu -i REP.ncu-rep --page source --csv --print-source sass > x.csv
       python tools/sass_stalls.py x.csv KERNEL_INDEX [TOP]
KERNEL_INDEX counts the "Kernel Name" blocks of the export (0-based)."""
import csv, io, sys
lines = open(sys.argv[1]).read().split("\n")
starts = [i for i, l in enumerate(lines) if l.startswith('"Kernel Name"')]
which = int(sys.argv[2])
s = starts[which]; e = starts[which + 1] if which + 1 < len(starts) else len(lines)
print(lines[s][:120])
rows = list(csv.reader(io.StringIO("\n".join(lines[s + 1:e]))))
hdr = rows[0]; data = [r for r in rows[1:] if len(r) == len(hdr)]
iS = hdr.index("Warp Stall Sampling (All Samples)"); iE = hdr.index("Instructions Executed")
stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_")]
tot = sum(float(r[iS] or 0) for r in data)
print("total samples", tot, "instrs", len(data), "warp-instr executed", sum(float(r[iE] or 0) for r in data))
agg = {hdr[i]: sum(float(r[i] or 0) for r in data) for i in stall_cols}
print(sorted(((round(v / tot * 100, 1), k) for k, v in agg.items() if v), reverse=True)[:12])
top = sorted(range(len(data)), key=lambda k: -float(data[k][iS] or 0))[:int(sys.argv[3]) if len(sys.argv) > 3 else 40]
for k in sorted(top):
    r = data[k]
    st = sorted(((float(r[i] or 0), hdr[i][6:]) for i in stall_cols if float(r[i] or 0) > 0), reverse=True)[:3]
    print(f"{k:5d} {r[iS]:>5} {r[iE]:>8} {r[1].strip()[:60]:60s} {st}")
