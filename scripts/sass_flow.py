#!/usr/bin/env python3
"""Per-instruction listing of an ncu source page: address, executions per message, stall
samples, source line, SASS.   usage: scripts/sass_flow.py <ncu-rep> <n_msgs> [min_exec_per_msg]"""
import csv, io, os, re, subprocess, sys
rep, nmsg = sys.argv[1], float(sys.argv[2])
thr = float(sys.argv[3]) if len(sys.argv) > 3 else 0.001
raw = subprocess.check_output(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"]).decode()
rows = list(csv.reader(io.StringIO(raw)))
h = rows[1]
ai, si, ei, ni = h.index("Address"), h.index("Source"), h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
base = None
tot_s = sum(float(r[ni] or 0) for r in rows[2:] if len(r) > ni)
for r in rows[2:]:
    if len(r) <= ei: continue
    a = int(r[ai], 16)
    base = a if base is None else base
    e = float(r[ei] or 0) / nmsg
    s = float(r[ni] or 0) / tot_s * 100
    if e >= thr or s > 0.2:
        print(f"{a-base:06x} {e:7.3f} {s:5.2f}%  {r[si].strip()[:110]}")
