#!/usr/bin/env python
"""Attribute ncu per-instruction counts to source lines.

usage: scripts/sass_hotspots.py <ncu-rep> <kernel-mangled-name> [top]
Joins `ncu --page source --print-source=sass` (per-address counts and stall
samples) with `nvdisasm -g -gi` line info of the in-tree liblob.so.
"""
import collections
import csv
import glob
import io
import os
import re
import subprocess
import sys
import tempfile

rep, fn = sys.argv[1], sys.argv[2]
dump = len(sys.argv) > 3 and sys.argv[3] == "dump"
alu_only = os.environ.get("ALU_ONLY") == "1"
ALU_OPS = ("ISETP", "SEL", "LOP3", "IADD3", "SHF", "PRMT", "IMNMX", "VIMNMX", "FLO", "POPC", "PLOP3", "P2R", "R2P",
           "VIADD", "LEA", "ICMP", "BMSK", "SGXT", "MOV ")
top = int(sys.argv[3]) if len(sys.argv) > 3 and not dump else 40
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
so = os.path.join(root, "paper_2308_13289_b200", "liblob.so")

raw = subprocess.check_output(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"]).decode()
rows = list(csv.reader(io.StringIO(raw)))
hdr = rows[1]
ai, ei = hdr.index("Address"), hdr.index("Instructions Executed")
si = hdr.index("Warp Stall Sampling (All Samples)")
counts, stalls = {}, {}
base = None
for r in rows[2:]:
    if len(r) <= ei:
        continue
    try:
        a = int(r[ai], 16)
    except ValueError:
        continue
    if base is None:
        base = a
    counts[a - base] = float(r[ei] or 0)
    stalls[a - base] = float(r[si] or 0)

d = tempfile.mkdtemp()
subprocess.check_call(["cuobjdump", "-xelf", "all", so], cwd=d, stdout=subprocess.DEVNULL)
cubin = glob.glob(os.path.join(d, "*.cubin"))[0]
dis = subprocess.check_output(["nvdisasm", "-g", "-gi", cubin]).decode().splitlines()
start = None
for i, l in enumerate(dis):
    if l.startswith(f".text.{fn}:"):
        start = i
        break
line_of = {}
cur_inner, cur_outer = None, None
pending = []
for l in dis[start + 1:]:
    if l.startswith("//-----") or l.startswith("\t.section"):
        break
    m = re.match(r'\s*//## File "([^"]+)", line (\d+)(?: inlined at "([^"]+)", line (\d+))?', l)
    if m:
        pending.append((os.path.basename(m.group(1)), int(m.group(2))))
        continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*)", l)
    if m:
        if pending:
            cur_inner = pending[0]
            cur_outer = pending[-1]
            pending = []
        line_of[int(m.group(1), 16)] = (cur_inner, cur_outer, m.group(2).split(";")[0].strip())

if dump:
    thr, norm = float(sys.argv[4]), float(sys.argv[5])
    for a in sorted(counts):
        if counts[a] >= thr:
            li = line_of.get(a, (None, None, ""))
            print(f"{a:06x} {counts[a] / norm:7.3f} {str(li[0][1]) if li[0] else '-':>4s} {li[2][:100]}")
    sys.exit(0)
src = open(os.path.join(root, "paper_2308_13289_b200", "csrc", "lob_kernels.cuh")).read().splitlines()
agg_i, agg_s = collections.Counter(), collections.Counter()
total = sum(counts.values())
for a, c in counts.items():
    if alu_only and not any(line_of.get(a, (None, None, ""))[2].lstrip("@!P0123456789T ").startswith(op)
                            for op in ALU_OPS):
        continue
    inner = line_of.get(a, (None, None, ""))[0]
    agg_i[inner] += c
    agg_s[inner] += stalls.get(a, 0)
print(f"total warp-instructions executed: {total:.4g}")
for k, v in agg_i.most_common(top):
    txt = src[k[1] - 1].strip()[:90] if k and k[0] == "lob_kernels.cuh" else ""
    print(f"{v / total * 100:6.2f}%  stall {agg_s[k] / max(1, sum(stalls.values())) * 100:5.1f}%  {k}  {txt}")

if len(sys.argv) > 4:
    want = int(sys.argv[4])
    for a in sorted(counts):
        li = line_of.get(a)
        if li and li[0] and li[0][1] == want and counts[a] > 0:
            print(f"{a:06x} {counts[a]:12.0f} outer={li[1]} {li[2]}")
