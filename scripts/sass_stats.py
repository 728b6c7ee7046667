#!/usr/bin/env python3
"""Per lob_step build: SASS instructions, BRA.DIV, STL/LDL, registers.  usage: sass_stats.py <so> [filter]"""
import re, subprocess, sys
so = sys.argv[1]; flt = sys.argv[2] if len(sys.argv) > 2 else "lob_step"
txt = subprocess.run(["cuobjdump", "-sass", so], capture_output=True, text=True).stdout
res = subprocess.run(["cuobjdump", "-res-usage", so], capture_output=True, text=True).stdout
regs = {}
cur = None
for line in res.splitlines():
    m = re.search(r"Function (\S+):", line)
    if m: cur = m.group(1); continue
    m = re.search(r"REG:(\d+) STACK:(\d+)", line)
    if m and cur: regs[cur] = (int(m.group(1)), int(m.group(2)))
cur = None; c = {}
for line in txt.splitlines():
    m = re.match(r"\s+Function : (\S+)", line)
    if m: cur = m.group(1); c[cur] = [0, 0, 0]; continue
    if cur and re.match(r"\s+/\*[0-9a-f]{4,}\*/", line):
        c[cur][0] += 1
        c[cur][1] += "BRA.DIV" in line
        c[cur][2] += ("STL" in line) or ("LDL" in line)
for k, v in c.items():
    if flt in k:
        m = re.search(r"lob_stepILi(\d+)ELi(\d+)ELi(\d+)ELi(\d+)", k)
        name = "<%s,%s,%s,%s>" % m.groups() if m else k
        print(f"{name:14s} instr {v[0]:6d} bra.div {v[1]:3d} stl/ldl {v[2]:3d} regs/stack {regs.get(k)}")
