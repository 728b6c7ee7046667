#!/usr/bin/env python
"""Per-kernel registers / stack / spills from the ptxas -v log."""
import re, sys
cur = None
for l in open(sys.argv[1] if len(sys.argv) > 1 else "paper_2308_13289_b200/ptxas.log"):
    m = re.search(r"Compiling entry function '(\S+)'", l)
    if m:
        cur = m.group(1); continue
    m = re.search(r"(\d+) bytes stack frame, (\d+) bytes spill stores, (\d+) bytes spill loads", l)
    if m and cur:
        st = m.groups()
    m = re.search(r"Used (\d+) registers", l)
    if m and cur:
        print(f"{cur[:48]:48s} regs={m.group(1):>4s} stack={st[0]:>4s} spill_st={st[1]:>4s} spill_ld={st[2]:>4s}")
        cur = None
