#!/usr/bin/env python3
"""SASS size per source line of one kernel (nvdisasm -g of the in-tree liblob.so).
usage: scripts/sass_lines.py <kernel-substring> [top]"""
import collections, os, re, subprocess, sys, tempfile
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pat, top = sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40
so = os.environ.get("LOB_SO", os.path.join(ROOT, "paper_2308_13289_b200/liblob.so"))
d = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", so], cwd=d, check=True, capture_output=True)
cub = [f for f in os.listdir(d) if f.endswith(".cubin")][0]
txt = subprocess.run(["nvdisasm", "-g", os.path.join(d, cub)], capture_output=True, text=True).stdout
cur_fn, cur, c = None, None, collections.Counter()
for line in txt.splitlines():
    m = re.match(r"\.text\.(\S+):", line)
    if m:
        cur_fn = m.group(1)
        continue
    if cur_fn is None or pat not in cur_fn:
        continue
    m = re.search(r'//## File "([^"]+)", line (\d+)', line)
    if m:
        cur = (os.path.basename(m.group(1)), int(m.group(2)))
        continue
    if re.match(r"\s+/\*[0-9a-f]{4,}\*/", line):
        c[cur] += 1
print("instructions:", sum(c.values()))
for k, v in c.most_common(top):
    print(f"{v:6d}  {k[0]}:{k[1]}" if k else f"{v:6d}  ?")
