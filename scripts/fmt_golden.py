#!/usr/bin/env python
"""Re-serialise golden JSON fixtures with innermost lists on one line (readable diffs)."""
import json
import re
import sys

for path in sys.argv[1:]:
    d = json.load(open(path))
    s = json.dumps(d, indent=1)
    # collapse lists that contain no nested containers
    s = re.sub(r"\[\s*([^\[\]\{\}]*?)\s*\]", lambda m: "[" + ", ".join(x.strip() for x in m.group(1).split(",")) + "]"
               if m.group(1).strip() else "[]", s)
    open(path, "w").write(s + "\n")
