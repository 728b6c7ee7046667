#!/usr/bin/env python
"""Wait counters of the side-split build (instrumented variant, -DLOB_SPLIT_STATS).

    LOB_LIB_OVERRIDE=variants/splitstats.so python scripts/split_stats.py [C2]
Sites: 0 = ring reuse window (chunk start), 1 = remainder of an own-side limit that may
trade, 2 = trade order before a fill.  Per site: waits, waits that spun, spin iterations.
"""
import ctypes
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import lobgen  # noqa: E402
from paper_2308_13289_b200 import LobBatch, lib  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
cfg = lobgen.CONFIGS[name]
msgs, init = lobgen.generate(cfg)
dm, di = torch.from_numpy(msgs).cuda(), torch.from_numpy(init).cuda()
b = LobBatch(cfg.n_books, cfg.capacity, cfg.trades_cap, cfg.l2_levels)
L = lib()
L.lob_split_stats_read.argtypes = [ctypes.c_void_p]
h = np.zeros((4, 3), np.uint64)
b.init(di, lobgen.INIT_TS, lobgen.INIT_TNS)
torch.cuda.synchronize()
assert L.lob_split_stats_read(h.ctypes.data) == 0
b.process(dm, cfg.n_steps, cfg.msgs_per_step)
torch.cuda.synchronize()
assert L.lob_split_stats_read(h.ctypes.data) == 0
n = cfg.n_books * cfg.n_msgs
out = {"config": name, "messages": n}
for s, nm in enumerate(["window", "remainder", "trade_order"]):
    out[nm] = {"waits_per_msg_per_warp": float(h[s, 0]) / (2 * n), "spun_frac": float(h[s, 1]) / max(1, float(h[s, 0])),
               "spins_per_spun": float(h[s, 2]) / max(1, float(h[s, 1]))}
print(json.dumps(out, indent=1))

# per-message cycles by class (lane 0 of each side's warp, first 8 books)
L.lob_split_trace_read.argtypes = [ctypes.c_void_p]
tr = np.zeros((8, 2, 10240), np.int64)
assert L.lob_split_trace_read(tr.ctypes.data) == 0
nm = min(cfg.n_msgs, 10240)
t = tr[:, :, :nm]
cyc, cls = t >> 4, t & 15
names = {0: "pad/bad", 1: "own cancel", 2: "own limit (no wait)", 3: "own limit (waited, traded)", 4: "own limit (waited, no trade)",
         5: "other cancel (skip)", 6: "other aggr, no fill", 7: "other aggr, fill"}
res = {}
for k, v in names.items():
    m = cls == k
    if m.sum():
        res[v] = {"share": float(m.mean()), "mean_cycles": float(cyc[m].mean()), "median": float(np.median(cyc[m]))}
res["mean_cycles_per_msg_per_warp"] = float(cyc.mean())
print(json.dumps(res, indent=1))
