#!/usr/bin/env python
"""Per-message cycle budget of the step kernel by message type (C2 chain).

Needs the instrumented variant (scripts/build_variant.sh WT trace -DLOB_TRACE_CYCLES)
loaded through LOB_LIB_OVERRIDE: it records clock64() at the start of every message
and around every L2 snapshot for the first 8 books of a launch.  One launch of the
config (mode B: all steps in one call, the other books running concurrently) gives
the timestamps; message i's cost is t[i+1] - t[i] (L2 snapshot time removed at step
ends; messages that close a 32-message staging chunk are reported separately).
Each message is classified by replaying the same 8 books one message per call
through the same library (book export before, counters after): limit resting
without a fill / limit with k fills / market with k fills / cancel exact OID /
cancel synthetic (G12) / cancel unknown / padding-malformed.

    LOB_LIB_OVERRIDE=variants/trace.so python scripts/cycle_budget.py [C2] > budget.json
"""
import collections
import ctypes
import json
import os
import statistics
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import lobgen  # noqa: E402
from paper_2308_13289_b200 import LobBatch, lib  # noqa: E402

TB, TM, TS = 8, 10240, 128


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "C2"
    cfg = lobgen.CONFIGS[name]
    K, S, M, L = cfg.n_books, cfg.n_steps, cfg.msgs_per_step, cfg.l2_levels
    n = cfg.n_msgs
    assert n <= TM and S <= TS
    msgs, init = lobgen.generate(cfg)
    dm, di = torch.from_numpy(msgs).cuda(), torch.from_numpy(init).cuda()
    b = LobBatch(K, cfg.capacity, cfg.trades_cap, L)
    for _ in range(3):
        b.init(di, lobgen.INIT_TS, lobgen.INIT_TNS)
        b.process(dm, S, M)
    torch.cuda.synchronize()
    tm = np.zeros((TB, TM), np.int64)
    tl = np.zeros((TB, TS, 2), np.int64)
    L_ = lib()
    L_.lob_trace_read.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
    assert L_.lob_trace_read(tm.ctypes.data, tl.ctypes.data) == 0
    # classification: the same 8 books, one message per call
    c = LobBatch(TB, cfg.capacity, cfg.trades_cap, L)
    c.init(di[:TB].contiguous(), lobgen.INIT_TS, lobgen.INIT_TNS)
    hm = msgs[:TB]
    cls = np.empty((TB, n), object)
    prev = c.stats().cpu().numpy()
    for i in range(n):
        book = c.book().cpu().numpy()
        c.process(torch.from_numpy(np.ascontiguousarray(hm[:, i:i + 1])).cuda(), 1, 1, l2=False)
        st = c.stats().cpu().numpy()
        d = st - prev
        prev = st
        for k in range(TB):
            T, Sd, Q, P, OID = (int(x) for x in hm[k, i, :5])
            fills = int(d[k, 2])
            if d[k, 1] or T == 0:
                cls[k, i] = "pad/bad"
            elif T in (2, 3):
                side = 1 if Sd == 1 else 0
                occ = book[k, side][:, 1] > 0
                if d[k, 6]:
                    cls[k, i] = "cancel unknown"
                elif (occ & (book[k, side][:, 2] == OID)).any():
                    cls[k, i] = "cancel exact OID"
                else:
                    cls[k, i] = "cancel synthetic (G12)"
            elif T == 1:
                f = "0" if fills == 0 else ("1" if fills == 1 else "2+")
                cls[k, i] = f"limit, {f} fills"
            else:
                cls[k, i] = "market, " + ("0" if fills == 0 else ("1" if fills == 1 else "2+")) + " fills"
    per = collections.defaultdict(list)
    boundary = []
    for k in range(TB):
        t = tm[k, :n]
        for i in range(n - 1):
            dt = int(t[i + 1] - t[i])
            if (i + 1) % M == 0:                      # an L2 snapshot sits between i and i+1
                s = i // M
                dt -= int(tl[k, s, 1] - tl[k, s, 0])
            if (i + 1) % 32 == 0:                     # chunk boundary: wait/decode/refill included
                boundary.append(dt)
                continue
            per[cls[k, i]].append(dt)
    l2c = [int(tl[k, s, 1] - tl[k, s, 0]) for k in range(TB) for s in range(S)]
    tot = sum(len(v) for v in per.values())
    out = {"config": name, "books_traced": TB, "messages_classified": tot,
           "note": "cycles from clock64 deltas of the instrumented build (lane 0); other books run concurrently",
           "classes": {}}
    budget = 0.0
    for k2, v in sorted(per.items(), key=lambda kv: -sum(kv[1])):
        m = statistics.mean(v)
        out["classes"][k2] = {"share": len(v) / tot, "mean_cycles": m, "median_cycles": statistics.median(v),
                              "p90_cycles": float(np.percentile(v, 90)), "cycles_per_msg_contrib": m * len(v) / tot}
        budget += m * len(v) / tot
    out["message_cycles_per_msg"] = budget
    out["chunk_boundary_extra_cycles"] = statistics.mean(boundary) - budget if boundary else None
    out["l2_snapshot_cycles"] = statistics.mean(l2c)
    out["l2_cycles_per_msg"] = statistics.mean(l2c) / M
    span = [int(tm[k, n - 1] - tm[k, 0]) for k in range(TB)]
    out["measured_cycles_per_msg_book"] = statistics.mean(span) / (n - 1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
