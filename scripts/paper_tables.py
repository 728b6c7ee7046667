#!/usr/bin/env python
"""Paper-shaped microbenchmarks (context, not targets): Tables 1, 2 and 4 of PAPER.md
re-run on this engine.  Books are filled to one third of capacity from a
synthetic L2 seed; every timing is CUDA events around whole library calls
(lob_init excluded), 1000 repetitions after warm-up, reported as median,
inter-quartile range and min, plus the op's device cost over a padding message
(median(op call) - median(padding call): the fixed launch cost cancels).

  Table 1: one book, one add / cancel / match message, N in {10,100,1000}
  Table 2: one book, N = 100, market order Q_a in {0,10,500,1000,10000}
  Table 4: the same message in 1000 identical books (the vmap shape),
                        time per call and effective ns per book-message
Prints one JSON document.
"""
import json
import os
import statistics
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2308_13289_b200 import LobBatch  # noqa: E402

REF, TICK = 1_000_000, 100


def seed(K, N):
    L0 = max(1, N // 3)
    rows = np.zeros((K, L0, 4), np.int32)
    for k in range(L0):
        rows[:, k] = [REF + (k + 1) * TICK, 300, REF - (k + 1) * TICK, 300]
    return torch.from_numpy(rows).cuda(), L0


def timed(b, init, msgs, reps=1000):
    """Per-call microseconds over `reps` calls: {median, q1, q3, min}."""
    st = torch.cuda.current_stream()
    es = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    for i in range(reps + 10):
        b.init(init, 34200, 0)
        if i >= 10:
            es[i - 10][0].record(st)
        b.process(msgs, 1, 1, l2=False)
        if i >= 10:
            es[i - 10][1].record(st)
    torch.cuda.synchronize()
    t = np.array([a.elapsed_time(z) * 1e3 for a, z in es])
    q1, med, q3 = np.percentile(t, [25, 50, 75])
    return {"median": float(med), "q1": float(q1), "q3": float(q3), "iqr": float(q3 - q1), "min": float(t.min())}


def with_device_cost(r, pad):
    r["device_us_over_padding"] = r["median"] - pad["median"]
    return r


def msg(T, S, Q, P, oid=777):
    return [T, S, Q, P, oid, 1, 34201, 0]


def cases(N):
    L0 = max(1, N // 3)
    return {
        "add": msg(1, 1, 100, REF - (L0 + 5) * TICK),           # passive bid below the book
        "cancel": msg(2, -1, 100, REF + TICK, 999999999),        # synthetic ask at the best price
        "match": msg(1, 1, 300 * 2, REF + 2 * TICK),             # crossing limit: takes two levels
    }


def run(reps=1000):
    out = {"note": "microseconds per library call; context only (PAPER.md Tables 1/2/4 were a 2080 Ti)",
           "reps": reps}
    pad = msg(0, 0, 0, 0, 0)
    t1 = {}
    for N in (10, 100, 1000):
        b = LobBatch(1, N, 64, 1)
        init, _ = seed(1, N)
        p0 = timed(b, init, torch.tensor([[pad]], dtype=torch.int32).cuda(), reps)
        t1[N] = {k: with_device_cost(timed(b, init, torch.tensor([[m]], dtype=torch.int32).cuda(), reps), p0)
                 for k, m in cases(N).items()}
        t1[N]["padding"] = p0
    out["table1_one_book_us"] = t1
    t2 = {}
    b = LobBatch(1, 100, 128, 1)
    init, _ = seed(1, 100)
    p0 = timed(b, init, torch.tensor([[pad]], dtype=torch.int32).cuda(), reps)
    for qa in (0, 10, 500, 1000, 10000):
        t2[qa] = with_device_cost(timed(b, init, torch.tensor([[msg(4, 1, qa, 0)]], dtype=torch.int32).cuda(), reps), p0)
    t2["padding"] = p0
    out["table2_market_us"] = t2
    t4 = {}
    for N in (10, 100, 1000):
        K = 1000
        b = LobBatch(K, N, 64, 1)
        init, _ = seed(K, N)
        p0 = timed(b, init, torch.tensor([[pad]] * K, dtype=torch.int32).cuda(), reps)
        row = {"padding": p0}
        for k, m in cases(N).items():
            r = with_device_cost(timed(b, init, torch.tensor([[m]] * K, dtype=torch.int32).cuda(), reps), p0)
            r["ns_per_book_message"] = r["median"] * 1e3 / K
            row[k] = r
        t4[N] = row
    out["table4_1000_books"] = t4
    return out


if __name__ == "__main__":
    print(json.dumps(run()))
