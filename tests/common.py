"""Test helpers shared by the oracle pins (-m "not gpu") and the GPU parity tests (-m gpu).

An *engine* is anything with the LobBatch/OracleBatch surface:
``init(init_l2, ts, tns)``, ``process(msgs, n_steps, msgs_per_step, l2=True)``,
``book()``, ``trades()``, ``l2()``, ``stats()``.
"""
from __future__ import annotations

import glob
import json
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
GOLDEN = os.path.join(HERE, "golden")
STAT_NAMES = ("msgs", "bad", "trades", "trades_dropped", "traded_qty", "cancelled_qty",
              "unknown_cancels", "add_overflow", "overflow_qty", "market_discarded_qty")


def golden_cases():
    """Yield (id, case dict) for every golden fixture (single-case files and 'cases' lists)."""
    out = []
    for path in sorted(glob.glob(os.path.join(GOLDEN, "*.json"))):
        base = os.path.basename(path)[:-5]
        if base.startswith("reward_"):   # NEXT N2 fixtures have their own schema
            continue
        doc = json.load(open(path))
        if "cases" in doc:
            for i, c in enumerate(doc["cases"]):
                out.append((f"{base}[{i}]", c))
        else:
            out.append((base, doc))
    return out


def _msgs(call):
    m = np.asarray(call["messages"], dtype=np.int32).reshape(-1, 8)
    return m


def _init(engine, case):
    init = case.get("init")
    if init:
        rows = np.asarray(init["rows"], np.int32)[None]
        engine.init(rows, init["ts"], init["tns"])
    else:
        engine.init(None, 0, 0)


def expected_book(spec, N):
    """{'asks': {slot: [6]}, 'bids': {...}} -> [2][N][6] with -1 elsewhere."""
    b = np.full((2, N, 6), -1, np.int32)
    for s, key in ((0, "asks"), (1, "bids")):
        for slot, rec in spec.get(key, {}).items():
            b[s, int(slot)] = rec
    return b


def run_golden_case(make_engine, case):
    """Replay a golden case on engine(s) built by make_engine(N, T_cap, L); assert every expectation."""
    N, T_cap, L = case["capacity"], case["trades_cap"], case["l2_levels"]
    eng = make_engine(N, T_cap, L)
    _init(eng, case)
    for ci, call in enumerate(case["calls"]):
        S, M = call["n_steps"], call["msgs_per_step"]
        msgs = _msgs(call)
        exp = call["expect"]
        if "l1_trace" in exp:
            l2, l1 = eng.process(msgs[None], S, M, l2=True, l1=True)
            np.testing.assert_array_equal(l1[0], np.asarray(exp["l1_trace"], np.int32),
                                          err_msg=f"call {ci} L1 trace")
        else:
            l2 = eng.process(msgs[None], S, M, l2=True)
        if "trades" in exp:
            tr, cnt = eng.trades()
            want = np.full((T_cap, 6), -1, np.int32)
            if exp["trades"]:
                want[:len(exp["trades"])] = exp["trades"]
            assert int(cnt[0]) == len(exp["trades"]), (ci, cnt[0], exp["trades"])
            np.testing.assert_array_equal(tr[0], want, err_msg=f"call {ci} trades")
        if "book" in exp:
            np.testing.assert_array_equal(eng.book()[0], expected_book(exp["book"], N),
                                          err_msg=f"call {ci} book")
        if "l2" in exp:
            np.testing.assert_array_equal(eng.l2()[0], np.asarray(exp["l2"], np.int32),
                                          err_msg=f"call {ci} l2")
        for s, rows in exp.get("l2_after_step", {}).items():
            np.testing.assert_array_equal(l2[0, int(s)], np.asarray(rows, np.int32),
                                          err_msg=f"call {ci} l2 after step {s}")
        if "stats" in exp:
            st = eng.stats()[0]
            for k, v in exp["stats"].items():
                assert int(st[STAT_NAMES.index(k)]) == v, (ci, k, int(st[STAT_NAMES.index(k)]), v)
        # book after an intermediate step: replay from scratch up to that step
        for s, spec in exp.get("book_after_step", {}).items():
            e2 = make_engine(N, T_cap, L)
            _init(e2, case)
            for prev in case["calls"][:ci]:
                e2.process(_msgs(prev)[None], prev["n_steps"], prev["msgs_per_step"], l2=False)
            k = (int(s) + 1) * M
            e2.process(msgs[None, :k], int(s) + 1, M, l2=False)
            np.testing.assert_array_equal(e2.book()[0], expected_book(spec, N),
                                          err_msg=f"call {ci} book after step {s}")


def run_engine(engine, cfg, msgs, init_l2, init_ts, init_tns, calls=1):
    """init + `calls` equal calls over the stream; returns dict of all outputs."""
    engine.init(init_l2, init_ts, init_tns)
    per = cfg.n_steps // calls
    l2s = []
    for c in range(calls):
        sl = msgs[:, c * per * cfg.msgs_per_step:(c + 1) * per * cfg.msgs_per_step]
        l2s.append(engine.process(np.ascontiguousarray(sl), per, cfg.msgs_per_step, l2=True))
    tr, cnt = engine.trades()
    return {"book": engine.book(), "trades": tr, "n_trades": cnt, "l2": np.concatenate(l2s, axis=1),
            "l2_now": engine.l2(), "stats": engine.stats()}


def assert_outputs_equal(a, b, books=None, what=""):
    for key in ("book", "trades", "n_trades", "l2", "l2_now", "stats"):
        x, y = np.asarray(a[key]), np.asarray(b[key])
        if books is not None:
            x = x[books] if x.shape[0] != len(books) else x
            y = y[books] if y.shape[0] != len(books) else y
        if not np.array_equal(x, y):
            bad = np.argwhere(x != y)
            raise AssertionError(f"{what}: {key} differs at {len(bad)} positions, first {bad[:5].tolist()}")


# Capacity contract (G6) in every padded geometry: the kernel pads N to NP = 32*W*KPL
# slots (N = 130 -> 256, 600 -> 1024, 1500 -> 2048); a saturating stream (passive limits
# on both sides, about 5N messages) drives every capacity band past N.
SATURATE_N = [16, 100, 130, 224, 250, 300, 480, 600, 896, 1025, 1500, 1920]


def saturate_cfg(N):
    import lobgen
    K = 48 if N <= 300 else (16 if N <= 1024 else 8)
    steps = -(-(5 * N) // 100)
    return lobgen.Config("sat", K, N, steps, 100, min(N // 4, 30), 64, 10, "saturate", 100 + N)
