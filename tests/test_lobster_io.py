"""NEXT row N4: LOBSTER ingestion (host side), -m "not gpu".

Pinned by SPEC.md's worked parsing/windowing examples,
an independent pure-Python parser (csv + decimal) on random files, a round trip
of generated streams, and the snapshot-fidelity invariant: the L2 of a
book initialised from a LOBSTER snapshot reproduces that snapshot."""
from __future__ import annotations

import csv
import decimal
import os
import time

import numpy as np
import pytest

import lobgen
import oracle
from paper_2308_13289_b200 import lobster


def _write(tmp_path, name, text):
    p = os.path.join(tmp_path, name)
    with open(p, "w") as f:
        f.write(text)
    return p


def test_spec_parse_examples(tmp_path):
    p = _write(tmp_path, "m.csv", "34200.189608000,1,11885113,21,2238100,1\n34200.5,3,42,10,1000,-1\n")
    m, rows, skipped = lobster.parse_messages(p)
    np.testing.assert_array_equal(m[0], [1, 1, 21, 2238100, 11885113, 0, 34200, 189608000])
    np.testing.assert_array_equal(m[1], [3, -1, 10, 1000, 42, 0, 34200, 500000000])
    assert rows.tolist() == [0, 1] and skipped.sum() == 0


def test_malformed_row_reports_row_number(tmp_path):
    p = _write(tmp_path, "m.csv", "34200.1,1,1,1,100,1\n34200.2,1,2,1,100\n")
    with pytest.raises(lobster.LobsterError, match="row 2"):
        lobster.parse_messages(p)


def test_executions_are_skipped_or_replayed(tmp_path):
    p = _write(tmp_path, "m.csv", "34200.1,1,1,5,100,1\n34200.2,4,1,2,100,1\n34200.3,5,9,1,100,1\n"
                                  "34200.4,6,0,0,0,1\n34200.5,7,0,0,0,1\n")
    m, _, sk = lobster.parse_messages(p)
    assert len(m) == 1 and sk.tolist() == [0, 0, 0, 0, 1, 1, 1, 1]
    m2, _, sk2 = lobster.parse_messages(p, exec_as_market=True)
    np.testing.assert_array_equal(m2[1], [4, -1, 2, 100, 1, 0, 34200, 200000000])          # aggressor side
    assert sk2.tolist() == [0, 0, 0, 0, 0, 1, 1, 1]


def test_nanosecond_rounding_half_even(tmp_path):
    p = _write(tmp_path, "m.csv", "1.0000000005,1,1,1,1,1\n1.0000000015,1,2,1,1,1\n1.00000000051,1,3,1,1,1\n"
                                  "1.9999999995,1,4,1,1,1\n")
    m, _, _ = lobster.parse_messages(p)
    assert m[:, 6:8].tolist() == [[1, 0], [1, 2], [1, 1], [2, 0]]


def _py_parse(path):
    """Independent reference: csv module + Decimal, same mapping."""
    out = []
    with open(path) as f:
        for row in csv.reader(f):
            if not row:
                continue
            t = decimal.Decimal(row[0])
            ts = int(t)
            tns = int(((t - ts) * 10**9).quantize(decimal.Decimal(1), rounding=decimal.ROUND_HALF_EVEN))
            if tns == 10**9:
                ts, tns = ts + 1, 0
            typ, oid, size, price, d = (int(x) for x in row[1:])
            if typ in (1, 2, 3):
                out.append([typ, d, size, price, oid, 0, ts, tns])
    return np.asarray(out, np.int32).reshape(-1, 8)


def test_native_parser_equals_python_reference(tmp_path):
    rng = np.random.default_rng(2)
    lines = []
    t = decimal.Decimal("34200")
    for i in range(5000):
        t += decimal.Decimal(int(rng.integers(0, 10**7))) / decimal.Decimal(10**int(rng.integers(3, 12)))
        lines.append(f"{t},{int(rng.integers(1, 8))},{int(rng.integers(1, 2**31 - 1))},{int(rng.integers(1, 10**5))},"
                     f"{int(rng.integers(1, 2**31 - 1))},{int(rng.choice([-1, 1]))}")
    p = _write(tmp_path, "r.csv", "\n".join(lines) + "\n")
    m, _, _ = lobster.parse_messages(p)
    np.testing.assert_array_equal(m, _py_parse(p))


def test_round_trip_of_generated_streams(tmp_path):
    cfg = lobgen.CONFIGS["C1"]
    msgs, _ = lobgen.generate(cfg)
    p = _write(tmp_path, "g.csv", lobster.format_messages(msgs[0]))
    m, _, _ = lobster.parse_messages(p)
    keep = msgs[0][np.isin(msgs[0][:, 0], [1, 2, 3])].copy()
    keep[:, 5] = 0                                                     # TIDs are not in LOBSTER files
    np.testing.assert_array_equal(m, keep)


def test_windowing_examples():
    """250 messages in one window and 100 per step -> 3 real steps, the third
    half padding; a message exactly at a boundary opens the later window."""
    n = 252                                       # +1 seed message, +1 boundary message
    msgs = np.zeros((n, 8), np.int32)
    msgs[:, 0] = 1
    msgs[:, 6] = 34200 + np.arange(n) // 10      # 10 messages per second
    msgs[-1, 6] = 34200 + 1800                    # exactly at the window boundary
    msgs[-1, 7] = 0
    rows = np.arange(n, dtype=np.int64)
    book = np.zeros((n, 10, 4), np.int32)
    book[:, 0] = [1001, 5, 999, 7]
    w = lobster.build_windows(msgs, rows, book, window_s=1800, msgs_per_step=100, start_s=34200, end_s=34200 + 3600)
    assert w.msgs.shape == (2, 300, 8)
    assert w.real_steps.tolist() == [3, 0]       # window 0: 251 - 1 seed = 250 -> 3 steps
    assert (w.msgs[0, 250:] == 0).all() and (w.msgs[0, :250, 0] == 1).all()
    np.testing.assert_array_equal(w.init_l2[0, 0], [1001, 5, 999, 7])
    np.testing.assert_array_equal(w.init_l2[1, 0], [1001, 5, 999, 7])   # boundary message seeds window 1
    np.testing.assert_array_equal(w.init_time[1], [34200 + 1800, 0])


def test_orderbook_sentinels_and_snapshot_fidelity(tmp_path):
    """LOBSTER empty-level sentinels map to absent levels; an oracle book
    initialised from the snapshot reproduces its L2 exactly."""
    rows = ["1001,50,999,40,1002,30,998,20,9999999999,0,-9999999999,0",
            "1001,50,999,40,1003,10,997,0,9999999999,0,-9999999999,0"]
    p = _write(tmp_path, "ob.csv", "\n".join(rows) + "\n")
    ob = lobster.parse_orderbook(p, 3)
    np.testing.assert_array_equal(ob[0], [[1001, 50, 999, 40], [1002, 30, 998, 20], [0, 0, 0, 0]])
    np.testing.assert_array_equal(ob[1, 1], [1003, 10, 0, 0])
    o = oracle.OracleBatch(2, 8, 4, 3)
    o.init(ob, 34200, 0)
    l2 = o.l2()
    want = ob.copy()
    want[want[..., 0] == 0, 0] = -1
    want[want[..., 2] == 0, 2] = -1
    np.testing.assert_array_equal(l2, want)


def test_parse_throughput_reported(tmp_path):
    """Measurement for N4: parse rate of the native parser on a synthetic day-sized file."""
    cfg = lobgen.CONFIGS["C4"].with_(n_books=200)
    msgs, _ = lobgen.generate(cfg)
    text = "".join(lobster.format_messages(msgs[k]) for k in range(200))
    p = _write(tmp_path, "big.csv", text)
    t0 = time.perf_counter()
    m, _, _ = lobster.parse_messages(p)
    dt = time.perf_counter() - t0
    assert len(m) > 100000
    print(f"\nlobster parse: {len(m) / dt:.3g} rows/s ({len(m)} rows, {os.path.getsize(p) / dt / 1e6:.0f} MB/s)")
