"""Pins for the host FNV-1a-64 used to check lob_digest: the published FNV-1a-64 test
vectors (the FNV reference test suite), and the vectorised form against the scalar one."""
import numpy as np

from digest import fnv1a64, fnv1a64_rows, state_digest


def test_known_vectors():
    assert fnv1a64(b"") == 0xCBF29CE484222325
    assert fnv1a64(b"a") == 0xAF63DC4C8601EC8C
    assert fnv1a64(b"foobar") == 0x85944171F73967E8


def test_rows_match_scalar():
    rng = np.random.default_rng(7)
    rows = rng.integers(0, 256, (9, 37), dtype=np.uint8)
    got = fnv1a64_rows(rows)
    assert [int(x) for x in got] == [fnv1a64(r.tobytes()) for r in rows]


def test_state_digest_byte_order():
    book = np.full((1, 2, 1, 6), -1, np.int32)
    book[0, 0, 0] = [1010, 5, -9000, -9000, 34200, 0]
    trades = np.full((1, 2, 6), -1, np.int32)
    counts = np.array([0], np.int32)
    stats = np.arange(10, dtype=np.int64).reshape(1, 10)
    raw = book.tobytes() + trades.tobytes() + counts.tobytes() + stats.tobytes()
    assert int(state_digest(book, trades, counts, stats)[0]) == fnv1a64(raw)
    book[0, 0, 0, 1] = 4                                   # any field changes the digest
    assert int(state_digest(book, trades, counts, stats)[0]) != fnv1a64(raw)
