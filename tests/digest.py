"""Host FNV-1a-64 for the lob_digest parity tests (include/lob.h): test infrastructure,
independent of the device kernel.  FNV-1a: h = offset basis; per byte h ^= b; h *= prime
(mod 2^64)."""
from __future__ import annotations

import numpy as np

FNV_OFFSET = 0xCBF29CE484222325
FNV_PRIME = 0x100000001B3


def fnv1a64(data: bytes) -> int:
    """Scalar reference, byte by byte."""
    h = FNV_OFFSET
    for b in data:
        h = ((h ^ b) * FNV_PRIME) & 0xFFFFFFFFFFFFFFFF
    return h


def fnv1a64_rows(rows: np.ndarray) -> np.ndarray:
    """FNV-1a-64 of every row of a [K][nbytes] uint8 array (vectorised over rows)."""
    rows = np.ascontiguousarray(rows, dtype=np.uint8)
    h = np.full(rows.shape[0], FNV_OFFSET, np.uint64)
    p = np.uint64(FNV_PRIME)
    with np.errstate(over="ignore"):
        for j in range(rows.shape[1]):
            h ^= rows[:, j]
            h *= p
    return h


def state_digest(book: np.ndarray, trades: np.ndarray, counts: np.ndarray, stats: np.ndarray) -> np.ndarray:
    """lob_digest's byte stream per book: book [2][N][6] i32, trades [T_cap][6] i32 (-1 tail),
    n_trades i32, counters [10] i64, all little-endian."""
    K = book.shape[0]
    parts = [np.ascontiguousarray(book, "<i4").reshape(K, -1).view(np.uint8),
             np.ascontiguousarray(trades, "<i4").reshape(K, -1).view(np.uint8),
             np.ascontiguousarray(counts, "<i4").reshape(K, 1).view(np.uint8),
             np.ascontiguousarray(stats, "<i8").reshape(K, -1).view(np.uint8)]
    return fnv1a64_rows(np.concatenate(parts, axis=1))
