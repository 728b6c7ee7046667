"""NEXT row N4: LOBSTER ingestion -> engine inputs (host side).

Parsing is native (``csrc/lobster_io.c`` -> ``liblobster.so``); this module only
cuts the parsed day into the paper's windows:

* fixed-duration, non-overlapping windows (default 30 minutes, half-open
  [start, end) on whole seconds after ``start_s``);
* inside a window, steps of exactly ``msgs_per_step`` messages (100 in the paper,
  P:L384); the last partial step and all steps up to the longest window are
  zero-padded (zero messages are no-ops, G21);
* the initial book of a window is the LOBSTER Level-2 row of the window's first
  message (one synthetic order per level), and the window's stream starts
  at the message AFTER it, because a LOBSTER orderbook row is the state after its
  message (reading G32).
"""
from __future__ import annotations

import ctypes
import os
import threading
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liblobster.so")
_lock = threading.Lock()
_lib = None


def _load():
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(_LIB_PATH):
                raise RuntimeError(f"{_LIB_PATH} is missing: run `make`")
            L = ctypes.CDLL(_LIB_PATH)
            L.lobster_parse_messages.restype = ctypes.c_int64
            L.lobster_parse_messages.argtypes = [ctypes.c_char_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32,
                                                 ctypes.c_void_p, ctypes.c_void_p]
            L.lobster_parse_orderbook.restype = ctypes.c_int64
            L.lobster_parse_orderbook.argtypes = [ctypes.c_char_p, ctypes.c_int32, ctypes.c_void_p, ctypes.c_int64]
            L.lobster_last_error.restype = ctypes.c_char_p
            _lib = L
    return _lib


class LobsterError(ValueError):
    pass


def parse_messages(path: str, exec_as_market: bool = False):
    """-> (msgs [n][8] int32 in Eq.6 order, source row [n] int64, skipped-per-type [8] int64)."""
    L = _load()
    p = os.fsencode(path)
    n = L.lobster_parse_messages(p, None, 0, int(exec_as_market), None, None)
    if n < 0:
        raise LobsterError(L.lobster_last_error().decode())
    out = np.empty((n, 8), np.int32)
    rows = np.empty((n,), np.int64)
    skipped = np.zeros((8,), np.int64)
    m = L.lobster_parse_messages(p, out.ctypes.data if n else None, n, int(exec_as_market),
                                 rows.ctypes.data if n else None, skipped.ctypes.data)
    if m != n:
        raise LobsterError(L.lobster_last_error().decode())
    return out, rows, skipped


def parse_orderbook(path: str, levels: int = 10) -> np.ndarray:
    """-> [rows][levels][4] int32 [ask_p, ask_q, bid_p, bid_q]; empty levels (0, 0)."""
    L = _load()
    p = os.fsencode(path)
    n = L.lobster_parse_orderbook(p, levels, None, 0)
    if n < 0:
        raise LobsterError(L.lobster_last_error().decode())
    out = np.empty((n, levels, 4), np.int32)
    m = L.lobster_parse_orderbook(p, levels, out.ctypes.data if n else None, n)
    if m != n:
        raise LobsterError(L.lobster_last_error().decode())
    return out


@dataclass
class Windows:
    msgs: np.ndarray          # [W][n_steps*msgs_per_step][8] int32, zero-padded
    init_l2: np.ndarray       # [W][levels][4] int32 (lob_init seed)
    init_time: np.ndarray     # [W][2] int32 (Ts, Tns) of the snapshot
    real_steps: np.ndarray    # [W] int32 steps that hold data
    n_steps: int
    msgs_per_step: int


def build_windows(msgs: np.ndarray, rows: np.ndarray, book: np.ndarray, window_s: int = 1800,
                  msgs_per_step: int = 100, start_s: int = 34200, end_s: int = 57600) -> Windows:
    """Cut parsed messages (and the orderbook rows they index) into windows."""
    if window_s <= 0 or msgs_per_step <= 0 or end_s <= start_s:
        raise ValueError("bad window parameters")
    nw = (end_s - start_s + window_s - 1) // window_s
    ts = msgs[:, 6].astype(np.int64)
    inside = (ts >= start_s) & (ts < end_s)
    widx = np.where(inside, (ts - start_s) // window_s, -1)
    per = []
    for w in range(nw):
        sel = np.nonzero(widx == w)[0]
        per.append(sel)
    counts = [max(0, len(sel) - 1) for sel in per]            # the first message seeds the book
    n_steps = max([(c + msgs_per_step - 1) // msgs_per_step for c in counts] + [1])
    levels = book.shape[1]
    out = np.zeros((nw, n_steps * msgs_per_step, 8), np.int32)
    init = np.zeros((nw, levels, 4), np.int32)
    init_time = np.zeros((nw, 2), np.int32)
    real = np.zeros((nw,), np.int32)
    for w, sel in enumerate(per):
        if len(sel) == 0:
            continue
        first = sel[0]
        init[w] = book[rows[first]]
        init_time[w] = msgs[first, 6:8]
        body = msgs[sel[1:]]
        out[w, :len(body)] = body
        real[w] = (len(body) + msgs_per_step - 1) // msgs_per_step
    return Windows(out, init, init_time, real, n_steps, msgs_per_step)


def format_messages(msgs: np.ndarray) -> str:
    """Engine messages (types 1-3) -> LOBSTER message CSV text (used by tests and tools)."""
    lines = []
    for m in msgs:
        T, S, Q, P, OID, _, Ts, Tns = (int(x) for x in m)
        if T not in (1, 2, 3):
            continue
        lines.append(f"{Ts}.{Tns:09d},{T},{OID},{Q},{P},{S}")
    return "\n".join(lines) + ("\n" if lines else "")
