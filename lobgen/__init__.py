"""Seeded synthetic LOBSTER-shaped streams (shared input plumbing; no method arithmetic).

Both the oracle and the CUDA path consume the buffers produced here; neither
side generates its own inputs.  The C core (``lobgen.c``) is integer-only and
deterministic per (seed, global book id).  Configs C1-C5 are BASELINE.json's
``configs`` made concrete.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading
from dataclasses import dataclass, replace

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "lobgen.c")
_LIB = os.path.join(_HERE, "liblobgen.so")
_lock = threading.Lock()
_lib = None

PROFILES = {"lobster": 0, "heavy_market": 1, "cancel_heavy": 2, "ties": 3, "overflow": 4,
            "synthetic": 5, "garbage": 6, "saturate": 7}
INIT_TS, INIT_TNS = 34200, 0          # 09:30:00 in LOBSTER seconds-after-midnight
TICK, REF0 = 100, 1_000_000


def build(force: bool = False) -> str:
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-Wall", "-shared", "-fPIC", "-pthread",
                               "-o", tmp, _SRC])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    with _lock:
        if _lib is None:
            build()
            lib = ctypes.CDLL(_LIB)
            lib.lobgen_generate.restype = ctypes.c_int
            lib.lobgen_generate.argtypes = [ctypes.c_uint64, ctypes.c_int64] + [ctypes.c_int32] * 7 + \
                [ctypes.c_void_p, ctypes.c_void_p]
            _lib = lib
    return _lib


@dataclass(frozen=True)
class Config:
    """One workload: K books of capacity N, n_steps x msgs_per_step messages per book."""
    name: str
    n_books: int
    capacity: int
    n_steps: int
    msgs_per_step: int
    init_levels: int
    trades_cap: int
    l2_levels: int
    profile: str
    seed: int
    occ_cap_pct: int = 90

    @property
    def n_msgs(self) -> int:
        return self.n_steps * self.msgs_per_step

    def with_(self, **kw) -> "Config":
        return replace(self, **kw)


CONFIGS = {
    # BASELINE.json configs[0]: 1 book, N=100, 1,000 messages; oracle in seconds
    "C1": Config("C1", 1, 100, 10, 100, 10, 1000, 10, "lobster", 1),
    # configs[1]: 1,000 books, N=100, 100 msgs/step, L2 top-10 each step (RL-env shape)
    "C2": Config("C2", 1000, 100, 100, 100, 10, 100, 10, "lobster", 2),
    # configs[2]: 16,384 books, 1,000 msgs/book, heavy market orders (deep sweeps)
    "C3": Config("C3", 16384, 100, 10, 100, 33, 1024, 10, "heavy_market", 3),
    # configs[3]: 65,536 books, cancel-heavy (order-id lookup dominated); the bench workload
    "C4": Config("C4", 65536, 100, 10, 100, 33, 512, 10, "cancel_heavy", 4),
    # configs[4]: capacity sweep x 4,096 books (register vs shared-memory regime)
    "C5_32": Config("C5_32", 4096, 32, 10, 100, 10, 1024, 10, "lobster", 5),
    "C5_100": Config("C5_100", 4096, 100, 10, 100, 33, 1024, 10, "lobster", 5),
    "C5_512": Config("C5_512", 4096, 512, 10, 100, 170, 1024, 10, "lobster", 5),
    "C5_2048": Config("C5_2048", 4096, 2048, 10, 100, 682, 1024, 10, "lobster", 5),
    # extra points of the same sweep (not BASELINE configs): the other kernel geometries
    "C5_256": Config("C5_256", 4096, 256, 10, 100, 85, 1024, 10, "lobster", 5),
    "C5_1024": Config("C5_1024", 4096, 1024, 10, 100, 341, 1024, 10, "lobster", 5),
}


def generate(cfg: Config, book_begin: int = 0, n_books: int | None = None,
             threads: int | None = None, msgs_out: np.ndarray | None = None,
             init_out: np.ndarray | None = None):
    """Return (msgs [n][n_msgs][8] int32, init_l2 [n][L0][4] int32 or None).

    ``book_begin`` is the GLOBAL id of the first book: book b's bytes depend only on
    (cfg.seed, b), so a shard of a multi-GPU run sees exactly its slice of the
    single-GPU stream.  ``msgs_out``/``init_out`` may be caller buffers (e.g. numpy
    views of pinned torch tensors) of the right shape.
    """
    lib = _load()
    n = cfg.n_books if n_books is None else int(n_books)
    if msgs_out is None:
        msgs_out = np.empty((n, cfg.n_msgs, 8), np.int32)
    assert msgs_out.shape == (n, cfg.n_msgs, 8) and msgs_out.dtype == np.int32
    assert msgs_out.flags.c_contiguous
    if cfg.init_levels > 0 and init_out is None:
        init_out = np.empty((n, cfg.init_levels, 4), np.int32)
    if init_out is not None:
        assert init_out.shape == (n, cfg.init_levels, 4) and init_out.flags.c_contiguous
    t = threads or min(32, os.cpu_count() or 1)
    rc = lib.lobgen_generate(cfg.seed, book_begin, n, cfg.capacity, cfg.n_msgs, cfg.init_levels,
                             PROFILES[cfg.profile], cfg.occ_cap_pct, t,
                             msgs_out.ctypes.data if n else None,
                             init_out.ctypes.data if (init_out is not None and n) else None)
    if rc != 0:
        raise ValueError("lobgen_generate: bad arguments")
    return msgs_out, init_out
