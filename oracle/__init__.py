"""CPU oracle for the JAX-LOB hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` leg may import this package.  The product path
(``paper_2308_13289_b200``) never imports it and has no CPU fallback.

The arithmetic lives in ``oracle/lob_oracle.c`` (plain C, one book at a time,
written in the order of PAPER.md Section 4); this module only marshals numpy
arrays into it.  ``OracleBatch`` mirrors the C ABI of ``include/lob.h`` so that
parity tests can drive both with the same calls.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading
from concurrent.futures import ThreadPoolExecutor

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "lob_oracle.c")
_LIB = os.path.join(_HERE, "liblob_oracle.so")
_lock = threading.Lock()
_lib = None

NSTATS = 10
STAT_NAMES = ("msgs", "bad", "trades", "trades_dropped", "traded_qty", "cancelled_qty",
              "unknown_cancels", "add_overflow", "overflow_qty", "market_discarded_qty")


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (building the checker is not using it)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-Wall", "-shared", "-fPIC",
                               "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


_variants = {}


def _declare(lib):
    P = ctypes.c_void_p
    i32 = ctypes.c_int32
    lib.oracle_create.restype = P
    lib.oracle_create.argtypes = [i32, i32, i32, i32, i32]
    lib.oracle_destroy.argtypes = [P]
    lib.oracle_init.restype = ctypes.c_int
    lib.oracle_init.argtypes = [P, i32, i32, P, i32, i32, i32]
    lib.oracle_process.restype = ctypes.c_int
    lib.oracle_process.argtypes = [P, i32, i32, P, i32, i32, P]
    lib.oracle_process_ex.restype = ctypes.c_int
    lib.oracle_process_ex.argtypes = [P, i32, i32, P, i32, i32, P, P]
    for name in ("oracle_get_book", "oracle_get_l2", "oracle_get_stats",
                 "oracle_get_violations"):
        getattr(lib, name).argtypes = [P, P]
    lib.oracle_get_trades.argtypes = [P, P, P]
    lib.oracle_step_reward.argtypes = [P, P, P, P, ctypes.c_double, P, P, P]
    lib.oracle_env_create.restype = P
    lib.oracle_env_create.argtypes = [i32]
    lib.oracle_env_destroy.argtypes = [P]
    lib.oracle_env_reset.argtypes = [P, P, P, i32, i32]
    lib.oracle_env_step.argtypes = [P, P, P, P, P, i32, P, P, P, P]
    lib.oracle_env_get.argtypes = [P, P, P]
    return lib


def _load(path: str | None = None):
    """The oracle library; `path` loads a separately compiled variant of lob_oracle.c
    (tests/test_oracle_mutations.py compiles deliberately broken copies to show that
    the pins catch them)."""
    global _lib
    with _lock:
        if path is not None:
            if path not in _variants:
                _variants[path] = _declare(ctypes.CDLL(path))
            return _variants[path]
        if _lib is None:
            build()
            _lib = _declare(ctypes.CDLL(_LIB))
    return _lib


def _ptr(a):
    return None if a is None else ctypes.c_void_p(a.ctypes.data)


class OracleBatch:
    """K independent books of capacity N (SURVEY 8(c) pseudo-code, in C)."""

    def __init__(self, n_books: int, capacity: int, trades_cap: int | None = None,
                 l2_levels: int = 10, check: bool = False, threads: int = 1, lib_path: str | None = None):
        self.lib = _load(lib_path)
        self.K, self.N = int(n_books), int(capacity)
        self.T_cap = self.N if trades_cap is None else int(trades_cap)
        self.L = int(l2_levels)
        self.threads = max(1, int(threads))
        self.ctx = self.lib.oracle_create(self.K, self.N, self.T_cap, self.L, int(bool(check)))
        if not self.ctx:
            raise ValueError("oracle_create: bad dimensions")
        self.init()

    def __del__(self):
        ctx, self.ctx = getattr(self, "ctx", None), None
        if ctx:
            self.lib.oracle_destroy(ctx)

    def _ranges(self):
        t = min(self.threads, max(1, self.K))
        step = (self.K + t - 1) // t
        return [(a, min(self.K, a + step)) for a in range(0, self.K, step)] or [(0, 0)]

    def init(self, init_l2: np.ndarray | None = None, init_ts: int = 0, init_tns: int = 0):
        L0 = 0
        if init_l2 is not None:
            init_l2 = np.ascontiguousarray(init_l2, dtype=np.int32)
            assert init_l2.ndim == 3 and init_l2.shape[0] == self.K and init_l2.shape[2] == 4
            L0 = init_l2.shape[1]
        rc = self.lib.oracle_init(self.ctx, 0, self.K, _ptr(init_l2), L0, int(init_ts), int(init_tns))
        if rc != 0:
            raise ValueError("oracle_init: init_levels must be <= capacity")

    def process(self, msgs: np.ndarray, n_steps: int, msgs_per_step: int, l2: bool = True,
                l1: bool = False):
        """Returns the per-step L2 [K][S][L][4] (or None); with l1=True returns
        (l2, l1) where l1 is the per-message Level-1 trace [K][S*M][4] (NEXT row N1)."""
        msgs = np.ascontiguousarray(msgs, dtype=np.int32)
        assert msgs.shape == (self.K, n_steps * msgs_per_step, 8), msgs.shape
        out = np.empty((self.K, n_steps, self.L, 4), np.int32) if l2 else None
        l1o = np.empty((self.K, n_steps * msgs_per_step, 4), np.int32) if l1 else None
        if self.threads == 1 or self.K <= 1:
            self.lib.oracle_process_ex(self.ctx, 0, self.K, _ptr(msgs), n_steps, msgs_per_step, _ptr(out),
                                       _ptr(l1o))
        else:
            with ThreadPoolExecutor(self.threads) as ex:   # ctypes releases the GIL
                list(ex.map(lambda r: self.lib.oracle_process_ex(
                    self.ctx, r[0], r[1], _ptr(msgs), n_steps, msgs_per_step, _ptr(out), _ptr(l1o)),
                    self._ranges()))
        return (out, l1o) if l1 else out

    def book(self) -> np.ndarray:
        out = np.empty((self.K, 2, self.N, 6), np.int32)
        self.lib.oracle_get_book(self.ctx, _ptr(out))
        return out

    def trades(self):
        out = np.empty((self.K, self.T_cap, 6), np.int32)
        cnt = np.empty((self.K,), np.int32)
        self.lib.oracle_get_trades(self.ctx, _ptr(out), _ptr(cnt))
        return out, cnt

    def l2(self) -> np.ndarray:
        out = np.empty((self.K, self.L, 4), np.int32)
        self.lib.oracle_get_l2(self.ctx, _ptr(out))
        return out

    def stats(self) -> np.ndarray:
        out = np.empty((self.K, NSTATS), np.int64)
        self.lib.oracle_get_stats(self.ctx, _ptr(out))
        return out

    def step_reward(self, agent_oids, p_init, side, lam: float):
        """NEXT row N2 over the last call's trade log: (reward f64[K], vwap f64[K], agent_qty i64[K])."""
        a = np.ascontiguousarray(agent_oids, dtype=np.int32).reshape(self.K, 2)
        pi = np.ascontiguousarray(p_init, dtype=np.float64).reshape(self.K)
        sd = np.ascontiguousarray(side, dtype=np.int32).reshape(self.K)
        r, v, q = np.empty(self.K), np.empty(self.K), np.empty(self.K, np.int64)
        self.lib.oracle_step_reward(self.ctx, _ptr(a), _ptr(pi), _ptr(sd), float(lam), _ptr(r), _ptr(v), _ptr(q))
        return r, v, q

    def violations(self) -> np.ndarray:
        out = np.empty((self.K,), np.int64)
        self.lib.oracle_get_violations(self.ctx, _ptr(out))
        return out


class EnvConfig(ctypes.Structure):
    """NEXT row N3 execution-env parameters (common to all envs)."""
    _fields_ = [("task_side", ctypes.c_int32), ("task_size", ctypes.c_int32), ("n_passive", ctypes.c_int32),
                ("tick", ctypes.c_int32), ("episode_s", ctypes.c_int32), ("agent_tid", ctypes.c_int32),
                ("oid_base", ctypes.c_int32), ("pad", ctypes.c_int32), ("lam", ctypes.c_double)]


class OracleEnv:
    """One execution environment per book of an OracleBatch (Sec.5.1.3, 5.2)."""

    def __init__(self, batch: OracleBatch, cfg: EnvConfig):
        self.b, self.cfg, self.lib = batch, cfg, batch.lib
        self.env = self.lib.oracle_env_create(batch.K)

    def __del__(self):
        e, self.env = getattr(self, "env", None), None
        if e:
            self.lib.oracle_env_destroy(e)

    def reset(self, init_ts: int, init_tns: int = 0):
        self.lib.oracle_env_reset(self.b.ctx, self.env, ctypes.byref(self.cfg), int(init_ts), int(init_tns))

    def step(self, actions, data, M: int):
        K = self.b.K
        a = np.ascontiguousarray(actions, dtype=np.float32).reshape(K, 4)
        d = np.ascontiguousarray(data, dtype=np.int32).reshape(K, M, 8)
        r, dn, ex = np.empty(K), np.empty(K, np.int32), np.empty(K, np.int64)
        am = np.empty((K, 8, 8), np.int32)
        self.lib.oracle_env_step(self.b.ctx, self.env, ctypes.byref(self.cfg), _ptr(a), _ptr(d), M, _ptr(r),
                                 _ptr(dn), _ptr(ex), _ptr(am))
        return r, dn, ex, am

    def state(self):
        out = np.empty((self.b.K, 16), np.int64)
        self.lib.oracle_env_get(self.b.ctx, self.env, _ptr(out))
        return out
