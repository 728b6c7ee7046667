"""Thin Python binding of the C ABI in ``include/lob.h`` (argument marshalling only).

Every step of the hot path runs in ``liblob.so`` (sm_100a CUDA kernels).  PyTorch
supplies device memory, streams and process groups; there is no CPU fallback:
constructing a ``LobBatch`` without the built library or without a CUDA device
raises.
"""
from __future__ import annotations

import ctypes
import os
import threading

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("LOB_LIB_OVERRIDE") or os.path.join(_HERE, "liblob.so")  # override: A/B experiments

LOB_NSTATS = 10
STAT_NAMES = ("msgs", "bad", "trades", "trades_dropped", "traded_qty", "cancelled_qty",
              "unknown_cancels", "add_overflow", "overflow_qty", "market_discarded_qty")
MAX_CAPACITY = 2048
MAX_L2_LEVELS = 32

_lock = threading.Lock()
_lib = None


class LobError(RuntimeError):
    pass


class _Config(ctypes.Structure):
    _fields_ = [("n_books", ctypes.c_int32), ("capacity", ctypes.c_int32),
                ("trades_cap", ctypes.c_int32), ("l2_levels", ctypes.c_int32),
                ("device", ctypes.c_int32)]


class EnvConfig(ctypes.Structure):
    """lob_env_config (include/lob.h): the execution task shared by all envs (NEXT row N3)."""
    _fields_ = [("task_side", ctypes.c_int32), ("task_size", ctypes.c_int32), ("n_passive", ctypes.c_int32),
                ("tick", ctypes.c_int32), ("episode_s", ctypes.c_int32), ("agent_tid", ctypes.c_int32),
                ("agent_oid_base", ctypes.c_int32), ("reserved", ctypes.c_int32), ("lam", ctypes.c_double)]


def lib():
    """Load liblob.so (built by ``make`` / ``__graft_entry__.build()``); raise if absent."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise LobError(f"{LIB_PATH} is missing: run `make` (or __graft_entry__.build()) first; "
                               "there is no CPU fallback")
            L = ctypes.CDLL(LIB_PATH)
            P, i32 = ctypes.c_void_p, ctypes.c_int32
            L.lob_state_bytes.restype = ctypes.c_size_t
            L.lob_state_bytes.argtypes = [ctypes.POINTER(_Config)]
            L.lob_create.restype = ctypes.c_int
            L.lob_create.argtypes = [ctypes.POINTER(P), ctypes.POINTER(_Config), P]
            L.lob_destroy.argtypes = [P]
            L.lob_init.restype = ctypes.c_int
            L.lob_init.argtypes = [P, P, i32, i32, i32, P]
            L.lob_process_messages.restype = ctypes.c_int
            L.lob_process_messages.argtypes = [P, P, i32, i32, P, P]
            if hasattr(L, "lob_process_messages_l1"):  # (absent only in old A/B builds)
                L.lob_process_messages_l1.restype = ctypes.c_int
                L.lob_process_messages_l1.argtypes = [P, P, i32, i32, P, P, P]
            L.lob_process_messages_host.restype = ctypes.c_int
            L.lob_process_messages_host.argtypes = [P, P, i32, i32, P, P, P, P, P, P, i32, P]
            L.lob_build_id.restype = ctypes.c_char_p
            for name in ("lob_get_l2", "lob_get_book", "lob_get_stats"):
                getattr(L, name).restype = ctypes.c_int
                getattr(L, name).argtypes = [P, P, P]
            L.lob_get_trades.restype = ctypes.c_int
            L.lob_get_trades.argtypes = [P, P, P, P]
            if hasattr(L, "lob_step_reward"):
                L.lob_step_reward.restype = ctypes.c_int
                L.lob_step_reward.argtypes = [P, P, P, P, ctypes.c_double, P, P, P, P]
            if hasattr(L, "lob_env_step"):
                L.lob_env_state_bytes.restype = ctypes.c_size_t
                L.lob_env_state_bytes.argtypes = [i32]
                L.lob_env_reset.restype = ctypes.c_int
                L.lob_env_reset.argtypes = [P, P, ctypes.POINTER(EnvConfig), i32, i32, P]
                L.lob_env_step.restype = ctypes.c_int
                L.lob_env_step.argtypes = [P, P, ctypes.POINTER(EnvConfig), P, P, i32, P, P, P, P, P, P]
            if hasattr(L, "lob_session_begin"):
                L.lob_session_begin.restype = ctypes.c_int
                L.lob_session_begin.argtypes = [P, P, ctypes.POINTER(EnvConfig), P, P, i32, i32, P, P, P, P, P, P]
                L.lob_session_step.restype = ctypes.c_int
                L.lob_session_step.argtypes = [P, P]
                L.lob_session_end.restype = ctypes.c_int
                L.lob_session_end.argtypes = [P, P]
            if hasattr(L, "lob_digest"):
                L.lob_digest.restype = ctypes.c_int
                L.lob_digest.argtypes = [P, P, P]
            L.lob_launch_count.restype = ctypes.c_int64
            L.lob_strerror.restype = ctypes.c_char_p
            L.lob_strerror.argtypes = [ctypes.c_int]
            L.lob_last_error.restype = ctypes.c_char_p
            _lib = L
    return _lib


def _check(rc: int, what: str):
    if rc != 0:
        L = lib()
        raise LobError(f"{what}: {L.lob_strerror(rc).decode()} ({L.lob_last_error().decode()})")


def launch_count() -> int:
    return int(lib().lob_launch_count())


def build_id() -> str:
    """Hash of the sources and flags liblob.so was built from (lob_build_id)."""
    return lib().lob_build_id().decode()


def _ptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream(stream=None):
    s = torch.cuda.current_stream() if stream is None else stream
    return ctypes.c_void_p(s.cuda_stream)


class _On:
    """Run a call's conversions, allocations and launch on ONE stream: ``stream=`` if
    given (made current for the block, so torch's copies and allocations are ordered
    with the kernel), else torch's current stream of the batch's device."""

    def __init__(self, device, stream):
        self.device, self.stream = device, stream

    def __enter__(self):
        self._d = torch.cuda.device(self.device)
        self._d.__enter__()
        self._s = torch.cuda.stream(self.stream) if self.stream is not None else None
        if self._s is not None:
            self._s.__enter__()
        return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)

    def __exit__(self, *a):
        if self._s is not None:
            self._s.__exit__(*a)
        self._d.__exit__(*a)


class LobBatch:
    """K independent limit-order books of capacity N on one GPU (the C ABI's lob_ctx).

    Tensors are int32 on the context's device in the layouts of include/lob.h.
    All calls are asynchronous on torch's current stream (or ``stream=``).
    """

    def __init__(self, n_books: int, capacity: int, trades_cap: int | None = None,
                 l2_levels: int = 10, device=None):
        if not torch.cuda.is_available():
            raise LobError("LobBatch needs a CUDA device; there is no CPU fallback")
        self.device = torch.device("cuda", torch.cuda.current_device()) if device is None \
            else torch.device(device)
        self.K, self.N = int(n_books), int(capacity)
        self.T_cap = self.N if trades_cap is None else int(trades_cap)
        self.L = int(l2_levels)
        L = lib()
        self._cfg = _Config(self.K, self.N, self.T_cap, self.L, self.device.index or 0)
        nbytes = L.lob_state_bytes(ctypes.byref(self._cfg))
        if nbytes == 0 and self.K > 0:
            raise LobError("invalid configuration (capacity 1..2048, l2_levels 1..32, K >= 0)")
        with torch.cuda.device(self.device):
            self.state = torch.empty(max(int(nbytes), 256) + 256, dtype=torch.uint8, device=self.device)
        off = (-self.state.data_ptr()) % 256
        self._state_ptr = ctypes.c_void_p(self.state.data_ptr() + off)
        self.ctx = ctypes.c_void_p()
        with torch.cuda.device(self.device):
            _check(L.lob_create(ctypes.byref(self.ctx), ctypes.byref(self._cfg), self._state_ptr),
                   "lob_create")
        self.last_l2 = None

    def __del__(self):
        ctx, self.ctx = getattr(self, "ctx", None), None
        if ctx:
            try:
                lib().lob_destroy(ctx)
            except Exception:
                pass

    def _dev(self, x, dtype=torch.int32):
        if x is None:
            return None
        t = torch.as_tensor(x)
        t = t.to(device=self.device, dtype=dtype, non_blocking=True)
        return t.contiguous()

    # ------------------------------------------------------------------ calls
    def init(self, init_l2=None, init_ts: int = 0, init_tns: int = 0, stream=None):
        """lob_init: empty books, optional synthetic L2 seed [K][L0][4]."""
        with _On(self.device, stream) as st:
            t = self._dev(init_l2)
            L0 = 0 if t is None else int(t.shape[1])
            if t is not None:
                assert t.shape == (self.K, L0, 4), t.shape
            _check(lib().lob_init(self.ctx, _ptr(t), L0, int(init_ts), int(init_tns), st), "lob_init")
        self._keep = t  # keep the input alive until the stream has consumed it

    def process(self, msgs, n_steps: int, msgs_per_step: int, l2: bool = True, l2_out=None,
                stream=None, l1: bool = False, l1_out=None):
        """lob_process_messages over msgs [K][n_steps*msgs_per_step][8]; returns L2 [K][S][L][4].

        With ``l1=True`` (lob_process_messages_l1, NEXT row N1) returns ``(l2, l1)`` where
        l1 [K][n_steps*msgs_per_step][4] is the Level-1 state after every message."""
        with _On(self.device, stream) as st:
            m = self._dev(msgs)
            assert m.shape == (self.K, n_steps * msgs_per_step, 8), m.shape
            out = l2_out
            if l2 and out is None:
                out = torch.empty((self.K, n_steps, self.L, 4), dtype=torch.int32, device=self.device)
            l1o = l1_out
            if l1 and l1o is None:
                l1o = torch.empty((self.K, n_steps * msgs_per_step, 4), dtype=torch.int32, device=self.device)
            if l1:
                _check(lib().lob_process_messages_l1(self.ctx, _ptr(m), int(n_steps), int(msgs_per_step),
                                                     _ptr(out) if l2 else None, _ptr(l1o), st),
                       "lob_process_messages_l1")
            else:
                _check(lib().lob_process_messages(self.ctx, _ptr(m), int(n_steps), int(msgs_per_step),
                                                  _ptr(out) if l2 else None, st),
                       "lob_process_messages")
        self._keep = m
        if l1:
            return (out if l2 else None), l1o
        return out if l2 else None

    def process_host(self, h_msgs, n_steps: int, msgs_per_step: int, h_l2_out=None,
                     h_stats_out=None, d_msgs_buf=None, d_l2_buf=None, chunks: int | None = None, stream=None,
                     h_trades_out=None, h_trade_counts_out=None):
        """lob_process_messages_host: pinned host messages in; pinned host L2 [K][S][L][4],
        counters [K][10], and the LOGGED trade rows packed book after book into
        ``h_trades_out`` (capacity [K*T_cap][6]) with per-book counts in
        ``h_trade_counts_out`` [K].  The caller synchronises the stream before reading.

        ``chunks`` (default: one per 1,024 books, at most 64): the book slices whose
        host->device copy overlaps the previous slice's kernel.  Measured on C4 (65,536
        books): 8 / 16 / 32 / 64 / 128 chunks reach 90 / 92 / 93 / 95 / 89 % of a plain
        pinned copy's bandwidth."""
        if chunks is None:
            chunks = max(1, min(64, self.K // 1024))
        assert h_msgs.device.type == "cpu" and h_msgs.dtype == torch.int32 and h_msgs.is_contiguous()
        for t in (h_l2_out, h_stats_out, h_trades_out, h_trade_counts_out):
            assert t is None or (t.device.type == "cpu" and t.is_contiguous() and t.is_pinned())
        if h_trades_out is not None:
            assert h_trades_out.dtype == torch.int32 and h_trades_out.numel() >= self.K * self.T_cap * 6
            assert h_trade_counts_out is not None and h_trade_counts_out.numel() == self.K
        with _On(self.device, stream) as st:
            _check(lib().lob_process_messages_host(
                self.ctx, _ptr(h_msgs), int(n_steps), int(msgs_per_step), _ptr(h_l2_out),
                _ptr(h_stats_out), _ptr(h_trades_out), _ptr(h_trade_counts_out), _ptr(d_msgs_buf),
                _ptr(d_l2_buf), int(chunks), st),
                "lob_process_messages_host")

    def step_reward(self, agent_oids, p_init, task_side, lam: float, stream=None):
        """lob_step_reward (NEXT row N2) over the last call's trade log.

        agent_oids [K][2] int32 (inclusive OID range), p_init [K] f64, task_side [K]
        int32 (-1 sell, +1 buy).  Returns (reward f64[K], vwap f64[K], agent_qty i64[K])."""
        with _On(self.device, stream) as st:
            a = self._dev(agent_oids)
            pi = self._dev(p_init, torch.float64)
            sd = self._dev(task_side)
            r = torch.empty((self.K,), dtype=torch.float64, device=self.device)
            v = torch.empty_like(r)
            q = torch.empty((self.K,), dtype=torch.int64, device=self.device)
            _check(lib().lob_step_reward(self.ctx, _ptr(a), _ptr(pi), _ptr(sd), float(lam), _ptr(r), _ptr(v),
                                         _ptr(q), st), "lob_step_reward")
        self._keep = (a, pi, sd)
        return r, v, q

    def l2(self, stream=None):
        with _On(self.device, stream) as st:
            out = torch.empty((self.K, self.L, 4), dtype=torch.int32, device=self.device)
            _check(lib().lob_get_l2(self.ctx, _ptr(out), st), "lob_get_l2")
        return out

    def trades(self, stream=None):
        with _On(self.device, stream) as st:
            out = torch.empty((self.K, self.T_cap, 6), dtype=torch.int32, device=self.device)
            cnt = torch.empty((self.K,), dtype=torch.int32, device=self.device)
            _check(lib().lob_get_trades(self.ctx, _ptr(out), _ptr(cnt), st), "lob_get_trades")
        return out, cnt

    def book(self, stream=None):
        with _On(self.device, stream) as st:
            out = torch.empty((self.K, 2, self.N, 6), dtype=torch.int32, device=self.device)
            _check(lib().lob_get_book(self.ctx, _ptr(out), st), "lob_get_book")
        return out

    def stats(self, stream=None):
        with _On(self.device, stream) as st:
            out = torch.empty((self.K, LOB_NSTATS), dtype=torch.int64, device=self.device)
            _check(lib().lob_get_stats(self.ctx, _ptr(out), st), "lob_get_stats")
        return out


    def digest(self, stream=None):
        """[K] per-book FNV-1a-64 of the exported book, trade log, n_trades and counters
        (lob_digest), as int64 bit patterns (torch has no uint64 arithmetic)."""
        with _On(self.device, stream) as st:
            out = torch.empty((self.K,), dtype=torch.int64, device=self.device)
            _check(lib().lob_digest(self.ctx, _ptr(out), st), "lob_digest")
        return out


class LobEnv:
    """Execution environments on the device, one per book of a LobBatch (NEXT row N3):
    lob_env_reset / lob_env_step (Sec.5.1.3 and 5.2)."""

    def __init__(self, batch: LobBatch, config: EnvConfig, msgs_per_step: int):
        self.b, self.cfg, self.M = batch, config, int(msgs_per_step)
        L = lib()
        n = L.lob_env_state_bytes(batch.K)
        self.state = torch.empty(max(int(n), 64), dtype=torch.uint8, device=batch.device)
        self.work = torch.empty((batch.K, 8, 8), dtype=torch.int32, device=batch.device)  # agent messages
        self.reward = torch.empty((batch.K,), dtype=torch.float64, device=batch.device)
        self.done = torch.empty((batch.K,), dtype=torch.int32, device=batch.device)
        self.executed = torch.empty((batch.K,), dtype=torch.int64, device=batch.device)

    def reset(self, init_ts: int, init_tns: int = 0, stream=None):
        with _On(self.b.device, stream) as st:
            _check(lib().lob_env_reset(self.b.ctx, _ptr(self.state), ctypes.byref(self.cfg), int(init_ts),
                                       int(init_tns), st), "lob_env_reset")

    def step(self, actions, data, l2_out=None, stream=None):
        """actions [K][4] f32, data [K][M][8] int32 -> (reward, done, executed) device tensors;
        ``self.work[:, :8]`` holds the agent's messages of the step."""
        with _On(self.b.device, stream) as st:
            a = self.b._dev(actions, torch.float32)
            d = self.b._dev(data)
            assert a.shape == (self.b.K, 4) and d.shape == (self.b.K, self.M, 8)
            _check(lib().lob_env_step(self.b.ctx, _ptr(self.state), ctypes.byref(self.cfg), _ptr(a), _ptr(d),
                                      self.M, _ptr(self.work), _ptr(self.reward), _ptr(self.done),
                                      _ptr(self.executed), _ptr(l2_out), st), "lob_env_step")
        self._keep = (a, d)
        return self.reward, self.done, self.executed


class LobSession:
    """A RESIDENT env session (NEXT row N3, residency; include/lob.h lob_session_*): one
    persistent launch keeps every book of ``env``'s batch on chip for an episode whose
    data messages ``data`` [K][n_steps][M][8] (or [K][n_steps*M][8]) are given up front;
    each ``step(actions)`` runs what one ``LobEnv.step`` runs, without reloading or
    storing a book.  Outputs are ``env``'s buffers (``env.reward``, ``env.done``,
    ``env.executed``, ``env.work``) and ``self.l2`` [K][L][4], overwritten every step and
    complete on the stream after ``step`` returns.  ``end()`` writes books and counters
    back.  Other calls on the batch while the session runs are not allowed, and so is a
    DEVICE-wide synchronize (``torch.cuda.synchronize()``): it would wait for the resident
    kernel, which waits for the next step -- synchronise the stream instead."""

    def __init__(self, env: LobEnv, data, n_steps: int, l2: bool = True, stream=None):
        self.env, self.b, self.n_steps = env, env.b, int(n_steps)
        b = self.b
        with _On(b.device, stream) as st:
            d = b._dev(data)
            assert d.numel() == b.K * self.n_steps * env.M * 8, d.shape
            self.data = d.reshape(b.K, self.n_steps * env.M, 8)
            self.actions = torch.zeros((b.K, 4), dtype=torch.float32, device=b.device)
            self.l2 = torch.empty((b.K, b.L, 4), dtype=torch.int32, device=b.device) if l2 else None
            _check(lib().lob_session_begin(b.ctx, _ptr(env.state), ctypes.byref(env.cfg), _ptr(self.actions),
                                           _ptr(self.data), self.n_steps, env.M, _ptr(env.work),
                                           _ptr(env.reward), _ptr(env.done), _ptr(env.executed), _ptr(self.l2),
                                           st), "lob_session_begin")
        self.active = True

    def step(self, actions=None, stream=None):
        """actions [K][4] f32 -> (reward, done, executed): env's buffers, this step's values.
        ``actions=None``: the caller has already written them into ``self.actions`` on the
        stream (e.g. the policy's output), so nothing is copied."""
        with _On(self.b.device, stream) as st:
            if actions is not None:
                a = torch.as_tensor(actions)
                self.actions.copy_(a.to(device=self.b.device, dtype=torch.float32, non_blocking=True))
            _check(lib().lob_session_step(self.b.ctx, st), "lob_session_step")
        return self.env.reward, self.env.done, self.env.executed

    def end(self, stream=None):
        if self.active:
            with _On(self.b.device, stream) as st:
                _check(lib().lob_session_end(self.b.ctx, st), "lob_session_end")
            self.active = False

