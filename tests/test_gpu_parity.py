"""GPU parity (-m gpu): the CUDA path, called through the C ABI, must equal the CPU
oracle element by element (bit-exact: every output is integer) on the same
seeded inputs."""
from __future__ import annotations

import numpy as np
import pytest
import torch

import lobgen
import oracle
from common import (SATURATE_N, STAT_NAMES, assert_outputs_equal, golden_cases, run_engine, run_golden_case,
                    saturate_cfg)

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    from gpu_engine import GpuEngine, make_gpu


def _both(cfg, n_books=None, calls=1, book_begin=0, threads=8):
    cfg = cfg if n_books is None else cfg.with_(n_books=n_books)
    msgs, init = lobgen.generate(cfg, book_begin=book_begin)
    g = run_engine(GpuEngine(cfg.n_books, cfg.capacity, cfg.trades_cap, cfg.l2_levels), cfg, msgs, init,
                   lobgen.INIT_TS, lobgen.INIT_TNS, calls)
    o = run_engine(oracle.OracleBatch(cfg.n_books, cfg.capacity, cfg.trades_cap, cfg.l2_levels, threads=threads),
                   cfg, msgs, init, lobgen.INIT_TS, lobgen.INIT_TNS, calls)
    return g, o


@pytest.mark.parametrize("cid,case", golden_cases(), ids=[c[0] for c in golden_cases()])
def test_golden_on_gpu(cid, case):
    run_golden_case(make_gpu, case)


def test_c1_full():
    g, o = _both(lobgen.CONFIGS["C1"])
    assert_outputs_equal(g, o, what="C1")


@pytest.mark.parametrize("calls", [1, 100])
def test_c2_modes(calls):
    # C2 at full size: mode B (one call of 100 steps) and mode A (one call per step)
    g, o = _both(lobgen.CONFIGS["C2"], calls=calls)
    assert_outputs_equal(g, o, what=f"C2 calls={calls}")


@pytest.mark.parametrize("name,n", [("C3", 1000), ("C4", 1500), ("C5_32", 700), ("C5_100", 700),
                                    ("C5_512", 150), ("C5_2048", 20)])
def test_configs_subset(name, n):
    # several persistent-grid waves' worth of books plus a ragged tail
    g, o = _both(lobgen.CONFIGS[name], n_books=n)
    assert_outputs_equal(g, o, what=name)


@pytest.mark.parametrize("profile,N", [("ties", 100), ("overflow", 16), ("synthetic", 100),
                                       ("garbage", 100), ("heavy_market", 64), ("lobster", 1),
                                       ("lobster", 33), ("lobster", 97), ("overflow", 130),
                                       ("garbage", 300), ("ties", 1024), ("garbage", 1024),
                                       ("garbage", 2000), ("synthetic", 1500)])
def test_profiles(profile, N):
    cfg = lobgen.Config("p", 333, N, 7, 37, min(N, 12), 50, 10, profile, 21 + N)
    g, o = _both(cfg)
    assert_outputs_equal(g, o, what=f"{profile} N={N}")


@pytest.mark.parametrize("N", [31, 32, 33, 64, 65, 96, 128, 129, 256, 257, 512, 513, 1024, 1025, 2047, 2048])
def test_geometry_boundaries(N):
    # every (rows per thread, warps per book) geometry and both sides of each boundary
    # (lob_api.cu geo_of: KPL = 1/2/3/4/8 with one warp, then 2/4/8 warps of 8 rows)
    for profile in ("ties", "overflow"):
        cfg = lobgen.Config("geo", 45, N, 4, 60, min(N, 10), 40, 10, profile, 7 * N + len(profile))
        g, o = _both(cfg)
        assert_outputs_equal(g, o, what=f"{profile} N={N}")


@pytest.mark.parametrize("profile,N,calls", [("ties", 100, 1), ("overflow", 100, 1), ("synthetic", 100, 3),
                                             ("garbage", 128, 1), ("heavy_market", 97, 2), ("cancel_heavy", 100, 7),
                                             ("lobster", 120, 1)])
def test_wide_build_row_bounds(monkeypatch, profile, N, calls):
    # the many-wave build (MODE 3: row-bounded scans, Engine::with_rows) forced on a
    # small batch of 4-row books: overflowing, tied, malformed and sweeping streams
    # move the row high-water mark up to the last (partial) row and back down
    monkeypatch.setenv("LOB_FORCE_WIDE", "1")
    cfg = lobgen.Config("w", 700, N, 8, 40, min(N, 40), 64, 10, profile, 3 * N + calls)
    g, o = _both(cfg, calls=calls)
    assert_outputs_equal(g, o, what=f"wide {profile} N={N} calls={calls}")


@pytest.mark.parametrize("N,cap,wide,calls", [(100, 1, False, 1), (100, 3, True, 4), (33, 2, False, 2),
                                             (200, 5, False, 1), (512, 3, False, 2), (1024, 2, False, 1)])
def test_dynamic_scheduling_small_grid(monkeypatch, N, cap, wide, calls):
    # LOB_GRID_CAP caps the persistent grid, so a few hundred books run through the
    # dynamic book scheduler (atomic claim + shared-word hand-off, counter re-arm
    # between launches) in every geometry and in the many-wave build
    monkeypatch.setenv("LOB_GRID_CAP", str(cap))
    if wide:
        monkeypatch.setenv("LOB_FORCE_WIDE", "1")
    K = 150 if N >= 512 else 400
    cfg = lobgen.Config("dyn", K, N, 4, 30, min(N, 20), 32, 10, "heavy_market" if N < 512 else "lobster", N + cap)
    g, o = _both(cfg, calls=calls)
    assert_outputs_equal(g, o, what=f"dyn N={N} cap={cap} wide={wide} calls={calls}")


@pytest.mark.parametrize("split", [0, 1])
@pytest.mark.parametrize("profile,N,Tcap,calls", [("heavy_market", 100, 1024, 1), ("heavy_market", 32, 5, 3),
                                                  ("lobster", 100, 100, 1), ("ties", 64, 1024, 2),
                                                  ("garbage", 256, 200, 1), ("synthetic", 512, 1024, 1),
                                                  ("overflow", 16, 1024, 4), ("cancel_heavy", 97, 0, 1),
                                                  ("saturate", 130, 1024, 1), ("heavy_market", 1, 1024, 1)])
def test_side_split_build(monkeypatch, split, profile, N, Tcap, calls):
    # the side-split build (lob_split.cuh: one warp per side, ring hand-off of Q_a',
    # trade-order waits) forced on (LOB_SPLIT_BPS large: also several waves of warp pairs)
    # and off (0: lob_step on a small batch); deep sweeps with every trade logged
    # (Tcap >= fills: the trade-order wait on every fill), tiny and empty logs, ties,
    # malformed messages, synthetic cancels, saturated sides, one-slot books
    monkeypatch.setenv("LOB_SPLIT_BPS", "100000" if split else "0")
    monkeypatch.setenv("LOB_SPLIT_MIN_MSGS", "0")
    K = 1900 if split and N <= 128 else 300
    cfg = lobgen.Config("s", K, N, 6, 64, min(N, 30), Tcap, 10, profile, 11 * N + Tcap + calls)
    g, o = _both(cfg, calls=calls)
    assert_outputs_equal(g, o, what=f"split={split} {profile} N={N} Tcap={Tcap} calls={calls}")


@pytest.mark.parametrize("M,steps,L", [(37, 9, 10), (1, 70, 3), (200, 3, 32), (33, 4, 1)])
def test_side_split_ragged_steps(monkeypatch, M, steps, L):
    # step ends in the middle of a staging chunk, one-message steps, steps spanning several
    # chunks, a ragged last chunk: the per-side L2 snapshots and the chunk-granular
    # progress / window logic of the side-split build
    monkeypatch.setenv("LOB_SPLIT_BPS", "100000")
    monkeypatch.setenv("LOB_SPLIT_MIN_MSGS", "0")
    cfg = lobgen.Config("sr", 257, 100, steps, M, 20, 512, L, "heavy_market", 7 * M + steps)
    g, o = _both(cfg)
    assert_outputs_equal(g, o, what=f"split ragged M={M} steps={steps} L={L}")


@pytest.mark.parametrize("L,Tcap", [(1, 0), (32, 3), (10, 1)])
def test_levels_and_tiny_trade_log(L, Tcap):
    cfg = lobgen.Config("p", 200, 100, 5, 50, 40, Tcap, L, "heavy_market", 5)
    g, o = _both(cfg)
    assert_outputs_equal(g, o, what=f"L={L} Tcap={Tcap}")


def test_empty_and_degenerate_calls():
    cfg = lobgen.Config("p", 65, 50, 3, 20, 5, 20, 5, "lobster", 8)
    msgs, init = lobgen.generate(cfg)
    for eng in (GpuEngine(65, 50, 20, 5), oracle.OracleBatch(65, 50, 20, 5)):
        eng.init(init, 1, 2)
        eng.process(msgs, 3, 20)
        eng.process(msgs[:, :0], 0, 20)          # no messages: clears the trade log only
    g, o = GpuEngine(65, 50, 20, 5), oracle.OracleBatch(65, 50, 20, 5)
    for eng in (g, o):
        eng.init(init, 1, 2)
        eng.process(msgs, 3, 20)
        eng.process(msgs[:, :0], 0, 20)
    np.testing.assert_array_equal(g.book(), o.book())
    np.testing.assert_array_equal(g.trades()[1], o.trades()[1])
    np.testing.assert_array_equal(g.trades()[0], o.trades()[0])
    np.testing.assert_array_equal(g.stats(), o.stats())
    # zero books
    z = GpuEngine(0, 100, 10, 10)
    z.init(None)
    z.process(np.zeros((0, 10, 8), np.int32), 1, 10)
    assert z.book().shape == (0, 2, 100, 6)


def test_determinism_clones_and_isolation():
    cfg = lobgen.CONFIGS["C1"]
    msgs, init = lobgen.generate(cfg.with_(n_books=4))
    K = 1000
    e = GpuEngine(K, 100, 1000, 10)
    e.init(np.repeat(init[:1], K, 0), lobgen.INIT_TS, lobgen.INIT_TNS)
    l2 = e.process(np.repeat(msgs[:1], K, 0), 10, 100)
    assert (l2 == l2[:1]).all() and (e.book() == e.book()[:1]).all()
    st = e.stats()
    assert (st == st[:1]).all()


@pytest.mark.parametrize("K", [300, 6000])
def test_cuda_graph_mode_a(K):
    # C2's RL shape, one call per step, captured once in a CUDA graph and replayed:
    # one wave of books (K = 300) and dynamic scheduling across waves (K = 6000)
    from paper_2308_13289_b200 import LobBatch
    cfg = lobgen.CONFIGS["C2"].with_(n_books=K, n_steps=6)
    msgs, init = lobgen.generate(cfg)
    M, L = cfg.msgs_per_step, cfg.l2_levels
    b = LobBatch(K, cfg.capacity, cfg.trades_cap, L)
    steps = [torch.from_numpy(np.ascontiguousarray(msgs[:, s * M:(s + 1) * M])).cuda() for s in range(cfg.n_steps)]
    ti = torch.from_numpy(init).cuda()
    l2 = torch.empty((cfg.n_steps, K, 1, L, 4), dtype=torch.int32, device="cuda")
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):  # warm-up outside capture
        b.init(ti, lobgen.INIT_TS, lobgen.INIT_TNS)
        b.process(steps[0], 1, M, l2_out=l2[0])
    torch.cuda.current_stream().wait_stream(side)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        b.init(ti, lobgen.INIT_TS, lobgen.INIT_TNS)
        for s in range(cfg.n_steps):
            b.process(steps[s], 1, M, l2_out=l2[s])
    for _ in range(2):  # replays are independent episodes from the same initial state
        l2.fill_(7)
        g.replay()
        torch.cuda.synchronize()
    o = oracle.OracleBatch(K, cfg.capacity, cfg.trades_cap, L, threads=8)
    want = run_engine(o, cfg, msgs, init, lobgen.INIT_TS, lobgen.INIT_TNS, calls=cfg.n_steps)
    np.testing.assert_array_equal(l2[:, :, 0].permute(1, 0, 2, 3).cpu().numpy(), want["l2"])
    np.testing.assert_array_equal(b.book().cpu().numpy(), want["book"])
    np.testing.assert_array_equal(b.stats().cpu().numpy(), want["stats"])
    tr, cnt = b.trades()
    np.testing.assert_array_equal(cnt.cpu().numpy(), want["n_trades"])
    np.testing.assert_array_equal(tr.cpu().numpy(), want["trades"])


def _host_buffers(cfg):
    K, S, L = cfg.n_books, cfg.n_steps, cfg.l2_levels
    pin = lambda shape, dt: torch.empty(shape, dtype=dt).pin_memory()
    return {"l2": pin((K, S, L, 4), torch.int32), "st": pin((K, 10), torch.int64),
            "tr": pin((K * cfg.trades_cap, 6), torch.int32), "cnt": pin((K,), torch.int32)}


def _check_host_outputs(h, a, l2a):
    """Host outputs of lob_process_messages_host against the device path `a`."""
    assert torch.equal(h["l2"], l2a.cpu())
    assert torch.equal(h["st"], a.stats().cpu())
    tr, cnt = a.trades()
    cnt = cnt.cpu()
    assert torch.equal(h["cnt"], cnt)
    n = int(cnt.sum())
    mask = torch.arange(tr.shape[1])[None, :] < cnt[:, None]          # logged rows, book order
    assert torch.equal(h["tr"][:n], tr.cpu()[mask])


@pytest.mark.parametrize("name,n,chunks,Tcap", [("C4", 3000, 5, None), ("C3", 1200, 3, None),
                                                ("C3", 700, 1, 2), ("C5_512", 150, 4, None),
                                                ("C4", 4500, None, None), ("C4", 2000, 64, None)])
def test_host_path_equals_device_path(name, n, chunks, Tcap):
    """The end-to-end call (pinned host buffers in and out, chunked copy/compute pipeline)
    returns exactly what the device path produces: per-step L2, counters, and every
    logged trade row packed book after book with its per-book count (Eq.3-4)."""
    cfg = lobgen.CONFIGS[name].with_(n_books=n)
    if Tcap is not None:
        cfg = cfg.with_(trades_cap=Tcap)
    msgs, init = lobgen.generate(cfg)
    from paper_2308_13289_b200 import LobBatch
    a = LobBatch(cfg.n_books, cfg.capacity, cfg.trades_cap, cfg.l2_levels)
    b = LobBatch(cfg.n_books, cfg.capacity, cfg.trades_cap, cfg.l2_levels)
    ti = torch.from_numpy(init)
    a.init(ti, lobgen.INIT_TS, lobgen.INIT_TNS)
    b.init(ti, lobgen.INIT_TS, lobgen.INIT_TNS)
    l2a = a.process(torch.from_numpy(msgs), cfg.n_steps, cfg.msgs_per_step)
    hm = torch.from_numpy(msgs).pin_memory()
    h = _host_buffers(cfg)
    h["tr"].fill_(-7)
    dm = torch.empty_like(hm, device="cuda")
    dl = torch.empty_like(h["l2"], device="cuda")
    b.process_host(hm, cfg.n_steps, cfg.msgs_per_step, h["l2"], h["st"], dm, dl, chunks=chunks,
                   h_trades_out=h["tr"], h_trade_counts_out=h["cnt"])
    torch.cuda.synchronize()
    _check_host_outputs(h, a, l2a)
    assert (h["tr"][int(h["cnt"].sum()):] == -7).all()            # nothing past the packed rows
    assert torch.equal(b.book(), a.book())
    # a second call continues the books (counters accumulate, the trade log is per call)
    l2a = a.process(torch.from_numpy(msgs), cfg.n_steps, cfg.msgs_per_step)
    b.process_host(hm, cfg.n_steps, cfg.msgs_per_step, h["l2"], h["st"], dm, dl, chunks=chunks,
                   h_trades_out=h["tr"], h_trade_counts_out=h["cnt"])
    torch.cuda.synchronize()
    _check_host_outputs(h, a, l2a)


def test_host_path_in_cuda_graph():
    """lob_init + lob_process_messages_host captured once into a CUDA graph (the context's
    copy streams fork from and join back to the capturing stream) and replayed: every
    replay returns the device path's outputs in the host buffers."""
    cfg = lobgen.CONFIGS["C4"].with_(n_books=2000)
    msgs, init = lobgen.generate(cfg)
    from paper_2308_13289_b200 import LobBatch
    a = LobBatch(cfg.n_books, cfg.capacity, cfg.trades_cap, cfg.l2_levels)
    a.init(torch.from_numpy(init), lobgen.INIT_TS, lobgen.INIT_TNS)
    l2a = a.process(torch.from_numpy(msgs), cfg.n_steps, cfg.msgs_per_step)
    b = LobBatch(cfg.n_books, cfg.capacity, cfg.trades_cap, cfg.l2_levels)
    hm = torch.from_numpy(msgs).pin_memory()
    ti = torch.from_numpy(init).cuda()
    h = _host_buffers(cfg)
    dm = torch.empty_like(hm, device="cuda")
    dl = torch.empty_like(h["l2"], device="cuda")

    def run():
        b.init(ti, lobgen.INIT_TS, lobgen.INIT_TNS)
        b.process_host(hm, cfg.n_steps, cfg.msgs_per_step, h["l2"], h["st"], dm, dl, chunks=4,
                       h_trades_out=h["tr"], h_trade_counts_out=h["cnt"])

    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        run()
    torch.cuda.current_stream().wait_stream(side)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        run()
    for _ in range(2):
        for t in h.values():
            t.fill_(-5)
        g.replay()
        torch.cuda.synchronize()
        _check_host_outputs(h, a, l2a)


def test_host_trades_need_pinned_memory():
    from paper_2308_13289_b200 import LobBatch, lib
    import ctypes
    cfg = lobgen.CONFIGS["C1"].with_(n_books=4)
    msgs, init = lobgen.generate(cfg)
    b = LobBatch(4, 100, cfg.trades_cap, 10)
    b.init(torch.from_numpy(init), lobgen.INIT_TS, lobgen.INIT_TNS)
    hm = torch.from_numpy(msgs).pin_memory()
    dm = torch.empty_like(hm, device="cuda")
    pageable = torch.empty((4 * cfg.trades_cap, 6), dtype=torch.int32)
    cnt = torch.empty((4,), dtype=torch.int32).pin_memory()
    rc = lib().lob_process_messages_host(b.ctx, ctypes.c_void_p(hm.data_ptr()), 10, 100, None, None,
                                         ctypes.c_void_p(pageable.data_ptr()), ctypes.c_void_p(cnt.data_ptr()),
                                         ctypes.c_void_p(dm.data_ptr()), None, 2,
                                         ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
    assert rc == -1 and b"pinned" in lib().lob_last_error()


def test_env_rejects_agent_oid_base_zero():
    from paper_2308_13289_b200 import EnvConfig, LobBatch, LobEnv, LobError
    b = LobBatch(2, 16, 16, 2)
    b.init(None, 0, 0)
    env = LobEnv(b, EnvConfig(task_side=-1, task_size=10, n_passive=1, tick=10, episode_s=60, agent_tid=1,
                              agent_oid_base=0, reserved=0, lam=0.0), 1)
    with pytest.raises(LobError):
        env.reset(34200, 0)


@pytest.mark.parametrize("name", ["C4", "C3", "C2", "C5_32", "C5_100", "C5_256", "C5_512", "C5_1024", "C5_2048"])
def test_full_size_sampled_books(name):
    """Every BASELINE.json config at its full size (C4: 65,536 books, the launch
    configuration bench.py times; C3: 16,384; C5: 4,096 at each capacity), sampled
    books recomputed one by one by the oracle."""
    cfg = lobgen.CONFIGS[name]
    msgs, init = lobgen.generate(cfg)
    e = GpuEngine(cfg.n_books, cfg.capacity, cfg.trades_cap, cfg.l2_levels)
    g = run_engine(e, cfg, msgs, init, lobgen.INIT_TS, lobgen.INIT_TNS)
    rng = np.random.default_rng(0)
    sample = np.unique(np.concatenate([[0, 1, cfg.n_books - 1], rng.integers(0, cfg.n_books, 61)]))
    o = oracle.OracleBatch(len(sample), cfg.capacity, cfg.trades_cap, cfg.l2_levels)
    want = run_engine(o, cfg, np.ascontiguousarray(msgs[sample]), np.ascontiguousarray(init[sample]),
                      lobgen.INIT_TS, lobgen.INIT_TNS)
    got = {k: v[sample] for k, v in g.items()}
    assert_outputs_equal(got, want, what=f"{name} full-size sample")
    from digest import state_digest
    dg = e.b.digest().cpu().numpy().view(np.uint64)
    np.testing.assert_array_equal(dg[sample], state_digest(want["book"], want["trades"], want["n_trades"],
                                                           want["stats"]))
    # properties that hold at any size, on every book
    st = g["stats"]
    assert (st[:, STAT_NAMES.index("msgs")] == cfg.n_msgs).all()
    assert (st[:, STAT_NAMES.index("trades")] == g["n_trades"] + st[:, STAT_NAMES.index("trades_dropped")]).all()
    l2 = g["l2"]
    both = (l2[..., 0] > 0) & (l2[..., 2] > 0)
    assert (l2[..., 0, 0][both[..., 0]] > l2[..., 0, 2][both[..., 0]]).all()  # never crossed


# ------------------------------------------- lob_digest (SURVEY.md 8(e) full-state fingerprint)
@pytest.mark.parametrize("name,n,profile,Tcap", [("C2", 60, None, None), ("C5_2048", 6, None, None),
                                                 ("C5_32", 300, "overflow", 3), ("C1", 1, "garbage", 0)])
def test_digest_matches_oracle_state(name, n, profile, Tcap):
    from digest import state_digest
    cfg = lobgen.CONFIGS[name].with_(n_books=n)
    if profile:
        cfg = cfg.with_(profile=profile)
    if Tcap is not None:
        cfg = cfg.with_(trades_cap=Tcap)
    msgs, init = lobgen.generate(cfg)
    e = GpuEngine(cfg.n_books, cfg.capacity, cfg.trades_cap, cfg.l2_levels)
    run_engine(e, cfg, msgs, init, lobgen.INIT_TS, lobgen.INIT_TNS)
    got = e.b.digest().cpu().numpy().view(np.uint64)
    o = oracle.OracleBatch(cfg.n_books, cfg.capacity, cfg.trades_cap, cfg.l2_levels, threads=8)
    w = run_engine(o, cfg, msgs, init, lobgen.INIT_TS, lobgen.INIT_TNS)
    want = state_digest(w["book"], w["trades"], w["n_trades"], w["stats"])
    np.testing.assert_array_equal(got, want)
    assert len(np.unique(got)) == cfg.n_books or cfg.n_books == 1   # books differ, so must digests


# ------------------------------------------- NEXT row N1: per-message Level-1 trace
@pytest.mark.parametrize("name,n,profile", [("C4", 700, None), ("C3", 400, None), ("C5_32", 300, None),
                                            ("C5_512", 80, None), ("C5_2048", 12, None),
                                            ("C1", 1, "ties"), ("C1", 1, "garbage"), ("C1", 1, "synthetic"),
                                            ("C5_100", 200, "overflow")])
def test_l1_trace(name, n, profile):
    cfg = lobgen.CONFIGS[name].with_(n_books=n)
    if profile:
        cfg = cfg.with_(profile=profile, n_books=150, capacity=60, init_levels=12)
    msgs, init = lobgen.generate(cfg)
    g = GpuEngine(cfg.n_books, cfg.capacity, cfg.trades_cap, cfg.l2_levels)
    o = oracle.OracleBatch(cfg.n_books, cfg.capacity, cfg.trades_cap, cfg.l2_levels, threads=8)
    res = []
    for e in (g, o):
        e.init(init, lobgen.INIT_TS, lobgen.INIT_TNS)
        l2, l1 = e.process(msgs, cfg.n_steps, cfg.msgs_per_step, l1=True)
        res.append((l2, l1, e.book(), e.stats()))
    for a, b, what in zip(res[0], res[1], ("l2", "l1", "book", "stats")):
        if not np.array_equal(a, b):
            bad = np.argwhere(a != b)
            raise AssertionError(f"{name}/{profile}: {what} differs at {len(bad)} positions, first {bad[:4].tolist()}")


# ------------------------------------------------- NEXT row N2: step reward epilogue
def test_reward_golden_on_gpu():
    from test_reward_pins import DOC, _run_fixture
    eng = _run_fixture(lambda K, N, T, L: GpuEngine(K, N, T, L))
    for c in DOC["cases"]:
        r, v, q = eng.step_reward([c["agent"]], [c["p_init"]], [c["side"]], c["lambda"])
        assert r[0] == c["reward"] and v[0] == c["vwap"] and q[0] == c["agent_qty"], c


@pytest.mark.parametrize("name,n", [("C3", 3000), ("C2", 1000), ("C5_512", 60)])
def test_reward_parity(name, n):
    """P_VWAP and the agent quantity are exact (bit-equal); R within 1e-12 of the
    magnitude of its terms (summation order differs: lane-strided + warp tree)."""
    cfg = lobgen.CONFIGS[name].with_(n_books=n, n_steps=1)
    msgs, init = lobgen.generate(cfg)
    rng = np.random.default_rng(7)
    lo = rng.integers(1, 60, n).astype(np.int32)
    agent = np.stack([lo, lo + rng.integers(0, 40, n).astype(np.int32)], 1)
    p_init = rng.uniform(9.9e5, 1.01e6, n)
    side = rng.choice([-1, 1], n).astype(np.int32)
    g = GpuEngine(n, cfg.capacity, cfg.trades_cap, cfg.l2_levels)
    o = oracle.OracleBatch(n, cfg.capacity, cfg.trades_cap, cfg.l2_levels, threads=8)
    for e in (g, o):
        e.init(init, lobgen.INIT_TS, lobgen.INIT_TNS)
        e.process(msgs, cfg.n_steps, cfg.msgs_per_step)
    tr, cnt = o.trades()
    for lam in (0.0, 1.0, 0.25):
        rg, vg, qg = g.step_reward(agent, p_init, side, lam)
        ro, vo, qo = o.step_reward(agent, p_init, side, lam)
        np.testing.assert_array_equal(vg, vo)
        np.testing.assert_array_equal(qg, qo)
        for k in range(n):
            t = tr[k, :cnt[k]]
            mine = ((t[:, 2] >= agent[k, 0]) & (t[:, 2] <= agent[k, 1])) | \
                   ((t[:, 3] >= agent[k, 0]) & (t[:, 3] <= agent[k, 1]))
            q = t[mine, 1].astype(np.float64)
            scale = (q * (np.abs(t[mine, 0]) + abs(vo[k]))).sum() + abs(lam) * (q * (abs(vo[k]) + p_init[k])).sum()
            assert abs(rg[k] - ro[k]) <= 1e-12 * max(scale, 1.0), (k, lam, rg[k], ro[k])


# ---------------------------------------------- NEXT row N4: LOBSTER files -> engine
def test_lobster_windows_end_to_end(tmp_path):
    """A synthetic LOBSTER day (message + orderbook CSV) is parsed, cut into windows
    (each window one independent book) and replayed on the GPU and the
    oracle: bit-exact."""
    import os
    from paper_2308_13289_b200 import lobster
    cfg = lobgen.CONFIGS["C4"].with_(n_books=1, n_steps=30, msgs_per_step=100)
    msgs, init = lobgen.generate(cfg)
    text = lobster.format_messages(msgs[0])
    mp = os.path.join(tmp_path, "day_message_10.csv")
    open(mp, "w").write(text)
    m, rows, _ = lobster.parse_messages(mp)
    rng = np.random.default_rng(4)
    ob = np.zeros((len(m), 40), np.int64)
    for lv in range(10):
        ob[:, 4 * lv:4 * lv + 4] = [lobgen.REF0 + (lv + 1) * 100, 0, lobgen.REF0 - (lv + 1) * 100, 0]
        ob[:, 4 * lv + 1] = rng.integers(1, 500, len(m))
        ob[:, 4 * lv + 3] = rng.integers(1, 500, len(m))
    obp = os.path.join(tmp_path, "day_orderbook_10.csv")
    np.savetxt(obp, ob, fmt="%d", delimiter=",")
    book = lobster.parse_orderbook(obp, 10)
    w = lobster.build_windows(m, rows, book, window_s=3, msgs_per_step=100, start_s=int(m[0, 6]),
                              end_s=int(m[-1, 6]) + 1)
    K = w.msgs.shape[0]
    assert K >= 2 and w.real_steps.sum() > 0
    g = GpuEngine(K, 100, 512, 10)
    o = oracle.OracleBatch(K, 100, 512, 10)
    res = []
    for e in (g, o):
        e.init(w.init_l2, 34200, 0)
        res.append((e.process(w.msgs, w.n_steps, w.msgs_per_step), e.book(), e.stats()))
    for a, b in zip(*res):
        np.testing.assert_array_equal(a, b)


# ------------------------------------------- NEXT row N3: execution-env step on device
def _env_pair(K, N, cfg_kw, init, Tcap=512, L=10):
    from paper_2308_13289_b200 import EnvConfig, LobEnv
    ge = GpuEngine(K, N, Tcap, L)
    oe = oracle.OracleBatch(K, N, Tcap, L)
    for e in (ge, oe):
        e.init(init, lobgen.INIT_TS, lobgen.INIT_TNS)
    gcfg = EnvConfig(**cfg_kw)
    ocfg = oracle.EnvConfig(cfg_kw["task_side"], cfg_kw["task_size"], cfg_kw["n_passive"], cfg_kw["tick"],
                            cfg_kw["episode_s"], cfg_kw["agent_tid"], cfg_kw["agent_oid_base"], 0, cfg_kw["lam"])
    return ge, oe, gcfg, ocfg, LobEnv


def test_env_golden_on_gpu():
    """The hand-derived N3 traces of tests/test_env_pins.py, on the device."""
    from test_env_pins import BASE, DATA1, INIT, NONE
    kw = dict(task_side=-1, task_size=10, n_passive=2, tick=10, episode_s=61, agent_tid=77,
              agent_oid_base=BASE, reserved=0, lam=1.0)
    from paper_2308_13289_b200 import EnvConfig, LobBatch, LobEnv
    b = LobBatch(1, 8, 16, 2)
    b.init(torch.from_numpy(INIT), 34200, 0)
    env = LobEnv(b, EnvConfig(**kw), 1)
    env.reset(34200, 0)
    r, d, x = env.step(np.array([[2.4, 1.6, 3.5, 0.5]], np.float32), DATA1)
    assert r.item() == -20.0 and x.item() == 4 and d.item() == 0
    np.testing.assert_array_equal(env.work[0, :3].cpu().numpy(), [[1, -1, 2, 990, BASE, 77, 34200, 0],
                                                                  [1, -1, 2, 1000, BASE + 1, 77, 34200, 0],
                                                                  [1, -1, 4, 1010, BASE + 2, 77, 34200, 0]])
    r, d, x = env.step(np.array([[9, 9, 9, 9]], np.float32), NONE)
    assert abs(r.item() + 65.0) < 1e-9 and x.item() == 10 and d.item() == 1
    assert env.work[0, 3].cpu().tolist() == [4, -1, 6, 0, BASE + 3, 77, 34201, 0]


@pytest.mark.parametrize("K,N,side,episode", [(1000, 100, -1, 1800), (500, 100, 1, 40), (64, 512, -1, 600),
                                               (24, 2048, 1, 600)])
def test_env_rollout_parity(K, N, side, episode):
    """Random actions over 12 steps of 100 data messages (the RL shape):
    agent messages, books, executed quantities and done flags bit-exact; rewards within
    1e-12 of the magnitude of their terms."""
    cfg = lobgen.Config("env", K, N, 12, 100, min(N // 3, 33), 512, 10, "lobster", 40 + K)
    msgs, init = lobgen.generate(cfg)
    kw = dict(task_side=side, task_size=3000, n_passive=2, tick=100, episode_s=episode, agent_tid=77,
              agent_oid_base=2_000_000_000, reserved=0, lam=0.5)
    ge, oe, gcfg, ocfg, LobEnv = _env_pair(K, N, kw, init)
    genv = LobEnv(ge.b, gcfg, 100)
    oenv = oracle.OracleEnv(oe, ocfg)
    genv.reset(lobgen.INIT_TS, lobgen.INIT_TNS)
    oenv.reset(lobgen.INIT_TS, lobgen.INIT_TNS)
    rng = np.random.default_rng(K)
    prev = np.zeros(K, np.int64)
    for s in range(cfg.n_steps):
        acts = rng.uniform(-100, 600, (K, 4)).astype(np.float32)
        acts[rng.random((K, 4)) < 0.03] = np.nan
        data = np.ascontiguousarray(msgs[:, s * 100:(s + 1) * 100])
        r, d, x = genv.step(torch.from_numpy(acts), torch.from_numpy(data))
        ro, do, xo, am = oenv.step(acts, data, 100)
        np.testing.assert_array_equal(genv.work[:, :8].cpu().numpy(), am, err_msg=f"agent msgs step {s}")
        np.testing.assert_array_equal(d.cpu().numpy(), do)
        np.testing.assert_array_equal(x.cpu().numpy(), xo)
        rg = r.cpu().numpy()
        # magnitude of eq:rewardfunc's terms: sum_j Q_j (|P_j| + |VWAP|) (1 + lambda), prices < 2e6
        scale = (xo - prev).astype(np.float64) * 4e6 * (1 + kw["lam"])
        prev = xo.copy()
        assert np.all(np.abs(rg - ro) <= 1e-12 * np.maximum(1.0, scale)), (s, np.abs(rg - ro).max())
        np.testing.assert_array_equal(ge.book(), oe.book())
        np.testing.assert_array_equal(ge.stats(), oe.stats())


def test_env_episode_in_cuda_graph():
    """A whole N3 episode (book init, env reset, 10 env steps) captured once in a CUDA
    graph and replayed twice: per-step rewards, done flags, executed quantities and the
    final books equal the oracle's eager rollout (rewards within 1e-12 of their terms)."""
    from paper_2308_13289_b200 import LobBatch
    K, N, S = 800, 100, 10
    cfg = lobgen.Config("env", K, N, S, 100, 33, 512, 10, "lobster", 91)
    msgs, init = lobgen.generate(cfg)
    kw = dict(task_side=1, task_size=2500, n_passive=2, tick=100, episode_s=900, agent_tid=77,
              agent_oid_base=2_000_000_000, reserved=0, lam=0.5)
    _, oe, gcfg, ocfg, LobEnv = _env_pair(K, N, kw, init)
    b = LobBatch(K, N, 512, 10)
    env = LobEnv(b, gcfg, 100)
    rng = np.random.default_rng(5)
    acts = [torch.from_numpy(rng.uniform(-50, 400, (K, 4)).astype(np.float32)).cuda() for _ in range(S)]
    data = [torch.from_numpy(np.ascontiguousarray(msgs[:, s * 100:(s + 1) * 100])).cuda() for s in range(S)]
    ti = torch.from_numpy(init).cuda()
    rew = torch.empty((S, K), dtype=torch.float64, device="cuda")
    dn = torch.empty((S, K), dtype=torch.int32, device="cuda")
    ex = torch.empty((S, K), dtype=torch.int64, device="cuda")

    def episode():
        b.init(ti, lobgen.INIT_TS, lobgen.INIT_TNS)
        env.reset(lobgen.INIT_TS, lobgen.INIT_TNS)
        for s in range(S):
            r, d, x = env.step(acts[s], data[s])
            rew[s].copy_(r)
            dn[s].copy_(d)
            ex[s].copy_(x)

    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        episode()
    torch.cuda.current_stream().wait_stream(side)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        episode()
    for _ in range(2):
        rew.fill_(float("nan"))
        g.replay()
        torch.cuda.synchronize()
    oenv = oracle.OracleEnv(oe, ocfg)
    oenv.reset(lobgen.INIT_TS, lobgen.INIT_TNS)
    prev = np.zeros(K, np.int64)
    for s in range(S):
        ro, do, xo, _ = oenv.step(acts[s].cpu().numpy(), np.ascontiguousarray(msgs[:, s * 100:(s + 1) * 100]), 100)
        np.testing.assert_array_equal(dn[s].cpu().numpy(), do)
        np.testing.assert_array_equal(ex[s].cpu().numpy(), xo)
        scale = (xo - prev).astype(np.float64) * 4e6 * (1 + kw["lam"])
        prev = xo.copy()
        assert np.all(np.abs(rew[s].cpu().numpy() - ro) <= 1e-12 * np.maximum(1.0, scale)), s
    np.testing.assert_array_equal(b.book().cpu().numpy(), oe.book())
    np.testing.assert_array_equal(b.stats().cpu().numpy(), oe.stats())


def _edge_stream(rng, n):
    """Messages at the value boundaries the kernel special-cases: empty sides, market
    orders (P rewritten to 0 / max_int at decode), limits at P = max_int (the empty-ask
    sentinel), Q = max_int, OIDs at -9000 / INT_MIN / INT_MAX, malformed codes."""
    IMAX, IMIN = 2**31 - 1, -2**31
    out = np.zeros((n, 8), np.int32)
    for i in range(n):
        k = rng.integers(0, 12)
        S = int(rng.choice([-1, 1]))
        ts, tns = 34200 + i // 7, int(rng.integers(0, 10**9))
        oid = int(rng.choice([i + 1, i + 1, i + 1, -9000, -9001, IMIN, IMAX, int(rng.integers(1, 40))]))
        if k == 0:
            out[i] = (4, S, int(rng.choice([1, 50, IMAX])), int(rng.integers(-5, 5)), oid, 7, ts, tns)  # market
        elif k == 1:
            out[i] = (1, S, int(rng.integers(1, 300)), IMAX, oid, 7, ts, tns)                           # limit at max_int
        elif k == 2:
            out[i] = (1, S, int(rng.choice([1, IMAX])), int(rng.choice([1, 2, IMAX - 1])), oid, 7, ts, tns)
        elif k in (3, 4):
            out[i] = (int(rng.choice([2, 3])), S, int(rng.choice([1, 10, IMAX])), int(rng.choice([1, IMAX, 100])),
                      int(rng.integers(1, i + 2)) if k == 3 else oid, 7, ts, tns)                         # cancels
        elif k == 5:
            out[i] = (int(rng.integers(-2, 7)), int(rng.integers(-2, 3)), int(rng.integers(-3, 3)),
                      int(rng.integers(-3, 3)), oid, 7, ts, tns)                                           # malformed / padding
        else:
            out[i] = (1, S, int(rng.integers(1, 500)), 1000 + int(rng.integers(-8, 8)) * 10, oid, 7, ts, tns)
    return out


@pytest.mark.parametrize("wide,N,l1", [(False, 100, False), (True, 100, False), (False, 100, True), (False, 7, False),
                                       (True, 128, False), (False, 300, False), (False, 1500, False)])
def test_edge_values_and_empty_sides(monkeypatch, wide, N, l1):
    if wide:
        monkeypatch.setenv("LOB_FORCE_WIDE", "1")
    K, S, M = 64, 6, 25
    rng = np.random.default_rng(N + 7 * wide + 3 * l1)
    msgs = np.stack([_edge_stream(rng, S * M) for _ in range(K)])
    g, o = GpuEngine(K, N, 40, 6), oracle.OracleBatch(K, N, 40, 6)
    res = []
    for e in (g, o):
        e.init(None, 0, 0)
        out = e.process(msgs, S, M, l2=True, l1=l1)
        tr, cnt = e.trades()
        res.append((out, e.book(), tr, cnt, e.stats(), e.l2()))
    for a, b, what in zip(res[0], res[1], ("out", "book", "trades", "n_trades", "stats", "l2_now")):
        if what == "out" and l1:
            np.testing.assert_array_equal(a[0], b[0], err_msg="l2")
            np.testing.assert_array_equal(a[1], b[1], err_msg="l1")
        else:
            np.testing.assert_array_equal(a, b, err_msg=what)
    assert res[0][4][:, STAT_NAMES.index("market_discarded_qty")].sum() > 0
    assert res[0][4][:, STAT_NAMES.index("bad")].sum() > 0


# ------------------------------------- capacity contract (G6) in every padded geometry
# geo_of pads N to NP = 32*W*KPL slots (e.g. N = 130 -> 256); the padding slots are
# empty and must never take an order (common.saturate_cfg: more passive limits than N).
@pytest.mark.parametrize("N", SATURATE_N)
@pytest.mark.parametrize("wide", [False, True])
def test_capacity_saturated(monkeypatch, N, wide):
    if wide and N > 128:
        pytest.skip("the many-wave build exists for 4-row books only")
    if wide:
        monkeypatch.setenv("LOB_FORCE_WIDE", "1")
    cfg = saturate_cfg(N)
    g, o = _both(cfg, calls=2 if cfg.n_steps % 2 == 0 else 1)
    assert_outputs_equal(g, o, what=f"saturate N={N}")
    ov = o["stats"][:, STAT_NAMES.index("add_overflow")]
    assert (ov > 0).mean() >= 0.5, "the stream must overflow most books"
    occ = (o["book"][..., 1] > 0).sum(-1)
    assert (occ <= N).all() and (occ.max() == N)


def _big_qty_stream(rng, n):
    """Limits with quantities up to max_int at a handful of prices (level volumes far past
    2^31), partial cancels and small market orders: the saturating L2 / L1 volume (G20)."""
    out = np.zeros((n, 8), np.int32)
    for i in range(n):
        S = int(rng.choice([-1, 1]))
        ts, tns = 34200 + i, 0
        k = rng.integers(0, 10)
        if k < 7:
            P = 1000 + S * -10 * int(rng.integers(1, 4))          # passive: asks above 1000, bids below
            Q = int(rng.choice([rng.integers(1 << 27, 2**31 - 1), rng.integers(1, 1 << 20)]))
            out[i] = (1, S, Q, P, i + 1, 7, ts, tns)
        elif k < 9:
            out[i] = (2, S, int(rng.integers(1, 1 << 30)), 0, int(rng.integers(1, i + 2)), 7, ts, tns)
        else:
            out[i] = (4, S, int(rng.integers(1, 1 << 29)), 0, i + 1, 7, ts, tns)
    return out


@pytest.mark.parametrize("N,l1,wide", [(100, False, False), (100, True, False), (100, False, True), (7, True, False),
                                       (300, False, False), (300, True, False), (1500, False, False),
                                       (1500, True, False)])
def test_l2_volume_saturation(monkeypatch, N, l1, wide):
    if wide:
        monkeypatch.setenv("LOB_FORCE_WIDE", "1")
    K, S, M = 40, 8, 30
    rng = np.random.default_rng(N + 11 * l1 + 5 * wide)
    msgs = np.stack([_big_qty_stream(rng, S * M) for _ in range(K)])
    g, o = GpuEngine(K, N, 64, 5), oracle.OracleBatch(K, N, 64, 5)
    res = []
    for e in (g, o):
        e.init(None, 0, 0)
        out = e.process(msgs, S, M, l2=True, l1=l1)
        res.append((out, e.book(), e.stats(), e.l2()))
    l2o = res[1][0][0] if l1 else res[1][0]
    assert (l2o[..., 1] == 2**31 - 1).any() and (l2o[..., 3] == 2**31 - 1).any()    # saturated levels occur
    assert (l2o[..., 1] >= 0).all() and (l2o[..., 3] >= 0).all()
    for a, b, what in zip(res[0], res[1], ("out", "book", "stats", "l2_now")):
        if what == "out" and l1:
            np.testing.assert_array_equal(a[0], b[0], err_msg="l2")
            np.testing.assert_array_equal(a[1], b[1], err_msg="l1")
        else:
            np.testing.assert_array_equal(a, b, err_msg=what)
