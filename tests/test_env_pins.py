"""NEXT row N3 (execution-env step, Sec.5.1.3 and 5.2) -- oracle pins.

The expected values below are derived by hand from the paper's rules (comments
give each step) on a 2-level initial book; they pin the action -> message mapping
(reading E1-E8), the forced market order, the
reward (eq:rewardfunc), the time update and termination
(P:L423)."""
from __future__ import annotations

import numpy as np
import pytest

import lobgen
import oracle

INIT = np.array([[[1010, 5, 990, 5], [1020, 5, 980, 5]]], np.int32)   # asks OIDs -9000/-9001, bids -9002/-9003
BASE = 1_000_000


def cfg(episode_s=600, side=-1, size=10, lam=1.0):
    return oracle.EnvConfig(task_side=side, task_size=size, n_passive=2, tick=10, episode_s=episode_s,
                            agent_tid=77, oid_base=BASE, pad=0, lam=lam)


def make(episode_s=600, **kw):
    b = oracle.OracleBatch(1, 8, 16, 2)
    b.init(INIT, 34200, 0)
    e = oracle.OracleEnv(b, cfg(episode_s, **kw))
    e.reset(34200, 0)
    return b, e


DATA1 = np.array([[[1, 1, 3, 1005, 5, 9, 34201, 0]]], np.int32)        # a data buy 3 @ 1005 at t = 34201 s
NONE = np.zeros((1, 1, 8), np.int32)


def test_step1_action_mapping_trades_reward():
    b, e = make()
    st = e.state()[0]
    assert st[13] == np.float64(1000.0).view(np.int64)                   # P_init = (1010 + 990) / 2
    # sizes rint half-even: 2.4 -> 2, 1.6 -> 2, 3.5 -> 4, 0.5 -> 0 (E2)
    r, dn, ex, am = e.step([[2.4, 1.6, 3.5, 0.5]], DATA1, 1)
    # sell task: far touch = best bid 990, mid = (1010+990)/2 = 1000, near touch = best ask 1010
    np.testing.assert_array_equal(am[0, :3], [[1, -1, 2, 990, BASE, 77, 34200, 0],
                                              [1, -1, 2, 1000, BASE + 1, 77, 34200, 0],
                                              [1, -1, 4, 1010, BASE + 2, 77, 34200, 0]])
    assert (am[0, 3:] == 0).all()
    tr, cnt = b.trades()
    # the far-touch sell fills 2 @ 990 against bid -9002; the data buy takes the agent's 2 @ 1000
    assert tr[0, :cnt[0]].tolist() == [[990, 2, BASE, -9002, 34200, 0], [1000, 2, 5, BASE + 1, 34201, 0]]
    # VWAP = (1980 + 2000) / 4 = 995; R = 2(990-995) + 2(1000-995) + 1*4*(995-1000) = -20
    assert r[0] == -20.0 and ex[0] == 4 and dn[0] == 0
    st = e.state()[0]
    assert st[3:5].tolist() == [34201, 0]                                 # time := last data message
    assert st[9:13].tolist() == [BASE, BASE + 1, BASE + 2, 0]             # orders to cancel next step (E1)
    book = b.book()[0]
    assert book[0, 3].tolist() == [1010, 4, BASE + 2, 77, 34200, 0]       # near-touch order rests


def test_step2_cancel_all_and_idle_action():
    b, e = make()
    e.step([[2.4, 1.6, 3.5, 0.5]], DATA1, 1)
    r, dn, ex, am = e.step([[0, 0, 0, 0]], NONE, 1)
    # cancel-all: the three orders of step 1 (two already filled -> unknown cancels)
    assert am[0, :3, 0].tolist() == [3, 3, 3] and am[0, :3, 4].tolist() == [BASE, BASE + 1, BASE + 2]
    assert am[0, :3, 2].tolist() == [2**31 - 1] * 3 and (am[0, 3:] == 0).all()
    assert r[0] == 0.0 and ex[0] == 4 and dn[0] == 0                      # no trades in the step (G31)
    st = b.stats()[0]
    assert st[6] == 2                                                    # unknown_cancels
    assert (b.book()[0, 0, :, 1] > 0).sum() == 2                          # only the two synthetic asks rest


def test_forced_market_order_and_completion():
    # episode of 61 s: after step 1 the time is 34201 s, 1 s >= 61 - 60 -> forced market order
    b, e = make(episode_s=61)
    e.step([[2.4, 1.6, 3.5, 0.5]], DATA1, 1)
    r, dn, ex, am = e.step([[9, 9, 9, 9]], NONE, 1)
    assert am[0, 3].tolist() == [4, -1, 6, 0, BASE + 3, 77, 34201, 0]     # remaining 10 - 4 = 6, limits replaced
    tr, cnt = b.trades()
    assert tr[0, :cnt[0]].tolist() == [[1005, 1, BASE + 3, 5, 34201, 0], [990, 3, BASE + 3, -9002, 34201, 0],
                                       [980, 2, BASE + 3, -9003, 34201, 0]]
    # all three trades are the agent's: advantage sums to ~0; drift = 6 (5935/6 - 1000) = -65
    assert abs(r[0] - (-65.0)) < 1e-9 and ex[0] == 10 and dn[0] == 1       # task complete
    # a finished env is idle: no agent messages, padding only -- the book does not change (E8)
    before = b.book().copy()
    r, dn, ex, am = e.step([[5, 5, 5, 5]], DATA1, 1)
    assert (am == 0).all() and r[0] == 0.0 and dn[0] == 1 and ex[0] == 10
    np.testing.assert_array_equal(b.book(), before)


def test_time_termination_and_buy_side():
    # buy task: far = best ask 1010, mid rounds DOWN to the tick (E5), passive = bid - 2 ticks
    b, e = make(episode_s=600, side=1, size=3)
    r, dn, ex, am = e.step([[0, 1, 0, 1]], np.array([[[2, -1, 1, 1010, 424242, 0, 34800, 1]]], np.int32), 1)
    np.testing.assert_array_equal(am[0, :2], [[1, 1, 1, 1000, BASE, 77, 34200, 0],
                                              [1, 1, 1, 970, BASE + 1, 77, 34200, 0]])
    # time 34800.000000001 - 34200 = 600 s + 1 ns > 600 s -> done (strict)
    assert dn[0] == 1 and ex[0] == 0


def test_caps_and_rounding_properties():
    cfg_ = lobgen.CONFIGS["C2"].with_(n_books=64, n_steps=5)
    msgs, init = lobgen.generate(cfg_)
    b = oracle.OracleBatch(64, 100, 1000, 10)
    b.init(init, lobgen.INIT_TS, lobgen.INIT_TNS)
    e = oracle.OracleEnv(b, oracle.EnvConfig(-1, 2000, 2, 100, 1800, 77, BASE, 0, 0.5))
    e.reset(lobgen.INIT_TS, lobgen.INIT_TNS)
    rng = np.random.default_rng(1)
    for s in range(5):
        acts = rng.uniform(-200, 900, (64, 4)).astype(np.float32)
        acts[rng.random((64, 4)) < 0.05] = np.nan
        r, dn, ex, am = e.step(acts, msgs[:, s * 100:(s + 1) * 100], 100)
        lim = am[:, :, 0] == 1
        assert ((am[:, :, 2] * lim).sum(1) <= 2000).all()                  # never more than the task (E3)
        assert (ex <= 2000).all() and np.isfinite(r).all()              # fills never exceed the task
    assert (e.state()[:, 5] > BASE).any()
