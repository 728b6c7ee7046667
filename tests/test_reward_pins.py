"""NEXT row N2 (step reward epilogue) -- oracle pins (-m "not gpu").

The oracle's double-precision reward is pinned by hand-derived values
(tests/golden/reward_examples.json) and by an exact rational recomputation of
eq:rewardfunc / eq:vwap (fractions.Fraction) on random steps: the double result
must be within 1e-12 of the exact value relative to the magnitude of its terms."""
from __future__ import annotations

import json
import os
from fractions import Fraction

import numpy as np
import pytest

import lobgen
import oracle

HERE = os.path.dirname(os.path.abspath(__file__))
DOC = json.load(open(os.path.join(HERE, "golden", "reward_examples.json")))


def _run_fixture(make):
    eng = make(1, DOC["capacity"], DOC["trades_cap"], DOC["l2_levels"])
    eng.init(None, 0, 0)
    m = np.asarray(DOC["messages"], np.int32)[None]
    eng.process(m, 1, m.shape[1])
    tr, cnt = eng.trades()
    assert tr[0, :cnt[0]].tolist() == DOC["expect_trades"]
    return eng


@pytest.mark.parametrize("i", range(len(DOC["cases"])))
def test_reward_golden(i):
    c = DOC["cases"][i]
    eng = _run_fixture(lambda K, N, T, L: oracle.OracleBatch(K, N, T, L))
    r, v, q = eng.step_reward([c["agent"]], [c["p_init"]], [c["side"]], c["lambda"])
    assert r[0] == c["reward"] and v[0] == c["vwap"] and q[0] == c["agent_qty"]


def exact_reward(trades, lo, hi, p_init, side, lam):
    """eq:rewardfunc and eq:vwap in exact rational arithmetic."""
    sq = sum(Fraction(int(t[1])) for t in trades)
    if sq == 0:
        return Fraction(0), Fraction(0), 0, Fraction(0)
    vwap = sum(Fraction(int(t[1])) * int(t[0]) for t in trades) / sq
    mine = [t for t in trades if lo <= t[2] <= hi or lo <= t[3] <= hi]
    p0 = Fraction(p_init)
    adv = sum(Fraction(int(t[1])) * (int(t[0]) - vwap) for t in mine)
    drift = sum(Fraction(int(t[1])) * (vwap - p0) for t in mine)
    r = adv + Fraction(lam) * drift
    scale = sum(Fraction(int(t[1])) * (abs(int(t[0])) + abs(vwap)) for t in mine) + \
        abs(Fraction(lam)) * sum(Fraction(int(t[1])) * (abs(vwap) + abs(p0)) for t in mine)
    return (-r if side == 1 else r), vwap, sum(int(t[1]) for t in mine), scale


def test_reward_matches_exact_rational():
    cfg = lobgen.CONFIGS["C3"].with_(n_books=64, n_steps=2, msgs_per_step=100)
    msgs, init = lobgen.generate(cfg)
    o = oracle.OracleBatch(64, cfg.capacity, cfg.trades_cap, cfg.l2_levels)
    o.init(init, lobgen.INIT_TS, lobgen.INIT_TNS)
    o.process(msgs, cfg.n_steps, cfg.msgs_per_step)
    tr, cnt = o.trades()
    rng = np.random.default_rng(3)
    lo = rng.integers(1, 150, 64).astype(np.int32)
    agent = np.stack([lo, lo + rng.integers(0, 60, 64).astype(np.int32)], 1)
    p_init = rng.uniform(9.9e5, 1.01e6, 64)
    side = rng.choice([-1, 1], 64).astype(np.int32)
    for lam in (0.0, 1.0, 0.37):
        r, v, q = o.step_reward(agent, p_init, side, lam)
        for k in range(64):
            er, ev, eq, scale = exact_reward(tr[k, :cnt[k]], agent[k, 0], agent[k, 1], p_init[k], side[k], lam)
            assert q[k] == eq
            assert abs(Fraction(v[k]) - ev) <= Fraction(1, 10**12) * max(abs(ev), 1)
            assert abs(Fraction(r[k]) - er) <= Fraction(1, 10**12) * max(scale, 1), (k, lam)


def test_reward_homogeneous_and_zero_cases():
    """Scaling every price and P_init by c scales R by c (homogeneity of eq:rewardfunc);
    lambda = 0 and all trades at one price gives R = 0."""
    base = np.asarray(DOC["messages"], np.int32)
    outs = []
    for c in (1, 7):
        m = base.copy()
        m[:, 3] *= c
        o = oracle.OracleBatch(1, 8, 8, 1)
        o.process(m[None], 1, m.shape[0])
        outs.append(o.step_reward([[500, 599]], [100.0 * c], [-1], 1.0)[0][0])
    assert outs[1] == 7 * outs[0]
    same = np.array([[1, 1, 5, 100, 1, 0, 1, 0], [4, -1, 3, 0, 9, 0, 2, 0], [4, -1, 2, 0, 10, 0, 3, 0]], np.int32)
    o = oracle.OracleBatch(1, 8, 8, 1)
    o.process(same[None], 1, 3)
    assert o.step_reward([[9, 9]], [90.0], [-1], 0.0)[0][0] == 0.0
