"""Do the oracle's pins bite?  (-m "not gpu")

Each case below is a plausible one-line bug in oracle/lob_oracle.c -- a dropped
term, a wrong sign or index, a mis-read of the paper.  The test compiles the mutated
copy with gcc, runs the pin battery against it (golden hand traces, the independent
FIFO engine, exhaustive tiny-input brute force, the L2 group-by, the invariant
checker) and requires at least one pin to fail.  The unmutated source must pass the
same battery.  A second test shows the C invariant checker is not vacuous: on
mutants that break an invariant, check mode reports violations."""
from __future__ import annotations

import itertools
import os
import subprocess

import numpy as np
import pytest

import lobgen
import oracle
from common import golden_cases, run_golden_case
from pins.fifo_engine import run_stream
from test_oracle_pins import _alphabet, _compare_with_fifo, _encode

SRC = os.path.join(os.path.dirname(oracle.__file__), "lob_oracle.c")

# (name, paper passage / reading it violates, original text, mutated text)
MUTANTS = [
    ("bid_is_min", "Eq.5 + G1 (best bid = max)",
     "is_ask ? (x[O_P] < y[O_P]) : (x[O_P] > y[O_P])", "is_ask ? (x[O_P] < y[O_P]) : (x[O_P] < y[O_P])"),
    ("highest_slot_tie", "G4 (equal keys: lowest slot)",
     "if (best < 0 || better(o, side + (size_t)best * O_NF, is_ask)) best = i;",
     "if (best < 0 || !better(side + (size_t)best * O_NF, o, is_ask)) best = i;"),
    ("tns_ignored", "P:L206 (earliest (Ts, Tns))", "return x[O_TNS] < y[O_TNS];", "return 0;"),
    ("synthetic_strict", "G12 (OID <= -9000)", "o[O_OID] <= -9000 && o[O_P] == P", "o[O_OID] < -9000 && o[O_P] == P"),
    ("synthetic_any_price", "P:L379 (synthetic cancel at the message price)",
     "o[O_OID] <= -9000 && o[O_P] == P", "o[O_OID] <= -9000"),
    ("trade_time_of_standing", "Eq.3 P:L195 (Ts_j = Ts_a)", "t[4] = m[M_TS];", "t[4] = os[O_TS];"),
    ("trade_oid_swapped", "Eq.3 P:L193-194 (OID_a, OID_s)", "t[2] = m[M_OID];", "t[2] = os[O_OID];"),
    ("no_sweep", "P:L204 (Q <= 0 -> all -1)", "if (Qs2 <= 0) set_empty(os);", ""),
    ("cancel_no_min", "G14 (cancelled += min(Q, Q_i))", "(Q < o[O_Q]) ? Q : o[O_Q];", "Q;"),
    ("cancel_opposite_side", "G16 (the message's side)", "cancel(X, b, own, m[M_P]", "cancel(X, b, opp, m[M_P]"),
    ("overlap_strict", "P:L215-216 (buy P_a >= P_s trades)",
     "(S == 1 && Pa < Ps) || (S == -1 && Pa > Ps)", "(S == 1 && Pa <= Ps) || (S == -1 && Pa >= Ps)"),
    ("market_price_swapped", "P:L290 (buy at max_int, sell at 0)",
     "(S == 1 ? INT32_MAX_ : 0)", "(S == 1 ? 0 : INT32_MAX_)"),
    ("oid_start_9001", "P:L379 (OIDs from -9000)", "int32_t oid = -9000;", "int32_t oid = -9001;"),
    ("l2_last_not_sum", "G23 (summed Q per level)", "if (occupied(o) && o[O_P] == best) sum += o[O_Q];",
     "if (occupied(o) && o[O_P] == best) sum = o[O_Q];"),
    ("highest_free_slot", "P:L175 + G3 (lowest empty slot)",
     "if (!occupied(own + (size_t)k * O_NF)) { i = k; break; }", "if (!occupied(own + (size_t)k * O_NF)) i = k;"),
    ("dropped_not_counted", "G8 (trades_dropped)", "b->c[C_TRADES_DROPPED]++;", ""),
    ("remainder_discarded_limit", "P:L288 (limit remainder rests)", "if (T == 1 && Qa > 0) {", "if (T == 9 && Qa > 0) {"),
    ("padding_counted_bad", "G21 (T = 0 is a silent no-op)", "if (T == 0) return;", "if (T == 0) { b->c[C_BAD]++; return; }"),
]


def _build(tmp, name, old, new):
    src = open(SRC).read()
    assert src.count(old) == 1, f"{name}: mutation site must be unique ({src.count(old)} matches)"
    path = os.path.join(tmp, f"m_{name}.c")
    open(path, "w").write(src.replace(old, new))
    so = os.path.join(tmp, f"liboracle_{name}.so")
    subprocess.check_call(["gcc", "-O1", "-std=c11", "-shared", "-fPIC", "-o", so, path, "-lm"])
    return so


def _battery(so):
    """Run the pins against the oracle in `so`; return the names of the pins that failed."""
    def mk(K, N, T=None, L=10, check=False, threads=1):
        return oracle.OracleBatch(K, N, T, L, check=check, threads=threads, lib_path=so)

    failed = []

    def pin(name, fn):
        try:
            fn()
        except AssertionError:
            failed.append(name)

    def golden():
        for _, case in golden_cases():
            run_golden_case(lambda N, T, L: mk(1, N, T, L, check=True), case)

    def fifo():
        for prof, init_levels in (("lobster", 10), ("synthetic", 33), ("ties", 10), ("heavy_market", 33)):
            cfg = lobgen.Config("mut", 6, 100, 5, 100, init_levels, 2000, 10, prof, 500)
            _compare_with_fifo(cfg, 6, make=mk)

    def brute():
        alpha = _alphabet()
        seqs = [s for n in range(1, 3) for s in itertools.product(alpha, repeat=n)]
        msgs = np.asarray([_encode(s, 2) for s in seqs], np.int32)
        o = mk(len(seqs), 2, 16, 3, check=True)
        l2 = o.process(msgs, 2, 1)
        assert (o.violations() == 0).all()
        tr, cnt = o.trades()
        for k in range(len(seqs)):
            ref, snaps = run_stream(msgs[k], 2, 1, 3)
            assert [tuple(t) for t in tr[k, :cnt[k]].tolist()] == ref.tape
            np.testing.assert_array_equal(l2[k], np.asarray(snaps, np.int32))

    def l2_groupby():
        cfg = lobgen.CONFIGS["C5_100"].with_(n_books=8)
        msgs, init = lobgen.generate(cfg)
        o = mk(8, cfg.capacity, cfg.trades_cap, 10)
        o.init(init, lobgen.INIT_TS, lobgen.INIT_TNS)
        o.process(msgs, cfg.n_steps, cfg.msgs_per_step, l2=False)
        book, l2 = o.book(), o.l2()
        for k in range(8):
            for s, cols in ((0, (0, 1)), (1, (2, 3))):
                occ = book[k, s][book[k, s, :, 1] > 0]
                prices, inv = np.unique(occ[:, 0], return_inverse=True)
                sums = np.bincount(inv, weights=occ[:, 1]).astype(np.int64)
                if s == 1:
                    prices, sums = prices[::-1], sums[::-1]
                want = np.full((10, 2), [-1, 0], np.int64)
                m = min(10, len(prices))
                want[:m, 0], want[:m, 1] = prices[:m], sums[:m]
                np.testing.assert_array_equal(l2[k][:, cols], want)

    for name, fn in (("golden", golden), ("fifo", fifo), ("brute_force", brute), ("l2_groupby", l2_groupby)):
        pin(name, fn)
    return failed


@pytest.fixture(scope="module")
def tmpdir_mod(tmp_path_factory):
    return str(tmp_path_factory.mktemp("mutants"))


def test_unmutated_oracle_passes_the_battery(tmpdir_mod):
    so = _build(tmpdir_mod, "none", "int32_t oid = -9000;", "int32_t oid = -9000;")
    assert _battery(so) == []


@pytest.mark.parametrize("name,why,old,new", MUTANTS, ids=[m[0] for m in MUTANTS])
def test_each_mutant_fails_a_pin(tmpdir_mod, name, why, old, new):
    so = _build(tmpdir_mod, name, old, new)
    failed = _battery(so)
    assert failed, f"mutant {name} ({why}) passed every pin"


@pytest.mark.parametrize("name", ["bid_is_min", "highest_slot_tie", "tns_ignored", "no_sweep", "cancel_no_min",
                                  "overlap_strict", "dropped_not_counted", "remainder_discarded_limit"])
def test_invariant_checker_is_not_vacuous(tmpdir_mod, name):
    """check mode (priority of every fill, sentinel discipline, never crossed, quantity
    conservation) must REPORT violations on mutants that break those invariants."""
    m = {x[0]: x for x in MUTANTS}[name]
    so = _build(tmpdir_mod, name, m[2], m[3])
    cfg = lobgen.Config("chk", 24, 50, 5, 100, 15, 8, 10, "ties", 9)
    msgs, init = lobgen.generate(cfg)
    o = oracle.OracleBatch(24, 50, 8, 10, check=True, lib_path=so)
    o.init(init, lobgen.INIT_TS, lobgen.INIT_TNS)
    o.process(msgs, cfg.n_steps, cfg.msgs_per_step)
    assert o.violations().sum() > 0, name
    good = oracle.OracleBatch(24, 50, 8, 10, check=True)
    good.init(init, lobgen.INIT_TS, lobgen.INIT_TNS)
    good.process(msgs, cfg.n_steps, cfg.msgs_per_step)
    assert good.violations().sum() == 0
