"""Pins for the CPU oracle (-m "not gpu"): the oracle is checked against things other
than itself -- hand-derived golden traces, an independent textbook FIFO engine,
exhaustive tiny-input brute force, closed forms and invariants."""
from __future__ import annotations

import itertools

import numpy as np
import pytest

import lobgen
import oracle
from common import STAT_NAMES, golden_cases, run_golden_case
from pins.fifo_engine import run_stream

ST = {n: i for i, n in enumerate(STAT_NAMES)}


def make_oracle(N, T_cap, L):
    return oracle.OracleBatch(1, N, T_cap, L, check=True)


# --------------------------------------------------------------- golden traces
@pytest.mark.parametrize("cid,case", golden_cases(), ids=[c[0] for c in golden_cases()])
def test_golden(cid, case):
    run_golden_case(make_oracle, case)


# ------------------------------------------------- independent FIFO sorted map
def _compare_with_fifo(cfg, n_books, make=oracle.OracleBatch, book_begin=0):
    msgs, init = lobgen.generate(cfg.with_(n_books=n_books), book_begin=book_begin)
    o = make(n_books, cfg.capacity, cfg.n_msgs * 4, cfg.l2_levels, check=True)
    o.init(init, lobgen.INIT_TS, lobgen.INIT_TNS)
    l2 = o.process(msgs, cfg.n_steps, cfg.msgs_per_step)
    tr, cnt = o.trades()
    book, st = o.book(), o.stats()
    assert (o.violations() == 0).all()
    assert (st[:, ST["add_overflow"]] == 0).all() and (st[:, ST["trades_dropped"]] == 0).all()
    for k in range(n_books):
        ref, snaps = run_stream(msgs[k], cfg.n_steps, cfg.msgs_per_step, cfg.l2_levels,
                                init[k] if init is not None else None, lobgen.INIT_TS, lobgen.INIT_TNS)
        assert [tuple(t) for t in tr[k, :cnt[k]].tolist()] == ref.tape, f"book {k} trade tape"
        np.testing.assert_array_equal(l2[k], np.asarray(snaps, np.int32), err_msg=f"book {k} L2")
        rest = []
        for s in (0, 1):
            for o_ in book[k, s]:
                if o_[1] > 0:
                    rest.append((s, *o_.tolist()))
        assert sorted((r[0], r[1], r[2], r[3], r[4], r[5], r[6]) for r in rest) == ref.resting(), k
        assert st[k, ST["cancelled_qty"]] == ref.cancelled
        assert st[k, ST["unknown_cancels"]] == ref.unknown
        assert st[k, ST["market_discarded_qty"]] == ref.discarded
        assert st[k, ST["bad"]] == ref.bad
        assert st[k, ST["trades"]] == len(ref.tape)
        assert st[k, ST["traded_qty"]] == sum(t[1] for t in ref.tape)


@pytest.mark.parametrize("profile,n_books", [("lobster", 48), ("cancel_heavy", 24),
                                             ("heavy_market", 24), ("synthetic", 24)])
def test_oracle_equals_fifo_engine(profile, n_books):
    # SPEC acceptance #1 shape: N=100, 1000-message streams, occupancy < N
    cfg = lobgen.Config("pin", n_books, 100, 10, 100, 33 if profile != "lobster" else 10,
                        4000, 10, profile, 1000 + n_books)
    _compare_with_fifo(cfg, n_books)


def test_oracle_equals_fifo_small_capacity():
    cfg = lobgen.Config("pin", 64, 12, 20, 10, 3, 2000, 5, "lobster", 77)
    _compare_with_fifo(cfg, 64)


# ------------------------------------------------------ exhaustive brute force
def _alphabet():
    out = []
    for S in (1, -1):
        for P in (1, 2, 3):
            for Q in (1, 2):
                out.append(("L", S, Q, P, None))
    for T in (2, 3):
        for S in (1, -1):
            for oid in (1, 2, 99):
                for Q in (1, 2):
                    out.append(("C" if T == 2 else "D", S, Q, 2, oid))
    for S in (1, -1):
        for Q in (1, 3):
            out.append(("M", S, Q, 0, None))
    return out


def _encode(seq, length):
    rows = []
    for i, (kind, S, Q, P, oid) in enumerate(seq):
        T = {"L": 1, "C": 2, "D": 3, "M": 4}[kind]
        OID = (i + 1) if oid is None else oid
        rows.append([T, S, Q, P, OID, 7, i + 1, 0])
    rows += [[0] * 8] * (length - len(seq))
    return rows


@pytest.mark.parametrize("N", [1, 2, 3])
def test_bruteforce_all_sequences_up_to_3(N):
    alpha = _alphabet()
    seqs = [s for n in range(1, 4) for s in itertools.product(alpha, repeat=n)]
    msgs = np.asarray([_encode(s, 3) for s in seqs], np.int32)
    K = len(seqs)
    o = oracle.OracleBatch(K, N, 16, 3, check=True)
    l2 = o.process(msgs, 3, 1)
    assert (o.violations() == 0).all()
    tr, cnt = o.trades()
    book, st = o.book(), o.stats()
    # sorted-map equality whenever the book cannot overflow (N >= number of messages)
    idx = [k for k, s in enumerate(seqs) if len(s) <= N]
    for k in idx:
        ref, snaps = run_stream(msgs[k], 3, 1, 3)
        assert [tuple(t) for t in tr[k, :cnt[k]].tolist()] == ref.tape
        np.testing.assert_array_equal(l2[k], np.asarray(snaps, np.int32))
        assert st[k, ST["unknown_cancels"]] == ref.unknown
        assert st[k, ST["market_discarded_qty"]] == ref.discarded


def _alphabet_array():
    """The 40-message alphabet as rows [T, S, Q, P, OID or 0 (= position-dependent)]."""
    T = {"L": 1, "C": 2, "D": 3, "M": 4}
    return np.asarray([[T[k], S, Q, P, 0 if oid is None else oid] for k, S, Q, P, oid in _alphabet()], np.int64)


def _encode_all(idx):
    """Vectorised _encode for sequences given as alphabet indices idx [n][length]."""
    a = _alphabet_array()
    n, length = idx.shape
    m = np.zeros((n, length, 8), np.int32)
    rows = a[idx]                                          # [n][length][5]
    pos = np.arange(1, length + 1)[None, :]
    m[..., :4] = rows[..., :4]
    m[..., 4] = np.where(rows[..., 4] == 0, pos, rows[..., 4])
    m[..., 5] = 7
    m[..., 6] = pos
    return m


@pytest.mark.slow
@pytest.mark.parametrize("N", [1, 2, 3])
def test_bruteforce_all_sequences_of_length_4(N):
    """Every sequence of exactly 4 messages over the 40-message alphabet (2,560,000 per
    capacity) in check mode: sentinel discipline, never crossed, priority of every fill,
    quantity conservation, fills = logged + dropped, unknown cancels leave the book
    bit-identical -- after every message.  (Shorter sequences: the length <= 3 test; at
    N < 4 the sorted-map FIFO comparison needs N >= length, see the N = 4 sample below.)"""
    n_alpha = len(_alphabet())
    total = n_alpha ** 4
    chunk = 160_000
    for c0 in range(0, total, chunk):
        flat = np.arange(c0, min(total, c0 + chunk))
        idx = np.stack([(flat // n_alpha ** p) % n_alpha for p in (3, 2, 1, 0)], 1)
        msgs = _encode_all(idx)
        o = oracle.OracleBatch(len(flat), N, 4, 3, check=True, threads=8)
        o.process(msgs, 4, 1, l2=False)
        v = o.violations()
        assert (v == 0).all(), (N, c0 + int(np.argmax(v)))
        st = o.stats()
        assert (st[:, ST["msgs"]] == 4).all()
        occ = (o.book()[..., 1] > 0).sum(-1)
        assert (occ <= N).all()


@pytest.mark.slow
def test_length_4_sample_equals_fifo_at_capacity_4():
    """A seeded sample of 25,000 length-4 sequences at N = 4 (no overflow possible):
    trade tape, per-step L2, unknown cancels and discarded market quantity equal the
    independent sorted-map FIFO engine's."""
    rng = np.random.default_rng(44)
    idx = rng.integers(0, len(_alphabet()), (25_000, 4))
    msgs = _encode_all(idx)
    o = oracle.OracleBatch(len(idx), 4, 16, 3, check=True, threads=8)
    l2 = o.process(msgs, 4, 1)
    assert (o.violations() == 0).all()
    tr, cnt = o.trades()
    st = o.stats()
    for k in range(len(idx)):
        ref, snaps = run_stream(msgs[k], 4, 1, 3)
        assert [tuple(t) for t in tr[k, :cnt[k]].tolist()] == ref.tape, k
        np.testing.assert_array_equal(l2[k], np.asarray(snaps, np.int32))
        assert st[k, ST["unknown_cancels"]] == ref.unknown
        assert st[k, ST["market_discarded_qty"]] == ref.discarded


def test_vectorised_encoding_matches_encode():
    rng = np.random.default_rng(3)
    alpha = _alphabet()
    idx = rng.integers(0, len(alpha), (50, 4))
    want = np.asarray([_encode([alpha[i] for i in row], 4) for row in idx], np.int32)
    np.testing.assert_array_equal(_encode_all(idx), want)


@pytest.mark.slow
@pytest.mark.parametrize("profile", ["lobster", "cancel_heavy", "heavy_market", "synthetic"])
def test_oracle_equals_fifo_engine_1024_streams(profile):
    """SPEC acceptance #1 at its stated size (>= 1000 random streams):
    4 profiles x 256 streams = 1,024 streams of 1,000 messages at N = 100, global book ids
    disjoint from the other FIFO tests."""
    cfg = lobgen.Config("pin1k", 256, 100, 10, 100, 33 if profile != "lobster" else 10, 4000, 10, profile, 7001)
    _compare_with_fifo(cfg, 256, book_begin=100_000)


def test_bruteforce_random_longer_sequences():
    rng = np.random.default_rng(5)
    alpha = _alphabet()
    K, length = 3000, 8
    seqs = [[alpha[i] for i in rng.integers(0, len(alpha), rng.integers(5, length + 1))] for _ in range(K)]
    msgs = np.asarray([_encode(s, length) for s in seqs], np.int32)
    for N in (2, 8):
        o = oracle.OracleBatch(K, N, 32, 3, check=True)
        l2 = o.process(msgs, length, 1)
        assert (o.violations() == 0).all()
        if N == 8:
            tr, cnt = o.trades()
            for k in range(0, K, 3):
                ref, snaps = run_stream(msgs[k], length, 1, 3)
                assert [tuple(t) for t in tr[k, :cnt[k]].tolist()] == ref.tape
                np.testing.assert_array_equal(l2[k], np.asarray(snaps, np.int32))


# ------------------------------------------------------------------ closed forms
def test_static_sweep_closed_form():
    """A market order against a static side trades the stable-sorted eligible prefix
    (price, then time, then slot) truncated at Q_a; traded = min(Q_a, sum Q)
    (P:L180-196 closed form q = min(Q_s, Q_a); Table 2 protocol P:L240-256)."""
    rng = np.random.default_rng(11)
    for trial in range(200):
        N = int(rng.integers(3, 40))
        n = int(rng.integers(1, N + 1))
        side = int(rng.choice([1, -1]))              # side of the resting orders
        P = rng.integers(100, 106, n)
        Q = rng.integers(1, 50, n)
        Ts = rng.integers(0, 4, n)                   # many ties on purpose
        Tns = rng.integers(0, 3, n)
        adds = np.stack([np.ones(n), np.full(n, side), Q, P, np.arange(1, n + 1), np.zeros(n), Ts, Tns], 1)
        # non-crossing: all orders on one side, so the adds only rest
        Qa = int(rng.integers(1, 60 * n))
        mkt = np.array([[4, -side, Qa, 0, 999, 0, 9, 9]])
        o = oracle.OracleBatch(1, N, 4 * N, 1)
        o.process(adds.astype(np.int32)[None], 1, n, l2=False)
        book = o.book()[0, 0 if side == -1 else 1]
        o.process(mkt.astype(np.int32)[None], 1, 1, l2=False)
        tr, cnt = o.trades()
        slots = np.nonzero(book[:, 1] > 0)[0]
        key_p = book[slots, 0] if side == -1 else -book[slots, 0]
        order = slots[np.lexsort((slots, book[slots, 5], book[slots, 4], key_p))]
        want, rem = [], Qa
        for s in order:
            if rem <= 0:
                break
            q = min(rem, int(book[s, 1]))
            want.append((int(book[s, 0]), q, 999, int(book[s, 2]), 9, 9))
            rem -= q
        assert [tuple(t) for t in tr[0, :cnt[0]].tolist()] == want, trial
        assert o.stats()[0, ST["traded_qty"]] == min(Qa, int(book[slots, 1].sum()))


def test_l2_is_group_by_sum():
    """L2 = top-L distinct prices with summed quantity (G23), via numpy group-by."""
    cfg = lobgen.CONFIGS["C5_512"].with_(n_books=16)
    msgs, init = lobgen.generate(cfg)
    o = oracle.OracleBatch(16, cfg.capacity, cfg.trades_cap, 10)
    o.init(init, lobgen.INIT_TS, lobgen.INIT_TNS)
    o.process(msgs, cfg.n_steps, cfg.msgs_per_step, l2=False)
    book, l2 = o.book(), o.l2()
    for k in range(16):
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


# --------------------------------------------------------------- invariants
@pytest.mark.parametrize("profile,N", [("lobster", 100), ("ties", 100), ("overflow", 16),
                                       ("synthetic", 64), ("garbage", 100), ("heavy_market", 100),
                                       ("cancel_heavy", 100), ("lobster", 1), ("lobster", 33)])
def test_invariants_hold(profile, N):
    cfg = lobgen.Config("inv", 32, N, 10, 100, min(N, 10), 256, 10, profile, 9)
    msgs, init = lobgen.generate(cfg)
    o = oracle.OracleBatch(32, N, 256, 10, check=True)
    o.init(init, lobgen.INIT_TS, lobgen.INIT_TNS)
    o.process(msgs, cfg.n_steps, cfg.msgs_per_step)
    assert (o.violations() == 0).all()
    st = o.stats()
    assert (st[:, ST["msgs"]] == cfg.n_msgs).all()
    if profile == "overflow":
        assert st[:, ST["add_overflow"]].sum() > 0
    if profile == "garbage":
        assert st[:, ST["bad"]].sum() > 0


# ---------------------------------------------------- batch determinism/isolation
def test_batch_determinism_and_isolation():
    """clones are identical; book k is its own serial fold;
    perturbing book i changes only book i."""
    cfg = lobgen.CONFIGS["C1"].with_(n_books=8)
    msgs, init = lobgen.generate(cfg)
    clones = np.repeat(msgs[:1], 50, axis=0)
    o = oracle.OracleBatch(50, 100, 1000, 10)
    o.init(np.repeat(init[:1], 50, 0), lobgen.INIT_TS, lobgen.INIT_TNS)
    l2 = o.process(clones, 10, 100)
    assert (o.book() == o.book()[:1]).all() and (l2 == l2[:1]).all()
    both = oracle.OracleBatch(8, 100, 1000, 10)
    both.init(init, lobgen.INIT_TS, lobgen.INIT_TNS)
    l2a = both.process(msgs, 10, 100)
    for k in (0, 5):
        one = oracle.OracleBatch(1, 100, 1000, 10)
        one.init(init[k:k + 1], lobgen.INIT_TS, lobgen.INIT_TNS)
        l2b = one.process(msgs[k:k + 1], 10, 100)
        np.testing.assert_array_equal(l2a[k], l2b[0])
        np.testing.assert_array_equal(both.book()[k], one.book()[0])
    pert = msgs.copy()
    pert[3, 10:20] = 0
    p = oracle.OracleBatch(8, 100, 1000, 10)
    p.init(init, lobgen.INIT_TS, lobgen.INIT_TNS)
    p.process(pert, 10, 100)
    changed = [k for k in range(8) if not np.array_equal(p.book()[k], both.book()[k])]
    assert changed == [3]


def test_generator_is_shard_invariant():
    cfg = lobgen.CONFIGS["C4"]
    a, ia = lobgen.generate(cfg, book_begin=0, n_books=64, threads=3)
    b, ib = lobgen.generate(cfg, book_begin=40, n_books=24, threads=1)
    np.testing.assert_array_equal(a[40:], b)
    np.testing.assert_array_equal(ia[40:], ib)


# ------------------------------------------------- NEXT row N1: Level-1 trace
@pytest.mark.parametrize("profile", ["lobster", "heavy_market", "cancel_heavy"])
def test_l1_trace_equals_fifo_top_of_book(profile):
    """Level-1 after every message equals the independent FIFO engine's
    top of book after that message."""
    cfg = lobgen.Config("l1", 12, 100, 4, 50, 20, 4000, 3, profile, 31)
    msgs, init = lobgen.generate(cfg)
    o = oracle.OracleBatch(12, 100, 4000, 3)
    o.init(init, lobgen.INIT_TS, lobgen.INIT_TNS)
    l2, l1 = o.process(msgs, cfg.n_steps, cfg.msgs_per_step, l1=True)
    assert l1.shape == (12, cfg.n_msgs, 4)
    for k in range(12):
        _, snaps = run_stream(msgs[k], cfg.n_msgs, 1, 1, init[k], lobgen.INIT_TS, lobgen.INIT_TNS)
        np.testing.assert_array_equal(l1[k], np.asarray(snaps, np.int32)[:, 0], err_msg=f"book {k}")
        # consistency with the per-step L2 (level 1 at the step boundaries)
        np.testing.assert_array_equal(l1[k, cfg.msgs_per_step - 1::cfg.msgs_per_step], l2[k, :, 0])


def test_saturate_profile_reaches_capacity():
    """The GPU capacity test (test_gpu_parity.py::test_capacity_saturated) is only
    meaningful if its streams saturate: on the oracle most books overflow (G6), some
    side ends exactly full, and no side ever holds more than N orders."""
    from common import SATURATE_N, saturate_cfg
    for N in SATURATE_N:
        cfg = saturate_cfg(N)
        msgs, init = lobgen.generate(cfg)
        o = oracle.OracleBatch(cfg.n_books, N, cfg.trades_cap, cfg.l2_levels, threads=8)
        o.init(init, lobgen.INIT_TS, lobgen.INIT_TNS)
        o.process(msgs, cfg.n_steps, cfg.msgs_per_step)
        st = o.stats()
        assert (st[:, STAT_NAMES.index("add_overflow")] > 0).mean() >= 0.5, N
        occ = (o.book()[..., 1] > 0).sum(-1)
        assert occ.max() == N and (occ <= N).all(), N


def test_l2_volume_saturates_at_int32_max():
    """G20: a level's volume is the exact int64 sum reported in the int32 field, saturated
    at INT32_MAX (32-bit fields).  Closed forms: 1.5e9 + 6e8 = 2.1e9 fits; 2^30 +
    2^30 = 2^31 does not (INT32_MAX); a level of three max-int orders is INT32_MAX, never a
    wrapped (negative) value; level 1 of the L1 trace is the same number."""
    IMAX = 2**31 - 1
    rows = [[1, -1, 1_500_000_000, 105, 1, 0, 1, 0], [1, -1, 600_000_000, 105, 2, 0, 2, 0],
            [1, -1, 2**30, 106, 3, 0, 3, 0], [1, -1, 2**30, 106, 4, 0, 4, 0],
            [1, 1, IMAX, 90, 5, 0, 5, 0], [1, 1, IMAX, 90, 6, 0, 6, 0], [1, 1, IMAX, 90, 7, 0, 7, 0],
            [1, 1, 5, 89, 8, 0, 8, 0]]
    o = oracle.OracleBatch(1, 8, 4, 3, check=True)
    l2, l1 = o.process(np.asarray(rows, np.int32)[None], 1, 8, l1=True)
    assert l2[0, 0].tolist() == [[105, 2_100_000_000, 90, IMAX], [106, IMAX, 89, 5], [-1, 0, -1, 0]]
    assert l1[0, -1].tolist() == [105, 2_100_000_000, 90, IMAX]
    assert l1[0, 5].tolist() == [105, 2_100_000_000, 90, IMAX]       # two max-int bids: 2^32 - 2 -> IMAX
    assert (o.violations() == 0).all()
