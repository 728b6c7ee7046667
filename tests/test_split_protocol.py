"""CPU model of the side-split build's hand-off protocol (lob_split.cuh).

The two warps of a book are modelled as Python generators that follow the kernel's
publication and wait rules step by step -- progress words published at chunk ends and
before every wait, the ring-reuse window at chunk starts, the parity-tagged remainder
ring (dummy entries written at decode time for messages the other warp never reads),
the trade-order wait while the log has room -- and a random scheduler interleaves them.
The checks are the properties the kernel relies on:
  * no schedule deadlocks (DESIGN.md 7d "No wait cycle");
  * a reader that accepts a ring entry by its parity bit always gets the entry of ITS
    message (no entry two passes old is ever mistaken for it);
  * trade records are numbered in message order (Eq.3-4) up to T_cap.
This checks the protocol, not the kernel: the kernel itself is compared with the oracle
bit for bit by the GPU tests (tests/test_gpu_parity.py::test_side_split_build).
"""
from __future__ import annotations

import random

import pytest

CH, RING = 32, 64


def _stream(rng, n, p_aggr=0.3, p_fill=0.4, p_sure=0.6):
    """Messages: (side, kind, fills, sure) -- kind 'c' cancel / 'l' limit / 'm' market;
    fills = trades the other side's warp makes; sure = the aggressor's bound proves no
    trade (only possible when fills == 0)."""
    out = []
    for _ in range(n):
        side = rng.randrange(2)
        u = rng.random()
        if u < p_aggr:
            kind = "l" if rng.random() < 0.8 else "m"
            fills = rng.randrange(1, 4) if rng.random() < p_fill else 0
            sure = kind == "l" and fills == 0 and rng.random() < p_sure
            out.append((side, kind, fills, sure))
        elif u < 0.95:
            out.append((side, "c", 0, False))
        else:
            out.append((-1, "pad", 0, False))
    return out


class _Book:
    def __init__(self, msgs, tcap):
        self.msgs, self.tcap = msgs, tcap
        self.prog = [0, 0]                  # published progress (messages finished)
        self.fills = [0, 0]                 # published fill counts
        self.ring = [[None] * RING, [None] * RING]   # ring[writer][slot] = message index
        self.trades = []                    # (message index, trade number)


def _warp(bk: _Book, X: int):
    """Generator for the warp of side X; yields a wait label while it waits, None per step."""
    Y = 1 - X
    msgs = bk.msgs
    n = len(msgs)
    nchunks = (n + CH - 1) // CH
    myfills = 0
    for c in range(nchunks):
        if c >= 2:                                       # ring reuse window
            bk.prog[X] = CH * c
            while not bk.prog[Y] >= CH * (c - 1):
                yield "window"
        cnt = min(CH, n - c * CH)
        for k in range(cnt):                             # decode: dummies for unread slots
            mk = c * CH + k
            side, kind, _, _ = msgs[mk]
            other_aggr = side == Y and kind in ("l", "m")
            if not other_aggr:
                bk.ring[X][mk % RING] = mk
        yield None
        for k in range(cnt):
            mi = c * CH + k
            side, kind, fills, sure = msgs[mi]
            if side == X and kind == "l" and not sure:  # own limit that may trade: the ring
                bk.prog[X] = mi
                while True:
                    e = bk.ring[Y][mi % RING]
                    if e is not None and (e // RING) % 2 == (mi // RING) % 2:
                        assert e == mi, f"warp {X} read the entry of message {e} for message {mi}"
                        break
                    yield "remainder"
            elif side == Y and kind in ("l", "m"):      # the other side aggresses: fills here
                if fills:
                    if myfills + bk.fills[Y] < bk.tcap:
                        bk.prog[X] = mi
                        while not bk.prog[Y] >= mi:
                            yield "trade order"
                    base = myfills + bk.fills[Y]
                    for f in range(fills):
                        if base + f < bk.tcap:
                            bk.trades.append((mi, base + f))
                    myfills += fills
                    bk.fills[X] = myfills
                bk.ring[X][mi % RING] = mi               # the entry (Q_a', bound) of message mi
            yield None
        bk.prog[X] = c * CH + cnt
        yield None


def _run(msgs, tcap, rng, bias=0.5):
    bk = _Book(msgs, tcap)
    warps = [_warp(bk, 0), _warp(bk, 1)]
    state = [None, None]                               # last yield (None or a wait label)
    alive = [True, True]
    stuck = 0
    while any(alive):
        live = [k for k in (0, 1) if alive[k]]
        i = live[0] if len(live) == 1 else (0 if rng.random() < bias else 1)
        try:
            state[i] = next(warps[i])
        except StopIteration:
            alive[i] = False
            continue
        # deadlock: every live warp has been waiting for many scheduling rounds in a row
        stuck = stuck + 1 if all(state[k] is not None for k in (0, 1) if alive[k]) else 0
        assert stuck < 10000, f"deadlock: {state}"
    return bk


@pytest.mark.parametrize("seed", range(40))
def test_split_protocol_random_schedules(seed):
    rng = random.Random(seed)
    n = rng.choice([1, 31, 32, 33, 64, 65, 200, 640])
    tcap = rng.choice([0, 1, 5, 100, 10 ** 6])
    msgs = _stream(rng, n, p_aggr=rng.choice([0.1, 0.3, 0.6]), p_fill=rng.choice([0.1, 0.5, 1.0]))
    for rep in range(5):
        bk = _run(msgs, tcap, random.Random(seed * 100 + rep))
        expect = []
        for mi, (side, kind, fills, _) in enumerate(msgs):
            expect += [mi] * (fills if side >= 0 and kind in ("l", "m") else 0)
        logged = sorted(bk.trades, key=lambda t: t[1])
        assert [t[1] for t in logged] == list(range(min(tcap, len(expect))))
        assert [t[0] for t in logged] == expect[:tcap], "trades out of message order"


@pytest.mark.parametrize("seed", range(12))
def test_split_protocol_biased_schedules(seed):
    # one warp is scheduled 20-100x as often as the other: it runs as far ahead as the
    # ring-reuse window lets it (without the window it overwrites entries still unread)
    rng = random.Random(1000 + seed)
    msgs = _stream(rng, 700, p_aggr=rng.choice([0.05, 0.2]), p_fill=0.5, p_sure=0.3)
    bias = rng.choice([0.95, 0.99, 0.01, 0.05])
    bk = _run(msgs, 10 ** 6, random.Random(seed), bias=bias)
    assert sorted(t[1] for t in bk.trades) == list(range(len(bk.trades)))


def test_split_protocol_skewed_schedule():
    # one warp runs far ahead whenever it can (the window and the waits must hold it)
    rng = random.Random(7)
    msgs = _stream(rng, 1000, p_aggr=0.4, p_fill=0.5)
    bk = _Book(msgs, 10 ** 6)
    w = [_warp(bk, 0), _warp(bk, 1)]
    alive, st = [True, True], [None, None]
    guard = 0
    while any(alive):
        guard += 1
        assert guard < 10 ** 6
        i = 0 if alive[0] and st[0] is None else 1
        if not alive[i]:
            i = 1 - i
        try:
            st[i] = next(w[i])
        except StopIteration:
            alive[i] = False
        if st[i] is not None and alive[1 - i]:         # waiting: let the other run
            try:
                st[1 - i] = next(w[1 - i])
            except StopIteration:
                alive[1 - i] = False
    assert len(bk.trades) == sum(f for s, k, f, _ in msgs if s >= 0 and k in ("l", "m"))
