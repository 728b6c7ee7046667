"""Independent textbook matching engine used to PIN the oracle (not the oracle itself).

A price-time-priority continuous double auction written from its textbook
definition (Gould et al. 2013, cited at P:L206): each side is a sorted map
price -> FIFO queue of orders in arrival order.  It shares nothing with
``oracle/lob_oracle.c`` (different language, different data structure: no
slots, no arrays, no -1 sentinels).

Where the paper's array engine is a plain CDA, the two must agree exactly:
streams with strictly increasing timestamps (so arrival order == time order),
no add overflow (occupancy < N) and no trade-log overflow (SPEC S:L141,
S:L575).  Paper rules mirrored here because they define the *method*, not the
array representation: market prices 0 / max_int, cancel == delete
(P:L289), the synthetic -9000 cancel fallback (reading G12), malformed
messages are no-ops (G22), zero messages are padding (G21).
"""
from __future__ import annotations

from collections import deque

from sortedcontainers import SortedDict

INT32_MAX = 2**31 - 1


class FifoBook:
    def __init__(self):
        self.asks = SortedDict()      # price -> deque[[oid, q, tid, ts, tns]]
        self.bids = SortedDict()
        self.index = [{}, {}]         # per side (0 asks, 1 bids): oid -> price
        self.tape = []                # every fill, in order
        self.cancelled = 0
        self.unknown = 0
        self.discarded = 0
        self.bad = 0

    # ----------------------------------------------------------------- helpers
    def _side(self, s):               # s: 0 asks, 1 bids
        return self.bids if s else self.asks

    def _best_price(self, s):
        side = self._side(s)
        if not side:
            return None
        return side.peekitem(-1)[0] if s else side.peekitem(0)[0]

    def _rest(self, s, price, order):
        side = self._side(s)
        if price not in side:
            side[price] = deque()
        side[price].append(order)
        self.index[s].setdefault(order[0], price)

    def _remove_empty_level(self, s, price):
        side = self._side(s)
        if not side[price]:
            del side[price]

    def seed(self, asks, bids, ts, tns):
        """Initial L2 snapshot: one order per level, OIDs -9000 descending."""
        oid = -9000
        for s, levels in ((0, asks), (1, bids)):
            for p, q in levels:
                if p > 0 and q > 0:
                    self._rest(s, p, [oid, q, -9000, ts, tns])
                    oid -= 1

    # ------------------------------------------------------------------ events
    def message(self, m):
        T, S, Q, P, OID, TID, Ts, Tns = (int(x) for x in m)
        if T == 0:
            return
        if T not in (1, 2, 3, 4) or S not in (1, -1):
            self.bad += 1
            return
        own = 1 if S == 1 else 0
        opp = 1 - own
        if T in (2, 3):
            if Q <= 0:
                self.bad += 1
                return
            self._cancel(own, P, OID, Q)
            return
        if T == 1 and P <= 0:
            self.bad += 1
            return
        limit = P if T == 1 else (INT32_MAX if S == 1 else 0)
        rem = Q
        while rem > 0:
            bp = self._best_price(opp)
            if bp is None:
                break
            if (S == 1 and limit < bp) or (S == -1 and limit > bp):
                break
            queue = self._side(opp)[bp]
            head = queue[0]
            fill = min(rem, head[1])
            self.tape.append((bp, fill, OID, head[0], Ts, Tns))
            head[1] -= fill
            rem -= fill
            if head[1] == 0:
                queue.popleft()
                self._drop_index(opp, head[0], bp)
                self._remove_empty_level(opp, bp)
        if rem > 0:
            if T == 1:
                self._rest(own, P, [OID, rem, TID, Ts, Tns])
            else:
                self.discarded += rem

    def _drop_index(self, s, oid, price):
        if self.index[s].get(oid) == price:
            # another live order might share the OID at a different price (not generated)
            del self.index[s][oid]

    def _find(self, s, oid):
        price = self.index[s].get(oid)
        if price is None:
            return None
        for o in self._side(s)[price]:
            if o[0] == oid:
                return price, o
        return None

    def _cancel(self, s, P, OID, Q):
        hit = self._find(s, OID)
        if hit is None:
            # synthetic initial order at the cancel's price (G12)
            side = self._side(s)
            if P in side:
                for o in side[P]:
                    if o[0] <= -9000:
                        hit = (P, o)
                        break
        if hit is None:
            self.unknown += 1
            return
        price, o = hit
        self.cancelled += min(Q, o[1])
        o[1] -= Q
        if o[1] <= 0:
            self._side(s)[price].remove(o)
            self._drop_index(s, o[0], price)
            self._remove_empty_level(s, price)

    # ------------------------------------------------------------------- views
    def l2(self, levels):
        rows = [[-1, 0, -1, 0] for _ in range(levels)]
        for k, p in enumerate(list(self.asks.keys())[:levels]):
            rows[k][0], rows[k][1] = p, sum(o[1] for o in self.asks[p])
        for k, p in enumerate(list(reversed(self.bids.keys()))[:levels]):
            rows[k][2], rows[k][3] = p, sum(o[1] for o in self.bids[p])
        return rows

    def resting(self):
        """Multiset of resting orders as sorted tuples (side, P, Q, OID, TID, Ts, Tns)."""
        out = []
        for s in (0, 1):
            for p, q in self._side(s).items():
                for o in q:
                    out.append((s, p, o[1], o[0], o[2], o[3], o[4]))
        return sorted(out)


def run_stream(msgs, n_steps, msgs_per_step, levels, init_rows=None, ts=0, tns=0):
    """Replay one book's stream; returns (engine, per-step L2 list)."""
    b = FifoBook()
    if init_rows is not None:
        b.seed([(r[0], r[1]) for r in init_rows], [(r[2], r[3]) for r in init_rows], ts, tns)
    snaps = []
    for s in range(n_steps):
        for i in range(msgs_per_step):
            b.message(msgs[s * msgs_per_step + i])
        snaps.append(b.l2(levels))
    return b, snaps
