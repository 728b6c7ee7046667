// lob_split.cuh -- the side-split step kernel for latency-bound launches (few books).
//
// When a launch has too few books to fill the SMs (C2: 1,000 books, the paper's RL
// shape), the time of a call is one book's serial per-message dependency chain
// (~500 cycles per message), not the issue rate.  This build gives each
// book TWO warps, one per side (warp ASK holds the asks, warp BID the bids; Eq.1-2,
// P:L161-166), that walk the same message stream concurrently.  Most messages touch one
// side only (a cancel its own side, a non-marketable limit its own side), so
// each warp does the work of its own side's messages and only reads past the others:
// the chain per book roughly halves.  The two warps meet only where the method couples
// the sides:
//   * an aggressive order (limit or market) of side S is matched against side 1-S first
//     (P:L206): the warp of side 1-S runs the fill loop, writes the trades and
//     publishes the remainder Q_a' (and its side's best price after the message) in a
//     64-entry ring; the warp of side S rests Q_a' > 0 -- market remainders are
//     discarded by the filling warp;
//   * the warp of side S needs that remainder only when the order MAY be marketable:
//     it keeps a bound on the other side's best price (the exact value published after
//     its last aggressive order, tightened by every later limit price of the other side --
//     the only way that side's best can improve), and a limit price outside the bound
//     rests without waiting.  C2: ~90 % of limits are passive (lobgen "lobster");
//   * trade records are in message order (Eq.3-4): before a fill at message i the
//     filling warp waits until the other warp has finished every message < i and numbers
//     its trades after the other warp's fills so far (the other warp cannot fill at a
//     message >= i before this one finishes i, by the same rule).
// Progress words (messages finished), the ring and the fill counts live in shared
// memory; waits are warp-uniform polling loops.  No wait cycle exists: a warp waits only
// for the other warp to reach a message index at or below its own (or, for the ring's
// reuse window, at most two chunks behind), see the proof in DESIGN.md 7d.
//
// Results are identical to lob_step's (the same parity tests): only the schedule of
// the two sides' work changes.  Used for one-warp geometries (N <= 512) when the launch
// has at most LOB_SPLIT_BPS books per SM (lob_api.cu), MODE 0 only (no L1 trace / env).
#pragma once
#include "lob_kernels.cuh"

namespace lobk {

#ifndef LOB_SPLIT_SLEEP  // back-off (ns) per poll of the other warp's progress
#define LOB_SPLIT_SLEEP 0
#endif
constexpr int SPLIT_RING = 64;  // remainder ring entries (2 staging chunks)

// one book (two warps) of the side-split build: byte offsets in its shared region
template <int KPL>
struct SplitLayout {
    static constexpr int NP = KPL * 32;
    static constexpr int STAGE = 0;                              // [2 sides][2][CH][32 B]
    static constexpr int BARS = STAGE + 2 * 2 * CH * 32;         // [2 sides][2] mbarriers
    static constexpr int COLD = BARS + 32;                       // [2 sides][NP] x 16 B
    static constexpr int SCR = COLD + 2 * NP * 16;               // [2 sides][128 B]: counters, bt
    static constexpr int SYN = SCR + 2 * 128;                    // prog[2], fills[2]
    static constexpr int RING = SYN + 16;                        // [2 sides][SPLIT_RING] int2
    static constexpr int BYTES = ((RING + 2 * SPLIT_RING * 8) + 127) / 128 * 128;
};
static_assert(8 * NST + 16 <= 128, "split scratch");

__device__ __forceinline__ int lds_acq(uint32_t a) {
    int v;
    asm volatile("ld.acquire.cta.shared.b32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
    return v;
}
// lane `who == 0` stores v with release semantics (orders this thread's earlier shared
// stores -- ring entry, fill count -- before it); a predicated store, no divergent branch
__device__ __forceinline__ void sts_rel_if0(int who, uint32_t a, int v) {
    asm volatile("{\n\t.reg .pred p;\n\tsetp.eq.s32 p, %0, 0;\n\t@p st.release.cta.shared.b32 [%1], %2;\n\t}" ::"r"(who),
                 "r"(a), "r"(v)
                 : "memory");
}
__device__ __forceinline__ unsigned long long lds64v(uint32_t a) {
    unsigned long long v;
    asm volatile("ld.volatile.shared.b64 %0, [%1];" : "=l"(v) : "r"(a) : "memory");
    return v;
}
__device__ __forceinline__ void sts64_if0(int who, uint32_t a, unsigned long long v) {
    asm volatile("{\n\t.reg .pred p;\n\tsetp.eq.s32 p, %0, 0;\n\t@p st.volatile.shared.b64 [%1], %2;\n\t}" ::"r"(who),
                 "r"(a), "l"(v)
                 : "memory");
}
#ifdef LOB_SPLIT_STATS  // instrumented variant only: [site][calls, spun, spin iterations]
__device__ unsigned long long g_split_stats[4][3];
__device__ long long g_split_trace[8][2][10240];  // (cycles << 4) | class, first 8 books
#endif
// every lane polls until the other warp's progress word reaches `target` (a warp
// reduction as the loop condition: a uniform loop for ptxas)
template <int SITE = 0>
__device__ __forceinline__ void wait_prog(uint32_t a, int target) {
#ifdef LOB_SPLIT_STATS
    unsigned long long it = 0;
    while (__reduce_min_sync(FULL, lds_acq(a) >= target ? 1u : 0u) == 0u) ++it;
    if ((threadIdx.x & 31) == 0) {
        atomicAdd(&g_split_stats[SITE][0], 1ull);
        if (it) { atomicAdd(&g_split_stats[SITE][1], 1ull); atomicAdd(&g_split_stats[SITE][2], it); }
    }
#else
    while (__reduce_min_sync(FULL, lds_acq(a) >= target ? 1u : 0u) == 0u) {
#if LOB_SPLIT_SLEEP
        __nanosleep(LOB_SPLIT_SLEEP);  // leave the issue slots to the warps doing work
#endif
    }
#endif
}

// The warp of side X of book b.  Y = the other side.
template <int KPL, int X>
__device__ __forceinline__ void split_side(const Params &p, unsigned char *region, int lb, int tid) {
    using BK = RegBook<KPL, 1>;
    using SL = SplitLayout<KPL>;
    constexpr int Y = 1 - X, NP = BK::NP;
    const uint32_t r0 = smem_u32(region);
    const uint32_t stage = r0 + SL::STAGE + X * 2 * CH * 32;
    const uint32_t bars = r0 + SL::BARS + 16 * X;
    const uint32_t sc = r0 + SL::SCR + 128 * X;
    const uint32_t prog_me = r0 + SL::SYN + 4 * X, prog_ot = r0 + SL::SYN + 4 * Y;
    const uint32_t fill_me = r0 + SL::SYN + 8 + 4 * X, fill_ot = r0 + SL::SYN + 8 + 4 * Y;
    const uint32_t ring_me = r0 + SL::RING + X * SPLIT_RING * 8, ring_ot = r0 + SL::RING + Y * SPLIT_RING * 8;
    const int b = p.book0 + lb;
    const int nmsg = p.n_steps * p.M;
    const int nchunks = (nmsg + CH - 1) / CH;
    const int4 *src = reinterpret_cast<const int4 *>(p.msgs + (size_t)lb * nmsg * 8);
    if (tid == 0) {
        fence_proxy_async();
#pragma unroll
        for (int c = 0; c < 2; ++c) {
            if (c < nchunks) {
                const int cnt = min(CH, nmsg - c * CH);
                mbar_arrive_expect_tx(bars + 8 * c, cnt * 32);
                bulk_g2s(stage + c * CH * 32, src + (size_t)c * CH * 2, cnt * 32, bars + 8 * c);
            }
        }
    }
    Engine<BK, false, true, false, (KPL <= 8)> e(p);
    e.bk.cold = r0 + SL::COLD;  // [2][NP] records: rec(X, slot) is this side's
    e.bk.tid = tid;
    e.tid = tid; e.book = b; e.ntr = 0; e.sc = sc; e.xph = 0;
    e.scp = region + SL::SCR + 128 * X;
    e.part_cxl = 0; e.part_trd = 0;
    e.lastPs = 0;
    {   // this side of the book (RegBook::load, one side)
        const int32_t *g = p.book + (size_t)b * 2 * NF * NP + X * NF * NP;
#pragma unroll
        for (int f = 0; f < 3; ++f)
#pragma unroll
            for (int j = 0; j < KPL; ++j) e.bk.v[X][f][j] = __ldcs(g + f * NP + j * 32 + tid);
#pragma unroll
        for (int j = 0; j < KPL; ++j) {
            const int *r = g + j * 32 + tid;
            e.bk.put_cold(X, j * 32 + tid, __ldcs(r + F_TID * NP), __ldcs(r + F_TS * NP), __ldcs(r + F_TNS * NP));
        }
        __syncwarp();
    }
    e.hr[X] = e.template top_row<X>();
    e.hr[Y] = KPL - 1;
    e.flb[0] = e.flb[1] = 0;
    e.frm[0] = e.frm[1] = NP;
    e.bslot[X] = e.bslot[Y] = BEST_INVALID;
    e.bP[X] = e.bP[Y] = 0;
    e.bV[0] = e.bV[1] = 0;
    // bound on side Y's best price: X = BID keeps a lower bound of the best ask (a bid at
    // P < bound cannot trade), X = ASK an upper bound of the best bid; "unknown" never
    // decides (prices are >= 1, G22)
    constexpr int UNKNOWN_Y = (Y == ASK) ? 0 : INT_MAX;     // bound on Y as X reads it
    constexpr int UNKNOWN_X = (X == ASK) ? 0 : INT_MAX;     // bound on X as Y reads it
    int ob = UNKNOWN_Y;
    int myfills = 0;
    int left = p.M, step = 0, mi = 0;
    for (int c = 0; c < nchunks; ++c) {
        const uint32_t slot = c & 1;
        // ring reuse window: entry i % 64 is rewritten at message i + 64, so the other
        // warp must be past message 32 (c - 1) - 1 before this warp starts chunk c
        if (c >= 2) {
            sts_rel_if0(tid, prog_me, mi);
            wait_prog<0>(prog_ot, CH * (c - 1));
        }
        mbar_wait(bars + 8 * slot, (c >> 1) & 1);
        const uint32_t mbase = stage + slot * CH * 32;
        int cnt = min(CH, nmsg - c * CH);
        // decode lane-parallel (lane k: message k of the chunk), then ONE vote picks the
        // messages this side acts on: its own cancels and limits, and every aggressive order
        // of the other side (matched against this side).  The other side's cancels, this
        // side's market orders (nothing rests) and padding are never visited.
        unsigned rel;
        {
            int dc = MC_PAD;
            if (tid < cnt) {
                const uint32_t m = mbase + 32u * (uint32_t)tid;
                const int4 d = msg_decode(lds128(m));
                sts32(m, d.x);
                sts32(m + 12u, d.w);
                dc = d.x;
            }
            const bool act = dc >= MC_CANCEL;
            const bool mine = (((dc & MC_BID) != 0) == (X == BID));
            const bool aggr = (dc & MC_AGGR) != 0, mkt = (dc & MC_MKT) != 0;
            // every ring slot gets an entry of its pass each pass, so a slot never holds one
            // two passes old (which would carry the same parity bit): messages the other warp
            // never reads get a dummy entry here; the other side's aggressive orders get
            // theirs when matched (the other warp finished chunk c - 2, the slot's previous
            // user: window above)
            if (tid < cnt && !(act && !mine && aggr)) {
                const int mk = c * CH + tid;
                sts64_if0(0, ring_me + 8u * (uint32_t)(mk & (SPLIT_RING - 1)),
                          (unsigned long long)((unsigned)(mk / SPLIT_RING) & 1u) << 31);
            }
            rel = __ballot_sync(FULL, act && (mine ? !(aggr && mkt) : aggr));
            if constexpr (X == ASK) {                                   // malformed (G22), counted once
                const int nbad = __popc(__ballot_sync(FULL, dc == MC_BAD));
                if (nbad && tid == 0) e.count(ST_BAD, nbad);
            }
        }
        __syncwarp();
        int k0 = 0;
        while (cnt > 0) {
            const int run = min(cnt, left);
            unsigned todo = rel & (run >= 32 ? FULL : (((1u << run) - 1u) << k0));
            while (todo != 0u) {
                const int k = __ffs(todo) - 1;
                todo &= todo - 1u;
                mi = c * CH + k;
                const uint32_t maddr = mbase + 32u * (uint32_t)k;
                const int4 a = lds128(maddr), bb = lds128(maddr + 16);
#ifdef LOB_SPLIT_STATS
                const long long t0 = clock64();
                int cls = 0;
#define SPLIT_CLS(x) cls = (x)
#else
#define SPLIT_CLS(x)
#endif
                const int code = a.x, Q = a.z, P = a.w;
                const bool bid = (code & MC_BID) != 0;
                if ((code & MC_AGGR) == 0) {                           // own cancel / delete
                    SPLIT_CLS(1);
                    e.template cancel<X>(Q, P, bb.x);
                } else if (bid == (X == BID)) {                        // own limit: its remainder rests here
                    int Qa = Q;
                    const bool sure = (X == BID) ? (P < ob) : (P > ob);
                    SPLIT_CLS(2);
                    if (!sure) {                                       // may trade: the other warp decides
                        SPLIT_CLS(3);
                        sts_rel_if0(tid, prog_me, mi);                 // (the other warp may wait on us)
                        const uint32_t ra = ring_ot + 8u * (uint32_t)(mi & (SPLIT_RING - 1));
                        const unsigned gen = (unsigned)(mi / SPLIT_RING) & 1u;
                        unsigned long long r = lds64v(ra);
                        while (__reduce_min_sync(FULL, (((unsigned)r >> 31) & 1u) == gen ? 1u : 0u) == 0u) r = lds64v(ra);
                        Qa = (int)((unsigned)r & (unsigned)INT_MAX);
                        ob = (int)(unsigned)(r >> 32);
                        SPLIT_CLS(Qa == Q ? 4 : 3);
                    }
                    if (Qa > 0) e.with_rows(e.hr[X], [&](auto R) {
                        e.template add_r<X, decltype(R)::value>(Qa, P, bb.x, bb.y, bb.z, bb.w);
                    });
                } else {                                               // the other side aggresses: fills here
                    if ((code & MC_MKT) == 0) ob = (X == ASK) ? max(ob, P) : min(ob, P);
                    int Qa = Q;
                    SPLIT_CLS(6);
                    const bool no_fill = e.bslot[X] != BEST_INVALID && (X == ASK ? (P < e.bP[X]) : (P > e.bP[X]));
                    e.lastPs = UNKNOWN_X;
                    if (!no_fill && Qa > 0) {
                        // trades stay in message order (Eq.4) -- unless the log is already
                        // full: the other warp's count only grows, so once this sum reaches
                        // T_cap no later fill is logged (G8) and only the counts matter
                        SPLIT_CLS(7);
                        if (myfills + lds32(fill_ot) < p.Tcap) {
                            sts_rel_if0(tid, prog_me, mi);
                            wait_prog<2>(prog_ot, mi);
                        }
                        e.ntr = myfills + lds32(fill_ot);
                        const int n0 = e.ntr;
                        e.with_rows(e.hr[X], [&](auto R) {
                            Qa = e.template fill_r<Y, decltype(R)::value>(P, Qa, bb.x, bb.z, bb.w);
                        });
                        myfills += e.ntr - n0;
                        sts32_if0(tid, fill_me, myfills);
                    }
                    if ((code & MC_MKT) != 0 && Qa > 0 && tid == 0) e.count(ST_DISCARDED, Qa);
                    const int after = e.bslot[X] == BEST_INVALID ? e.lastPs : e.bP[X];
                    // the ring entry: one 64-bit store, single-copy atomic -- Q_a' >= 0 with
                    // the pass parity of message mi in bit 31 (the reader's flag), the bound
                    const unsigned gen = (unsigned)(mi / SPLIT_RING) & 1u;
                    sts64_if0(tid, ring_me + 8u * (uint32_t)(mi & (SPLIT_RING - 1)),
                              ((unsigned long long)(unsigned)after << 32) | (gen << 31) | (unsigned)(Qa > 0 ? Qa : 0));
                }
#ifdef LOB_SPLIT_STATS
                if (tid == 0 && lb < 8 && mi < 10240) g_split_trace[lb][X][mi] = ((clock64() - t0) << 4) | cls;
#endif
            }
            k0 += run;
            cnt -= run;
            left -= run;
            if (left == 0) {                                           // step end: this side's L2 (G23)
                left = p.M;
                if (p.l2out) {
                    int op, oq;
                    e.template l2_side<X>(p.L, op, oq);
                    int32_t *dst = p.l2out + (((size_t)lb * p.n_steps + step) * p.L) * 4 + 2 * X;
                    if (tid < p.L) *reinterpret_cast<int2 *>(dst + 4 * tid) = make_int2(op, oq);
                }
                ++step;
            }
        }
        mi = c * CH + k0;
        sts_rel_if0(tid, prog_me, mi);  // chunk done: progress for the other warp's waits
        __syncwarp();
        if (tid == 0 && c + 2 < nchunks) {
            fence_proxy_async();
            const int cn = min(CH, nmsg - (c + 2) * CH);
            mbar_arrive_expect_tx(bars + 8 * slot, cn * 32);
            bulk_g2s(stage + slot * CH * 32, src + (size_t)(c + 2) * CH * 2, cn * 32, bars + 8 * slot);
        }
    }
    {   // this side back to HBM (RegBook::store, one side)
        int32_t *g = p.book + (size_t)b * 2 * NF * NP + X * NF * NP;
#pragma unroll
        for (int j = 0; j < KPL; ++j) {
            const bool occ = e.bk.v[X][F_Q][j] > 0;
            int *r = g + j * 32 + tid;
#pragma unroll
            for (int f = 0; f < 3; ++f) __stcs(r + f * NP, occ ? e.bk.v[X][f][j] : -1);
            const int4 cr = lds128(e.bk.rec(X, j * 32 + tid));
            __stcs(r + F_TID * NP, occ ? cr.y : -1);
            __stcs(r + F_TS * NP, occ ? cr.z : -1);
            __stcs(r + F_TNS * NP, occ ? cr.w : -1);
        }
    }
    long long cx = e.part_cxl, tq = e.part_trd;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        cx += __shfl_xor_sync(FULL, cx, o);
        tq += __shfl_xor_sync(FULL, tq, o);
    }
    __syncwarp();
    if (tid == 0) {
        e.count(ST_CANCELLED_QTY, cx);
        e.count(ST_TRADED_QTY, tq);
        e.count(ST_TRADES, myfills);
    }
}

template <int KPL, int G>
__global__ void __launch_bounds__(64 * G) lob_step_split(const Params p) {
    using SL = SplitLayout<KPL>;
    extern __shared__ __align__(128) unsigned char dyn[];
    const int warp = (int)__reduce_min_sync(FULL, threadIdx.x / 32);  // uniform (see lob_step)
    const int g = warp >> 1, side = warp & 1;
    const int tid = (int)opaque(threadIdx.x % 32);
    unsigned char *region = dyn + g * SL::BYTES;
    const uint32_t r0 = smem_u32(region);
    const int lb = blockIdx.x * G + g;
    if (tid < NST) sts64(r0 + SL::SCR + 128 * side + 8u * tid, 0);
    if (tid == 0) {
        mbar_init(r0 + SL::BARS + 16 * side, 1);
        mbar_init(r0 + SL::BARS + 16 * side + 8, 1);
        sts32(r0 + SL::SYN + 4 * side, 0);
        sts32(r0 + SL::SYN + 8 + 4 * side, 0);
        fence_mbar_init();
    }
    // ring entries start with parity 1: message i of the first pass (parity 0) is absent
    for (int k = tid; k < SPLIT_RING; k += 32) sts64_if0(0, r0 + SL::RING + side * SPLIT_RING * 8 + 8u * k, 1ull << 31);
    __syncthreads();
    if (lb < p.nb) {
        if (side == ASK) split_side<KPL, ASK>(p, region, lb, tid);
        else split_side<KPL, BID>(p, region, lb, tid);
    }
    __syncthreads();
    if (lb < p.nb && side == ASK && tid < NST) {   // both sides' counters, once per book
        const int b = p.book0 + lb;
        long long v = lds64(r0 + SL::SCR + 8u * tid) + lds64(r0 + SL::SCR + 128 + 8u * tid);
        const int fills = lds32(r0 + SL::SCR + 8u * ST_TRADES) + lds32(r0 + SL::SCR + 128 + 8u * ST_TRADES);
        const int logged = min(fills, p.Tcap);
        if (tid == ST_DROPPED) v += fills - logged;
        if (tid == ST_MSGS) v += p.n_steps * p.M;
        p.stats[(size_t)b * NST + tid] += v;
        if (tid == 0) p.ntrades[b] = logged;
    }
}

}  // namespace lobk
