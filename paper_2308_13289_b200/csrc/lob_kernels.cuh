// lob_kernels.cuh -- sm_100a device code for the batched limit-order-book hot path.
//
// One warp owns one book (messages within a book are strictly
// serial; books are independent).  The book's two sides (Eq.1) are
// held in REGISTERS for capacity N <= 128 (RegBook, KPL = slots per lane) and
// in SHARED MEMORY above that (SmemBook).  Slot i of a side lives in lane
// (i % 32), register/row (i / 32) -- "interleaved", so that every
// lowest-index search (free slot P:L175 / G3, order-id lookup P:L177) is a
// ballot + find-first-set per row, and the lowest-slot tie-break of the best
// order (G4) is the lowest set lane of the first row that has a candidate.
//
// Messages (Eq.6) stream HBM -> shared memory through a per-warp double buffer
// filled by 1-D bulk async copies (cp.async.bulk, the TMA bulk path, SASS
// UBLKCP) completing on an mbarrier; every lane reads the current message
// with two broadcast 16-byte shared loads.  Dispatch is warp-uniform on
// (T, S) -- the paper's 8 explicit cases -- so no lane diverges.
//
// The best standing order per side (Eq.5 + G1/G4) is cached (warp-uniform)
// and recomputed with __reduce_min_sync / __ballot_sync only when the cached
// order leaves the book; adds update it by one key comparison.
//
// Counters: lane c owns counter c (int64), so an increment is one predicated
// add and no per-counter register is spent on every lane.
#pragma once
#include <climits>
#include <cstdint>
#include <cuda_runtime.h>

namespace lobk {

constexpr unsigned FULL = 0xffffffffu;
enum { F_P = 0, F_Q, F_OID, F_TID, F_TS, F_TNS, NF };  // Eq.2 field order
enum { ASK = 0, BID = 1 };                               // side 0 = A, side 1 = B
enum {
    ST_MSGS = 0, ST_BAD, ST_TRADES, ST_DROPPED, ST_TRADED_QTY, ST_CANCELLED_QTY, ST_UNKNOWN,
    ST_ADD_OVF, ST_OVF_QTY, ST_DISCARDED, NST
};
constexpr int CH = 64;  // messages per staging chunk (2 KiB); two chunks per warp

struct Params {
    int32_t *book;         // [K][2][NF][NP] SoA, slot i at [i] (i = row*32 + lane)
    int32_t *trades;       // [K][Tcap][6]
    int32_t *ntrades;      // [K]
    long long *stats;      // [K][NST]
    const int32_t *msgs;   // [nb][n_steps*M][8]  (relative to book0)
    int32_t *l2out;        // [nb][n_steps][L][4] or null (relative to book0)
    int N, NP, Tcap, L, n_steps, M;
    int book0, nb;         // books [book0, book0+nb) of the state
};

// ------------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "LAB_WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra LAB_WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
// 1-D bulk copy global -> shared (TMA bulk engine), completes tx bytes on `bar`
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

// ---------------------------------------------------------------- book storage
// RegBook: v[s][f][j] is slot (j*32 + lane) of side s.  All indices in loops
// are compile-time after unrolling; runtime (warp-uniform) rows go through
// select chains so nothing spills to local memory.
template <int KPL_>
struct RegBook {
    static constexpr int KPL = KPL_;
    int32_t v[2][NF][KPL_];
    __device__ __forceinline__ int32_t at(int s, int f, int j) const { return v[s][f][j]; }
    __device__ __forceinline__ int32_t get(int s, int f, int j) const {
        int32_t r = v[s][f][0];
#pragma unroll
        for (int jj = 1; jj < KPL_; ++jj)
            if (j == jj) r = v[s][f][jj];
        return r;
    }
    __device__ __forceinline__ void put(int s, int f, int j, int32_t x) {
#pragma unroll
        for (int jj = 0; jj < KPL_; ++jj)
            if (j == jj) v[s][f][jj] = x;
    }
    __device__ __forceinline__ void load(const int32_t *g, int NP, int lane) {
#pragma unroll
        for (int s = 0; s < 2; ++s)
#pragma unroll
            for (int f = 0; f < NF; ++f)
#pragma unroll
                for (int j = 0; j < KPL_; ++j) v[s][f][j] = __ldcs(g + (s * NF + f) * NP + j * 32 + lane);
    }
    __device__ __forceinline__ void store(int32_t *g, int NP, int lane) const {
#pragma unroll
        for (int s = 0; s < 2; ++s)
#pragma unroll
            for (int j = 0; j < KPL_; ++j) {
                const bool occ = v[s][F_Q][j] > 0;
#pragma unroll
                for (int f = 0; f < NF; ++f) __stcs(g + (s * NF + f) * NP + j * 32 + lane, occ ? v[s][f][j] : -1);
            }
    }
};

// SmemBook: the same interleaved layout in this warp's shared-memory region.
template <int KPL_>
struct SmemBook {
    static constexpr int KPL = KPL_;
    int32_t *base;  // already offset by lane
    __device__ __forceinline__ int32_t at(int s, int f, int j) const { return base[(s * NF + f) * (KPL_ * 32) + j * 32]; }
    __device__ __forceinline__ int32_t get(int s, int f, int j) const { return at(s, f, j); }
    __device__ __forceinline__ void put(int s, int f, int j, int32_t x) { base[(s * NF + f) * (KPL_ * 32) + j * 32] = x; }
    __device__ __forceinline__ void load(const int32_t *g, int NP, int lane) {
        for (int i = 0; i < 2 * NF * KPL_; ++i) base[i * 32] = g[i * 32 + lane];
        __syncwarp();
    }
    __device__ __forceinline__ void store(int32_t *g, int NP, int lane) const {
        __syncwarp();
        for (int s = 0; s < 2; ++s)
            for (int j = 0; j < KPL_; ++j) {
                const bool occ = at(s, F_Q, j) > 0;
                for (int f = 0; f < NF; ++f) g[(s * NF + f) * NP + j * 32 + lane] = occ ? at(s, f, j) : -1;
            }
    }
};

// ------------------------------------------------------------------ the engine
template <class BK>
struct Engine {
    static constexpr int KPL = BK::KPL;
    BK bk;
    int lane, N, Tcap, ntr;
    int32_t *tlog;  // this book's trade log [Tcap][6]
    // warp-uniform best-order cache per side (Eq.5 + G1/G4)
    int bslot[2], bP[2], bTS[2], bTNS[2];
    bool bval[2];
    long long cnt;       // lane c owns counter c
    long long part_cxl;  // cancelled quantity accumulated on the owner lane

    __device__ __forceinline__ void add_cnt(int c, long long x) {
        if (lane == c) cnt += x;
    }
    __device__ __forceinline__ bool valid(int j) const { return j * 32 + lane < N; }

    // Best(o_s) of side SD over occupied slots: price (ask min / bid max,
    // Eq.5 + G1), then earliest (Ts, Tns), then lowest slot (G4).
    template <int SD>
    __device__ __forceinline__ void recompute_best() {
        int lk = INT_MAX, lts = 0, ltns = 0, lj = -1;
#pragma unroll
        for (int j = 0; j < KPL; ++j) {
            if (bk.at(SD, F_Q, j) > 0) {
                const int p = bk.at(SD, F_P, j);
                const int k = (SD == ASK) ? p : ~p;  // bids: larger price = smaller key
                const int ts = bk.at(SD, F_TS, j), tns = bk.at(SD, F_TNS, j);
                const bool better = (lj < 0) || k < lk || (k == lk && (ts < lts || (ts == lts && tns < ltns)));
                if (better) { lk = k; lts = ts; ltns = tns; lj = j; }
            }
        }
        const bool has = lj >= 0;
        if (!__any_sync(FULL, has)) { bval[SD] = true; bslot[SD] = -1; return; }
        const int m = __reduce_min_sync(FULL, has ? lk : INT_MAX);
        unsigned c = __ballot_sync(FULL, has && lk == m);
        if (c & (c - 1)) {
            const bool in = (c >> lane) & 1u;
            const int t = __reduce_min_sync(FULL, in ? lts : INT_MAX);
            c = __ballot_sync(FULL, in && lts == t);
            if (c & (c - 1)) {
                const bool in2 = (c >> lane) & 1u;
                const int t2 = __reduce_min_sync(FULL, in2 ? ltns : INT_MAX);
                c = __ballot_sync(FULL, in2 && ltns == t2);
            }
        }
        int slot;
        if (c & (c - 1)) {
            const bool in3 = (c >> lane) & 1u;
            slot = (int)__reduce_min_sync(FULL, in3 ? (unsigned)(lj * 32 + lane) : 0xffffffffu);
        } else {
            const int w = __ffs(c) - 1;
            slot = __shfl_sync(FULL, lj, w) * 32 + w;
        }
        const int w = slot & 31;
        bslot[SD] = slot;
        bP[SD] = (SD == ASK) ? m : ~m;
        bTS[SD] = __shfl_sync(FULL, lts, w);
        bTNS[SD] = __shfl_sync(FULL, ltns, w);
        bval[SD] = true;
    }

    // A new order at `slot` on side SD: keep the cache exact (G4 key order).
    template <int SD>
    __device__ __forceinline__ void note_add(int slot, int p, int ts, int tns) {
        if (!bval[SD]) return;
        if (bslot[SD] < 0) {
            bslot[SD] = slot; bP[SD] = p; bTS[SD] = ts; bTNS[SD] = tns;
            return;
        }
        const int kn = (SD == ASK) ? p : ~p, kb = (SD == ASK) ? bP[SD] : ~bP[SD];
        const bool better =
            kn < kb ||
            (kn == kb && (ts < bTS[SD] || (ts == bTS[SD] && (tns < bTNS[SD] || (tns == bTNS[SD] && slot < bslot[SD])))));
        if (better) { bslot[SD] = slot; bP[SD] = p; bTS[SD] = ts; bTNS[SD] = tns; }
    }

    // Cancellation (cancel == delete P:L289): lowest occupied slot with
    // OID == msg OID on the message's side (G16), else the lowest synthetic
    // order (OID <= -9000, G12) at the message price.
    template <int SD>
    __device__ __forceinline__ void cancel(int mQ, int mP, int mOID) {
        if (mQ <= 0) { add_cnt(ST_BAD, 1); return; }  // G22
        int slot = -1;
#pragma unroll
        for (int j = 0; j < KPL; ++j) {
            const unsigned f = __ballot_sync(FULL, bk.at(SD, F_Q, j) > 0 && bk.at(SD, F_OID, j) == mOID);
            if (slot < 0 && f) slot = j * 32 + __ffs(f) - 1;
        }
        if (slot < 0) {
#pragma unroll
            for (int j = 0; j < KPL; ++j) {
                const unsigned f = __ballot_sync(FULL, bk.at(SD, F_Q, j) > 0 && bk.at(SD, F_OID, j) <= -9000 &&
                                                           bk.at(SD, F_P, j) == mP);
                if (slot < 0 && f) slot = j * 32 + __ffs(f) - 1;
            }
        }
        if (slot < 0) { add_cnt(ST_UNKNOWN, 1); return; }  // G15
        const int oj = slot >> 5;
        if (lane == (slot & 31)) {
            const int qi = bk.get(SD, F_Q, oj);
            part_cxl += (mQ < qi) ? mQ : qi;  // G14
            bk.put(SD, F_Q, oj, qi - mQ);     // Q <= 0 -> empty
        }
        if (bval[SD] && bslot[SD] == slot) bval[SD] = false;
    }

    // Limit (T=1) or market (T=4) order of side OWN.
    template <int OWN, bool MARKET>
    __device__ __forceinline__ void aggress(int mQ, int mP, int mOID, int mTID, int mTS, int mTNS) {
        constexpr int OPP = 1 - OWN;
        if (!MARKET && mP <= 0) { add_cnt(ST_BAD, 1); return; }  // G22
        const int Pa = MARKET ? (OWN == BID ? INT_MAX : 0) : mP;   // P_m = 0 / max_int (G18)
        int Qa = mQ;
        while (Qa > 0) {
            if (!bval[OPP]) recompute_best<OPP>();
            if (bslot[OPP] < 0) break;                              // side empty
            const int Ps = bP[OPP];
            if (OWN == BID ? (Pa < Ps) : (Pa > Ps)) break;          // prices do not overlap
            const int s = bslot[OPP], ol = s & 31, oj = s >> 5;
            const int Qs = __shfl_sync(FULL, bk.get(OPP, F_Q, oj), ol);
            const int Qs2 = (Qs - Qa > 0) ? (Qs - Qa) : 0;            // Q_s' = max(0, Q_s - Q_a)
            const int q = Qs - Qs2;                                   // Q_j = Q_s - Q_s'
            Qa = Qa - Qs;                                             // Q_a' = Q_a - Q_s
            if (ntr < Tcap) {                                         // Eq.3 record, Eq.4 cap (G8)
                if (lane == ol) {
                    int2 *t = reinterpret_cast<int2 *>(tlog + (size_t)ntr * 6);
                    t[0] = make_int2(Ps, q);
                    t[1] = make_int2(mOID, bk.get(OPP, F_OID, oj));
                    t[2] = make_int2(mTS, mTNS);
                }
                ++ntr;
            } else {
                add_cnt(ST_DROPPED, 1);
            }
            add_cnt(ST_TRADED_QTY, q);
            if (lane == ol) bk.put(OPP, F_Q, oj, Qs2);              // filled order removed (G10)
            if (Qs2 == 0) bval[OPP] = false;
        }
        if (!MARKET) {
            if (Qa > 0) {                                            // remainder rests
                int slot = -1;
#pragma unroll
                for (int j = 0; j < KPL; ++j) {
                    const unsigned f = __ballot_sync(FULL, valid(j) && bk.at(OWN, F_Q, j) <= 0);
                    if (slot < 0 && f) slot = j * 32 + __ffs(f) - 1;  // lowest empty slot (G3)
                }
                if (slot < 0) {                                      // side saturated (G6)
                    add_cnt(ST_ADD_OVF, 1);
                    add_cnt(ST_OVF_QTY, Qa);
                } else {
                    const int oj = slot >> 5;
                    if (lane == (slot & 31)) {                       // G27
                        bk.put(OWN, F_P, oj, mP); bk.put(OWN, F_Q, oj, Qa); bk.put(OWN, F_OID, oj, mOID);
                        bk.put(OWN, F_TID, oj, mTID); bk.put(OWN, F_TS, oj, mTS); bk.put(OWN, F_TNS, oj, mTNS);
                    }
                    note_add<OWN>(slot, mP, mTS, mTNS);
                }
            }
        } else if (Qa > 0) {
            add_cnt(ST_DISCARDED, Qa);
        }
    }

    __device__ __forceinline__ void message(const int4 a, const int4 b) {
        const int T = a.x, S = a.y, Q = a.z, P = a.w;
        if (T == 0) return;                                          // padding (G21)
        // the paper's 8 (type x side) cases; cancel and delete share one
        const unsigned t = (unsigned)(T - 1);
        const int c = (S == 1) ? 0 : (S == -1) ? 1 : 2;
        if (t > 3u || c == 2) { add_cnt(ST_BAD, 1); return; }          // G22
        switch (t * 2 + c) {
            case 0: aggress<BID, false>(Q, P, b.x, b.y, b.z, b.w); break;
            case 1: aggress<ASK, false>(Q, P, b.x, b.y, b.z, b.w); break;
            case 2:
            case 4: cancel<BID>(Q, P, b.x); break;
            case 3:
            case 5: cancel<ASK>(Q, P, b.x); break;
            case 6: aggress<BID, true>(Q, P, b.x, b.y, b.z, b.w); break;
            default: aggress<ASK, true>(Q, P, b.x, b.y, b.z, b.w); break;
        }
    }

    // L2 (G23): k-th best distinct price per side and its summed quantity;
    // lane k keeps level k.  Absent levels are (-1, 0).
    template <int SD>
    __device__ __forceinline__ void l2_side(int L, int &outp, int &outq) const {
        outp = -1; outq = 0;
        int prev = 0;
        bool have_prev = false;
        for (int k = 0; k < L; ++k) {
            int lk = INT_MAX;
            bool lf = false;
#pragma unroll
            for (int j = 0; j < KPL; ++j) {
                if (bk.at(SD, F_Q, j) > 0) {
                    const int p = bk.at(SD, F_P, j);
                    const int key = (SD == ASK) ? p : ~p;
                    if ((!have_prev || key > prev) && (!lf || key < lk)) { lk = key; lf = true; }
                }
            }
            if (!__any_sync(FULL, lf)) break;
            const int m = __reduce_min_sync(FULL, lf ? lk : INT_MAX);
            unsigned lq = 0;
#pragma unroll
            for (int j = 0; j < KPL; ++j) {
                const int p = bk.at(SD, F_P, j);
                const int key = (SD == ASK) ? p : ~p;
                if (bk.at(SD, F_Q, j) > 0 && key == m) lq += (unsigned)bk.at(SD, F_Q, j);
            }
            const unsigned qs = __reduce_add_sync(FULL, lq);
            if (lane == k) { outp = (SD == ASK) ? m : ~m; outq = (int)qs; }
            prev = m;
            have_prev = true;
        }
    }
    __device__ __forceinline__ void l2_write(int32_t *dst, int L) const {
        int ap, aq, bp, bq;
        l2_side<ASK>(L, ap, aq);
        l2_side<BID>(L, bp, bq);
        if (lane < L) reinterpret_cast<int4 *>(dst)[lane] = make_int4(ap, aq, bp, bq);
    }
};

// ------------------------------------------------------------------ step kernel
// Persistent: each warp walks books w, w + total_warps, ...
template <class BK, int WARPS>
__device__ __forceinline__ void run_books(const Params &p, BK &bk, int32_t *stage /*[2][CH][8]*/, uint64_t *bars,
                                          uint32_t &chunk_seq) {
    const int lane = threadIdx.x & 31;
    const int gw = blockIdx.x * WARPS + (threadIdx.x >> 5);
    const int nw = gridDim.x * WARPS;
    const int nmsg = p.n_steps * p.M;
    const int nchunks = (nmsg + CH - 1) / CH;
    for (int lb = gw; lb < p.nb; lb += nw) {
        const int b = p.book0 + lb;
        const int4 *src = reinterpret_cast<const int4 *>(p.msgs + (size_t)lb * nmsg * 8);
        // prologue: first two chunks in flight before the book is even loaded
        __syncwarp();
        if (lane == 0) {
            fence_proxy_async();  // previous generic reads of the buffers before async writes
#pragma unroll
            for (int c = 0; c < 2; ++c) {
                if (c < nchunks) {
                    const uint32_t slot = (chunk_seq + c) & 1;
                    const int cnt = min(CH, nmsg - c * CH);
                    mbar_arrive_expect_tx(&bars[slot], cnt * 32);
                    bulk_g2s(stage + slot * CH * 8, src + (size_t)c * CH * 2, cnt * 32, &bars[slot]);
                }
            }
        }
        Engine<BK> e;
        e.bk = bk;
        e.bk.load(p.book + (size_t)b * 2 * NF * p.NP, p.NP, lane);
        e.lane = lane; e.N = p.N; e.Tcap = p.Tcap; e.ntr = 0;
        e.tlog = p.trades + (size_t)b * p.Tcap * 6;
        e.bval[0] = e.bval[1] = false;
        e.bslot[0] = e.bslot[1] = -1;
        e.bP[0] = e.bP[1] = e.bTS[0] = e.bTS[1] = e.bTNS[0] = e.bTNS[1] = 0;
        e.cnt = 0; e.part_cxl = 0;
        int left = p.M, step = 0;
        for (int c = 0; c < nchunks; ++c) {
            const uint32_t seq = chunk_seq + c, slot = seq & 1;
            mbar_wait(&bars[slot], (seq >> 1) & 1);
            const int4 *buf = reinterpret_cast<const int4 *>(stage + slot * CH * 8);
            const int cnt = min(CH, nmsg - c * CH);
            for (int i = 0; i < cnt; ++i) {
                const int4 a = buf[2 * i], bb = buf[2 * i + 1];
                e.message(a, bb);
                if (--left == 0) {                     // end of a step: L2 snapshot (G23)
                    left = p.M;
                    if (p.l2out) e.l2_write(p.l2out + (((size_t)lb * p.n_steps + step) * p.L) * 4, p.L);
                    ++step;
                }
            }
            __syncwarp();
            if (lane == 0 && c + 2 < nchunks) {      // refill this buffer with chunk c+2
                fence_proxy_async();
                const int cn = min(CH, nmsg - (c + 2) * CH);
                mbar_arrive_expect_tx(&bars[slot], cn * 32);
                bulk_g2s(stage + slot * CH * 8, src + (size_t)(c + 2) * CH * 2, cn * 32, &bars[slot]);
            }
        }
        chunk_seq += nchunks;
        // writeback: book, trade count, counters (msgs += nmsg; trades = logged + dropped)
        e.bk.store(p.book + (size_t)b * 2 * NF * p.NP, p.NP, lane);
        long long cx = e.part_cxl;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) cx += __shfl_xor_sync(FULL, cx, o);
        const long long dropped = __shfl_sync(FULL, e.cnt, ST_DROPPED);
        if (lane == ST_CANCELLED_QTY) e.cnt += cx;
        if (lane == ST_MSGS) e.cnt += nmsg;
        if (lane == ST_TRADES) e.cnt += e.ntr + dropped;
        if (lane < NST) p.stats[(size_t)b * NST + lane] += e.cnt;
        if (lane == 0) p.ntrades[b] = e.ntr;
        bk = e.bk;  // keep the smem base pointer for the next book
    }
}

template <int KPL, int WARPS>
__global__ void __launch_bounds__(WARPS * 32) lob_step_reg(const Params p) {
    __shared__ __align__(128) int32_t stage[WARPS][2][CH][8];
    __shared__ __align__(8) uint64_t bars[WARPS][2];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0) {
        mbar_init(&bars[w][0], 1);
        mbar_init(&bars[w][1], 1);
        fence_mbar_init();
    }
    __syncwarp();
    uint32_t seq = 0;
    RegBook<KPL> bk;
    run_books<RegBook<KPL>, WARPS>(p, bk, &stage[w][0][0][0], bars[w], seq);
}

template <int KPL>
__global__ void __launch_bounds__(32) lob_step_smem(const Params p) {
    extern __shared__ __align__(128) int32_t dyn[];
    int32_t *stage = dyn;                                          // [2][CH][8]
    uint64_t *bars = reinterpret_cast<uint64_t *>(dyn + 2 * CH * 8);
    int32_t *bookmem = dyn + 2 * CH * 8 + 8;                       // [2][NF][KPL*32]
    const int lane = threadIdx.x & 31;
    if (lane == 0) {
        mbar_init(&bars[0], 1);
        mbar_init(&bars[1], 1);
        fence_mbar_init();
    }
    __syncwarp();
    uint32_t seq = 0;
    SmemBook<KPL> bk;
    bk.base = bookmem + lane;
    run_books<SmemBook<KPL>, 1>(p, bk, stage, bars, seq);
}

// ------------------------------------------------------------- init / exports
// a0: -1 everywhere, counters 0, then one synthetic order per
// populated L2 level (G24).  One warp per book.
__global__ void lob_init_kernel(int32_t *book, int32_t *trades, int32_t *ntrades, long long *stats, int K, int N,
                                int NP, int Tcap, const int32_t *init_l2, int L0, int ts, int tns) {
    const int lane = threadIdx.x & 31;
    const int b = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (b >= K) return;
    int32_t *bb = book + (size_t)b * 2 * NF * NP;
    for (int i = lane; i < 2 * NF * NP; i += 32) bb[i] = -1;
    int32_t *tb = trades + (size_t)b * Tcap * 6;
    for (int i = lane; i < Tcap * 6; i += 32) tb[i] = -1;
    if (lane == 0) ntrades[b] = 0;
    if (lane < NST) stats[(size_t)b * NST + lane] = 0;
    __syncwarp();
    if (!init_l2) return;
    const int32_t *rows = init_l2 + (size_t)b * L0 * 4;
    int oid_base = -9000;
    for (int s = 0; s < 2; ++s) {       // asks (s=0) best->worst, then bids
        int placed = 0;
        for (int r0 = 0; r0 < L0; r0 += 32) {
            const int r = r0 + lane;
            int p = 0, q = 0;
            if (r < L0) { p = rows[r * 4 + 2 * s]; q = rows[r * 4 + 2 * s + 1]; }
            const bool pop = r < L0 && p > 0 && q > 0;
            const unsigned m = __ballot_sync(FULL, pop);
            const int idx = placed + __popc(m & ((1u << lane) - 1));
            if (pop && idx < N) {
                int32_t *o = bb + s * NF * NP + idx;
                o[F_P * NP] = p; o[F_Q * NP] = q; o[F_OID * NP] = oid_base - idx;
                o[F_TID * NP] = -9000; o[F_TS * NP] = ts; o[F_TNS * NP] = tns;
            }
            placed += __popc(m);
        }
        oid_base -= placed;
    }
}

// book export: SoA (internal) -> [K][2][N][6] AoS; one thread per (book, side, slot)
__global__ void lob_export_book(const int32_t *book, int32_t *out, int K, int N, int NP) {
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= (long long)K * 2 * N) return;
    const int i = (int)(t % N);
    const long long bs = t / N;  // book*2 + side
    const int32_t *src = book + bs * NF * NP + i;
    const bool occ = src[F_Q * NP] > 0;
    int32_t *dst = out + t * 6;
#pragma unroll
    for (int f = 0; f < NF; ++f) dst[f] = occ ? src[f * NP] : -1;
}

// trades export: rows >= count become -1 here, not on the hot path
__global__ void lob_export_trades(const int32_t *trades, const int32_t *ntrades, int32_t *out, int32_t *counts, int K,
                                  int Tcap) {
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long total = (long long)K * Tcap * 6;
    if (t < total) {
        const long long b = t / ((long long)Tcap * 6);
        const int row = (int)((t / 6) % Tcap);
        out[t] = row < ntrades[b] ? trades[t] : -1;
    }
    if (counts && t < K) counts[t] = ntrades[t];
}

// current L2 of every book, computed from the stored state (warp per book)
template <int KPL>
__global__ void lob_export_l2_reg(const int32_t *book, int32_t *out, int K, int N, int NP, int L) {
    const int lane = threadIdx.x & 31;
    const int b = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (b >= K) return;
    Engine<RegBook<KPL>> e;
    e.lane = lane; e.N = N;
    e.bk.load(book + (size_t)b * 2 * NF * NP, NP, lane);
    e.l2_write(out + (size_t)b * L * 4, L);
}
template <int KPL>
__global__ void lob_export_l2_smem(const int32_t *book, int32_t *out, int K, int N, int NP, int L) {
    const int lane = threadIdx.x & 31;
    const int b = blockIdx.x;
    if (b >= K) return;
    Engine<SmemBook<KPL>> e;
    e.lane = lane; e.N = N;
    e.bk.base = const_cast<int32_t *>(book) + (size_t)b * 2 * NF * NP + lane;  // read in place (global)
    e.l2_write(out + (size_t)b * L * 4, L);
}

}  // namespace lobk
