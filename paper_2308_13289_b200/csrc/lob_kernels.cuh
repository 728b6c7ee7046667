// lob_kernels.cuh -- sm_100a device code for the batched limit-order-book hot path.
//
// One warp owns one book (messages within a book are strictly
// serial; books are independent).  Slot i of a side (Eq.1) lives in
// lane (i % 32), row (i / 32) -- "interleaved" -- so that:
//   * every lowest-index search (free slot P:L175/G3, order-id lookup P:L177,
//     lowest-slot tie-break G4) is one lane-local scan plus ONE __reduce_min_sync
//     over (row*32 + lane), which directly yields the warp-uniform slot;
//   * the row of a selected slot is warp-uniform, so register writes branch
//     on it (no per-lane select chains, no local memory).
// Fields the method scans on every message -- P, Q, OID (Eq.2) -- are held in
// REGISTERS for capacity N <= 128 (RegBook); the fields read only on rare
// paths -- TID, Ts, Tns -- live in a per-warp SHARED-MEMORY region, where any
// lane reads any slot with a broadcast load.  Above N = 128 the whole book is
// in shared memory (SmemBook).
//
// Messages (Eq.6) stream HBM -> shared memory through a per-warp double buffer
// filled by 1-D bulk async copies (cp.async.bulk: the TMA bulk path, SASS
// UBLKCP) completing on an mbarrier; every lane reads the current message with
// two broadcast 16-byte shared loads.  Dispatch is warp-uniform on (T, S) --
// the paper's 8 explicit cases -- so no lane diverges.
//
// The best standing order of each side (Eq.5 + G1/G4) is cached (warp-uniform)
// and recomputed with warp reductions only after the cached order leaves the
// book; an add updates it by one key comparison.
#pragma once
#include <climits>
#include <cstdint>
#include <cuda_runtime.h>

#include <type_traits>

namespace lobk {

constexpr unsigned FULL = 0xffffffffu;
enum { F_P = 0, F_Q, F_OID, F_TID, F_TS, F_TNS, NF };  // Eq.2 field order
enum { ASK = 0, BID = 1 };                               // side 0 = A, side 1 = B
enum {
    ST_MSGS = 0, ST_BAD, ST_TRADES, ST_DROPPED, ST_TRADED_QTY, ST_CANCELLED_QTY, ST_UNKNOWN,
    ST_ADD_OVF, ST_OVF_QTY, ST_DISCARDED, NST
};
constexpr int CH = 32;  // messages per staging chunk (1 KiB); two chunks per warp
constexpr int BEST_INVALID = -2, BEST_EMPTY = -1;

template <int I>
using IC = std::integral_constant<int, I>;

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
// Hide how a value was computed so the register allocator keeps it instead of
// rematerialising it (e.g. shared addresses from SR_TID / SR_CgaCtaId) in the loop.
__device__ __forceinline__ uint32_t opaque(uint32_t x) {
    asm volatile("mov.b32 %0, %0;" : "+r"(x));
    return x;
}
__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

// 32-bit shared-window addresses keep smem pointers in one register each (no
// generic-pointer rematerialisation in the message loop).
__device__ __forceinline__ int lds32(uint32_t a) {
    int v;
    asm volatile("ld.shared.b32 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ void sts32(uint32_t a, int v) {
    asm volatile("st.shared.b32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
__device__ __forceinline__ long long lds64(uint32_t a) {
    long long v;
    asm volatile("ld.shared.b64 %0, [%1];" : "=l"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ void sts64(uint32_t a, long long v) {
    asm volatile("st.shared.b64 [%0], %1;" ::"r"(a), "l"(v) : "memory");
}

__device__ __forceinline__ int2 lds64x2(uint32_t a) {
    int2 v;
    asm volatile("ld.shared.v2.b32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(a));
    return v;
}
__device__ __forceinline__ int4 lds128(uint32_t a) {
    int4 v;
    asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
    return v;
}
__device__ __forceinline__ void sts128(uint32_t a, int4 v) {
    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
                 : "memory");
}

// ---------------------------------------------------------------- book storage
// RegBook: hot fields P, Q, OID of slot (j*32 + lane) in registers v[s][f][j];
// cold fields in shared memory, one 16-byte record per slot: cold[s][slot] =
// {Ts, Tns, TID, 0}, so an add is one vector store and a time read one load.
template <int KPL_>
struct RegBook {
    static constexpr int KPL = KPL_;
    static constexpr int UNR = KPL_;
    static constexpr bool kRegs = true;
    int32_t v[2][3][KPL_];
    uint32_t cold;  // shared address of this warp's [2][NP][4] region
    int lane;
    static constexpr int cold_words() { return 2 * KPL_ * 32 * 4; }
    __device__ __forceinline__ int32_t hot(int s, int f, int j) const { return v[s][f][j]; }
    __device__ __forceinline__ void set_hot(int s, int f, int j, int32_t x) { v[s][f][j] = x; }
    __device__ __forceinline__ uint32_t rec(int s, int slot) const { return cold + 16u * (uint32_t)(s * KPL_ * 32 + slot); }
    __device__ __forceinline__ int2 times(int s, int slot) const { return lds64x2(rec(s, slot)); }
    __device__ __forceinline__ void put_cold(int s, int slot, int tid, int ts, int tns) const {
        sts128(rec(s, slot), make_int4(ts, tns, tid, 0));
    }
    // run f(row) with the warp-uniform row as a compile-time constant
    template <class F>
    __device__ __forceinline__ void row(int j, F &&f) {
        if constexpr (KPL_ == 1) {
            f(IC<0>{});
        } else {
            switch (j) {
                case 0: f(IC<0>{}); break;
                case 1: f(IC<1>{}); break;
                case 2: if constexpr (KPL_ > 2) f(IC<2>{}); break;
                default: if constexpr (KPL_ > 3) f(IC<(KPL_ > 3 ? 3 : 0)>{}); break;
            }
        }
    }
    // value of field f in row j (warp-uniform j), branch-free select chain
    __device__ __forceinline__ int32_t get(int s, int f, int j) const {
        int32_t r = v[s][f][0];
#pragma unroll
        for (int jj = 1; jj < KPL_; ++jj) r = (j == jj) ? v[s][f][jj] : r;
        return r;
    }
    __device__ __forceinline__ void put_if(bool pred, int s, int f, int j, int32_t x) {
#pragma unroll
        for (int jj = 0; jj < KPL_; ++jj)
            if (pred && j == jj) v[s][f][jj] = x;
    }
    __device__ __forceinline__ void load(const int32_t *g, int NP) {
#pragma unroll
        for (int s = 0; s < 2; ++s) {
#pragma unroll
            for (int f = 0; f < 3; ++f)
#pragma unroll
                for (int j = 0; j < KPL_; ++j) v[s][f][j] = __ldcs(g + (s * NF + f) * NP + j * 32 + lane);
#pragma unroll
            for (int j = 0; j < KPL_; ++j) {
                const int *r = g + s * NF * NP + j * 32 + lane;
                put_cold(s, j * 32 + lane, __ldcs(r + F_TID * NP), __ldcs(r + F_TS * NP), __ldcs(r + F_TNS * NP));
            }
        }
        __syncwarp();
    }
    __device__ __forceinline__ void store(int32_t *g, int NP) const {
        __syncwarp();
#pragma unroll
        for (int s = 0; s < 2; ++s)
#pragma unroll
            for (int j = 0; j < KPL_; ++j) {
                const bool occ = v[s][F_Q][j] > 0;  // empty slots are all -1
                int *r = g + s * NF * NP + j * 32 + lane;
#pragma unroll
                for (int f = 0; f < 3; ++f) __stcs(r + f * NP, occ ? v[s][f][j] : -1);
                const int4 c = lds128(rec(s, j * 32 + lane));
                __stcs(r + F_TID * NP, occ ? c.z : -1);
                __stcs(r + F_TS * NP, occ ? c.x : -1);
                __stcs(r + F_TNS * NP, occ ? c.y : -1);
            }
    }
};

// SmemBook: every field in this warp's shared-memory region [2][NF][NP].
template <int KPL_>
struct SmemBook {
    static constexpr int KPL = KPL_;
    static constexpr int UNR = 4;
    static constexpr bool kRegs = false;
    uint32_t cold;  // shared address of the whole book region [2][NF][NP]
    int lane;
    static constexpr int cold_words() { return 2 * NF * KPL_ * 32; }
    __device__ __forceinline__ uint32_t cold_addr(int s, int f, int slot) const {
        return cold + 4u * (uint32_t)((s * NF + f) * (KPL_ * 32) + slot);
    }
    __device__ __forceinline__ int32_t ld(int s, int f, int slot) const { return lds32(cold_addr(s, f, slot)); }
    __device__ __forceinline__ void st(int s, int f, int slot, int32_t x) const { sts32(cold_addr(s, f, slot), x); }
    __device__ __forceinline__ int32_t hot(int s, int f, int j) const { return ld(s, f, j * 32 + lane); }
    __device__ __forceinline__ void set_hot(int s, int f, int j, int32_t x) { st(s, f, j * 32 + lane, x); }
    __device__ __forceinline__ int2 times(int s, int slot) const { return make_int2(ld(s, F_TS, slot), ld(s, F_TNS, slot)); }
    __device__ __forceinline__ void put_cold(int s, int slot, int tid, int ts, int tns) const {
        st(s, F_TID, slot, tid); st(s, F_TS, slot, ts); st(s, F_TNS, slot, tns);
    }
    __device__ __forceinline__ int32_t get(int s, int f, int j) const { return hot(s, f, j); }
    __device__ __forceinline__ void put_if(bool pred, int s, int f, int j, int32_t x) {
        if (pred) set_hot(s, f, j, x);
    }
    template <class F>
    __device__ __forceinline__ void row(int j, F &&f) { f(j); }
    __device__ __forceinline__ void load(const int32_t *g, int NP) {
        for (int i = lane; i < 2 * NF * KPL_ * 32; i += 32) sts32(cold + 4u * i, __ldcs(g + i));
        __syncwarp();
    }
    __device__ __forceinline__ void store(int32_t *g, int NP) const {
        __syncwarp();
        for (int s = 0; s < 2; ++s)
            for (int j = 0; j < KPL_; ++j) {
                const bool occ = hot(s, F_Q, j) > 0;
                for (int f = 0; f < NF; ++f) __stcs(g + (s * NF + f) * NP + j * 32 + lane, occ ? hot(s, f, j) : -1);
            }
    }
};

// ------------------------------------------------------------------ the engine
template <class BK>
struct Engine {
    static constexpr int KPL = BK::KPL;
    static constexpr int UNR = BK::UNR;
    BK bk;
    int lane, N, Tcap, ntr;
    int32_t *tlog;          // this book's trade log [Tcap][6]
    uint32_t sc;            // shared address: this warp's counters [NST] int64 (lane 0 only),
                            // then the best orders' times bt[side][Ts, Tns] (every lane, same value)
    // warp-uniform best-order cache per side (Eq.5 + G1/G4): slot or BEST_*, price
    int bslot[2], bP[2];
    long long part_cxl;     // cancelled quantity, accumulated on the owner lane (G14)
    long long part_trd;     // traded quantity, accumulated on the owner lane

    __device__ __forceinline__ void count(int c, long long x) {  // lane 0 only
        sts64(sc + 8u * c, lds64(sc + 8u * c) + x);
    }
    __device__ __forceinline__ bool valid(int j) const { return j < KPL - 1 || j * 32 + lane < N; }
    __device__ __forceinline__ uint32_t bt_addr(int sd, int k) const { return sc + 8u * NST + 4u * (2 * sd + k); }

    // Lowest slot whose lane-local predicate holds, or -1: one reduction over
    // (row*32 + lane), which is exactly the slot index (interleaved layout).
    template <class Pred>
    __device__ __forceinline__ int lowest(Pred pred) const {
        unsigned loc = 0xffffffffu;
#pragma unroll UNR
        for (int j = KPL - 1; j >= 0; --j)
            if (pred(j)) loc = (unsigned)(j * 32 + lane);
        return (int)__reduce_min_sync(FULL, loc);
    }

    // Best(o_s) of side SD over occupied slots: price (ask min / bid max,
    // Eq.5 + G1), then earliest (Ts, Tns), then lowest slot (G4).
    template <int SD>
    __device__ __forceinline__ void recompute_best() {
        int lk = INT_MAX;
        bool has = false;
#pragma unroll UNR
        for (int j = 0; j < KPL; ++j) {
            const int q = bk.hot(SD, F_Q, j), p = bk.hot(SD, F_P, j);
            const int k = (SD == ASK) ? p : ~p;  // bids: larger price = smaller key
            if (q > 0) { lk = min(lk, k); has = true; }
        }
        if (!__any_sync(FULL, has)) { bslot[SD] = BEST_EMPTY; return; }
        const int m = __reduce_min_sync(FULL, has ? lk : INT_MAX);
        // candidates at the best price: lane-local earliest (Ts, Tns, row)
        int lts = INT_MAX, ltns = INT_MAX, lj = -1, lc = 0;
#pragma unroll UNR
        for (int j = 0; j < KPL; ++j) {
            const int q = bk.hot(SD, F_Q, j), p = bk.hot(SD, F_P, j);
            const int k = (SD == ASK) ? p : ~p;
            if (q > 0 && k == m) {
                const int s = j * 32 + lane;
                const int2 t2 = bk.times(SD, s);
                const int ts = t2.x, tns = t2.y;
                if (lj < 0 || ts < lts || (ts == lts && tns < ltns)) { lts = ts; ltns = tns; lj = j; }
                ++lc;
            }
        }
        const unsigned loc = lj < 0 ? 0xffffffffu : (unsigned)(lj * 32 + lane);
        int slot;
        if (__reduce_add_sync(FULL, (unsigned)lc) == 1) {
            slot = (int)__reduce_min_sync(FULL, loc);
        } else {
            const bool in = lj >= 0;
            const int t = __reduce_min_sync(FULL, in ? lts : INT_MAX);
            const bool in2 = in && lts == t;
            const int t2 = __reduce_min_sync(FULL, in2 ? ltns : INT_MAX);
            slot = (int)__reduce_min_sync(FULL, (in2 && ltns == t2) ? loc : 0xffffffffu);
        }
        bslot[SD] = slot;
        bP[SD] = (SD == ASK) ? m : ~m;
        const int2 bt = bk.times(SD, slot);              // broadcast shared load
        sts32(bt_addr(SD, 0), bt.x);
        sts32(bt_addr(SD, 1), bt.y);
    }

    // A new order at `slot` on side SD: keep the cache exact (G4 key order).
    template <int SD>
    __device__ __forceinline__ void note_add(int slot, int p, int ts, int tns) {
        const int bs = bslot[SD];
        if (bs == BEST_INVALID) return;
        bool better = bs == BEST_EMPTY;
        if (!better) {
            const int kn = (SD == ASK) ? p : ~p, kb = (SD == ASK) ? bP[SD] : ~bP[SD];
            better = kn < kb;
            if (kn == kb) {                      // same price: time, then slot (G4)
                const int bts = lds32(bt_addr(SD, 0)), btns = lds32(bt_addr(SD, 1));
                better = ts < bts || (ts == bts && (tns < btns || (tns == btns && slot < bs)));
            }
        }
        if (better) {
            bslot[SD] = slot; bP[SD] = p;
            sts32(bt_addr(SD, 0), ts);
            sts32(bt_addr(SD, 1), tns);
        }
    }

    // Cancellation (cancel == delete P:L289): lowest occupied slot with
    // OID == msg OID on the message's side (G16), else the lowest synthetic
    // order (OID <= -9000, G12) at the message price.
    template <int SD>
    __device__ __forceinline__ void cancel(int mQ, int mP, int mOID) {
        if (mQ <= 0) { if (lane == 0) count(ST_BAD, 1); return; }  // G22
        int slot = lowest([&](int j) { return bk.hot(SD, F_Q, j) > 0 && bk.hot(SD, F_OID, j) == mOID; });
        if (slot < 0)
            slot = lowest([&](int j) {
                return bk.hot(SD, F_Q, j) > 0 && bk.hot(SD, F_OID, j) <= -9000 && bk.hot(SD, F_P, j) == mP;
            });
        if (slot < 0) { if (lane == 0) count(ST_UNKNOWN, 1); return; }  // G15
        const bool own = lane == (slot & 31);
        const int j = slot >> 5;
        const int qi = bk.get(SD, F_Q, j);
        if (own) part_cxl += (mQ < qi) ? mQ : qi;              // G14
        bk.put_if(own, SD, F_Q, j, qi - mQ);                   // Q <= 0 -> empty
        if (bslot[SD] == slot) bslot[SD] = BEST_INVALID;
        if constexpr (!BK::kRegs) __syncwarp();
    }

    // Limit (T=1) or market (T=4) order of side OWN.
    template <int OWN>
    __device__ __forceinline__ void aggress(bool market, int mQ, int mP, int mOID, int mTID, int mTS, int mTNS) {
        constexpr int OPP = 1 - OWN;
        if (!market && mP <= 0) { if (lane == 0) count(ST_BAD, 1); return; }  // G22
        const int Pa = market ? (OWN == BID ? INT_MAX : 0) : mP;  // P_m = 0 / max_int (G18)
        int Qa = mQ;
        while (Qa > 0) {
            if (bslot[OPP] == BEST_INVALID) recompute_best<OPP>();
            const int s = bslot[OPP];
            if (s < 0) break;                                       // side empty
            const int Ps = bP[OPP];
            if (OWN == BID ? (Pa < Ps) : (Pa > Ps)) break;          // prices do not overlap
            const int ol = s & 31;
            const bool own = lane == ol;
            const int sj = s >> 5;
            int Qs, myoid;
            if constexpr (BK::kRegs) {   // the owner's registers; Q broadcast by shuffle
                myoid = bk.get(OPP, F_OID, sj);
                Qs = __shfl_sync(FULL, bk.get(OPP, F_Q, sj), ol);
            } else {                     // shared memory: every lane reads the slot
                Qs = bk.ld(OPP, F_Q, s);
                myoid = bk.ld(OPP, F_OID, s);
            }
            const int Qs2 = (Qs - Qa > 0) ? (Qs - Qa) : 0;            // Q_s' = max(0, Q_s - Q_a)
            const int q = Qs - Qs2;                                   // Q_j = Q_s - Q_s'
            Qa = Qa - Qs;                                             // Q_a' = Q_a - Q_s
            if (own) {
                if (ntr < Tcap) {                                     // Eq.3 record, Eq.4 cap (G8)
                    int2 *t = reinterpret_cast<int2 *>(tlog + (size_t)ntr * 6);
                    t[0] = make_int2(Ps, q);
                    t[1] = make_int2(mOID, myoid);
                    t[2] = make_int2(mTS, mTNS);
                }
                part_trd += q;
            }
            ++ntr;                                                    // fills this call (logged = min(ntr, Tcap))
            bk.put_if(own, OPP, F_Q, sj, Qs2);                      // filled order removed (G10)
            if (Qs2 == 0) bslot[OPP] = BEST_INVALID;
            if constexpr (!BK::kRegs) __syncwarp();
        }
        if (Qa <= 0) return;
        if (market) {
            if (lane == 0) count(ST_DISCARDED, Qa);
            return;
        }
        // remainder rests as one new order in the lowest empty slot (G3)
        const int slot = lowest([&](int j) { return valid(j) && bk.hot(OWN, F_Q, j) <= 0; });
        if (slot < 0) {                                              // side saturated (G6)
            if (lane == 0) { count(ST_ADD_OVF, 1); count(ST_OVF_QTY, Qa); }
            return;
        }
        const bool own = lane == (slot & 31);
        bk.row(slot >> 5, [&](auto J) {                              // G27
            if (own) {
                bk.set_hot(OWN, F_P, J, mP);
                bk.set_hot(OWN, F_Q, J, Qa);
                bk.set_hot(OWN, F_OID, J, mOID);
            }
        });
        // every lane stores the same value, so each lane later reads its own write
        bk.put_cold(OWN, slot, mTID, mTS, mTNS);
        if constexpr (!BK::kRegs) __syncwarp();
        note_add<OWN>(slot, mP, mTS, mTNS);
    }

    __device__ __forceinline__ void message(const int4 a, const int4 b) {
        const int T = a.x, S = a.y, Q = a.z, P = a.w;
        // T in 1..4 and S in {-1, +1}; T = 0 is padding (G21), anything else malformed (G22)
        const unsigned t1 = (unsigned)(T - 1);
        if (!((t1 < 4u) & ((((unsigned)(S + 1)) & ~2u) == 0u))) {
            if (T != 0 && lane == 0) count(ST_BAD, 1);
            return;
        }
        // the paper's 8 (type x side) cases; cancel and delete share one
        if (t1 - 1u < 2u) {
            if (S == 1) cancel<BID>(Q, P, b.x);
            else cancel<ASK>(Q, P, b.x);
        } else {
            if (S == 1) aggress<BID>(T == 4, Q, P, b.x, b.y, b.z, b.w);
            else aggress<ASK>(T == 4, Q, P, b.x, b.y, b.z, b.w);
        }
    }

    // L2 (G23): k-th best distinct price per side and its summed quantity;
    // lane k keeps level k.  Absent levels are (-1, 0).  Each level takes the
    // warp minimum of the remaining keys and retires every slot at that price.
    template <int SD>
    __device__ __forceinline__ void l2_side(int L, int &outp, int &outq) const {
        if constexpr (!BK::kRegs) {
            l2_side_scan<SD>(L, outp, outq);
            return;
        }
        outp = -1; outq = 0;
        int key[KPL];
        bool any = false;
#pragma unroll UNR
        for (int j = 0; j < KPL; ++j) {
            const int p = bk.hot(SD, F_P, j);
            const bool occ = bk.hot(SD, F_Q, j) > 0;
            key[j] = occ ? ((SD == ASK) ? p : ~p) : INT_MAX;
            any |= occ;
        }
        unsigned live = __ballot_sync(FULL, any);
        for (int k = 0; k < L && live; ++k) {
            int lk = key[0];
#pragma unroll UNR
            for (int j = 1; j < KPL; ++j) lk = min(lk, key[j]);
            const int m = __reduce_min_sync(FULL, lk);
            unsigned lq = 0;
            bool left = false;
#pragma unroll UNR
            for (int j = 0; j < KPL; ++j) {
                const bool hit = key[j] == m;
                if (hit) { lq += (unsigned)bk.hot(SD, F_Q, j); key[j] = INT_MAX; }
                left |= key[j] != INT_MAX;
            }
            const unsigned qs = __reduce_add_sync(FULL, lq);
            if (lane == k) { outp = (SD == ASK) ? m : ~m; outq = (int)qs; }
            live = __ballot_sync(FULL, left);
        }
    }
    // shared-memory books: rescan with a "strictly worse than the previous level" filter
    template <int SD>
    __device__ __forceinline__ void l2_side_scan(int L, int &outp, int &outq) const {
        outp = -1; outq = 0;
        int prev = 0;
        bool have_prev = false;
        for (int k = 0; k < L; ++k) {
            int lk = INT_MAX;
            bool lf = false;
#pragma unroll UNR
            for (int j = 0; j < KPL; ++j) {
                const int p = bk.hot(SD, F_P, j);
                const int key = (SD == ASK) ? p : ~p;
                if (bk.hot(SD, F_Q, j) > 0 && (!have_prev || key > prev)) { lk = min(lk, key); lf = true; }
            }
            if (!__any_sync(FULL, lf)) break;
            const int m = __reduce_min_sync(FULL, lf ? lk : INT_MAX);
            unsigned lq = 0;
#pragma unroll UNR
            for (int j = 0; j < KPL; ++j) {
                const int p = bk.hot(SD, F_P, j);
                const int key = (SD == ASK) ? p : ~p;
                if (bk.hot(SD, F_Q, j) > 0 && key == m) lq += (unsigned)bk.hot(SD, F_Q, j);
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
// Per-warp shared scratch: counters [NST] int64 + best times [2][2] int32.
constexpr int SCRATCH_BYTES = 8 * NST + 16;

// Persistent: each warp walks books w, w + total_warps, ...
template <class BK, int WARPS>
__device__ __forceinline__ void run_books(const Params &p, BK &bk, int32_t *stage /*[2][CH][8]*/, uint64_t *bars,
                                          uint32_t scratch) {
    const int lane = (int)opaque(threadIdx.x & 31);
    const int gw = blockIdx.x * WARPS + (threadIdx.x >> 5);
    const int nw = gridDim.x * WARPS;
    const int nmsg = p.n_steps * p.M;
    const int nchunks = (nmsg + CH - 1) / CH;
    uint32_t chunk_seq = 0;
    const uint32_t stage_u32 = opaque(smem_u32(stage));
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
        if (lane < NST) sts64(scratch + 8u * lane, 0);
        Engine<BK> e;
        e.bk = bk;
        e.bk.load(p.book + (size_t)b * 2 * NF * p.NP, p.NP);
        e.lane = lane; e.N = p.N; e.Tcap = p.Tcap; e.ntr = 0; e.sc = scratch;
        e.tlog = p.trades + (size_t)b * p.Tcap * 6;
        e.bslot[0] = e.bslot[1] = BEST_INVALID;
        e.bP[0] = e.bP[1] = 0;
        e.part_cxl = 0; e.part_trd = 0;
        int left = p.M, step = 0;
        for (int c = 0; c < nchunks; ++c) {
            const uint32_t seq = chunk_seq + c, slot = seq & 1;
            mbar_wait(&bars[slot], (seq >> 1) & 1);
            uint32_t maddr = stage_u32 + slot * CH * 32;
            int cnt = min(CH, nmsg - c * CH);
            while (cnt > 0) {                          // runs up to the next chunk or step end
                const int run = min(cnt, left);
                const uint32_t mend = maddr + 32u * run;
                do {
                    const int4 a = lds128(maddr), bb = lds128(maddr + 16);
                    e.message(a, bb);
                    maddr += 32;
                } while (maddr != mend);
                cnt -= run;
                left -= run;
                if (left == 0) {                       // end of a step: L2 snapshot (G23)
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
        e.bk.store(p.book + (size_t)b * 2 * NF * p.NP, p.NP);
        long long cx = e.part_cxl, tq = e.part_trd;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            cx += __shfl_xor_sync(FULL, cx, o);
            tq += __shfl_xor_sync(FULL, tq, o);
        }
        __syncwarp();
        const int logged = min(e.ntr, p.Tcap);
        if (lane < NST) {
            long long v = lds64(scratch + 8u * lane);
            if (lane == ST_CANCELLED_QTY) v += cx;
            if (lane == ST_TRADED_QTY) v += tq;
            if (lane == ST_DROPPED) v += e.ntr - logged;
            if (lane == ST_MSGS) v += nmsg;
            if (lane == ST_TRADES) v += e.ntr;             // fills = logged + dropped
            p.stats[(size_t)b * NST + lane] += v;
        }
        if (lane == 0) p.ntrades[b] = logged;
    }
}

// minimum resident CTAs per SM: caps registers without spills
#ifndef MINB_REG
#define MINB_REG 6
#endif
template <int KPL, int WARPS>
__global__ void __launch_bounds__(WARPS * 32, (KPL <= 2 ? 8 : MINB_REG)) lob_step_reg(const Params p) {
    __shared__ __align__(128) int32_t stage[WARPS][2][CH][8];
    __shared__ __align__(16) int32_t cold[WARPS][RegBook<KPL>::cold_words()];
    __shared__ __align__(8) uint64_t bars[WARPS][2];
    __shared__ __align__(16) unsigned char scratch[WARPS][SCRATCH_BYTES];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0) {
        mbar_init(&bars[w][0], 1);
        mbar_init(&bars[w][1], 1);
        fence_mbar_init();
    }
    __syncwarp();
    RegBook<KPL> bk;
    bk.cold = opaque(smem_u32(cold[w]));
    bk.lane = (int)opaque(lane);
    run_books<RegBook<KPL>, WARPS>(p, bk, &stage[w][0][0][0], bars[w], opaque(smem_u32(scratch[w])));
}

template <int KPL>
__global__ void __launch_bounds__(32) lob_step_smem(const Params p) {
    extern __shared__ __align__(128) int32_t dyn[];
    int32_t *stage = dyn;                                          // [2][CH][8]
    uint64_t *bars = reinterpret_cast<uint64_t *>(dyn + 2 * CH * 8);
    const uint32_t scratch = opaque(smem_u32(dyn + 2 * CH * 8 + 4));  // SCRATCH_BYTES
    int32_t *bookmem = dyn + 2 * CH * 8 + 4 + SCRATCH_BYTES / 4;  // [2][NF][KPL*32]
    const int lane = threadIdx.x & 31;
    if (lane == 0) {
        mbar_init(&bars[0], 1);
        mbar_init(&bars[1], 1);
        fence_mbar_init();
    }
    __syncwarp();
    SmemBook<KPL> bk;
    bk.cold = opaque(smem_u32(bookmem));
    bk.lane = lane;
    run_books<SmemBook<KPL>, 1>(p, bk, stage, bars, scratch);
}
constexpr int smem_step_bytes(int kpl) { return (2 * CH * 8 + 4) * 4 + SCRATCH_BYTES + 2 * NF * kpl * 32 * 4; }

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

// current L2 of every book from the stored state: one warp per book, book in smem
template <int KPL>
__global__ void __launch_bounds__(32) lob_export_l2(const int32_t *book, int32_t *out, int K, int N, int NP, int L) {
    extern __shared__ __align__(16) int32_t bookmem[];
    const int lane = threadIdx.x & 31;
    const int b = blockIdx.x;
    if (b >= K) return;
    Engine<SmemBook<KPL>> e;
    e.lane = lane; e.N = N;
    e.bk.cold = smem_u32(bookmem);
    e.bk.lane = lane;
    e.bk.load(book + (size_t)b * 2 * NF * NP, NP);
    e.l2_write(out + (size_t)b * L * 4, L);
}

}  // namespace lobk
