// lob_kernels.cuh -- sm_100a device code for the batched limit-order-book hot path.
//
// A GROUP of W warps (GT = 32*W threads) owns one book (PAPER.md P:L320:
// messages within a book are strictly serial; books are independent).  W = 1
// for capacity N <= 512 (one warp per book, several books per CTA); larger books
// have W = 4 warps of one CTA (8 or 16 rows each; lob_api.cu geo_of).  Slot i of a side (Eq.1,
// P:L161-163) lives in thread (i % GT), row (i / GT) -- "interleaved" -- so:
//   * every lowest-index search (free slot P:L175/G3, order-id lookup P:L177,
//     lowest-slot tie-break G4) is a thread-local select over rows plus ONE
//     group minimum (__reduce_min_sync, and for W > 1 a shared-memory exchange
//     across the W warps) of (row*GT + tid), which IS the warp-uniform slot;
//   * the row of a selected slot is uniform, so the owner thread updates its
//     registers with predicated selects (no local memory, no divergence).
// The fields every message scans -- P, Q, OID (Eq.2) -- are REGISTERS (KPL rows
// per side per thread); TID, Ts, Tns, read only when a new best order must be
// found or written on an add, are one 16-byte shared-memory record per slot
// that any thread reads with a broadcast load.
//
// Messages (Eq.6) stream HBM -> shared memory through a per-book double buffer
// filled by 1-D bulk async copies (cp.async.bulk: the TMA bulk engine, SASS
// UBLKCP) completing on an mbarrier; every thread reads the current message with
// two broadcast 16-byte shared loads.  Dispatch is uniform on (T, S) -- the
// paper's 8 explicit cases -- so no thread diverges.
//
// The best standing order of each side (Eq.5 + G1/G4) is cached (uniform) and
// recomputed with group reductions only after the cached order leaves the book;
// an add updates it with one key comparison.
#pragma once
#include <climits>
#include <cstdint>
#include <cuda_runtime.h>

#include <type_traits>

// Build options measured by A/B (scripts/ab_pairs.sh); the defaults are the kept ones.
#ifndef LOB_CXL2_W    // books of >= this many warps cancel in ONE combined exact / synthetic
#define LOB_CXL2_W 2    // pass (C5 N = 1024 / 2048 +1.4 %; one-warp books: C4 -7 %, C2 -4.5 %,
#endif                  // C5 N = 256 / 512 -1 %)
#ifndef LOB_R16   // row bounds of 16-row books: 1 = {8,16} (C5 N = 512 +24 %, N = 2048 +5 % over
#define LOB_R16 1 // 0 = {4,8,16}); 2 = {16} (-25 %), 3 = {4,16} (-46 %, -23 %)
#endif
#ifndef LOB_ROWR   // the add's register write through a compare chain (not the row switch)
#define LOB_ROWR 4  // for books of <= LOB_ROWR rows at the full row bound (C2 +0.5 %, C3 +0.4 %, C4 -0.1 %)
#endif
#ifndef LOB_SYNC_READER  // one-warp books: the __syncwarp that publishes a new order's cold
#define LOB_SYNC_READER 1   // record runs where other lanes read records (the arg-best), not per
#endif                      // add (C2 +1.6 %, C3 / C5 N = 100 +0.8 %, N = 256 +1.9 %; racecheck clean)
#ifndef LOB_ADDSEL  // books of >= this many rows write an add's registers by predicated selects
#define LOB_ADDSEL 8    // over the bounded rows instead of a compare-and-branch chain (C5 N = 256 /
#endif              // 512 / 1024 +1.3 / +2.4 / +2.4 %, N = 2048 +-0; 4-row books: C4 -3 %, C2 -3 %)
#ifndef LOB_X4  // 4-warp books: cross-warp reductions finish with one broadcast load
#define LOB_X4 1
#endif
#ifndef LOB_FREEHINT  // multi-warp books: an add takes a known lowest empty slot without a search
#define LOB_FREEHINT 1  // (C5 N = 1024 / 2048 +1.1 %)
#endif
#ifndef LOB_FREEHINT_KPL  // ... and one-warp books of at least this many rows
#define LOB_FREEHINT_KPL 99
#endif
#ifndef LOB_TREE  // get_r as a select tree for row bounds >= LOB_TREE (0 = never; 16: C5 N = 512
#define LOB_TREE 0  // +6 % before the {8,16} row bounds, +-0 after)
#endif
#ifndef LOB_R16W  // 16-row multi-warp books: lower row bound (0: the one-warp {8, 16}); {6, 8, 16}:
#define LOB_R16W 6  // C5 N = 2048 +10 % (682 resting orders fill 5.3 rows of 128 slots)
#endif
#ifndef LOB_R8W  // 8-row multi-warp books: an extra lower row bound (0: none); {3, 4, 8}:
#define LOB_R8W 3  // C5 N = 1024 +7 % (128 slots per row: 341 resting orders fill 2.7 rows)
#endif
#ifndef LOB_R16W8  // ... with a middle bound of 8 rows ({6, 16} measured the same)
#define LOB_R16W8 1
#endif
#ifndef LOB_R16LO  // 16-row one-warp books: lower row bound (7: C5 N = 512 +0.8 %, 6: -33 %)
#define LOB_R16LO 8
#endif
#ifndef LOB_R8    // row bounds of 8-row books: 0 = {2,4,8}, 1 = {4,8} (C5 N = 256 +13 %, N = 1024 +4 %),
#define LOB_R8 1  // 2 = {2,8} (-10 %, -16 %)
#endif
namespace lobk {

constexpr unsigned FULL = 0xffffffffu;
enum { F_P = 0, F_Q, F_OID, F_TID, F_TS, F_TNS, NF };  // Eq.2 field order
enum { ASK = 0, BID = 1 };                               // side 0 = A, side 1 = B
enum {
    ST_MSGS = 0, ST_BAD, ST_TRADES, ST_DROPPED, ST_TRADED_QTY, ST_CANCELLED_QTY, ST_UNKNOWN,
    ST_ADD_OVF, ST_OVF_QTY, ST_DISCARDED, NST
};
constexpr int CH = 32;  // messages per staging chunk (1 KiB); two chunks per book
constexpr int BEST_INVALID = -2, BEST_EMPTY = -1;

template <int I>
using IC = std::integral_constant<int, I>;

// Dispatch code of a message (Eq.6 [T, S, Q, P, ...]), computed once per message
// lane-parallel over a staged chunk and written over T: 0 = padding (T = 0, G21),
// 1 = malformed (T not in 1..4, S not +-1, cancel/delete Q <= 0, limit P <= 0: G22),
// else MC_CANCEL | MC_AGGR (limit / market) | MC_MKT (market) | MC_BID (S = +1).
enum { MC_PAD = 0, MC_BAD = 1, MC_CANCEL = 2, MC_BID = 1, MC_AGGR = 4, MC_MKT = 8 };
__device__ __forceinline__ int msg_code(const int4 a) {
    const int T = a.x, S = a.y, Q = a.z, P = a.w;
    if (T == 0) return MC_PAD;
    const bool ok_ts = ((unsigned)(T - 1) < 4u) & ((((unsigned)(S + 1)) & ~2u) == 0u);
    const bool cxl = (unsigned)(T - 2) < 2u;                 // cancel == delete
    const bool ok = ok_ts && (cxl ? Q > 0 : (T == 4 || P > 0));
    if (!ok) return MC_BAD;
    return MC_CANCEL | (S == 1 ? MC_BID : 0) | (cxl ? 0 : MC_AGGR) | (T == 4 ? MC_MKT : 0);
}

// A message in Eq.6 form made ready for dispatch: the code over T, and a market
// order's price replaced by the price it matches at (P_m = 0 for a sell, max_int for a
// buy: P:L290, G18).
__device__ __forceinline__ int4 msg_decode(int4 a) {
    const int c = msg_code(a);
    if ((c & MC_MKT) != 0) a.w = (c & MC_BID) ? INT_MAX : 0;
    a.x = c;
    return a;
}

// NEXT row N3 (execution env, Sec.5.1.3 / 5.2): the task shared by all envs
// and the per-env state (see lob_env.cuh, include/lob.h lob_env_config)
struct EnvCfg {  // == lob_env_config (include/lob.h)
    int task_side, task_size, n_passive, tick, episode_s, agent_tid, oid_base, reserved;
    double lam;
};
struct EnvState {  // 64 bytes per env
    long long executed;
    double p_init;
    int init_ts, init_tns, cur_ts, cur_tns, next_oid, done, last_ask, last_bid;
    int live[4];
};
static_assert(sizeof(EnvState) == 64, "env state layout");

__device__ __forceinline__ long long env_elapsed_ns(const EnvState &e) {
    return ((long long)e.cur_ts - e.init_ts) * 1000000000LL + ((long long)e.cur_tns - e.init_tns);
}

struct Params {
    int32_t *book;         // [K][2][NF][NP] SoA, slot i at [i] (i = row*GT + tid)
    int32_t *trades;       // [K][Tcap][6]
    int32_t *ntrades;      // [K]
    long long *stats;      // [K][NST]
    const int32_t *msgs;   // [nb][n_steps*M][8]  (relative to book0)
    int32_t *l2out;        // [nb][n_steps][L][4] or null (relative to book0)
    int32_t *l1out;        // [nb][n_steps*M][4] or null: Level-1 after every message (NEXT N1)
    unsigned *sched;       // [2]: next book, finished groups (zero between launches)
    int N, NP, Tcap, L, n_steps, M;
    int book0, nb;         // books [book0, book0+nb) of the state
};
// MODE 2 only (fused env step, NEXT N3; Params::msgs = the step's data messages).  A
// separate kernel parameter, so the other modes' parameter block is unchanged.
struct EnvParams {
    EnvState *env;         // [K]
    const float *actions;  // [K][4]
    int32_t *agent_out;    // [K][8][8]: the agent's messages of the step, zero-padded
    double *reward;        // [K] or null
    int32_t *done;         // [K] or null
    long long *executed;   // [K] or null
    EnvCfg ec;
};

// ------------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ unsigned mbar_try(uint32_t bar, uint32_t parity) {
    unsigned ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(bar), "r"(parity)
        : "memory");
    return ok;
}
// every thread of the warp waits for the phase; the loop condition is a warp reduction,
// so ptxas sees a uniform loop (a per-thread spin would leave the warp "possibly
// diverged" for its convergence analysis: reconvergence barriers and divergence checks
// around every later branch and collective)
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    while (__reduce_min_sync(0xffffffffu, mbar_try(bar, parity)) == 0u) {
    }
}
// 1-D bulk copy global -> shared (TMA bulk engine), completes tx bytes on `bar`
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void *src, uint32_t bytes, uint32_t bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                 "l"(src), "r"(bytes), "r"(bar)
                 : "memory");
}
// Hide how a value was computed so the register allocator keeps it instead of
// rematerialising it (e.g. shared addresses from SR_TID / SR_CgaCtaId) in the loop.
__device__ __forceinline__ uint32_t opaque(uint32_t x) {
    asm volatile("mov.b32 %0, %0;" : "+r"(x));
    return x;
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }

// 32-bit shared-window addresses keep smem pointers in one register each.
__device__ __forceinline__ int lds32(uint32_t a) {
    int v;
    asm volatile("ld.shared.b32 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ void sts32(uint32_t a, int v) { asm volatile("st.shared.b32 [%0], %1;" ::"r"(a), "r"(v) : "memory"); }
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

// Single-writer stores as predicated instructions inside one asm block (all lanes
// execute it, only lane `who == 0` / the lane whose `pred` holds writes): no
// lane-divergent branch in the message loop, so ptxas proves the whole message body
// uniform and dispatches it on the uniform datapath (R2UR + ULOP3 + BRA.U).  Used by
// the many-wave build (MODE 3: C4 +1.6 %); the other builds measured slower with it.
__device__ __forceinline__ void sts32_if0(int who, uint32_t a, int v) {
    asm volatile("{\n\t.reg .pred p;\n\tsetp.eq.s32 p, %0, 0;\n\t@p st.shared.b32 [%1], %2;\n\t}" ::"r"(who), "r"(a),
                 "r"(v)
                 : "memory");
}
__device__ __forceinline__ void sts128_if0(int who, uint32_t a, int4 v) {
    asm volatile("{\n\t.reg .pred p;\n\tsetp.eq.s32 p, %0, 0;\n\t@p st.shared.v4.b32 [%1], {%2, %3, %4, %5};\n\t}" ::"r"(who),
                 "r"(a), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
                 : "memory");
}
__device__ __forceinline__ void add64_if0(int who, uint32_t a, long long x) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t.reg .b64 v;\n\tsetp.eq.s32 p, %0, 0;\n\t@p ld.shared.b64 v, [%1];\n\t"
        "@p add.s64 v, v, %2;\n\t@p st.shared.b64 [%1], v;\n\t}" ::"r"(who),
        "r"(a), "l"(x)
        : "memory");
}
// a 16-byte global record by lane `who == 0`
__device__ __forceinline__ void stg128_if0(int who, int32_t *g, int4 v) {
    asm volatile("{\n\t.reg .pred p;\n\tsetp.eq.s32 p, %0, 0;\n\t@p st.global.v4.b32 [%1], {%2, %3, %4, %5};\n\t}" ::"r"(who),
                 "l"(g), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
                 : "memory");
}
// the Eq.3 trade record (24 bytes) by the lane whose `pred` holds
__device__ __forceinline__ void trade_store_if(bool pred, int2 *t, int2 a, int2 b, int2 c) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %0, 0;\n\t@p st.global.v2.b32 [%1], {%2, %3};\n\t"
        "@p st.global.v2.b32 [%1+8], {%4, %5};\n\t@p st.global.v2.b32 [%1+16], {%6, %7};\n\t}" ::"r"((unsigned)pred),
        "l"(t), "r"(a.x), "r"(a.y), "r"(b.x), "r"(b.y), "r"(c.x), "r"(c.y)
        : "memory");
}

// ------------------------------------------------------------ group primitives
// Barrier over the book's threads: the warp itself, or the whole CTA (W > 1
// books own their CTA).
template <int W>
__device__ __forceinline__ void group_sync() {
    if constexpr (W == 1) __syncwarp();
    else __syncthreads();
}

// ---------------------------------------------------------------- book storage
// Hot fields P, Q, OID of slot (j*GT + tid) in registers v[s][f][j]; cold
// fields in shared memory, one 16-byte record per slot: {OID, TID, Ts, Tns}
// (the message quad as loaded; its OID word is not read).
template <int KPL_, int W_>
struct RegBook {
    static constexpr int KPL = KPL_, W = W_, GT = 32 * W_, NP = KPL_ * 32 * W_;
    int32_t v[2][3][KPL_];
    uint32_t cold;  // shared address of this book's [2][NP] x 16 B records
    int tid;        // thread index within the book group
    __device__ __forceinline__ int32_t hot(int s, int f, int j) const { return v[s][f][j]; }
    __device__ __forceinline__ uint32_t rec(int s, int slot) const { return cold + 16u * (uint32_t)(s * NP + slot); }
    // record = the message's second quad in Eq.6 order {OID, TID, Ts, Tns}: an add stores
    // it as loaded, without reordering moves (the OID word is unused here)
    __device__ __forceinline__ int2 times(int s, int slot) const { return lds64x2(rec(s, slot) + 8u); }
    __device__ __forceinline__ void put_cold(int s, int slot, const int4 b) const { sts128(rec(s, slot), b); }
    __device__ __forceinline__ void put_cold(int s, int slot, int tid_, int ts, int tns) const {
        sts128(rec(s, slot), make_int4(0, tid_, ts, tns));
    }
    // run f(row) with the uniform row as a compile-time constant
    template <class F>
    __device__ __forceinline__ void row(int j, F &&f) {
        if constexpr (KPL_ == 1) {
            f(IC<0>{});
        } else {
            switch (j) {
                case 0: f(IC<0>{}); break;
                case 1: f(IC<1>{}); break;
                case 2: if constexpr (KPL_ > 2) f(IC<2>{}); break;
                case 3: if constexpr (KPL_ > 3) f(IC<(KPL_ > 3 ? 3 : 0)>{}); break;
                case 4: if constexpr (KPL_ > 4) f(IC<(KPL_ > 4 ? 4 : 0)>{}); break;
                case 5: if constexpr (KPL_ > 5) f(IC<(KPL_ > 5 ? 5 : 0)>{}); break;
                case 6: if constexpr (KPL_ > 6) f(IC<(KPL_ > 6 ? 6 : 0)>{}); break;
                case 7: if constexpr (KPL_ > 7) f(IC<(KPL_ > 7 ? 7 : 0)>{}); break;
            case 8: if constexpr (KPL_ > 8) f(IC<(KPL_ > 8 ? 8 : 0)>{}); break;
            case 9: if constexpr (KPL_ > 9) f(IC<(KPL_ > 9 ? 9 : 0)>{}); break;
            case 10: if constexpr (KPL_ > 10) f(IC<(KPL_ > 10 ? 10 : 0)>{}); break;
            case 11: if constexpr (KPL_ > 11) f(IC<(KPL_ > 11 ? 11 : 0)>{}); break;
            case 12: if constexpr (KPL_ > 12) f(IC<(KPL_ > 12 ? 12 : 0)>{}); break;
            case 13: if constexpr (KPL_ > 13) f(IC<(KPL_ > 13 ? 13 : 0)>{}); break;
            case 14: if constexpr (KPL_ > 14) f(IC<(KPL_ > 14 ? 14 : 0)>{}); break;
            default: if constexpr (KPL_ > 15) f(IC<(KPL_ > 15 ? 15 : 0)>{}); break;
            }
        }
    }
    // f(row) for a uniform row j known to be below RR: a compare chain, no jump table
    template <int RR, int J0 = 0, class F>
    __device__ __forceinline__ void row_r(int j, F &&f) {
        if constexpr (J0 + 1 >= RR) {
            f(IC<J0>{});
        } else {
            if (j == J0) f(IC<J0>{});
            else row_r<RR, J0 + 1>(j, f);
        }
    }
    // value of field f in row j (uniform j), branch-free select chain
    __device__ __forceinline__ int32_t get(int s, int f, int j) const {
        int32_t r = v[s][f][0];
#pragma unroll
        for (int jj = 1; jj < KPL_; ++jj) r = (j == jj) ? v[s][f][jj] : r;
        return r;
    }
    // the same for a row known to be below R.  LOB_TREE: a binary select tree on the
    // bits of j (depth log2 R, one bit test per level) instead of the serial chain
    template <int LO, int NN>
    __device__ __forceinline__ int32_t sel_tree(int s, int f, int j) const {
        if constexpr (NN == 1) {
            return v[s][f][LO];
        } else {
            constexpr int H = NN > 8 ? 8 : (NN > 4 ? 4 : (NN > 2 ? 2 : 1));  // largest power of 2 < NN
            return (j & H) ? sel_tree<LO + H, NN - H>(s, f, j) : sel_tree<LO, H>(s, f, j);
        }
    }
    template <int R>
    __device__ __forceinline__ int32_t get_r(int s, int f, int j) const {
#if LOB_TREE
        if constexpr (R >= LOB_TREE) return sel_tree<0, R>(s, f, j);
#endif
        int32_t r = v[s][f][0];
#pragma unroll
        for (int jj = 1; jj < R; ++jj) r = (j == jj) ? v[s][f][jj] : r;
        return r;
    }
    template <int R>
    __device__ __forceinline__ void put_if_r(bool pred, int s, int f, int j, int32_t x) {
#pragma unroll
        for (int jj = 0; jj < R; ++jj)
            if (pred && j == jj) v[s][f][jj] = x;
    }
    __device__ __forceinline__ void load(const int32_t *g) {
#pragma unroll
        for (int s = 0; s < 2; ++s) {
#pragma unroll
            for (int f = 0; f < 3; ++f)
#pragma unroll
                for (int j = 0; j < KPL_; ++j) v[s][f][j] = __ldcs(g + (s * NF + f) * NP + j * GT + tid);
#pragma unroll
            for (int j = 0; j < KPL_; ++j) {
                const int *r = g + s * NF * NP + j * GT + tid;
                put_cold(s, j * GT + tid, __ldcs(r + F_TID * NP), __ldcs(r + F_TS * NP), __ldcs(r + F_TNS * NP));
            }
        }
        group_sync<W_>();  // records are read by every thread of the book from here on
    }
    __device__ __forceinline__ void store(int32_t *g) const {
#pragma unroll
        for (int s = 0; s < 2; ++s)
#pragma unroll
            for (int j = 0; j < KPL_; ++j) {
                const bool occ = v[s][F_Q][j] > 0;  // empty slots are all -1
                int *r = g + s * NF * NP + j * GT + tid;
#pragma unroll
                for (int f = 0; f < 3; ++f) __stcs(r + f * NP, occ ? v[s][f][j] : -1);
                const int4 c = lds128(rec(s, j * GT + tid));
                __stcs(r + F_TID * NP, occ ? c.y : -1);
                __stcs(r + F_TS * NP, occ ? c.z : -1);
                __stcs(r + F_TNS * NP, occ ? c.w : -1);
            }
    }
};

// ------------------------------------------------------------------ the engine
template <class BK, bool TL1 = false, bool ROWS = false, bool PRED = false, bool PREDT = PRED>
struct Engine {
    static constexpr int KPL = BK::KPL, W = BK::W, GT = BK::GT;
    BK bk;
    const Params &p;
    int tid, book, ntr;
    const unsigned char *scp;  // the same scratch through a shared-memory pointer (uniform loads)
    uint32_t sc;            // shared: counters [NST] int64 (thread 0 only), best times bt[2][2] int32,
                            //         cross-warp exchange xb[2][W] u32, next-book word
    int xph;                // exchange buffer phase (uniform)
    // uniform best-order cache per side (Eq.5 + G1/G4): slot or BEST_*, and its price
    int bslot[2], bP[2];
    // best order's (Ts, Tns): uniform registers for multi-warp books (no barriers),
    // shared memory for warp books (4 registers fewer in the 64-register kernel)
    static constexpr bool kBtRegs = (W > 1);
    // where a new order's cold record is published to the other lanes (LOB_SYNC_READER):
    // at the reader (the arg-best), except in the many-wave build (PRED), where the
    // per-add __syncwarp measured as fast (C4 -0.2 % the other way)
    static constexpr bool kSyncReader = LOB_SYNC_READER && W == 1 && !PRED;
    int bTS[2], bTNS[2];
    int hr[2];              // row high-water mark per side (see with_rows)
    // W > 1 (LOB_FREEHINT): the add's lowest empty slot (G3) without a search where
    // possible.  Invariant per side: every empty slot below flb is >= frm (frm = NP: none),
    // and frm is empty -- so frm, when below NP, IS the lowest empty slot.  A searched add
    // at s sets flb = s + 1, frm = NP; an add at frm sets flb = frm + 1, frm = NP; a removal
    // (cancel or fill emptying slot r < flb) lowers frm to r.
    static constexpr bool kFreeHint = LOB_FREEHINT && (W > 1 || KPL >= LOB_FREEHINT_KPL);
    int flb[2], frm[2];
    unsigned long long bV[2];  // TL1: total quantity at the cached best price (its L1 volume,
                               // exact in 64 bits; reported saturated at INT32_MAX, G20)
    long long part_cxl;     // cancelled quantity, accumulated on the owner thread (G14)
    long long part_trd;     // traded quantity, accumulated on the owner thread
    int lastPs;             // price of the last fill (side-split build: a bound on the side's
                            // best after its best order was filled away; lob_split.cuh)

    __device__ __forceinline__ Engine(const Params &p_) : p(p_) {}

    __device__ __forceinline__ void count(int c, long long x) {  // thread 0 only
        sts64(sc + 8u * c, lds64(sc + 8u * c) + x);
    }
    __device__ __forceinline__ uint32_t bt_addr(int sd, int k) const { return sc + 8u * NST + 4u * (2 * sd + k); }

    // ---- group reductions: warp REDUX, then (W > 1) one exchange through shared memory
    // (two phases of 16 B per warp, alternated so one barrier per exchange suffices)
    __device__ __forceinline__ uint32_t xbase() const { return sc + 8u * NST + 16u + 16u * (uint32_t)(xph * W); }
    // after the barrier lane k < W holds warp k's partial and the other lanes `ident`,
    // so a second warp REDUX finishes the group reduction
    __device__ __forceinline__ unsigned exchange(unsigned r, unsigned ident) {
        const uint32_t base = xbase();
        if ((tid & 31) == 0) sts32(base + 16u * (tid >> 5), (int)r);
        __syncthreads();
        const int lane = tid & 31;
        const unsigned v = lane < W ? (unsigned)lds32(base + 16u * lane) : ident;
        xph ^= 1;  // the other buffer next time: no write-after-read race with one barrier
        return v;
    }
    // W = 4 (LOB_X4): the four warp partials side by side, read by every lane with ONE
    // 16-byte broadcast load and combined in registers (no second warp reduction)
    static constexpr bool kX4 = (W == 4) && LOB_X4;
    __device__ __forceinline__ int4 exchange4(unsigned r) {
        const uint32_t base = xbase();
        if ((tid & 31) == 0) sts32(base + 4u * (tid >> 5), (int)r);
        __syncthreads();
        const int4 v = lds128(base);
        xph ^= 1;
        return v;
    }
    // two warp-reduced values per warp: warp k's pair lands in (a.x, a.y) / (a.z, a.w) /
    // (b.x, b.y) / (b.z, b.w) for k = 0..3
    __device__ __forceinline__ void exchange_pair4(unsigned r0, unsigned r1, int4 &a, int4 &b) {
        const uint32_t base = xbase();
        if ((tid & 31) == 0) sts64(base + 8u * (tid >> 5), (long long)(((unsigned long long)r1 << 32) | r0));
        __syncthreads();
        a = lds128(base);
        b = lds128(base + 16u);
        xph ^= 1;
    }
    __device__ __forceinline__ unsigned gmin_u(unsigned x) {
        const unsigned r = __reduce_min_sync(FULL, x);
        if constexpr (W == 1) return r;
        else if constexpr (kX4) {
            const int4 v = exchange4(r);
            return min(min((unsigned)v.x, (unsigned)v.y), min((unsigned)v.z, (unsigned)v.w));
        } else return __reduce_min_sync(FULL, exchange(r, 0xffffffffu));
    }
    __device__ __forceinline__ int gmin_i(int x) {
        const int r = __reduce_min_sync(FULL, x);
        if constexpr (W == 1) return r;
        else if constexpr (kX4) {
            const int4 v = exchange4((unsigned)r);
            return min(min(v.x, v.y), min(v.z, v.w));
        } else return __reduce_min_sync(FULL, (int)exchange((unsigned)r, (unsigned)INT_MAX));
    }
    __device__ __forceinline__ unsigned gadd(unsigned x) {
        const unsigned r = __reduce_add_sync(FULL, x);
        if constexpr (W == 1) return r;
        else if constexpr (kX4) {
            const int4 v = exchange4(r);
            return ((unsigned)v.x + (unsigned)v.y) + ((unsigned)v.z + (unsigned)v.w);
        } else return __reduce_add_sync(FULL, exchange(r, 0u));
    }
    // exact group sum of per-thread partials < 2^35 (sums of up to 16 int32 quantities):
    // two 32-bit reductions of the high and low 16-bit halves (each total < 2^27)
    __device__ __forceinline__ unsigned long long gadd64(unsigned long long x) {
        const unsigned hi = gadd((unsigned)(x >> 16)), lo = gadd((unsigned)(x & 0xffffu));
        return ((unsigned long long)hi << 16) + lo;
    }
    // any thread of the group
    __device__ __forceinline__ bool gany(bool x) {
        if constexpr (W == 1) return __any_sync(FULL, x);
        else return gmin_u(x ? 0u : 1u) == 0u;
    }
    // a level volume as reported (G20): the exact sum saturated at INT32_MAX
    static __device__ __forceinline__ int sat32(unsigned long long v) {
        return v > (unsigned long long)INT_MAX ? INT_MAX : (int)v;
    }
    // value held by thread `owner` of the group, to every thread
    __device__ __forceinline__ int bcast(int x, int owner) {
        if constexpr (W == 1) {
            return __shfl_sync(FULL, x, owner);
        } else {
            const uint32_t base = xbase();
            if (tid == owner) sts32(base, x);
            __syncthreads();
            // a plain load from a uniform shared address: the compiler then knows the
            // value (and the fill loop it controls) is uniform
            const int r = *reinterpret_cast<const int *>(scp + (8 * NST + 16 + 16 * xph * W));
            xph ^= 1;
            return r;
        }
    }

    static __device__ __forceinline__ bool found(int slot) { return (unsigned)slot < (unsigned)BK::NP; }

    // Row high-water mark: every occupied slot of side s lies in rows 0..hr[s] (-1: no
    // order).  Orders take the lowest empty slot (G3), so a book of n orders fills the
    // low rows; a scan over occupied slots runs over the first R rows only, R the
    // smallest of {2, 4, KPL} above hr (one uniform branch; rows between hr and R are
    // empty, so scanning them is harmless).  Raised on every add, lowered to the exact
    // value at every L2 snapshot.
    // ROWS = false (latency-bound launches: one wave of few books): always all rows --
    // the branch costs more latency than the skipped rows save (C2: -4 %).
    template <class F>
    __device__ __forceinline__ void with_rows(int h, F &&f) {
        if constexpr (KPL <= 2 || !ROWS) {
            f(IC<KPL>{});
        } else if constexpr (KPL <= 4) {
#if LOB_R4 == 1
            f(IC<KPL>{});
#else
            if (h < 2) f(IC<2>{});
            else f(IC<KPL>{});
#endif
        } else if constexpr (KPL <= 8) {
#if LOB_R8 == 1
            if constexpr (W > 1 && LOB_R8W > 0) {  // multi-warp books: {LOB_R8W, 4, 8}
                if (h < LOB_R8W) f(IC<LOB_R8W>{});
                else if (h < 4) f(IC<4>{});
                else f(IC<KPL>{});
            } else {
                if (h < 4) f(IC<4>{});
                else f(IC<KPL>{});
            }
#elif LOB_R8 == 2
            if (h < 2) f(IC<2>{});
            else f(IC<KPL>{});
#else
            if (h < 2) f(IC<2>{});
            else if (h < 4) f(IC<4>{});
            else f(IC<KPL>{});
#endif
        } else {
#if LOB_R16 == 2
            f(IC<KPL>{});
#elif LOB_R16 == 3
            if (h < 4) f(IC<4>{});
            else f(IC<KPL>{});
#elif LOB_R16 == 0
            if (h < 4) f(IC<4>{});
            else if (h < 8) f(IC<8>{});
            else f(IC<KPL>{});
#else  // {8, 16}: C5 N = 512 +24 %, N = 2048 +5 % over {4, 8, 16} (fewer code copies)
            if constexpr (W > 1 && LOB_R16W > 0) {  // multi-warp books: {LOB_R16W, (8,) 16}
                if (h < LOB_R16W) f(IC<LOB_R16W>{});
#if LOB_R16W8
                else if (h < 8) f(IC<8>{});
#endif
                else f(IC<KPL>{});
            } else {
                if (h < LOB_R16LO) f(IC<LOB_R16LO>{});
                else f(IC<KPL>{});
            }
#endif
        }
    }
    // highest occupied row of side s (group-uniform), -1 if none
    template <int SD>
    __device__ __forceinline__ int top_row() {
        int hl = -1;
#pragma unroll
        for (int j = 0; j < KPL; ++j)
            if (bk.hot(SD, F_Q, j) > 0) hl = j;
        return (KPL - 1) - (int)gmin_u((unsigned)(KPL - 1 - hl));
    }
    __device__ __forceinline__ void init_rows() {
        flb[0] = flb[1] = 0;
        frm[0] = frm[1] = BK::NP;
        if constexpr (ROWS) {
            hr[ASK] = top_row<ASK>();
            hr[BID] = top_row<BID>();
        } else {
            hr[ASK] = hr[BID] = KPL - 1;
        }
    }
    // Lowest slot of rows 0..R-1 whose thread-local predicate holds, or a value >= NP
    // (none, see found): the select chain picks a constant row (KPL = none), then ONE
    // group minimum of (row*GT + tid), which is exactly the slot index (interleaved
    // layout) -- one multiply-add instead of one add per row.
    template <int R, class Pred>
    __device__ __forceinline__ int lowest_rows(Pred pred) {
        unsigned r = KPL;
#pragma unroll
        for (int j = R - 1; j >= 0; --j)
            if (pred(j)) r = (unsigned)j;
        return (int)gmin_u(r * GT + (unsigned)tid);
    }
    // the same, also capturing the Q of this thread's lowest matching row into q
    template <int SD, int R, class Pred>
    __device__ __forceinline__ int lowest_rows_q(int &q, Pred pred) {
        unsigned r = KPL;
#pragma unroll
        for (int j = R - 1; j >= 0; --j)
            if (pred(j)) { r = (unsigned)j; q = bk.hot(SD, F_Q, j); }
        return (int)gmin_u(r * GT + (unsigned)tid);
    }
    // Best(o_s) of side SD over occupied slots: price (ask min / bid max,
    // Eq.5 + G1), then earliest (Ts, Tns), then lowest slot (G4).
    template <int SD>
    __device__ __forceinline__ void recompute_best() {
        with_rows(hr[SD], [&](auto R) { recompute_best_r<SD, R>(); });
    }
    template <int SD, int R>
    __device__ __forceinline__ void recompute_best_r() {
        if constexpr (W > 1) {
            recompute_best_multi<SD, R>();
            return;
        }
        // offset price key (resting prices are >= 1, G22): < 0xffffffff for every
        // occupied slot, so the all-ones minimum means "side empty" (no vote needed)
        unsigned lk = 0xffffffffu;
#pragma unroll
        for (int j = 0; j < R; ++j) {
            const int q = bk.hot(SD, F_Q, j), p = bk.hot(SD, F_P, j);
            const unsigned k = (SD == ASK) ? (unsigned)(p - 1) : (unsigned)(INT_MAX - p);
            if (q > 0) lk = min(lk, k);
        }
        const unsigned m = gmin_u(lk);
        if (m == 0xffffffffu) { set_empty<SD>(); return; }
        if constexpr (kSyncReader) __syncwarp();  // cold records written by lane 0 (add_r)
        // candidates at the best price: thread-local earliest (Ts, Tns, row)
        int lts = INT_MAX, ltns = INT_MAX, lj = -1, lc = 0;
        unsigned long long lv = 0;
#pragma unroll
        for (int j = 0; j < R; ++j) {
            const int q = bk.hot(SD, F_Q, j), p = bk.hot(SD, F_P, j);
            const unsigned k = (SD == ASK) ? (unsigned)(p - 1) : (unsigned)(INT_MAX - p);
            if (q > 0 && k == m) {
                const int2 t2 = bk.times(SD, j * GT + tid);
                if (lj < 0 || t2.x < lts || (t2.x == lts && t2.y < ltns)) { lts = t2.x; ltns = t2.y; lj = j; }
                ++lc;
                if constexpr (TL1) lv += (unsigned)q;
            }
        }
        if constexpr (TL1) bV[SD] = gadd64(lv);
        const unsigned loc = lj < 0 ? 0xffffffffu : (unsigned)(lj * GT + tid);
        int slot;
        if (gadd((unsigned)lc) == 1) {
            slot = (int)gmin_u(loc);
        } else {
            const bool in = lj >= 0;
            const int t = gmin_i(in ? lts : INT_MAX);
            const bool in2 = in && lts == t;
            const int t2 = gmin_i(in2 ? ltns : INT_MAX);
            slot = (int)gmin_u((in2 && ltns == t2) ? loc : 0xffffffffu);
        }
        bslot[SD] = slot;
        bP[SD] = (SD == ASK) ? (int)(m + 1u) : (int)(INT_MAX - (int)m);
        const int2 bt = bk.times(SD, slot);  // broadcast shared load
        set_bt<SD>(bt.x, bt.y);
    }
    // W > 1: the same key order with two barriers instead of four to six.  Resting
    // prices are >= 1 (G22), so the offset key below is < 0xffffffff for every
    // occupied slot and the all-ones value doubles as "side empty".  The time
    // tie-break runs as a warp-level lexicographic (Ts, Tns, slot) minimum whose W
    // winners are exchanged once.
    template <int SD, int R>
    __device__ __forceinline__ void recompute_best_multi() {
        unsigned lk = 0xffffffffu;
#pragma unroll
        for (int j = 0; j < R; ++j) {
            const int q = bk.hot(SD, F_Q, j), p = bk.hot(SD, F_P, j);
            const unsigned k = (SD == ASK) ? (unsigned)(p - 1) : (unsigned)(INT_MAX - p);
            if (q > 0) lk = min(lk, k);
        }
        const unsigned m = gmin_u(lk);
        if (m == 0xffffffffu) { set_empty<SD>(); return; }
        int lts = INT_MAX, ltns = INT_MAX, lj = -1;
        unsigned long long lv = 0;
#pragma unroll
        for (int j = 0; j < R; ++j) {
            const int q = bk.hot(SD, F_Q, j), p = bk.hot(SD, F_P, j);
            const unsigned k = (SD == ASK) ? (unsigned)(p - 1) : (unsigned)(INT_MAX - p);
            if (q > 0 && k == m) {
                const int2 t2 = bk.times(SD, j * GT + tid);
                if (lj < 0 || t2.x < lts || (t2.x == lts && t2.y < ltns)) { lts = t2.x; ltns = t2.y; lj = j; }
                if constexpr (TL1) lv += (unsigned)q;
            }
        }
        if constexpr (TL1) bV[SD] = gadd64(lv);
        const bool in = lj >= 0;
        const int w1 = __reduce_min_sync(FULL, in ? lts : INT_MAX);
        const bool in1 = in && lts == w1;
        const int w2 = __reduce_min_sync(FULL, in1 ? ltns : INT_MAX);
        const unsigned w3 = __reduce_min_sync(FULL, (in1 && ltns == w2) ? (unsigned)(lj * GT + tid) : 0xffffffffu);
        const uint32_t base = xbase();
        if ((tid & 31) == 0) sts128(base + 16u * (tid >> 5), make_int4(w1, w2, (int)w3, 0));
        __syncthreads();
        const int lane = tid & 31;  // lane k < W takes warp k's winner; the same REDUXes again
        const int4 c = lane < W ? lds128(base + 16u * lane) : make_int4(INT_MAX, INT_MAX, -1, 0);
        xph ^= 1;
        const int b1 = __reduce_min_sync(FULL, c.x);
        const bool c1 = c.x == b1;
        const int b2 = __reduce_min_sync(FULL, c1 ? c.y : INT_MAX);
        const unsigned b3 = __reduce_min_sync(FULL, (c1 && c.y == b2) ? (unsigned)c.z : 0xffffffffu);
        bslot[SD] = (int)b3;
        bP[SD] = (SD == ASK) ? (int)(m + 1u) : (int)(INT_MAX - (int)m);
        set_bt<SD>(b1, b2);
    }

    // an empty side's cached price never overlaps a limit price (1 .. INT_MAX-1 for a
    // buy against asks, >= 1 for a sell against bids), so the marketability test needs
    // no separate emptiness check
    template <int SD>
    __device__ __forceinline__ void set_empty() {
        bslot[SD] = BEST_EMPTY;
        bP[SD] = (SD == ASK) ? INT_MAX : 0;
    }
    template <int SD>
    __device__ __forceinline__ void set_bt(int ts, int tns) {
        if constexpr (kBtRegs) {
            bTS[SD] = ts; bTNS[SD] = tns;
        } else {
            group_sync<W>();                 // earlier readers of bt are done
            if constexpr (PRED) {            // one writer, published to the group
                sts32_if0(tid, bt_addr(SD, 0), ts);
                sts32_if0(tid, bt_addr(SD, 1), tns);
            } else if (tid == 0) {
                sts32(bt_addr(SD, 0), ts);
                sts32(bt_addr(SD, 1), tns);
            }
            group_sync<W>();
        }
    }

    // A new order at `slot` on side SD: keep the cache exact (G4 key order).
    template <int SD>
    __device__ __forceinline__ void note_add(int slot, int p, int ts, int tns, int q) {
        const int bs = bslot[SD];
        if (bs == BEST_INVALID) return;
        bool better = bs == BEST_EMPTY;
        if (!better) {
            const int kn = (SD == ASK) ? p : ~p, kb = (SD == ASK) ? bP[SD] : ~bP[SD];
            better = kn < kb;
            if (kn == kb) {  // same price: time, then slot (G4)
                const int bts = kBtRegs ? bTS[SD] : lds32(bt_addr(SD, 0));
                const int btns = kBtRegs ? bTNS[SD] : lds32(bt_addr(SD, 1));
                better = ts < bts || (ts == bts && (tns < btns || (tns == btns && slot < bs)));
            }
        }
        if (better) {
            bslot[SD] = slot; bP[SD] = p;
            set_bt<SD>(ts, tns);
        }
    }

    // Cancellation (cancel == delete P:L289): lowest occupied slot with
    // OID == msg OID on the message's side (G16), else the lowest synthetic
    // order (OID <= -9000, G12) at the message price.
    template <int SD>
    __device__ __forceinline__ void cancel(int mQ, int mP, int mOID) {
        // one row-bound branch for the whole cancel: scans and owner update over R rows
        with_rows(hr[SD], [&](auto R) { cancel_r<SD, R>(mQ, mP, mOID); });
    }
    // the cancelled order: its slot (or none, >= NP) and, on the owner thread, its Q
    template <int SD, int R>
    __device__ __forceinline__ int cancel_find(int mP, int mOID, int &qi, int mQ, bool &emptied) {
        if constexpr (W >= LOB_CXL2_W) {
            // ONE pass, ONE group minimum: each thread's lowest exact-OID row and lowest
            // synthetic row at P (with their Q), keyed so that any exact match in the group
            // beats every synthetic one: exact -> slot, synthetic -> NP + slot, none -> 2 NP.
            // The owner's captured Q is the found order's (its lowest match is the slot).
            unsigned rex = KPL, rsy = KPL;
            int qex = 0, qsy = 0;
#pragma unroll
            for (int j = R - 1; j >= 0; --j) {
                const int q = bk.hot(SD, F_Q, j), o = bk.hot(SD, F_OID, j);
                if (q > 0 && o == mOID) { rex = (unsigned)j; qex = q; }
                if (q > 0 && o <= -9000 && bk.hot(SD, F_P, j) == mP) { rsy = (unsigned)j; qsy = q; }
            }
            const unsigned key = rex < (unsigned)KPL
                                     ? rex * GT + (unsigned)tid
                                     : (rsy < (unsigned)KPL ? (unsigned)BK::NP + rsy * GT + (unsigned)tid : 2u * BK::NP);
            if constexpr (kFreeHint) {
                // bit 0: the cancel empties the found order (min(Q, Q_i) = Q_i) --
                // the owner's key wins the minimum, so the bit arrives uniform
                const int qo = rex < (unsigned)KPL ? qex : qsy;
                const unsigned k2 = gmin_u(key * 2u + (qo <= mQ ? 1u : 0u));
                const unsigned k = k2 >> 1;
                emptied = (k2 & 1u) != 0u;
                const bool exact = k < (unsigned)BK::NP;
                qi = exact ? qex : qsy;
                return (int)(exact ? k : k - BK::NP);
            } else {
                const unsigned k = gmin_u(key);
                const bool exact = k < (unsigned)BK::NP;
                qi = exact ? qex : qsy;
                return (int)(exact ? k : k - BK::NP);  // >= NP when neither exists
            }
        } else {
            // exact OID first, then the synthetic fallback (G12); the scans capture
            // the Q of each thread's lowest matching row (the owner's is the found order's):
            // no select chain after the reduction (C5 N = 512 +8 %, C4 / C2 +0.3 %)
            if constexpr (kFreeHint) {  // the same two passes, bit 0 of the key: the cancel empties it
                const auto pass = [&](auto pred) {
                    unsigned r = KPL;
#pragma unroll
                    for (int j = R - 1; j >= 0; --j)
                        if (pred(j)) { r = (unsigned)j; qi = bk.hot(SD, F_Q, j); }
                    const unsigned k2 = gmin_u((r * GT + (unsigned)tid) * 2u + (qi <= mQ ? 1u : 0u));
                    emptied = (k2 & 1u) != 0u;
                    return (int)(k2 >> 1);
                };
                int slot = pass([&](int j) { return bk.hot(SD, F_Q, j) > 0 && bk.hot(SD, F_OID, j) == mOID; });
                if (!found(slot))
                    slot = pass([&](int j) {
                        return bk.hot(SD, F_Q, j) > 0 && bk.hot(SD, F_OID, j) <= -9000 && bk.hot(SD, F_P, j) == mP;
                    });
                return slot;
            }
            int slot = lowest_rows_q<SD, R>(qi, [&](int j) { return bk.hot(SD, F_Q, j) > 0 && bk.hot(SD, F_OID, j) == mOID; });
            if (!found(slot))
                slot = lowest_rows_q<SD, R>(qi, [&](int j) {
                    return bk.hot(SD, F_Q, j) > 0 && bk.hot(SD, F_OID, j) <= -9000 && bk.hot(SD, F_P, j) == mP;
                });
            return slot;
        }
    }
    template <int SD, int R>
    __device__ __forceinline__ void cancel_r(int mQ, int mP, int mOID) {
        int qi = 0;
        bool emptied = false;
        const int slot = cancel_find<SD, R>(mP, mOID, qi, mQ, emptied);
        if (!found(slot)) {                        // G15
            if constexpr (PRED) add64_if0(tid, sc + 8u * ST_UNKNOWN, 1);
            else if (tid == 0) count(ST_UNKNOWN, 1);
            return;
        }
        const bool own = tid == (slot & (GT - 1));
        const int j = slot / GT;                   // the slot is occupied: its row is below R
        const int cq = (mQ < qi) ? mQ : qi;
        if (own) part_cxl += cq;                   // G14
        bk.template put_if_r<R>(own, SD, F_Q, j, qi - mQ);  // Q <= 0 -> empty
        if constexpr (TL1) {                       // the level volume loses what was cancelled there
            const int d = bcast(bk.get(SD, F_P, j) == bP[SD] ? cq : 0, slot & (GT - 1));
            if (bslot[SD] >= 0) bV[SD] -= (unsigned long long)d;
        }
        if (bslot[SD] == slot) bslot[SD] = BEST_INVALID;
        if constexpr (kFreeHint)
            if (emptied && slot < flb[SD]) frm[SD] = min(frm[SD], slot);
    }

    // Limit (T=1) or market (T=4) order of side OWN.
    template <int OWN>
    __device__ __forceinline__ void aggress(bool market, int mQ, int mP, int mOID, int mTID, int mTS, int mTNS) {
        constexpr int OPP = 1 - OWN;
        const int Pa = mP;  // a market order's P is already 0 / max_int (G18; msg_decode)
        int Qa = mQ;
        // the cached best decides most messages without a scan: a side known empty, or
        // no price overlap with its best order
        const bool no_fill = bslot[OPP] != BEST_INVALID && (OWN == BID ? (Pa < bP[OPP]) : (Pa > bP[OPP]));
        // the opposite side's row bound is fixed during the fills (they only remove)
        if (!no_fill && Qa > 0) with_rows(hr[OPP], [&](auto R) { Qa = fill_r<OWN, R>(Pa, Qa, mOID, mTS, mTNS); });
        if (Qa <= 0) return;
        if (market) {
            if (tid == 0) count(ST_DISCARDED, Qa);
            return;
        }
        // remainder rests as one new order in the lowest empty slot (G3)
        with_rows(hr[OWN], [&](auto R) { add_r<OWN, R>(Qa, mP, mOID, mTID, mTS, mTNS); });
    }
    // the fill loop against the opposite side (rows 0..R-1); returns the remainder Q_a'
    template <int OWN, int R>
    __device__ __forceinline__ int fill_r(int Pa, int Qa, int mOID, int mTS, int mTNS) {
        constexpr int OPP = 1 - OWN;
        while (Qa > 0) {
            if (bslot[OPP] == BEST_INVALID) recompute_best_r<OPP, R>();
            const int s = bslot[OPP];
            if (s < 0) break;                                      // side empty
            const int Ps = bP[OPP];
            if (OWN == BID ? (Pa < Ps) : (Pa > Ps)) break;         // prices do not overlap
            lastPs = Ps;
            const int ol = s & (GT - 1);
            const bool own = tid == ol;
            const int sj = s / GT;
            const int myoid = bk.template get_r<R>(OPP, F_OID, sj);  // meaningful on the owner
            const int Qs = bcast(bk.template get_r<R>(OPP, F_Q, sj), ol);
            const int Qs2 = (Qs - Qa > 0) ? (Qs - Qa) : 0;           // Q_s' = max(0, Q_s - Q_a)
            const int q = Qs - Qs2;                                  // Q_j = Q_s - Q_s'
            Qa = Qa - Qs;                                            // Q_a' = Q_a - Q_s
            if constexpr (PREDT) {                                   // Eq.3 record, Eq.4 cap (G8)
                trade_store_if(own && ntr < p.Tcap,
                               reinterpret_cast<int2 *>(p.trades + ((size_t)book * p.Tcap + ntr) * 6),
                               make_int2(Ps, q), make_int2(mOID, myoid), make_int2(mTS, mTNS));
                if (own) part_trd += q;
            } else if (own) {
                if (ntr < p.Tcap) {
                    int2 *t = reinterpret_cast<int2 *>(p.trades + ((size_t)book * p.Tcap + ntr) * 6);
                    t[0] = make_int2(Ps, q);
                    t[1] = make_int2(mOID, myoid);
                    t[2] = make_int2(mTS, mTNS);
                }
                part_trd += q;
            }
            ++ntr;                                                   // fills this call (logged = min(ntr, Tcap))
            bk.template put_if_r<R>(own, OPP, F_Q, sj, Qs2);         // filled order removed (G10)
            if constexpr (TL1) bV[OPP] -= (unsigned long long)q;
            if (Qs2 == 0) {
                bslot[OPP] = BEST_INVALID;
                if constexpr (kFreeHint)
                    if (s < flb[OPP]) frm[OPP] = min(frm[OPP], s);
            }
        }
        return Qa;
    }
    // the add over the row bound R: free slot in rows 0..R-1, else row R's first slot.
    // Capacity (G6): the geometry pads N to NP >= N slots, and the padding slots are
    // empty (-1), so the group minimum may land on one; slot indices grow with the row,
    // so the minimum over all empty slots is below N exactly when a free slot < N
    // exists -- ONE compare against N after the reduction decides saturation.
    template <int OWN, int R>
    __device__ __forceinline__ void add_r(int Qa, int mP, int mOID, int mTID, int mTS, int mTNS) {
        int slot;
        if (kFreeHint && frm[OWN] < BK::NP) {
            slot = frm[OWN];                                         // the lowest empty slot, known
        } else {
            unsigned r = KPL;
            if constexpr (R < KPL) r = (unsigned)R;
#pragma unroll
            for (int j = R - 1; j >= 0; --j)
                if (bk.hot(OWN, F_Q, j) <= 0) r = (unsigned)j;
            slot = (int)gmin_u(r * GT + (unsigned)tid);
            if (slot >= p.N) {                                       // side saturated (G6)
                if (tid == 0) { count(ST_ADD_OVF, 1); count(ST_OVF_QTY, Qa); }
                return;
            }
        }
        if constexpr (kFreeHint) { flb[OWN] = slot + 1; frm[OWN] = BK::NP; }
        const bool own = tid == (slot & (GT - 1));
        if constexpr (ROWS) hr[OWN] = max(hr[OWN], slot / GT);
        const auto put = [&](auto J) {                               // G27
            if (own) {
                bk.v[OWN][F_P][J] = mP;
                bk.v[OWN][F_Q][J] = Qa;
                bk.v[OWN][F_OID][J] = mOID;
            }
        };
        // the slot's row is at most R: a compare chain instead of the jump table
        if constexpr (KPL >= LOB_ADDSEL) {
            // predicated selects over rows 0..R (independent: no branch chain)
            constexpr int RR = R < KPL ? R + 1 : KPL;
            bk.template put_if_r<RR>(own, OWN, F_P, slot / GT, mP);
            bk.template put_if_r<RR>(own, OWN, F_Q, slot / GT, Qa);
            bk.template put_if_r<RR>(own, OWN, F_OID, slot / GT, mOID);
        } else if constexpr (R < KPL) bk.template row_r<R + 1>(slot / GT, put);
        else if constexpr (KPL <= LOB_ROWR) bk.template row_r<KPL>(slot / GT, put);
        else bk.row(slot / GT, put);
        if constexpr (PRED) sts128_if0(tid, bk.rec(OWN, slot), make_int4(mOID, mTID, mTS, mTNS));  // one writer
        else if (tid == 0) bk.put_cold(OWN, slot, make_int4(mOID, mTID, mTS, mTNS));
        // W = 1: __syncwarp publishes it to the lanes' next cold reads.  W > 1: cold
        // records are read only inside recompute_best_multi, after its first barrier,
        // and every such read completes before its second barrier, so the barriers
        // already order this write against earlier and later reads.
        if constexpr (W == 1 && !kSyncReader) group_sync<W>();
        if constexpr (TL1) {  // level volume: a new best level, or one more order at the best price
            const int ob = bslot[OWN], op = bP[OWN];
            const bool lvl = ob == BEST_EMPTY || (ob >= 0 && ((OWN == ASK) ? mP < op : mP > op));
            const bool same = ob >= 0 && mP == op;
            bV[OWN] = lvl ? (unsigned long long)Qa : (same ? bV[OWN] + (unsigned long long)Qa : bV[OWN]);
        }
        note_add<OWN>(slot, mP, mTS, mTNS, Qa);
    }

    // NEXT N1: Level-1 after the message: the cached best of each side
    // (recomputed if stale) and its level volume; absent side (-1, 0)
    __device__ __forceinline__ void l1_write(int32_t *dst) {
        if (bslot[ASK] == BEST_INVALID) recompute_best<ASK>();
        if (bslot[BID] == BEST_INVALID) recompute_best<BID>();
        const bool a = bslot[ASK] >= 0, b = bslot[BID] >= 0;
        // predicated store (no lane-divergent branch in the message loop)
        stg128_if0(tid, dst,
                   make_int4(a ? bP[ASK] : -1, a ? sat32(bV[ASK]) : 0, b ? bP[BID] : -1, b ? sat32(bV[BID]) : 0));
    }

    // A message whose first word holds its dispatch code (msg_code) instead of T.
    __device__ __forceinline__ void message_coded(const int4 a, const int4 b) {
        const int c = a.x, Q = a.z, P = a.w;
        // the paper's 8 (type x side) cases; cancel and delete share one.  The
        // order type is tested first (padding / malformed last: C4 +2 %), except for the
        // 16-row build, where that order measured 8 % slower (code layout)
        if constexpr (KPL > 8) {
            if (c < MC_CANCEL) {                               // padding (G21) / malformed (G22)
                if (c == MC_BAD && tid == 0) count(ST_BAD, 1);
                return;
            }
        }
        if (c & MC_AGGR) {
            if ((c & MC_BID) != 0) aggress<BID>(c & MC_MKT, Q, P, b.x, b.y, b.z, b.w);
            else aggress<ASK>(c & MC_MKT, Q, P, b.x, b.y, b.z, b.w);
        } else if (KPL > 8 || c >= MC_CANCEL) {
            if ((c & MC_BID) != 0) cancel<BID>(Q, P, b.x);
            else cancel<ASK>(Q, P, b.x);
        } else if (c == MC_BAD && tid == 0) {                   // malformed (G22); padding (G21) is a no-op
            count(ST_BAD, 1);
        }
    }
    // A message in Eq.6 form (the env agent's own orders).
    __device__ __forceinline__ void message(const int4 a, const int4 b) {
        message_coded(msg_decode(a), b);
    }

    // L2 (G23): k-th best distinct price per side and its summed quantity;
    // thread k keeps level k.  Absent levels are (-1, 0).  Each level takes the
    // group minimum of the remaining keys and retires every slot at that price.
    template <int SD, int R>
    __device__ __forceinline__ void l2_rows(int L, int &outp, int &outq) {
        // offset price keys as in recompute_best: all-ones = no (further) level
        unsigned key[R];
        int hl = -1;
#pragma unroll
        for (int j = 0; j < R; ++j) {
            const int p = bk.hot(SD, F_P, j);
            const bool occ = bk.hot(SD, F_Q, j) > 0;
            key[j] = occ ? ((SD == ASK) ? (unsigned)(p - 1) : (unsigned)(INT_MAX - p)) : 0xffffffffu;
            if (occ) hl = j;
        }
        if constexpr (kX4) {
            // 4-warp books: level k's volume and level k+1's price travel in ONE exchange
            // (the next minimum needs only this thread's keys once level k is retired), and
            // the row bound rides with level 0's price: L + 1 barriers instead of 2 L + 1
            unsigned lk = key[0];
#pragma unroll
            for (int j = 1; j < R; ++j) lk = min(lk, key[j]);
            int4 a, b;
            exchange_pair4(__reduce_min_sync(FULL, (unsigned)(KPL - 1 - hl)), __reduce_min_sync(FULL, lk), a, b);
            if constexpr (ROWS) hr[SD] = (KPL - 1) - (int)min(min((unsigned)a.x, (unsigned)a.z), min((unsigned)b.x, (unsigned)b.z));
            unsigned m = min(min((unsigned)a.y, (unsigned)a.w), min((unsigned)b.y, (unsigned)b.w));
            for (int k = 0; k < L; ++k) {
                if (m == 0xffffffffu) break;
                unsigned lq = 0, nk = 0xffffffffu;
#pragma unroll
                for (int j = 0; j < R; ++j) {
                    if (key[j] == m) { lq += (unsigned)bk.hot(SD, F_Q, j); key[j] = 0xffffffffu; }
                    nk = min(nk, key[j]);
                }
                exchange_pair4(__reduce_add_sync(FULL, lq), __reduce_min_sync(FULL, nk), a, b);
                const unsigned qs = ((unsigned)a.x + (unsigned)a.z) + ((unsigned)b.x + (unsigned)b.z);
                if (tid == k) { outp = (SD == ASK) ? (int)(m + 1u) : (int)(INT_MAX - (int)m); outq = (int)qs; }
                m = min(min((unsigned)a.y, (unsigned)a.w), min((unsigned)b.y, (unsigned)b.w));
            }
            return;
        }
        if constexpr (ROWS) hr[SD] = (KPL - 1) - (int)gmin_u((unsigned)(KPL - 1 - hl));  // exact row bound again
        for (int k = 0; k < L; ++k) {
            unsigned lk = key[0];
#pragma unroll
            for (int j = 1; j < R; ++j) lk = min(lk, key[j]);
            const unsigned m = gmin_u(lk);
            if (m == 0xffffffffu) break;
            unsigned lq = 0;
#pragma unroll
            for (int j = 0; j < R; ++j)
                if (key[j] == m) { lq += (unsigned)bk.hot(SD, F_Q, j); key[j] = 0xffffffffu; }
            const unsigned qs = gadd(lq);
            if (tid == k) { outp = (SD == ASK) ? (int)(m + 1u) : (int)(INT_MAX - (int)m); outq = (int)qs; }
        }
    }
    // L2 over the first R rows only (with_rows).  Volume (G20): the exact sum, saturated
    // at INT32_MAX.  While every resting Q on the side is below 2^20 no level can reach
    // 2^31 (N <= 2048) and the 32-bit sums above are exact; otherwise (one vote per
    // snapshot decides, uniformly) the volumes are recomputed in 64 bits -- a rare path
    // kept outside the row-specialised code.
    template <int SD>
    __device__ __forceinline__ void l2_side(int L, int &outp, int &outq) {
        outp = -1; outq = 0;
        const int h = hr[SD];
        if (h < 0) return;
#if LOB_L2FULL
        if constexpr (KPL >= 8) l2_rows<SD, KPL>(L, outp, outq);
        else
#endif
        with_rows(h, [&](auto R) { l2_rows<SD, R>(L, outp, outq); });
        bool bg = false;
#pragma unroll
        for (int j = 0; j < KPL; ++j) bg |= bk.hot(SD, F_Q, j) >= (1 << 20);
        if (gany(bg)) {
            for (int k = 0; k < L; ++k) {
                const int pk = bcast(tid == k ? outp : 0, k);   // level k's price (-1: absent)
                if (pk < 0) break;
                unsigned long long l64 = 0;
#pragma unroll
                for (int j = 0; j < KPL; ++j)
                    if (bk.hot(SD, F_Q, j) > 0 && bk.hot(SD, F_P, j) == pk) l64 += (unsigned)bk.hot(SD, F_Q, j);
                const int v = sat32(gadd64(l64));
                if (tid == k) outq = v;
            }
        }
    }
    __device__ __forceinline__ void l2_write(int32_t *dst, int L) {
        int ap, aq, bp, bq;
        l2_side<ASK>(L, ap, aq);
        l2_side<BID>(L, bp, bq);
        if (tid < L) reinterpret_cast<int4 *>(dst)[tid] = make_int4(ap, aq, bp, bq);
    }
};

// ------------------------------------------------------------------ step kernel
// Per-book shared scratch: counters [NST] int64, best times [2][2] int32,
// cross-warp exchange buffers [2][W] u32.
template <int W>
constexpr int scratch_bytes() { return 8 * NST + 16 + (W == 1 ? 8 : 32 * W) + 8; }

__device__ __forceinline__ double warp_sum(double x) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(FULL, x, o);
    return x;
}

// ---------------------------------------------------- NEXT N3: fused env step
// The agent's action -> at most 8 messages, processed before the step's data
// (P:L417-418): cancel (delete) the previous step's orders (E1); then either the
// forced market order one minute before the end or one limit order per
// positive size at the far-touch / mid / near-touch / passive prices (P:L476-493,
// P:L457-465; E2-E6).  Every price comes from the book as it was before the
// first agent message.  All values are group-uniform; the messages are also
// written to agent_out (thread 0) for observability.
template <class E>
__device__ __forceinline__ void env_agent(E &e, EnvState &es, const Params &p, const EnvParams &ep, int b, int tid) {
    const EnvCfg &c = ep.ec;
    int4 *out = reinterpret_cast<int4 *>(ep.agent_out + (size_t)b * 64);
    int n = 0;
    if (!es.done) {
        if (e.bslot[ASK] == BEST_INVALID) e.template recompute_best<ASK>();
        if (e.bslot[BID] == BEST_INVALID) e.template recompute_best<BID>();
        int ask = e.bslot[ASK] >= 0 ? e.bP[ASK] : -1, bid = e.bslot[BID] >= 0 ? e.bP[BID] : -1;
        const int S = c.task_side;
        long long remaining = (long long)c.task_size - es.executed;
        const bool forced = remaining > 0 && env_elapsed_ns(es) >= ((long long)c.episode_s - 60) * 1000000000LL;
        const bool limits = remaining > 0 && !forced;
        int pr0 = 0, pr1 = 0, pr2 = 0, pr3 = 0;
        if (limits) {
            if (ask > 0) es.last_ask = ask; else ask = es.last_ask;  // E6
            if (bid > 0) es.last_bid = bid; else bid = es.last_bid;
            const int far = (S == -1) ? bid : ask, near = (S == -1) ? ask : bid;
            pr0 = far;
            pr2 = near;
            pr3 = near > 0 ? near - S * c.n_passive * c.tick : 0;
            if (ask > 0 && bid > 0) {  // E5: the tick at or beyond the mid, away from the spread
                const long long twice = (long long)ask + bid, t2 = 2LL * c.tick;
                const long long q = twice / t2, rmd = twice % t2;
                pr1 = (int)((S == -1 && rmd) ? (q + 1) * c.tick : q * c.tick);
            }
        }
        const int l0 = es.live[0], l1 = es.live[1], l2 = es.live[2], l3 = es.live[3];
        int n0 = 0, n1 = 0, n2 = 0, n3 = 0, li = 0;
        for (int k = 0; k < 9; ++k) {
            int T = 0, Q = 0, P = 0, O = 0;
            if (k < 4) {  // E1
                const int l = k == 0 ? l0 : (k == 1 ? l1 : (k == 2 ? l2 : l3));
                if (l != 0) { T = 3; Q = INT_MAX; O = l; }
            } else if (k == 4) {
                if (forced) { T = 4; Q = (int)(remaining > INT_MAX ? INT_MAX : remaining); O = es.next_oid++; }
            } else if (limits) {
                const int j = k - 5;
                // L2-coherent load: a resident session (lob_session.cuh) reads a buffer the
                // caller rewrites between steps, which a stale L1 line would hide
                const float x = __ldcg(ep.actions + 4 * (size_t)b + j);
                long long q = 0;  // E2: round half-even, NaN / negative -> 0
                if (x == x && x > 0.0f) q = (x >= 2147483647.0f) ? 2147483647LL : (long long)__float2int_rn(x);
                if (q > remaining) q = remaining;  // E3
                const int pr = j == 0 ? pr0 : (j == 1 ? pr1 : (j == 2 ? pr2 : pr3));
                if (q > 0 && pr > 0) {
                    remaining -= q;
                    T = 1; Q = (int)q; P = pr; O = es.next_oid++;
                    n0 = li == 0 ? O : n0; n1 = li == 1 ? O : n1; n2 = li == 2 ? O : n2; n3 = li == 3 ? O : n3;
                    ++li;
                }
            }
            if (T != 0) {
                const int4 a = make_int4(T, S, Q, P), bb = make_int4(O, c.agent_tid, es.cur_ts, es.cur_tns);
                if (tid == 0) { out[2 * n] = a; out[2 * n + 1] = bb; }
                ++n;
                e.message(a, bb);
            }
        }
        es.live[0] = n0; es.live[1] = n1; es.live[2] = n2; es.live[3] = n3;
    }
    if (tid == 0)
        for (int i = n; i < 8; ++i) out[2 * i] = out[2 * i + 1] = make_int4(0, 0, 0, 0);
}

// After the step: reward over the step's logged trades (eq:rewardfunc / eq:vwap,
// P:L498-506, agent = OIDs [oid_base, next_oid), G29; the same sums as
// lob_reward_kernel), executed quantity, time := the last data message,
// termination.  The group's first warp; trades were written
// by their owner threads, hence the barrier.
// the group's first warp: reward, executed quantity, time, termination
__device__ __forceinline__ void env_post_warp(const Params &p, const EnvParams &ep, int b, int tid, int n,
                                              bool have_last, int last_ts, int last_tns) {
    const EnvCfg &c = ep.ec;
    EnvState es = ep.env[b];
    const int lane = tid;
    if (es.done) {  // finished before this step (E8)
        if (lane == 0) {
            if (ep.reward) ep.reward[b] = 0.0;
            if (ep.done) ep.done[b] = 1;
            if (ep.executed) ep.executed[b] = es.executed;
        }
    } else {
        const int2 *t = reinterpret_cast<const int2 *>(p.trades + (size_t)b * p.Tcap * 6);
        double sqp = 0.0, sq = 0.0;
        for (int i = lane; i < n; i += 32) {
            const int2 pq = t[3 * i];
            sqp += (double)pq.y * (double)pq.x;
            sq += (double)pq.y;
        }
        sqp = warp_sum(sqp);
        sq = warp_sum(sq);
        const double v = sq > 0.0 ? sqp / sq : 0.0;
        const int lo = c.oid_base, hi = es.next_oid - 1;
        double adv = 0.0, drift = 0.0;
        long long qa = 0;
        for (int i = lane; i < n && sq > 0.0; i += 32) {
            const int2 pq = t[3 * i], oo = t[3 * i + 1];
            if ((oo.x >= lo && oo.x <= hi) || (oo.y >= lo && oo.y <= hi)) {
                adv += (double)pq.y * ((double)pq.x - v);
                drift += (double)pq.y * (v - es.p_init);
                qa += pq.y;
            }
        }
        adv = warp_sum(adv);
        drift = warp_sum(drift);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) qa += __shfl_xor_sync(FULL, qa, o);
        if (lane == 0) {
            es.executed += qa;
            if (have_last) { es.cur_ts = last_ts; es.cur_tns = last_tns; }
            es.done = (es.executed >= c.task_size) || (env_elapsed_ns(es) > (long long)c.episode_s * 1000000000LL);
            const double r = adv + c.lam * drift;
            if (ep.reward) ep.reward[b] = c.task_side == 1 ? -r : r;
            if (ep.done) ep.done[b] = es.done;
            if (ep.executed) ep.executed[b] = es.executed;
            ep.env[b] = es;
        }
    }
}

template <int W>
__device__ __forceinline__ void env_post(const Params &p, const EnvParams &ep, int b, int tid, int n, bool have_last,
                                         int last_ts, int last_tns) {
    group_sync<W>();  // also publishes env_agent's state write (thread 0)
    // no early returns: a data-dependent exit here made ptxas treat the whole persistent
    // loop as possibly diverged (reconvergence barriers and divergence checks throughout)
    if constexpr (W == 1) env_post_warp(p, ep, b, tid, n, have_last, last_ts, last_tns);
    else if (tid < 32) env_post_warp(p, ep, b, tid, n, have_last, last_ts, last_tns);
}

#ifdef LOB_TRACE_CYCLES
// instrumented variant only: clock64 at the start of every message and around every L2
// snapshot of the first LOB_TRACE_BOOKS books of a launch (scripts/cycle_budget.py)
constexpr int LOB_TRACE_BOOKS = 8, LOB_TRACE_MSGS = 10240, LOB_TRACE_STEPS = 128;
__device__ long long g_trace_msg[LOB_TRACE_BOOKS][LOB_TRACE_MSGS];
__device__ long long g_trace_l2[LOB_TRACE_BOOKS][LOB_TRACE_STEPS][2];
#endif

// Dynamic shared memory of one CTA of G books of (KPL, W).
template <int KPL, int W, int G>
constexpr int step_smem_bytes() {
    return G * (2 * CH * 32 + 16 + 2 * KPL * 32 * W * 16 + ((scratch_bytes<W>() + 15) / 16) * 16);
}

#ifndef MINB4
#define MINB4 7
#endif
#ifndef MINB16  // 16-row one-warp books (MODE 0): register budget of 4 CTAs/SM (128 registers;
#define MINB16 4   // shared memory still allows 3): C5 N = 512 +1 % over the 168-register build
#endif
#ifndef MINB8W  // 8-row 4-warp books: CTAs (books) per SM the registers are sized for
#define MINB8W 5  // (5: 96 registers, C5 N = 1024 +8 % over 4; 6: +4 %; the L1 / env builds keep 4)
#endif
#ifndef MINB8
#define MINB8 5  // 8-row one-warp books: 5 CTAs/SM (102 registers): C5 N = 256 +3 % over 3 (128 registers)
#endif
// Persistent: group g of CTA b starts with book b*G + g, then takes books from the
// dynamic counter.  MODE 0 (and 3): L2 per step; MODE 1 also writes the Level-1
// trace (NEXT N1); MODE 2 is one fused execution-env step (NEXT N3, env_agent /
// env_post).
// MODE 3 = MODE 0 built for 8 CTAs/SM (64 registers); chosen by the host for many-wave
// batches of 4-row books.  (With the uniform persistent loop MODE 0 also fits in 64
// registers without spills, so the two now compile alike; MODE 3 keeps the hard cap.)
// resident CTAs per SM the register budget is sized for
template <int KPL, int W, int MODE>
constexpr int step_min_blocks() {
    return MODE == 3 ? 8 : (KPL <= 2 ? 7 : (KPL <= 4 ? MINB4 : (W == 1 ? (KPL > 8 ? (MODE == 0 ? MINB16 : 3) : MINB8) : (KPL > 8 ? 12 / W : (MODE == 0 ? MINB8W : 16 / W)))));
}
template <int KPL, int W, int G, int MODE>
__global__ void __launch_bounds__(32 * W * G, step_min_blocks<KPL, W, MODE>())
    lob_step(const Params p, const EnvParams ep) {
    using BK = RegBook<KPL, W>;
    constexpr bool TL1 = MODE == 1, ENV = MODE == 2;
    // row-bounded scans (Engine::with_rows) in every build: C4 +4.5 %, C3 +10 %, C5
    // N = 256 +3 %, N = 2048 +9 %, C2 -0.5 % (measured with the uniform persistent loop;
    // before it, the extra branch cost C2 4 %)
    constexpr bool kRows = true;
    extern __shared__ __align__(128) unsigned char dyn[];
    // the group index through a warp reduction: ptxas then knows it (and every shared
    // address below) is warp-uniform, so messages loaded from those addresses are
    // uniform and the dispatch branches need no reconvergence (BSSY/BSYNC) and the
    // warp collectives no divergence check (BRA.DIV).  Kept even when G = 1 (the
    // value is then 0): a one-warp build without this opening collective compiled
    // with 66 divergence checks.
    const int g = (int)__reduce_min_sync(FULL, threadIdx.x / (32 * W));
    const int tid = (int)opaque(threadIdx.x % (32 * W));
    // carve this group's region: stage [2][CH][32 B] | bars [2] | cold [2][NP][16 B] | scratch
    unsigned char *base = dyn + g * (step_smem_bytes<KPL, W, G>() / G);
    const uint32_t stage = smem_u32(base);
    const uint32_t bars = smem_u32(base + 2 * CH * 32);
    const uint32_t cold = smem_u32(base + 2 * CH * 32 + 16);
    const uint32_t scratch = smem_u32(base + 2 * CH * 32 + 16 + 2 * BK::NP * 16);
    if (tid == 0) {
        mbar_init(bars, 1);
        mbar_init(bars + 8, 1);
        fence_mbar_init();
    }
    group_sync<W>();
    const int nmsg = p.n_steps * p.M;
    const int nchunks = (nmsg + CH - 1) / CH;
    uint32_t chunk_seq = 0;
    // dynamic book scheduling: deep sweeps make books unequal, so after its first
    // (static) book a group takes the next one from a global counter when it is free
    constexpr int next_off = 2 * CH * 32 + 16 + 2 * BK::NP * 16 + 8 * NST + 16 + (W == 1 ? 8 : 32 * W);
    const int groups = gridDim.x * G;
    const bool multi = groups < p.nb;  // more books than groups: dynamic scheduling (sched counters)
    int lb = blockIdx.x * G + g;
    while (lb < p.nb) {
        const int b = p.book0 + lb;
        const int4 *src = reinterpret_cast<const int4 *>(p.msgs + (size_t)lb * nmsg * 8);
        // prologue: the first two chunks are in flight before the book is loaded
        group_sync<W>();
        if (tid == 0) {
            fence_proxy_async();  // earlier generic reads of the buffers before async writes
#pragma unroll
            for (int c = 0; c < 2; ++c) {
                if (c < nchunks) {
                    const uint32_t slot = (chunk_seq + c) & 1;
                    const int cnt = min(CH, nmsg - c * CH);
                    mbar_arrive_expect_tx(bars + 8 * slot, cnt * 32);
                    bulk_g2s(stage + slot * CH * 32, src + (size_t)c * CH * 2, cnt * 32, bars + 8 * slot);
                }
            }
        }
        if (tid < NST) sts64(scratch + 8u * tid, 0);
        // predicated single-writer stores (sts32_if0 ...): all of them in the many-wave
        // build, the trade record in every one-warp build up to 8 rows (C2 +3 %, C3 +2 %,
        // env step -7 %; measured slower for the 16-row build and the other stores)
        Engine<BK, TL1, kRows, MODE == 3, MODE == 3 || (W == 1 && KPL <= 8)> e(p);
        e.bk.cold = cold;
        e.bk.tid = tid;
        e.tid = tid; e.book = b; e.ntr = 0; e.sc = scratch; e.xph = 0;
        e.scp = base + 2 * CH * 32 + 16 + 2 * BK::NP * 16;
        e.part_cxl = 0; e.part_trd = 0;
        e.bk.load(p.book + (size_t)b * 2 * NF * BK::NP);
        e.init_rows();
        e.bslot[0] = e.bslot[1] = BEST_INVALID;
        e.bP[0] = e.bP[1] = 0;
        e.bV[0] = e.bV[1] = 0;
        int32_t *l1dst = TL1 ? p.l1out + (size_t)lb * nmsg * 4 : nullptr;
        int left = p.M, step = 0;
        [[maybe_unused]] int last_ts = 0, last_tns = 0;
        [[maybe_unused]] bool idle = false, have_last = false;
        if constexpr (ENV) {  // the agent's messages go first
            EnvState es = ep.env[b];
            idle = es.done != 0;  // a finished env only sees padding (E8)
            env_agent(e, es, p, ep, b, tid);
            if (tid == 0) ep.env[b] = es;  // re-read by env_post: not live across the message loop
            if (nmsg == 0 && p.l2out) e.l2_write(p.l2out + (size_t)lb * p.L * 4, p.L);
        }
        for (int c = 0; c < nchunks; ++c) {
            const uint32_t seq = chunk_seq + c, slot = seq & 1;
            mbar_wait(bars + 8 * slot, (seq >> 1) & 1);
            uint32_t maddr = stage + slot * CH * 32;
            int cnt = min(CH, nmsg - c * CH);
            // decode the chunk lane-parallel: message i's T becomes its dispatch code
            if (tid < cnt) {
                const uint32_t m = maddr + 32u * (uint32_t)tid;
                const int4 d = msg_decode(lds128(m));
                sts32(m, d.x);
                sts32(m + 12u, d.w);
            }
            group_sync<W>();
            while (cnt > 0) {  // runs up to the next chunk or step end
                const int run = min(cnt, left);
                const uint32_t mend = maddr + 32u * run;
                do {
                    const int4 a = lds128(maddr), bb = lds128(maddr + 16);
#ifdef LOB_TRACE_CYCLES  // instrumented variant only (scripts/cycle_budget.py): message start times
                    if (tid == 0 && lb < LOB_TRACE_BOOKS) {
                        const int mi = c * CH + (int)((maddr - (stage + slot * CH * 32)) >> 5);
                        if (mi < LOB_TRACE_MSGS) g_trace_msg[lb][mi] = clock64();
                    }
#endif
                    if constexpr (ENV) {
                        if (!idle) {
                            e.message_coded(a, bb);
                            if (a.x != 0) { last_ts = bb.z; last_tns = bb.w; have_last = true; }
                        }
                    } else {
                        e.message_coded(a, bb);
                    }
                    if constexpr (TL1) {
                        e.l1_write(l1dst);
                        l1dst += 4;
                    }
                    maddr += 32;
                } while (maddr != mend);
                cnt -= run;
                left -= run;
                if (left == 0) {  // end of a step: L2 snapshot (G23)
                    left = p.M;
#ifdef LOB_TRACE_CYCLES
                    const long long tl0 = clock64();
#endif
                    if (p.l2out) e.l2_write(p.l2out + (((size_t)lb * p.n_steps + step) * p.L) * 4, p.L);
#ifdef LOB_TRACE_CYCLES
                    if (tid == 0 && lb < LOB_TRACE_BOOKS && step < LOB_TRACE_STEPS) {
                        g_trace_l2[lb][step][0] = tl0;
                        g_trace_l2[lb][step][1] = clock64();
                    }
#endif
                    ++step;
                }
            }
            group_sync<W>();  // every thread is done with this buffer
            if (tid == 0 && c + 2 < nchunks) {  // refill it with chunk c+2
                fence_proxy_async();
                const int cn = min(CH, nmsg - (c + 2) * CH);
                mbar_arrive_expect_tx(bars + 8 * slot, cn * 32);
                bulk_g2s(stage + slot * CH * 32, src + (size_t)(c + 2) * CH * 2, cn * 32, bars + 8 * slot);
            }
        }
        chunk_seq += nchunks;
        // writeback: book, trade count, counters (msgs += nmsg; trades = logged + dropped)
        e.bk.store(p.book + (size_t)b * 2 * NF * BK::NP);
        long long cx = e.part_cxl, tq = e.part_trd;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            cx += __shfl_xor_sync(FULL, cx, o);
            tq += __shfl_xor_sync(FULL, tq, o);
        }
        group_sync<W>();
        if ((tid & 31) == 0) {  // one add per warp (rare: once per book)
            atomicAdd(reinterpret_cast<unsigned long long *>(base + 2 * CH * 32 + 16 + 2 * BK::NP * 16) +
                          ST_CANCELLED_QTY, (unsigned long long)cx);
            atomicAdd(reinterpret_cast<unsigned long long *>(base + 2 * CH * 32 + 16 + 2 * BK::NP * 16) +
                          ST_TRADED_QTY, (unsigned long long)tq);
        }
        group_sync<W>();
        const int logged = min(e.ntr, p.Tcap);
        if (tid < NST) {
            long long v = lds64(scratch + 8u * tid);
            if (tid == ST_DROPPED) v += e.ntr - logged;
            if (tid == ST_MSGS) v += nmsg + (ENV ? 8 : 0);  // env: 8 agent rows + data (E8)
            if (tid == ST_TRADES) v += e.ntr;  // fills = logged + dropped
            p.stats[(size_t)b * NST + tid] += v;
        }
        if (tid == 0) p.ntrades[b] = logged;
        if constexpr (ENV) env_post<W>(p, ep, b, tid, logged, have_last, last_ts, last_tns);
        if (!multi) break;  // one wave: every book had a group of its own
        // the next book: claimed by thread 0 with an atomic, handed to the group through a
        // plain shared-memory word.  An atomic's result counts as thread-divergent in the
        // compiler's uniformity analysis (and a shuffle or reduction of it stays so), which
        // would make the whole persistent loop "possibly diverged": reconvergence barriers
        // around every branch and a divergence check before every warp collective (~2x
        // the control instructions).  A load from a uniform shared address is uniform.
        int *next_word = reinterpret_cast<int *>(base + next_off);
        if (tid == 0) *next_word = groups + (int)atomicAdd(p.sched, 1u);
        group_sync<W>();
        lb = *next_word;
    }
    // the last group to finish re-arms the counters for the next launch
    if (multi && tid == 0) {
        __threadfence();
        if (atomicAdd(p.sched + 1, 1u) == gridDim.x * G - 1) {
            atomicExch(p.sched, 0u);
            atomicExch(p.sched + 1, 0u);
        }
    }
}

// ------------------------------------------------------------- init / exports
// a0: -1 everywhere, counters 0, then one synthetic order per
// populated L2 level (G24).  One warp per book.
__global__ void lob_init_kernel(int32_t *book, int32_t *trades, int32_t *ntrades, long long *stats, unsigned *sched,
                                int K, int N, int NP, int Tcap, const int32_t *init_l2, int L0, int ts, int tns) {
    const int lane = threadIdx.x & 31;
    const int b = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (blockIdx.x == 0 && threadIdx.x < 2) sched[threadIdx.x] = 0u;
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
    for (int s = 0; s < 2; ++s) {  // asks (s=0) best->worst, then bids
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

// NEXT row N2: step reward over the last call's trade log (one env step), one warp
// per book.  P_VWAP = sum_i Q_i P_i / sum_i Q_i (eq:vwap): both sums are
// exact in double (integer products < 2^53), so P_VWAP is correctly rounded whatever
// the summation order.  R = sum_j Q_j (P_j - P_VWAP) + lambda sum_j Q_j (P_VWAP -
// P_init) over the agent's trades j (eq:rewardfunc; agent = aggressor or
// standing OID in the book's range, G29); buy task negates (G30); no trades -> 0 (G31).
__global__ void lob_reward_kernel(const int32_t *trades, const int32_t *ntrades, int K, int Tcap,
                                  const int32_t *agent, const double *p_init, const int32_t *side, double lambda,
                                  double *reward, double *vwap, long long *agent_qty) {
    const int lane = threadIdx.x & 31;
    const int b = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (b >= K) return;
    const int n = ntrades[b];
    const int2 *t = reinterpret_cast<const int2 *>(trades + (size_t)b * Tcap * 6);
    double sqp = 0.0, sq = 0.0;
    for (int i = lane; i < n; i += 32) {
        const int2 pq = t[3 * i];
        sqp += (double)pq.y * (double)pq.x;
        sq += (double)pq.y;
    }
    sqp = warp_sum(sqp);
    sq = warp_sum(sq);
    const double v = sq > 0.0 ? sqp / sq : 0.0;
    const int lo = agent[2 * b], hi = agent[2 * b + 1];
    const double p0 = p_init[b];
    double adv = 0.0, drift = 0.0;
    long long qa = 0;
    for (int i = lane; i < n && sq > 0.0; i += 32) {
        const int2 pq = t[3 * i], oo = t[3 * i + 1];
        if ((oo.x >= lo && oo.x <= hi) || (oo.y >= lo && oo.y <= hi)) {
            adv += (double)pq.y * ((double)pq.x - v);
            drift += (double)pq.y * (v - p0);
            qa += pq.y;
        }
    }
    adv = warp_sum(adv);
    drift = warp_sum(drift);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) qa += __shfl_xor_sync(FULL, qa, o);
    if (lane == 0) {
        const double r = adv + lambda * drift;
        if (reward) reward[b] = side[b] == 1 ? -r : r;
        if (vwap) vwap[b] = v;
        if (agent_qty) agent_qty[b] = qa;
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

// Host path (lob_process_messages_host): packed copy of the logged trade rows.
// Row offsets of books [b0, b0+nb): an exclusive scan of the logged-row counts,
// continuing the running total tro[K] of the earlier chunks (one CTA of 1024 threads).
__global__ void __launch_bounds__(1024) lob_trade_offsets(const int32_t *ntrades, long long *tro, int b0, int nb,
                                                          int K) {
    __shared__ long long wsum[32];
    const int t = threadIdx.x, lane = t & 31, w = t >> 5;
    long long base = tro[K];
    for (int i0 = 0; i0 < nb; i0 += 1024) {
        const int i = i0 + t;
        const long long c = i < nb ? ntrades[b0 + i] : 0;
        long long x = c;  // inclusive warp scan
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const long long y = __shfl_up_sync(FULL, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) wsum[w] = x;
        __syncthreads();
        if (w == 0) {
            long long v = wsum[lane];
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const long long y = __shfl_up_sync(FULL, v, o);
                if (lane >= o) v += y;
            }
            wsum[lane] = v;  // inclusive over warps
        }
        __syncthreads();
        const long long before = (w > 0 ? wsum[w - 1] : 0) + x - c;
        if (i < nb) tro[b0 + i] = base + before;
        base += wsum[31];
        __syncthreads();
    }
    if (t == 0) tro[K] = base;
}
// One warp per book: its logged rows (24 B each, contiguous) to row tro[b] of `dst`
// (8-byte words, coalesced; `dst` may be mapped pinned host memory).
__global__ void lob_pack_trades(const int32_t *trades, const int32_t *ntrades, const long long *tro, int b0, int nb,
                                int Tcap, int2 *dst) {
    const long long gw = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (gw >= nb) return;
    const int b = b0 + (int)gw;
    const int n = ntrades[b] * 3;  // int2 words
    const int2 *src = reinterpret_cast<const int2 *>(trades + (size_t)b * Tcap * 6);
    int2 *d = dst + tro[b] * 3;
    for (int i = lane; i < n; i += 32) d[i] = src[i];
}

// per-book FNV-1a-64 over the exported state (include/lob.h lob_digest): one thread per book
__device__ __forceinline__ unsigned long long fnv1a_word(unsigned long long h, uint32_t w) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        h ^= (w >> (8 * k)) & 0xffu;
        h *= 0x100000001b3ULL;
    }
    return h;
}

__global__ void lob_digest_kernel(const int32_t *book, const int32_t *trades, const int32_t *ntrades,
                                  const long long *stats, unsigned long long *out, int K, int N, int NP, int Tcap) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= K) return;
    unsigned long long h = 0xcbf29ce484222325ULL;
    const int32_t *bk = book + (size_t)b * 2 * NF * NP;
    for (int s = 0; s < 2; ++s)
        for (int i = 0; i < N; ++i) {
            const int32_t *src = bk + s * NF * NP + i;
            const bool occ = src[F_Q * NP] > 0;
#pragma unroll
            for (int f = 0; f < NF; ++f) h = fnv1a_word(h, occ ? (uint32_t)src[f * NP] : 0xffffffffu);
        }
    const int nt = ntrades[b];
    const int32_t *tr = trades + (size_t)b * Tcap * 6;
    for (int r = 0; r < Tcap; ++r)
#pragma unroll
        for (int f = 0; f < 6; ++f) h = fnv1a_word(h, r < nt ? (uint32_t)tr[r * 6 + f] : 0xffffffffu);
    h = fnv1a_word(h, (uint32_t)nt);
    for (int c = 0; c < NST; ++c) {
        const unsigned long long v = (unsigned long long)stats[(size_t)b * NST + c];
        h = fnv1a_word(fnv1a_word(h, (uint32_t)v), (uint32_t)(v >> 32));
    }
    out[b] = h;
}

// current L2 of every book from the stored state: one group per book (G = 1)
template <int KPL, int W>
__global__ void __launch_bounds__(32 * W) lob_export_l2(const int32_t *book, int32_t *out, int K, int N, int L) {
    using BK = RegBook<KPL, W>;
    extern __shared__ __align__(128) unsigned char dyn[];
    const int b = blockIdx.x;
    if (b >= K) return;
    Params p{};
    p.N = N;
    Engine<BK> e(p);
    e.tid = threadIdx.x; e.xph = 0;
    e.bk.tid = threadIdx.x;
    e.bk.cold = smem_u32(dyn);
    e.sc = smem_u32(dyn + 2 * BK::NP * 16);
    e.scp = dyn + 2 * BK::NP * 16;
    e.bk.load(book + (size_t)b * 2 * NF * BK::NP);
    e.init_rows();
    e.l2_write(out + (size_t)b * L * 4, L);
}
template <int KPL, int W>
constexpr int export_l2_smem_bytes() { return 2 * KPL * 32 * W * 16 + scratch_bytes<W>(); }

}  // namespace lobk
