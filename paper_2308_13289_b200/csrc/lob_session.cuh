// lob_session.cuh -- NEXT row N3, residency ("a persistent kernel for
// K <~ 7k"): a resident env session.  ONE persistent launch keeps
// every book (registers + shared-memory cold records) on chip for a whole episode;
// the caller's stream drives it step by step through two device words:
//   go    written by the caller's stream (cuStreamWriteValue32): step s (1-based) is
//         released when go >= s; bit 31 (SESSION_STOP) ends the session;
//   done  CTAs that have finished a step, cumulative: after step s every CTA has added
//         1 s times, so the caller's stream waits for done >= s*grid
//         (cuStreamWaitValue32, cyclic >=) before reading the step's outputs.
// Per step and book, in the order of a lob_env_step launch (lob_kernels.cuh MODE 2):
// the agent's messages from the actions (env_agent), the step's data
// messages (the episode's data are given up front: [K][n_steps][M][8], streamed by the
// same double-buffered bulk copies, so the next step's first chunks are already in
// shared memory when it is released), the post-step L2, then reward / executed / time
// / termination (env_post).  The trade log and its count are per step (G9); the book
// and the counters are written back when the session ends.
#pragma once
#include "lob_kernels.cuh"

namespace lobk {

constexpr unsigned SESSION_STOP = 0x80000000u;
#ifndef SESS_POLL_NS
#define SESS_POLL_NS 32  // back-off between polls of the step flag / the done counter
#endif

struct SessionParams {
    const unsigned *go;  // step flag (caller's stream)
    unsigned *done;      // CTAs that finished a step (cumulative; its own 128-byte line)
    int n_steps;         // steps of episode data
};

__device__ __forceinline__ unsigned ld_acquire_gpu(const unsigned *p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// a release reduction: the CTA's writes (ordered before it by the barrier) are visible
// to whoever acquires the counter -- no separate full fence
__device__ __forceinline__ void red_release_gpu_add(unsigned *p, unsigned v) {
    asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_release_gpu(unsigned *p, unsigned v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// The caller's side of a step, ONE tiny launch on the caller's stream: release step s
// (a release store: every earlier write of the stream, e.g. the actions, is visible to
// the session's acquire), then -- unless target is 0 -- spin until `done` reaches
// target (cyclic >=), so later work on the stream sees the step's outputs.  Measured
// against stream memory operations (cuStreamWriteValue32 + cuStreamWaitValue32, A/B hook
// LOB_SESSION_MEMOPS=1): 13.1 us of fixed time per step at 1,000 envs, this launch 11.7
// us from an eager host loop and 9.3 us inside a CUDA graph (scripts/session_overhead.py).
__global__ void lob_session_sync_kernel(unsigned *go, unsigned s, const unsigned *done, unsigned target) {
    if (threadIdx.x != 0) return;
    st_release_gpu(go, s);
    if (target == 0u) return;
    while ((int)(ld_acquire_gpu(done) - target) < 0) __nanosleep(SESS_POLL_NS);
}

// Step boundary of a whole CTA (every group, with or without a book, calls it):
//  1. a CTA barrier: every group has written the finished step's outputs;
//  2. (signal) thread 0 publishes them (fence, release) and adds 1 to `done` -- ONE
//     counter update per CTA, and the counter sits on its own 128-byte line, away from
//     `go`, so neither the updates nor the polls queue behind each other in L2;
//  3. warp 0 alone polls `go` until step s is released (or the session stopped) -- one
//     poller per CTA -- with a warp-uniform loop (every lane loads, a reduction decides;
//     a lane-0 spin loop cost ptxas its uniformity proof of the whole kernel).  Lanes
//     never disagree: the flag moves to s (release) or to STOP, never both while a step
//     is pending, since the caller's stream writes STOP only after its wait for the
//     previous step;
//  4. the flag goes to every group through a shared word behind a second CTA barrier
//     (a load from a uniform shared address is uniform).
__device__ __forceinline__ unsigned session_step_sync(const SessionParams &sp, unsigned s, bool signal,
                                                      unsigned *word) {
    __syncthreads();
    if (signal && threadIdx.x == 0) red_release_gpu_add(sp.done, 1u);
    const unsigned wid = __reduce_min_sync(FULL, threadIdx.x / 32u);  // uniform
    if (wid == 0u) {
        unsigned v = ld_acquire_gpu(sp.go);
        while (__reduce_min_sync(FULL, ((v & SESSION_STOP) != 0u || v >= s) ? 1u : 0u) == 0u) {
            __nanosleep(SESS_POLL_NS);
            v = ld_acquire_gpu(sp.go);
        }
        v = __reduce_max_sync(FULL, v);
        if (threadIdx.x == 0) *word = v;
    }
    __syncthreads();
    return *word;  // rewritten only after the next step's first barrier
}

// One wave only, so occupancy matters less than for lob_step: books of up to 128 orders
// get 96 registers (5 CTAs/SM: up to 2,960 resident books; no spills -- at 72 registers
// the per-step state spilled 40 bytes); larger books the lob_step budget.
template <int KPL, int W, int G>
__global__ void __launch_bounds__(32 * W * G, (KPL <= 4 ? 5 : (W == 1 ? 3 : (KPL > 8 ? 12 / W : 16 / W))))
    lob_session(const Params p, const EnvParams ep, const SessionParams sp) {
    using BK = RegBook<KPL, W>;
    extern __shared__ __align__(128) unsigned char dyn[];
    const int g = (int)__reduce_min_sync(FULL, threadIdx.x / (32 * W));  // uniform (see lob_step)
    const int tid = (int)opaque(threadIdx.x % (32 * W));
    unsigned char *base = dyn + g * (step_smem_bytes<KPL, W, G>() / G);
    const uint32_t stage = smem_u32(base);
    const uint32_t bars = smem_u32(base + 2 * CH * 32);
    const uint32_t cold = smem_u32(base + 2 * CH * 32 + 16);
    const uint32_t scratch = smem_u32(base + 2 * CH * 32 + 16 + 2 * BK::NP * 16);
    constexpr int word_off = 2 * CH * 32 + 16 + 2 * BK::NP * 16 + 8 * NST + 16 + (W == 1 ? 8 : 32 * W);
    unsigned *word = reinterpret_cast<unsigned *>(dyn + word_off);  // group 0's: one per CTA
    const int lb = blockIdx.x * G + g;  // one book per group for the whole session
    // a group without a book (the grid's last CTA) still joins every CTA barrier
    const bool has = lb < p.nb;         // uniform
    const int b = p.book0 + (has ? lb : 0);
    const int M = p.M;
    const int nmsg = sp.n_steps * M;
    const int nchunks = (nmsg + CH - 1) / CH;
    const int4 *src = reinterpret_cast<const int4 *>(p.msgs + (size_t)(has ? lb : 0) * nmsg * 8);
    Engine<BK, false, true, false, (W == 1 && KPL <= 8)> e(p);
    if (has) {
        if (tid == 0) {
            mbar_init(bars, 1);
            mbar_init(bars + 8, 1);
            fence_mbar_init();
        }
        group_sync<W>();
        if (tid == 0) {
#pragma unroll
            for (int c = 0; c < 2; ++c) {
                if (c < nchunks) {
                    const int cnt = min(CH, nmsg - c * CH);
                    mbar_arrive_expect_tx(bars + 8 * c, cnt * 32);
                    bulk_g2s(stage + c * CH * 32, src + (size_t)c * CH * 2, cnt * 32, bars + 8 * c);
                }
            }
        }
        if (tid < NST) sts64(scratch + 8u * tid, 0);
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
    }
    int steps_done = 0, last_ts = 0, last_tns = 0;
    bool have_last = false, idle = false;
    // one iteration per step: the CTA's step boundary (signal of the previous step, wait
    // for the release), the agent's messages, the step's M data messages (chunk refills
    // inline), L2 / reward.  The per-step work with lane-guarded stores stays outside the
    // message loop (inside it, such a branch costs ptxas its uniformity proof:
    // reconvergence barriers around every message).
    int c = -1, avail = 0;  // current chunk, its unprocessed messages
    uint32_t maddr = stage;
    for (; steps_done < sp.n_steps; ++steps_done) {
        if ((session_step_sync(sp, (unsigned)steps_done + 1u, steps_done > 0, word) & SESSION_STOP) != 0u) break;
        if (!has) continue;
        e.ntr = 0;  // a new step: a new trade log (G9)
        have_last = false;
        {
            EnvState es = ep.env[b];
            idle = es.done != 0;  // E8
            env_agent(e, es, p, ep, b, tid);
            if (tid == 0) ep.env[b] = es;
        }
        int left = M;
        while (left > 0) {
            if (avail == 0) {  // next chunk; the finished one's buffer takes chunk c + 2
                if (c >= 0) {
                    group_sync<W>();
                    if (tid == 0 && c + 2 < nchunks) {
                        const uint32_t sl = c & 1;
                        fence_proxy_async();
                        const int cn = min(CH, nmsg - (c + 2) * CH);
                        mbar_arrive_expect_tx(bars + 8 * sl, cn * 32);
                        bulk_g2s(stage + sl * CH * 32, src + (size_t)(c + 2) * CH * 2, cn * 32, bars + 8 * sl);
                    }
                }
                ++c;
                mbar_wait(bars + 8 * (c & 1), (c >> 1) & 1);
                maddr = stage + (c & 1) * CH * 32;
                avail = min(CH, nmsg - c * CH);
                if (tid < avail) {  // lane-parallel decode (lob_step)
                    const uint32_t m = maddr + 32u * (uint32_t)tid;
                    const int4 d = msg_decode(lds128(m));
                    sts32(m, d.x);
                    sts32(m + 12u, d.w);
                }
                group_sync<W>();
            }
            const int run = min(avail, left);
            const uint32_t mend = maddr + 32u * run;
            if (!idle) {
                do {
                    const int4 a = lds128(maddr), bb = lds128(maddr + 16);
                    e.message_coded(a, bb);
                    if (a.x != 0) { last_ts = bb.z; last_tns = bb.w; have_last = true; }
                    maddr += 32;
                } while (maddr != mend);
            } else {
                maddr = mend;
            }
            avail -= run;
            left -= run;
        }
        // end of the step: L2, reward / time / termination (published at the next boundary)
        if (p.l2out) e.l2_write(p.l2out + (size_t)lb * p.L * 4, p.L);
        const int logged = min(e.ntr, p.Tcap);
        if (tid == 0) {  // fills = logged + dropped (G8)
            p.ntrades[b] = logged;
            e.count(ST_TRADES, e.ntr);
            e.count(ST_DROPPED, e.ntr - logged);
        }
        env_post<W>(p, ep, b, tid, logged, have_last, last_ts, last_tns);
    }
    if (steps_done == sp.n_steps) {  // the last step's signal (the loop ended without a boundary)
        __syncthreads();
        if (threadIdx.x == 0) red_release_gpu_add(sp.done, 1u);
    }
    if (!has) return;
    // chunks still in flight land before the CTA exits (stopped sessions)
    // (chunks c + 1 and, before the first chunk, 1 were requested but not consumed)
    const int last = min(nchunks - 1, c < 0 ? 1 : c + 1);
    for (int k = c + 1; k <= last; ++k) mbar_wait(bars + 8 * (k & 1), (k >> 1) & 1);
    // writeback: book, counters (each finished step counts its 8 agent rows and M data
    // messages, as lob_env_step does)
    e.bk.store(p.book + (size_t)b * 2 * NF * BK::NP);
    long long cx = e.part_cxl, tq = e.part_trd;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        cx += __shfl_xor_sync(FULL, cx, o);
        tq += __shfl_xor_sync(FULL, tq, o);
    }
    group_sync<W>();
    if ((tid & 31) == 0) {
        unsigned long long *ctr = reinterpret_cast<unsigned long long *>(base + 2 * CH * 32 + 16 + 2 * BK::NP * 16);
        atomicAdd(ctr + ST_CANCELLED_QTY, (unsigned long long)cx);
        atomicAdd(ctr + ST_TRADED_QTY, (unsigned long long)tq);
    }
    group_sync<W>();
    if (tid < NST) {
        long long v = lds64(scratch + 8u * tid);
        if (tid == ST_MSGS) v += (long long)steps_done * (M + 8);
        p.stats[(size_t)b * NST + tid] += v;
    }
}

}  // namespace lobk
