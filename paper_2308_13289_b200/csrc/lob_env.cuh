// lob_env.cuh -- NEXT row N3: the execution-environment step on the device
// (Sec.5.1.3 and 5.2), one env per book.  lob_env_reset_kernel sets up an
// episode; a step is ONE launch of lob_step<..., MODE = 2> (lob_kernels.cuh):
//   env_agent   the agent's action -> at most 8 messages, processed first
//               (P:L476-493);
//   the engine  over the step's data messages (one call = one step, G9);
//   env_post    reward (eq:rewardfunc, N2), executed quantity, time update
//               (P:L419), termination.
// Readings E1-E8: DESIGN.md.
#pragma once
#include "lob_kernels.cuh"

namespace lobk {

// best ask / bid price of book b from the stored SoA state (-1 if a side is empty)
__device__ __forceinline__ void book_best(const int32_t *bk, int N, int NP, int lane, int &ask, int &bid) {
    int r[2];
#pragma unroll
    for (int s = 0; s < 2; ++s) {
        int lk = INT_MAX;
        bool has = false;
        for (int i = lane; i < N; i += 32) {
            const int q = bk[(s * NF + F_Q) * NP + i], p = bk[(s * NF + F_P) * NP + i];
            if (q > 0) { lk = min(lk, s == ASK ? p : ~p); has = true; }
        }
        const bool any = __any_sync(FULL, has);
        const int m = __reduce_min_sync(FULL, has ? lk : INT_MAX);
        r[s] = any ? (s == ASK ? m : ~m) : -1;
    }
    ask = r[ASK];
    bid = r[BID];
}

// after lob_init: P_init = (P_ask + P_bid) / 2 of the initial book (E7)
__global__ void lob_env_reset_kernel(const int32_t *book, int N, int NP, int K, EnvState *env, EnvCfg c, int ts,
                                     int tns) {
    const int lane = threadIdx.x & 31;
    const int k = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (k >= K) return;
    int ask, bid;
    book_best(book + (size_t)k * 2 * NF * NP, N, NP, lane, ask, bid);
    if (lane == 0) {
        EnvState e;
        e.executed = 0;
        e.init_ts = e.cur_ts = ts;
        e.init_tns = e.cur_tns = tns;
        e.next_oid = c.oid_base;
        e.done = 0;
        e.last_ask = ask;
        e.last_bid = bid;
        e.live[0] = e.live[1] = e.live[2] = e.live[3] = 0;
        const int a = ask > 0 ? ask : bid, b = bid > 0 ? bid : ask;
        e.p_init = a > 0 ? ((double)a + (double)b) / 2.0 : 0.0;
        env[k] = e;
    }
}

}  // namespace lobk
