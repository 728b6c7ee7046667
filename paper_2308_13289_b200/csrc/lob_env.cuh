// lob_env.cuh -- NEXT row N3: the execution-environment step on the device
// (Sec.5.1.3 and 5.2), one env per book.  A step is three launches on the
// caller's stream (graph-capturable):
//   lob_env_actions_kernel  the agent's action -> at most 8 messages (cancel the
//                           previous step's orders; the forced market order one
//                           minute before the end or one limit per
//                           positive size at far-touch / mid / near-touch /
//                           passive prices), followed by
//                           the step's data messages, into one
//                           stream per book;
//   lob_step                the engine over that stream (one call = one step, G9);
//   lob_env_post_kernel     reward (eq:rewardfunc, N2), executed quantity, time
//                           update, termination.
// Readings E1-E8: DESIGN.md.
#pragma once
#include "lob_kernels.cuh"

namespace lobk {

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

__device__ __forceinline__ long long env_elapsed_ns(const EnvState &e) {
    return ((long long)e.cur_ts - e.init_ts) * 1000000000LL + ((long long)e.cur_tns - e.init_tns);
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

// one warp per env: agent messages into work[k][0..8), data into work[k][8..8+M)
__global__ void lob_env_actions_kernel(const int32_t *book, int N, int NP, int K, EnvState *env, EnvCfg c,
                                       const float *actions, const int32_t *data, int M, int32_t *work) {
    const int lane = threadIdx.x & 31;
    const int k = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (k >= K) return;
    EnvState e = env[k];
    int ask, bid;
    book_best(book + (size_t)k * 2 * NF * NP, N, NP, lane, ask, bid);
    int4 *w = reinterpret_cast<int4 *>(work + (size_t)k * (8 + M) * 8);
    if (lane == 0) {
        int m[8][8];
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
            for (int f = 0; f < 8; ++f) m[i][f] = 0;
        int n = 0;
        const int S = c.task_side;
        if (!e.done) {
#pragma unroll
            for (int i = 0; i < 4; ++i)  // E1: cancel (delete) the previous step's orders
                if (e.live[i] != 0) {
                    m[n][0] = 3; m[n][1] = S; m[n][2] = INT_MAX; m[n][4] = e.live[i]; m[n][5] = c.agent_tid;
                    m[n][6] = e.cur_ts; m[n][7] = e.cur_tns;
                    ++n;
                    e.live[i] = 0;
                }
            long long remaining = (long long)c.task_size - e.executed;
            if (remaining > 0) {
                if (env_elapsed_ns(e) >= ((long long)c.episode_s - 60) * 1000000000LL) {
                    m[n][0] = 4; m[n][1] = S; m[n][2] = (int)(remaining > INT_MAX ? INT_MAX : remaining);
                    m[n][4] = e.next_oid++; m[n][5] = c.agent_tid; m[n][6] = e.cur_ts; m[n][7] = e.cur_tns;
                    ++n;
                } else {
                    if (ask > 0) e.last_ask = ask; else ask = e.last_ask;  // E6
                    if (bid > 0) e.last_bid = bid; else bid = e.last_bid;
                    const int far = (S == -1) ? bid : ask, near = (S == -1) ? ask : bid;
                    const int passive = near > 0 ? near - S * c.n_passive * c.tick : 0;
                    int mid = 0;  // E5: the tick at or beyond the mid, away from the spread
                    if (ask > 0 && bid > 0) {
                        const long long twice = (long long)ask + bid, t2 = 2LL * c.tick;
                        const long long q = twice / t2, rmd = twice % t2;
                        mid = (int)((S == -1 && rmd) ? (q + 1) * c.tick : q * c.tick);
                    }
                    const int price[4] = {far, mid, near, passive};
                    int li = 0;
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const float x = actions[4 * k + j];
                        long long q = 0;  // E2: round half-even, NaN / negative -> 0
                        if (x == x && x > 0.0f) q = (x >= 2147483647.0f) ? 2147483647LL : (long long)__float2int_rn(x);
                        if (q > remaining) q = remaining;  // E3
                        if (q <= 0 || price[j] <= 0) continue;
                        remaining -= q;
                        m[n][0] = 1; m[n][1] = S; m[n][2] = (int)q; m[n][3] = price[j]; m[n][4] = e.next_oid;
                        m[n][5] = c.agent_tid; m[n][6] = e.cur_ts; m[n][7] = e.cur_tns;
                        ++n;
                        e.live[li++] = e.next_oid++;
                    }
                }
            }
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            w[2 * i] = make_int4(m[i][0], m[i][1], m[i][2], m[i][3]);
            w[2 * i + 1] = make_int4(m[i][4], m[i][5], m[i][6], m[i][7]);
        }
        env[k] = e;
    }
    // the step's data messages; a finished env gets padding only (E8)
    const int4 *d = reinterpret_cast<const int4 *>(data + (size_t)k * M * 8);
    for (int i = lane; i < 2 * M; i += 32) w[16 + i] = e.done ? make_int4(0, 0, 0, 0) : d[i];
}

// one warp per env, after lob_step over the work stream
__global__ void lob_env_post_kernel(const int32_t *trades, const int32_t *ntrades, int Tcap, int K, EnvState *env,
                                    EnvCfg c, const int32_t *data, int M, double *reward, int32_t *done,
                                    long long *executed) {
    const int lane = threadIdx.x & 31;
    const int k = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (k >= K) return;
    EnvState e = env[k];
    if (e.done) {  // finished before this step (E8)
        if (lane == 0) {
            if (reward) reward[k] = 0.0;
            if (done) done[k] = 1;
            if (executed) executed[k] = e.executed;
        }
        return;
    }
    // reward over the step's trades, agent = OIDs [oid_base, next_oid) (G29): same sums as lob_reward_kernel
    const int n = ntrades[k];
    const int2 *t = reinterpret_cast<const int2 *>(trades + (size_t)k * Tcap * 6);
    double sqp = 0.0, sq = 0.0;
    for (int i = lane; i < n; i += 32) {
        const int2 pq = t[3 * i];
        sqp += (double)pq.y * (double)pq.x;
        sq += (double)pq.y;
    }
    sqp = warp_sum(sqp);
    sq = warp_sum(sq);
    const double v = sq > 0.0 ? sqp / sq : 0.0;
    const int lo = c.oid_base, hi = e.next_oid - 1;
    double adv = 0.0, drift = 0.0;
    long long qa = 0;
    for (int i = lane; i < n && sq > 0.0; i += 32) {
        const int2 pq = t[3 * i], oo = t[3 * i + 1];
        if ((oo.x >= lo && oo.x <= hi) || (oo.y >= lo && oo.y <= hi)) {
            adv += (double)pq.y * ((double)pq.x - v);
            drift += (double)pq.y * (v - e.p_init);
            qa += pq.y;
        }
    }
    adv = warp_sum(adv);
    drift = warp_sum(drift);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) qa += __shfl_xor_sync(FULL, qa, o);
    // the time of the last (non-padding) data message
    int last = -1;
    for (int base = ((M - 1) / 32) * 32; base >= 0 && last < 0; base -= 32) {
        const int i = base + lane;
        const bool nz = i < M && data[((size_t)k * M + i) * 8] != 0;
        const unsigned bl = __ballot_sync(FULL, nz);
        if (bl) last = base + 31 - __clz(bl);
    }
    if (lane == 0) {
        e.executed += qa;
        if (last >= 0) {
            e.cur_ts = data[((size_t)k * M + last) * 8 + 6];
            e.cur_tns = data[((size_t)k * M + last) * 8 + 7];
        }
        e.done = (e.executed >= c.task_size) || (env_elapsed_ns(e) > (long long)c.episode_s * 1000000000LL);
        const double r = adv + c.lam * drift;
        if (reward) reward[k] = c.task_side == 1 ? -r : r;
        if (done) done[k] = e.done;
        if (executed) executed[k] = e.executed;
        env[k] = e;
    }
}

}  // namespace lobk
