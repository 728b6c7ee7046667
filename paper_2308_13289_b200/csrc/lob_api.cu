// lob_api.cu -- host shim of the C ABI declared in include/lob.h.
// Validation, state layout, launch configuration; all compute is in
// lob_kernels.cuh.  No CPU fallback: every entry point either launches the
// sm_100a kernels or returns an error.
#include <cuda.h>  // driver types for the stream memory operations (entry points via the runtime)
#include <cuda_runtime.h>

#include <atomic>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <new>

#include "../../include/lob.h"
#include "lob_kernels.cuh"
#include "lob_env.cuh"
#include "lob_session.cuh"
#include "lob_split.cuh"

using namespace lobk;

static_assert((int)NST == (int)LOB_NSTATS, "counter layout");
static_assert(F_P == 0 && F_TNS == 5, "field order");
static_assert(sizeof(lob_env_config) == sizeof(EnvCfg), "env config layout");

namespace {
thread_local char g_err[512] = "";
std::atomic<long long> g_launches{0};

int fail(int code, const char *fmt, const char *detail = "") {
    snprintf(g_err, sizeof(g_err), fmt, detail);
    return code;
}
int cuda_fail(cudaError_t e, const char *where) {
    snprintf(g_err, sizeof(g_err), "%s: %s", where, cudaGetErrorString(e));
    return LOB_ECUDA;
}

// Book geometry: KPL register rows per thread and side, W warps per book.
//   N <= 128:  KPL = ceil(N/32), W = 1 (4 books per CTA)
//   N <= 256:  KPL = 8,  W = 1 (4 books per CTA)
//   N <= 512:  KPL = 16, W = 1 (4 books per CTA; 3 CTAs/SM)
//   N <= 1024: KPL = 8,  W = 4 (one book per CTA)
//   N <= 2048: KPL = 16, W = 4 (one book per CTA)
// (measured per capacity band: the row high-water mark keeps most scans short, so
// fewer warps with more rows win wherever the registers allow -- N = 512 +38 %,
// N = 2048 +26 % over 8-row books of 2 / 8 warps; 16 rows x 2 warps lost at 1024)
struct Geo {
    int kpl, w;
};
Geo geo_of(int N) {
    if (N <= 128) return {(N + 31) / 32, 1};
    if (N <= 256) return {8, 1};
    if (N <= 512) return {16, 1};
    if (N <= 1024) return {8, 4};
    return {16, 4};
}

struct Layout {
    int NP;
    size_t off_book, off_trades, off_ntr, off_stats, off_sched, off_tro, off_sess, total;
};

bool layout_of(const lob_config *c, Layout *L) {
    if (!c || c->n_books < 0 || c->capacity < 1 || c->capacity > LOB_MAX_CAPACITY || c->trades_cap < 0 ||
        c->l2_levels < 1 || c->l2_levels > LOB_MAX_L2_LEVELS)
        return false;
    const size_t K = (size_t)c->n_books;
    const Geo g = geo_of(c->capacity);
    L->NP = 32 * g.kpl * g.w;
    auto al = [](size_t x) { return (x + 255) & ~(size_t)255; };
    L->off_book = 0;
    L->off_trades = al(L->off_book + K * 2 * NF * L->NP * sizeof(int32_t));
    L->off_ntr = al(L->off_trades + K * (size_t)c->trades_cap * 6 * sizeof(int32_t));
    L->off_stats = al(L->off_ntr + K * sizeof(int32_t));
    L->off_sched = al(L->off_stats + K * NST * sizeof(long long));
    // host path only: per-book row offsets of the packed trade copy + the running total
    L->off_tro = al(L->off_sched + 2 * sizeof(unsigned));
    // resident env session: the step flag and the finished book-step counter
    L->off_sess = al(L->off_tro + (K + 1) * sizeof(long long));
    L->total = al(L->off_sess + 256);  // go and done on separate 128-byte lines
    return true;
}
}  // namespace

struct lob_ctx {
    lob_config cfg;
    Layout lay;
    char *state;
    int sm_count;
    Geo geo;
    int grid_cap[4];  // persistent grid: resident CTAs of the step kernel, per MODE
    long long split_max;  // side-split build (lob_split.cuh) for launches of at most this many
                          // books (LOB_SPLIT_BPS books per SM; 0 = never) ...
    long long split_min_msgs;  // ... of at least this many messages per book (LOB_SPLIT_MIN_MSGS)
    bool force_wide;  // test hook (env LOB_FORCE_WIDE=1): MODE 3 for every 4-row batch
    int grid_limit;   // test hook (env LOB_GRID_CAP=n): at most n CTAs per step launch, so
                      // small batches exercise the dynamic book scheduler
    // lob_process_messages_host: copy streams and fork/join events, created on first use
    // and kept for the context's lifetime (none per call)
    cudaStream_t h2d = nullptr, d2h = nullptr;
    cudaEvent_t ev_start = nullptr, ev_h = nullptr, ev_k = nullptr;
    // resident env session (lob_session_*): its stream, the join event, the step count
    cudaStream_t sess = nullptr;
    cudaEvent_t ev_sess = nullptr;
    bool sess_active = false;
    int sess_step = 0, sess_nsteps = 0, sess_grid_cap = 0, sess_grid = 0;
    bool sess_memops = false;
    int32_t *book() const { return reinterpret_cast<int32_t *>(state + lay.off_book); }
    int32_t *trades() const { return reinterpret_cast<int32_t *>(state + lay.off_trades); }
    int32_t *ntr() const { return reinterpret_cast<int32_t *>(state + lay.off_ntr); }
    long long *stats() const { return reinterpret_cast<long long *>(state + lay.off_stats); }
    unsigned *sched() const { return reinterpret_cast<unsigned *>(state + lay.off_sched); }
    long long *tro() const { return reinterpret_cast<long long *>(state + lay.off_tro); }
    unsigned *sess_go() const { return reinterpret_cast<unsigned *>(state + lay.off_sess); }
    unsigned *sess_done() const { return sess_go() + 32; }
};

#ifndef G16
#define G16 4
#endif
// The side-split build (lob_split.cuh) for latency-bound launches: at most LOB_SPLIT_BPS
// books per SM and at least LOB_SPLIT_MIN_MSGS messages per book.  Measured on B200
// (profiles/r02_v32_split_sweep.txt): C2 (1,000 books x 10,000 messages) +5 %; C1 -6 %,
// C4 batches of 592 - 4,736 books (1,000 messages) -5 ... -38 %, so only long streams of
// few books take it.
#ifndef LOB_SPLIT_BPS
#define LOB_SPLIT_BPS 8
#endif
#ifndef LOB_SPLIT_MIN_MSGS
#define LOB_SPLIT_MIN_MSGS 4096
#endif
constexpr int GS = 2;  // books (warp pairs) per CTA of the side-split build
namespace {
// call f(IC<KPL>, IC<W>, IC<G>) for the compiled geometry (G = books per CTA)
template <class F>
void for_geo(Geo g, F &&f) {
    if (g.w == 1) {
        switch (g.kpl) {
            case 1: f(IC<1>(), IC<1>(), IC<4>()); break;
            case 2: f(IC<2>(), IC<1>(), IC<4>()); break;
            case 3: f(IC<3>(), IC<1>(), IC<4>()); break;
            case 4: f(IC<4>(), IC<1>(), IC<4>()); break;
            case 8: f(IC<8>(), IC<1>(), IC<4>()); break;
            default: f(IC<16>(), IC<1>(), IC<G16>()); break;
        }
    } else {
        if (g.kpl == 8) f(IC<8>(), IC<4>(), IC<1>());
        else f(IC<16>(), IC<4>(), IC<1>());
    }
}

int check_ctx(lob_ctx *ctx) {
    if (!ctx) return fail(LOB_EINVAL, "null context%s");
    int dev = -1;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
    if (dev != ctx->cfg.device) return fail(LOB_EINVAL, "context device is not the current device%s");
    return LOB_OK;
}

int after_launch(const char *what) {
    g_launches.fetch_add(1, std::memory_order_relaxed);
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? LOB_OK : cuda_fail(e, what);
}

unsigned blocks_for(long long threads, int bs) { return (unsigned)((threads + bs - 1) / bs); }

int launch_step(lob_ctx *ctx, const int32_t *d_msgs, int32_t n_steps, int32_t M, int32_t *d_l2, int book0, int nb,
                cudaStream_t st, int32_t *d_l1 = nullptr, const EnvParams *env = nullptr) {
    if (nb <= 0) return LOB_OK;
    Params p;
    const EnvParams ep = env ? *env : EnvParams{};
    p.book = ctx->book(); p.trades = ctx->trades(); p.ntrades = ctx->ntr(); p.stats = ctx->stats();
    p.msgs = d_msgs; p.l2out = d_l2; p.l1out = d_l1; p.sched = ctx->sched();
    p.N = ctx->cfg.capacity; p.NP = ctx->lay.NP; p.Tcap = ctx->cfg.trades_cap; p.L = ctx->cfg.l2_levels;
    p.n_steps = n_steps; p.M = M; p.book0 = book0; p.nb = nb;
    int rc = LOB_OK;
    for_geo(ctx->geo, [&](auto kc, auto wc, auto gc) {
        constexpr int KPL = decltype(kc)::value, W = decltype(wc)::value, G = decltype(gc)::value;
        const unsigned need = blocks_for(nb, G);
        constexpr bool kWide = KPL == 4 && W == 1;  // MODE 3 exists for 4-row warp books only
        // many waves of books: the 8-CTA/SM build (occupancy beats its extra spills)
        const bool wide = kWide && !env && !d_l1 && (ctx->force_wide || (long long)nb >= 8LL * ctx->grid_cap[0] * G);
        const unsigned cap = (unsigned)ctx->grid_cap[env ? 2 : (d_l1 ? 1 : (wide ? 3 : 0))];
        unsigned grid = need < cap ? need : cap;
        if (ctx->grid_limit > 0 && grid > (unsigned)ctx->grid_limit) grid = (unsigned)ctx->grid_limit;
        const int smem = step_smem_bytes<KPL, W, G>();
        if constexpr (W == 1) {
            if (!env && !d_l1 && nb <= ctx->split_max && (long long)n_steps * M >= ctx->split_min_msgs &&
                !ctx->force_wide && ctx->grid_limit == 0) {  // few books: one warp per side (lob_split.cuh)
                lob_step_split<KPL, GS><<<blocks_for(nb, GS), 64 * GS, GS * SplitLayout<KPL>::BYTES, st>>>(p);
                rc = after_launch("lob_step_split kernel");
                return;
            }
        }
        if (env) lob_step<KPL, W, G, 2><<<grid, 32 * W * G, smem, st>>>(p, ep);
        else if (d_l1) lob_step<KPL, W, G, 1><<<grid, 32 * W * G, smem, st>>>(p, ep);
        else if constexpr (kWide) {
            if (wide) lob_step<KPL, W, G, 3><<<grid, 32 * W * G, smem, st>>>(p, ep);
            else lob_step<KPL, W, G, 0><<<grid, 32 * W * G, smem, st>>>(p, ep);
        } else {
            lob_step<KPL, W, G, 0><<<grid, 32 * W * G, smem, st>>>(p, ep);
        }
        rc = after_launch("lob_step kernel");
    });
    return rc;
}
}  // namespace

extern "C" {

size_t lob_state_bytes(const lob_config *cfg) {
    Layout L;
    return layout_of(cfg, &L) ? L.total : 0;
}

int lob_create(lob_ctx **out, const lob_config *cfg, void *d_state) {
    if (!out) return fail(LOB_EINVAL, "out is null%s");
    *out = nullptr;
    if (cfg && cfg->capacity > LOB_MAX_CAPACITY) return fail(LOB_EUNSUPPORTED, "capacity > LOB_MAX_CAPACITY%s");
    Layout L;
    if (!layout_of(cfg, &L)) return fail(LOB_EINVAL, "invalid lob_config%s");
    if (!d_state && cfg->n_books > 0) return fail(LOB_EINVAL, "state is null%s");
    if (reinterpret_cast<uintptr_t>(d_state) % 256) return fail(LOB_EINVAL, "state must be 256-byte aligned%s");
    int dev = -1;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
    if (dev != cfg->device) return fail(LOB_EINVAL, "cfg.device is not the current device%s");
    int sms = 0;
    e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (e != cudaSuccess) return cuda_fail(e, "cudaDeviceGetAttribute");
    lob_ctx *c = new (std::nothrow) lob_ctx();
    if (!c) return fail(LOB_ENOMEM, "host allocation failed%s");
    c->cfg = *cfg;
    c->lay = L;
    c->state = static_cast<char *>(d_state);
    c->sm_count = sms;
    c->geo = geo_of(cfg->capacity);
    {
        const char *fw = getenv("LOB_FORCE_WIDE");
        c->force_wide = fw && fw[0] == '1';
        const char *gc = getenv("LOB_GRID_CAP");
        c->grid_limit = gc ? atoi(gc) : 0;
        const char *sb = getenv("LOB_SPLIT_BPS");
        c->split_max = (long long)sms * (sb ? atoi(sb) : LOB_SPLIT_BPS);
        const char *sm = getenv("LOB_SPLIT_MIN_MSGS");
        c->split_min_msgs = sm ? atoll(sm) : LOB_SPLIT_MIN_MSGS;
    }
    int per_sm[4] = {1, 1, 1, 1}, sess_per_sm = 0;
    int rc = LOB_OK;
    for_geo(c->geo, [&](auto kc, auto wc, auto gc) {
        constexpr int KPL = decltype(kc)::value, W = decltype(wc)::value, G = decltype(gc)::value;
        constexpr int smem = step_smem_bytes<KPL, W, G>();
        e = cudaFuncSetAttribute(lob_step<KPL, W, G, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(lob_step<KPL, W, G, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(lob_step<KPL, W, G, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e == cudaSuccess)
            e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm[0], lob_step<KPL, W, G, 0>, 32 * W * G, smem);
        if (e == cudaSuccess)
            e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm[1], lob_step<KPL, W, G, 1>, 32 * W * G, smem);
        if (e == cudaSuccess)
            e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm[2], lob_step<KPL, W, G, 2>, 32 * W * G, smem);
        if constexpr (KPL == 4 && W == 1) {
            if (e == cudaSuccess)
                e = cudaFuncSetAttribute(lob_step<KPL, W, G, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
            if (e == cudaSuccess)
                e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm[3], lob_step<KPL, W, G, 3>, 32 * W * G,
                                                                  smem);
        }
        if constexpr (W == 1) {
            if (e == cudaSuccess)
                e = cudaFuncSetAttribute(lob_step_split<KPL, GS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         GS * SplitLayout<KPL>::BYTES);
        }
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(lob_session<KPL, W, G>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e == cudaSuccess)
            e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&sess_per_sm, lob_session<KPL, W, G>, 32 * W * G, smem);
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(lob_export_l2<KPL, W>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     export_l2_smem_bytes<KPL, W>());
        if (e != cudaSuccess) rc = cuda_fail(e, "kernel attribute / occupancy query");
    });
    if (rc != LOB_OK) { delete c; return rc; }
    {
        // load the session's step kernel now: under lazy module loading (the CUDA 12
        // default) its first launch would otherwise load the module while a resident
        // session kernel spins, and the load waits for the device -- a deadlock
        cudaFuncAttributes fa;
        e = cudaFuncGetAttributes(&fa, lob_session_sync_kernel);
        if (e != cudaSuccess) { delete c; return cuda_fail(e, "lob_session_sync_kernel attributes"); }
    }
    for (int m = 0; m < 4; ++m) c->grid_cap[m] = sms * (per_sm[m] > 0 ? per_sm[m] : 1);
    c->sess_grid_cap = sms * sess_per_sm;
    *out = c;
    return LOB_OK;
}

void lob_destroy(lob_ctx *ctx) {
    if (!ctx) return;
    if (ctx->sess_active) {  // a session still running: stop it (synchronously) before the streams go
        const unsigned stop = SESSION_STOP | (unsigned)ctx->sess_step;
        cudaMemcpy(ctx->sess_go(), &stop, sizeof stop, cudaMemcpyHostToDevice);
        cudaStreamSynchronize(ctx->sess);
    }
    if (ctx->sess) cudaStreamDestroy(ctx->sess);
    if (ctx->ev_sess) cudaEventDestroy(ctx->ev_sess);
    if (ctx->h2d) cudaStreamDestroy(ctx->h2d);
    if (ctx->d2h) cudaStreamDestroy(ctx->d2h);
    for (cudaEvent_t e : {ctx->ev_start, ctx->ev_h, ctx->ev_k})
        if (e) cudaEventDestroy(e);
    delete ctx;
}

int lob_init(lob_ctx *ctx, const int32_t *d_init_l2, int32_t init_levels, int32_t init_ts, int32_t init_tns,
             void *stream) {
    int rc = check_ctx(ctx);
    if (rc) return rc;
    if (init_levels < 0 || init_levels > ctx->cfg.capacity) return fail(LOB_EINVAL, "init_levels must be in 0..capacity%s");
    if (d_init_l2 && init_levels == 0) d_init_l2 = nullptr;
    const int K = ctx->cfg.n_books;
    if (K == 0) return LOB_OK;
    const int wpb = 8;
    lob_init_kernel<<<blocks_for(K, wpb), wpb * 32, 0, (cudaStream_t)stream>>>(
        ctx->book(), ctx->trades(), ctx->ntr(), ctx->stats(), ctx->sched(), K, ctx->cfg.capacity, ctx->lay.NP,
        ctx->cfg.trades_cap,
        d_init_l2, init_levels, init_ts, init_tns);
    return after_launch("lob_init_kernel");
}

int lob_process_messages(lob_ctx *ctx, const int32_t *d_msgs, int32_t n_steps, int32_t msgs_per_step,
                         int32_t *d_l2_out, void *stream) {
    int rc = check_ctx(ctx);
    if (rc) return rc;
    if (n_steps < 0 || msgs_per_step < 0) return fail(LOB_EINVAL, "negative n_steps/msgs_per_step%s");
    const long long nmsg = (long long)n_steps * msgs_per_step;
    if (nmsg > (1ll << 30)) return fail(LOB_EINVAL, "n_steps*msgs_per_step overflows%s");
    if (nmsg > 0 && !d_msgs && ctx->cfg.n_books > 0) return fail(LOB_EINVAL, "d_msgs is null%s");
    if (reinterpret_cast<uintptr_t>(d_msgs) % 16) return fail(LOB_EINVAL, "d_msgs must be 16-byte aligned%s");
    if (reinterpret_cast<uintptr_t>(d_l2_out) % 16) return fail(LOB_EINVAL, "d_l2_out must be 16-byte aligned%s");
    if (msgs_per_step == 0) n_steps = 0;
    return launch_step(ctx, d_msgs, n_steps, msgs_per_step, n_steps > 0 ? d_l2_out : nullptr, 0, ctx->cfg.n_books,
                       (cudaStream_t)stream);
}

int lob_process_messages_l1(lob_ctx *ctx, const int32_t *d_msgs, int32_t n_steps, int32_t msgs_per_step,
                            int32_t *d_l2_out, int32_t *d_l1_out, void *stream) {
    int rc = check_ctx(ctx);
    if (rc) return rc;
    if (n_steps < 0 || msgs_per_step < 0) return fail(LOB_EINVAL, "negative n_steps/msgs_per_step%s");
    const long long nmsg = (long long)n_steps * msgs_per_step;
    if (nmsg > (1ll << 30)) return fail(LOB_EINVAL, "n_steps*msgs_per_step overflows%s");
    if (nmsg > 0 && ctx->cfg.n_books > 0 && (!d_msgs || !d_l1_out)) return fail(LOB_EINVAL, "d_msgs or d_l1_out is null%s");
    if (reinterpret_cast<uintptr_t>(d_msgs) % 16 || reinterpret_cast<uintptr_t>(d_l2_out) % 16 ||
        reinterpret_cast<uintptr_t>(d_l1_out) % 16)
        return fail(LOB_EINVAL, "buffers must be 16-byte aligned%s");
    if (msgs_per_step == 0) n_steps = 0;
    return launch_step(ctx, d_msgs, n_steps, msgs_per_step, n_steps > 0 ? d_l2_out : nullptr, 0, ctx->cfg.n_books,
                       (cudaStream_t)stream, n_steps > 0 ? d_l1_out : nullptr);
}

int lob_process_messages_host(lob_ctx *ctx, const int32_t *h_msgs, int32_t n_steps, int32_t msgs_per_step,
                              int32_t *h_l2_out, int64_t *h_stats_out, int32_t *h_trades_out,
                              int32_t *h_trade_counts_out, int32_t *d_msgs_buf, int32_t *d_l2_buf, int32_t chunks,
                              void *stream) {
    int rc = check_ctx(ctx);
    if (rc) return rc;
    if (n_steps < 0 || msgs_per_step < 0 || chunks < 1) return fail(LOB_EINVAL, "bad n_steps/msgs_per_step/chunks%s");
    const long long nmsg = (long long)n_steps * msgs_per_step;
    if (nmsg > (1ll << 30)) return fail(LOB_EINVAL, "n_steps*msgs_per_step overflows%s");
    const int K = ctx->cfg.n_books;
    if (K == 0) return LOB_OK;
    if ((nmsg > 0 && (!h_msgs || !d_msgs_buf)) || (h_l2_out && !d_l2_buf))
        return fail(LOB_EINVAL, "null buffer%s");
    if (h_trades_out && !h_trade_counts_out) return fail(LOB_EINVAL, "h_trades_out needs h_trade_counts_out%s");
    if (reinterpret_cast<uintptr_t>(d_msgs_buf) % 16 || reinterpret_cast<uintptr_t>(d_l2_buf) % 16 ||
        reinterpret_cast<uintptr_t>(h_trades_out) % 8)
        return fail(LOB_EINVAL, "misaligned buffer%s");
    // the packed trade rows are written by a kernel straight into the caller's pinned
    // host buffer (mapped through unified addressing): only logged rows cross PCIe
    int2 *trades_dst = nullptr;
    if (h_trades_out && ctx->cfg.trades_cap > 0) {
        void *dp = nullptr;
        if (cudaHostGetDevicePointer(&dp, h_trades_out, 0) != cudaSuccess) {
            cudaGetLastError();
            return fail(LOB_EINVAL, "h_trades_out must be pinned (page-locked, mapped) host memory%s");
        }
        trades_dst = static_cast<int2 *>(dp);
    }
    if (msgs_per_step == 0) n_steps = 0;
    cudaStream_t st = (cudaStream_t)stream;
    cudaError_t e = cudaSuccess;
    if (!ctx->h2d) {  // first use: the context's copy streams and events
        e = cudaStreamCreateWithFlags(&ctx->h2d, cudaStreamNonBlocking);
        if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&ctx->d2h, cudaStreamNonBlocking);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ctx->ev_start, cudaEventDisableTiming);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ctx->ev_h, cudaEventDisableTiming);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ctx->ev_k, cudaEventDisableTiming);
        if (e != cudaSuccess) return cuda_fail(e, "copy stream / event creation");
    }
    cudaStream_t h2d = ctx->h2d, d2h = ctx->d2h;
    const int L = ctx->cfg.l2_levels, Tcap = ctx->cfg.trades_cap;
    const size_t msg_bytes_pb = (size_t)nmsg * 8 * sizeof(int32_t);
    const size_t l2_bytes_pb = (size_t)n_steps * L * 4 * sizeof(int32_t);
    const int per = (K + chunks - 1) / chunks;
    // checked enqueue: the first failing CUDA call sets rc (later calls are skipped)
    auto ck = [&](cudaError_t r, const char *what) {
        if (rc == LOB_OK && r != cudaSuccess) rc = cuda_fail(r, what);
        return rc == LOB_OK;
    };
    // Three-stage pipeline over book chunks: H2D(i) on `h2d`, kernel(i) on the caller's
    // stream after H2D(i), then on `d2h` after kernel(i): the L2 copy and the trade
    // packing of chunk i.  Copies of neighbouring chunks overlap the kernels on the two
    // copy engines.  Fork/join through events only, so the whole call can be captured
    // into a CUDA graph from the caller's stream.
    ck(cudaEventRecord(ctx->ev_start, st), "event record");
    ck(cudaStreamWaitEvent(h2d, ctx->ev_start, 0), "stream wait");
    ck(cudaStreamWaitEvent(d2h, ctx->ev_start, 0), "stream wait");
    if (trades_dst) ck(cudaMemsetAsync(ctx->tro() + K, 0, sizeof(long long), d2h), "memset");
    for (int i = 0; i < chunks && rc == LOB_OK; ++i) {
        const int b0 = i * per, nb = (b0 + per <= K) ? per : K - b0;
        if (nb <= 0) break;
        if (msg_bytes_pb)
            ck(cudaMemcpyAsync((char *)d_msgs_buf + (size_t)b0 * msg_bytes_pb,
                               (const char *)h_msgs + (size_t)b0 * msg_bytes_pb, (size_t)nb * msg_bytes_pb,
                               cudaMemcpyHostToDevice, h2d), "H2D messages");
        ck(cudaEventRecord(ctx->ev_h, h2d), "event record");  // a wait captures the event's
        ck(cudaStreamWaitEvent(st, ctx->ev_h, 0), "stream wait");  // state at the wait call
        if (rc) break;
        rc = launch_step(ctx, d_msgs_buf + (size_t)b0 * nmsg * 8, n_steps, msgs_per_step,
                         (h_l2_out && n_steps) ? d_l2_buf + (size_t)b0 * n_steps * L * 4 : nullptr, b0, nb, st);
        if (rc) break;
        const bool l2c = h_l2_out && l2_bytes_pb;
        if (l2c || trades_dst) {
            ck(cudaEventRecord(ctx->ev_k, st), "event record");
            ck(cudaStreamWaitEvent(d2h, ctx->ev_k, 0), "stream wait");
        }
        if (l2c)
            ck(cudaMemcpyAsync((char *)h_l2_out + (size_t)b0 * l2_bytes_pb, (char *)d_l2_buf + (size_t)b0 * l2_bytes_pb,
                               (size_t)nb * l2_bytes_pb, cudaMemcpyDeviceToHost, d2h), "D2H L2");
        if (trades_dst && rc == LOB_OK) {
            // row offsets of this chunk's books after every earlier chunk's rows, then the
            // logged rows of each book to host row offs[b] (books in order: packed)
            lob_trade_offsets<<<1, 1024, 0, d2h>>>(ctx->ntr(), ctx->tro(), b0, nb, K);
            rc = after_launch("lob_trade_offsets");
            if (rc == LOB_OK) {
                lob_pack_trades<<<blocks_for((long long)nb * 32, 256), 256, 0, d2h>>>(ctx->trades(), ctx->ntr(),
                                                                                      ctx->tro(), b0, nb, Tcap,
                                                                                      trades_dst);
                rc = after_launch("lob_pack_trades");
            }
        }
    }
    // join: the caller's stream continues after every D2H (also on failure, so the
    // context's streams never run ahead of the caller's)
    cudaError_t j1 = cudaEventRecord(ctx->ev_h, d2h);
    cudaError_t j2 = j1 == cudaSuccess ? cudaStreamWaitEvent(st, ctx->ev_h, 0) : j1;
    ck(j2, "join");
    if (rc == LOB_OK && h_stats_out)
        ck(cudaMemcpyAsync(h_stats_out, ctx->stats(), (size_t)K * NST * sizeof(long long), cudaMemcpyDeviceToHost, st),
           "D2H stats");
    if (rc == LOB_OK && h_trade_counts_out)
        ck(cudaMemcpyAsync(h_trade_counts_out, ctx->ntr(), (size_t)K * sizeof(int32_t), cudaMemcpyDeviceToHost, st),
           "D2H trade counts");
    return rc;
}

int lob_step_reward(lob_ctx *ctx, const int32_t *d_agent_oids, const double *d_p_init, const int32_t *d_task_side,
                    double lambda, double *d_reward, double *d_vwap, int64_t *d_agent_qty, void *stream) {
    int rc = check_ctx(ctx);
    if (rc) return rc;
    const int K = ctx->cfg.n_books;
    if (K == 0) return LOB_OK;
    if (!d_agent_oids || !d_p_init || !d_task_side) return fail(LOB_EINVAL, "agent range, p_init and side are required%s");
    if (reinterpret_cast<uintptr_t>(d_p_init) % 8 || reinterpret_cast<uintptr_t>(d_reward) % 8 ||
        reinterpret_cast<uintptr_t>(d_vwap) % 8 || reinterpret_cast<uintptr_t>(d_agent_qty) % 8)
        return fail(LOB_EINVAL, "double / int64 buffers must be 8-byte aligned%s");
    const int wpb = 8;
    lob_reward_kernel<<<blocks_for(K, wpb), wpb * 32, 0, (cudaStream_t)stream>>>(
        ctx->trades(), ctx->ntr(), K, ctx->cfg.trades_cap, d_agent_oids, d_p_init, d_task_side, lambda, d_reward,
        d_vwap, reinterpret_cast<long long *>(d_agent_qty));
    return after_launch("lob_reward_kernel");
}

size_t lob_env_state_bytes(int32_t n_envs) { return n_envs < 0 ? 0 : (size_t)n_envs * sizeof(EnvState); }

// agent_oid_base > 0: a live agent order is remembered by its OID with 0 meaning "none"
// (EnvState::live), so the agent's OIDs base, base+1, ... must never include 0 (E4)
static int env_cfg_ok(const lob_env_config *c) {
    return c && (c->task_side == 1 || c->task_side == -1) && c->task_size > 0 && c->tick > 0 && c->n_passive >= 0 &&
           c->episode_s > 0 && c->agent_oid_base > 0;
}

int lob_env_reset(lob_ctx *ctx, void *d_env, const lob_env_config *cfg, int32_t init_ts, int32_t init_tns,
                  void *stream) {
    int rc = check_ctx(ctx);
    if (rc) return rc;
    if (!env_cfg_ok(cfg)) return fail(LOB_EINVAL, "invalid lob_env_config%s");
    const int K = ctx->cfg.n_books;
    if (K == 0) return LOB_OK;
    if (!d_env || reinterpret_cast<uintptr_t>(d_env) % 16) return fail(LOB_EINVAL, "d_env null or misaligned%s");
    EnvCfg c;
    memcpy(&c, cfg, sizeof c);
    lob_env_reset_kernel<<<blocks_for(K, 8), 256, 0, (cudaStream_t)stream>>>(
        ctx->book(), ctx->cfg.capacity, ctx->lay.NP, K, static_cast<EnvState *>(d_env), c, init_ts, init_tns);
    return after_launch("lob_env_reset_kernel");
}

int lob_env_step(lob_ctx *ctx, void *d_env, const lob_env_config *cfg, const float *d_actions,
                 const int32_t *d_data, int32_t msgs_per_step, int32_t *d_work, double *d_reward, int32_t *d_done,
                 int64_t *d_executed, int32_t *d_l2_out, void *stream) {
    int rc = check_ctx(ctx);
    if (rc) return rc;
    if (!env_cfg_ok(cfg)) return fail(LOB_EINVAL, "invalid lob_env_config%s");
    if (msgs_per_step < 0 || msgs_per_step > (1 << 24)) return fail(LOB_EINVAL, "bad msgs_per_step%s");
    const int K = ctx->cfg.n_books;
    if (K == 0) return LOB_OK;
    if (!d_env || !d_actions || !d_work || (msgs_per_step > 0 && !d_data))
        return fail(LOB_EINVAL, "env, actions, work and data buffers are required%s");
    if (reinterpret_cast<uintptr_t>(d_env) % 16 || reinterpret_cast<uintptr_t>(d_work) % 16 ||
        reinterpret_cast<uintptr_t>(d_data) % 16 || reinterpret_cast<uintptr_t>(d_l2_out) % 16 ||
        reinterpret_cast<uintptr_t>(d_reward) % 8 || reinterpret_cast<uintptr_t>(d_executed) % 8)
        return fail(LOB_EINVAL, "misaligned buffer%s");
    EnvParams ep{};
    memcpy(&ep.ec, cfg, sizeof ep.ec);
    ep.env = static_cast<EnvState *>(d_env);
    ep.actions = d_actions;
    ep.agent_out = d_work;
    ep.reward = d_reward;
    ep.done = d_done;
    ep.executed = reinterpret_cast<long long *>(d_executed);
    // one fused launch: agent messages, the step's data, reward / time / termination
    return launch_step(ctx, d_data, 1, msgs_per_step, d_l2_out, 0, K, (cudaStream_t)stream, nullptr, &ep);
}

// ---------------------------------------------------------------- resident env session
namespace {
typedef CUresult (*PFN_write32)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
typedef CUresult (*PFN_wait32)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
PFN_write32 g_write32 = nullptr;
PFN_wait32 g_wait32 = nullptr;

// the driver's stream memory operations, through the runtime's entry-point query (no
// link-time dependency on libcuda)
int stream_memops() {
    if (g_write32 && g_wait32) return LOB_OK;
    void *w = nullptr, *t = nullptr;
    cudaDriverEntryPointQueryResult q1 = cudaDriverEntryPointSymbolNotFound, q2 = q1;
    cudaError_t e = cudaGetDriverEntryPoint("cuStreamWriteValue32", &w, cudaEnableDefault, &q1);
    if (e == cudaSuccess) e = cudaGetDriverEntryPoint("cuStreamWaitValue32", &t, cudaEnableDefault, &q2);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGetDriverEntryPoint");
    if (q1 != cudaDriverEntryPointSuccess || q2 != cudaDriverEntryPointSuccess || !w || !t)
        return fail(LOB_EUNSUPPORTED, "stream memory operations (cuStreamWriteValue32/cuStreamWaitValue32) unavailable%s");
    g_write32 = reinterpret_cast<PFN_write32>(w);
    g_wait32 = reinterpret_cast<PFN_wait32>(t);
    return LOB_OK;
}
int cu_fail(CUresult r, const char *where) {
    snprintf(g_err, sizeof(g_err), "%s: CUresult %d", where, (int)r);
    return LOB_ECUDA;
}
}  // namespace

int lob_session_begin(lob_ctx *ctx, void *d_env, const lob_env_config *cfg, const float *d_actions,
                      const int32_t *d_data, int32_t n_steps, int32_t msgs_per_step, int32_t *d_work,
                      double *d_reward, int32_t *d_done, int64_t *d_executed, int32_t *d_l2_out, void *stream) {
    int rc = check_ctx(ctx);
    if (rc) return rc;
    if (ctx->sess_active) return fail(LOB_EINVAL, "a session is already running on this context%s");
    if (!env_cfg_ok(cfg)) return fail(LOB_EINVAL, "invalid lob_env_config%s");
    const int K = ctx->cfg.n_books;
    if (K == 0) return fail(LOB_EINVAL, "a session needs at least one book%s");
    if (n_steps < 1 || msgs_per_step < 1 || (long long)n_steps * msgs_per_step > (1ll << 30))
        return fail(LOB_EINVAL, "bad n_steps/msgs_per_step%s");
    if (!d_env || !d_actions || !d_data || !d_work)
        return fail(LOB_EINVAL, "env, actions, data and work buffers are required%s");
    if (reinterpret_cast<uintptr_t>(d_env) % 16 || reinterpret_cast<uintptr_t>(d_work) % 16 ||
        reinterpret_cast<uintptr_t>(d_data) % 16 || reinterpret_cast<uintptr_t>(d_l2_out) % 16 ||
        reinterpret_cast<uintptr_t>(d_reward) % 8 || reinterpret_cast<uintptr_t>(d_executed) % 8)
        return fail(LOB_EINVAL, "misaligned buffer%s");
    {
        const char *mo = getenv("LOB_SESSION_MEMOPS");  // A/B hook: stream memory operations
        ctx->sess_memops = mo && mo[0] == '1';
    }
    if (ctx->sess_memops) {
        rc = stream_memops();
        if (rc) return rc;
    }
    int G = 1;
    for_geo(ctx->geo, [&](auto, auto, auto gc) { G = decltype(gc)::value; });
    const long long grid = (K + G - 1) / G;
    if (grid > ctx->sess_grid_cap)  // every book must stay resident: one wave only
        return fail(LOB_EUNSUPPORTED, "too many books for a resident session (one wave of the GPU)%s");
    cudaStream_t st = (cudaStream_t)stream;
    cudaError_t e = cudaSuccess;
    if (!ctx->sess) {
        e = cudaStreamCreateWithFlags(&ctx->sess, cudaStreamNonBlocking);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ctx->ev_sess, cudaEventDisableTiming);
        if (e != cudaSuccess) return cuda_fail(e, "session stream / event creation");
    }
    e = cudaMemsetAsync(ctx->sess_go(), 0, 256, st);
    if (e == cudaSuccess) e = cudaEventRecord(ctx->ev_sess, st);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(ctx->sess, ctx->ev_sess, 0);
    if (e != cudaSuccess) return cuda_fail(e, "session fork");
    Params p;
    p.book = ctx->book(); p.trades = ctx->trades(); p.ntrades = ctx->ntr(); p.stats = ctx->stats();
    p.msgs = d_data; p.l2out = d_l2_out; p.l1out = nullptr; p.sched = ctx->sched();
    p.N = ctx->cfg.capacity; p.NP = ctx->lay.NP; p.Tcap = ctx->cfg.trades_cap; p.L = ctx->cfg.l2_levels;
    p.n_steps = 1; p.M = msgs_per_step; p.book0 = 0; p.nb = K;
    EnvParams ep{};
    memcpy(&ep.ec, cfg, sizeof ep.ec);
    ep.env = static_cast<EnvState *>(d_env);
    ep.actions = d_actions;
    ep.agent_out = d_work;
    ep.reward = d_reward;
    ep.done = d_done;
    ep.executed = reinterpret_cast<long long *>(d_executed);
    SessionParams sp{ctx->sess_go(), ctx->sess_done(), n_steps};
    // An ordinary launch: the grid fits one wave (checked above), so every CTA becomes
    // resident as soon as the SMs it needs are free.  (A cooperative launch measured as a
    // device-exclusive kernel here: the caller's step launch queued behind it.)
    for_geo(ctx->geo, [&](auto kc, auto wc, auto gc) {
        constexpr int KPL = decltype(kc)::value, W = decltype(wc)::value, GG = decltype(gc)::value;
        lob_session<KPL, W, GG><<<(unsigned)grid, 32 * W * GG, step_smem_bytes<KPL, W, GG>(), ctx->sess>>>(p, ep, sp);
    });
    rc = after_launch("lob_session launch");
    if (rc) return rc;
    ctx->sess_active = true;
    ctx->sess_step = 0;
    ctx->sess_nsteps = n_steps;
    ctx->sess_grid = (int)grid;
    return LOB_OK;
}

int lob_session_step(lob_ctx *ctx, void *stream) {
    int rc = check_ctx(ctx);
    if (rc) return rc;
    if (!ctx->sess_active) return fail(LOB_EINVAL, "no session running%s");
    if (ctx->sess_step >= ctx->sess_nsteps) return fail(LOB_EINVAL, "the session's episode data are exhausted%s");
    const unsigned s = (unsigned)(ctx->sess_step + 1);
    // the step's outputs are complete when every CTA has finished it (one count per CTA)
    const unsigned target = s * (unsigned)ctx->sess_grid;
    if (ctx->sess_memops) {
        CUstream st = (CUstream)stream;
        CUresult r = g_write32(st, (CUdeviceptr)ctx->sess_go(), s, 0);  // release step s (fenced)
        if (r != CUDA_SUCCESS) return cu_fail(r, "cuStreamWriteValue32");
        r = g_wait32(st, (CUdeviceptr)ctx->sess_done(), target, CU_STREAM_WAIT_VALUE_GEQ);
        if (r != CUDA_SUCCESS) return cu_fail(r, "cuStreamWaitValue32");
    } else {
        lob_session_sync_kernel<<<1, 32, 0, (cudaStream_t)stream>>>(ctx->sess_go(), s, ctx->sess_done(), target);
        rc = after_launch("lob_session_sync_kernel");
        if (rc) return rc;
    }
    ctx->sess_step = (int)s;
    return LOB_OK;
}

int lob_session_end(lob_ctx *ctx, void *stream) {
    int rc = check_ctx(ctx);
    if (rc) return rc;
    if (!ctx->sess_active) return fail(LOB_EINVAL, "no session running%s");
    cudaStream_t st = (cudaStream_t)stream;
    if (ctx->sess_step < ctx->sess_nsteps) {  // the kernel is waiting for a step: stop it
        const unsigned stop = SESSION_STOP | (unsigned)ctx->sess_step;
        if (ctx->sess_memops) {
            CUresult r = g_write32((CUstream)st, (CUdeviceptr)ctx->sess_go(), stop, 0);
            if (r != CUDA_SUCCESS) return cu_fail(r, "cuStreamWriteValue32");
        } else {
            lob_session_sync_kernel<<<1, 32, 0, st>>>(ctx->sess_go(), stop, ctx->sess_done(), 0u);
            rc = after_launch("lob_session_sync_kernel");
            if (rc) return rc;
        }
    }
    // join: the caller's stream continues after the kernel has written the books back
    cudaError_t e = cudaEventRecord(ctx->ev_sess, ctx->sess);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(st, ctx->ev_sess, 0);
    ctx->sess_active = false;
    return e == cudaSuccess ? LOB_OK : cuda_fail(e, "session join");
}

int lob_get_l2(lob_ctx *ctx, int32_t *d_out, void *stream) {
    int rc = check_ctx(ctx);
    if (rc) return rc;
    const int K = ctx->cfg.n_books;
    if (K == 0) return LOB_OK;
    if (!d_out || reinterpret_cast<uintptr_t>(d_out) % 16) return fail(LOB_EINVAL, "d_out null or misaligned%s");
    for_geo(ctx->geo, [&](auto kc, auto wc, auto) {
        constexpr int KPL = decltype(kc)::value, W = decltype(wc)::value;
        lob_export_l2<KPL, W><<<K, 32 * W, export_l2_smem_bytes<KPL, W>(), (cudaStream_t)stream>>>(
            ctx->book(), d_out, K, ctx->cfg.capacity, ctx->cfg.l2_levels);
        rc = after_launch("lob_export_l2");
    });
    return rc;
}

int lob_get_trades(lob_ctx *ctx, int32_t *d_out, int32_t *d_counts, void *stream) {
    int rc = check_ctx(ctx);
    if (rc) return rc;
    const int K = ctx->cfg.n_books;
    if (K == 0) return LOB_OK;
    if (!d_out && ctx->cfg.trades_cap > 0) return fail(LOB_EINVAL, "d_out is null%s");
    const long long n = (long long)K * ctx->cfg.trades_cap * 6;
    const long long threads = n > K ? n : K;
    lob_export_trades<<<blocks_for(threads, 256), 256, 0, (cudaStream_t)stream>>>(ctx->trades(), ctx->ntr(), d_out,
                                                                                   d_counts, K, ctx->cfg.trades_cap);
    return after_launch("lob_export_trades");
}

int lob_get_book(lob_ctx *ctx, int32_t *d_out, void *stream) {
    int rc = check_ctx(ctx);
    if (rc) return rc;
    const int K = ctx->cfg.n_books;
    if (K == 0) return LOB_OK;
    if (!d_out) return fail(LOB_EINVAL, "d_out is null%s");
    lob_export_book<<<blocks_for((long long)K * 2 * ctx->cfg.capacity, 256), 256, 0, (cudaStream_t)stream>>>(
        ctx->book(), d_out, K, ctx->cfg.capacity, ctx->lay.NP);
    return after_launch("lob_export_book");
}

int lob_get_stats(lob_ctx *ctx, int64_t *d_out, void *stream) {
    int rc = check_ctx(ctx);
    if (rc) return rc;
    const int K = ctx->cfg.n_books;
    if (K == 0) return LOB_OK;
    if (!d_out) return fail(LOB_EINVAL, "d_out is null%s");
    cudaError_t e = cudaMemcpyAsync(d_out, ctx->stats(), (size_t)K * NST * sizeof(long long), cudaMemcpyDeviceToDevice,
                                    (cudaStream_t)stream);
    return e == cudaSuccess ? LOB_OK : cuda_fail(e, "lob_get_stats copy");
}

int lob_digest(lob_ctx *ctx, uint64_t *d_out, void *stream) {
    int rc = check_ctx(ctx);
    if (rc) return rc;
    const int K = ctx->cfg.n_books;
    if (K == 0) return LOB_OK;
    if (!d_out) return fail(LOB_EINVAL, "d_out is null%s");
    lob_digest_kernel<<<blocks_for(K, 128), 128, 0, (cudaStream_t)stream>>>(
        ctx->book(), ctx->trades(), ctx->ntr(), ctx->stats(), reinterpret_cast<unsigned long long *>(d_out), K,
        ctx->cfg.capacity, ctx->lay.NP, ctx->cfg.trades_cap);
    return after_launch("lob_digest_kernel");
}

int64_t lob_launch_count(void) { return g_launches.load(); }

#ifndef LOB_BUILD_ID
#define LOB_BUILD_ID "unknown"
#endif
const char *lob_build_id(void) { return LOB_BUILD_ID; }

#ifdef LOB_TRACE_CYCLES
// instrumented variant only (not in include/lob.h): copy the cycle trace of the last launch
int lob_trace_read(int64_t *h_msg, int64_t *h_l2) {
    cudaError_t e = cudaMemcpyFromSymbol(h_msg, g_trace_msg, sizeof(g_trace_msg));
    if (e == cudaSuccess) e = cudaMemcpyFromSymbol(h_l2, g_trace_l2, sizeof(g_trace_l2));
    return e == cudaSuccess ? LOB_OK : cuda_fail(e, "trace read");
}
#endif

#ifdef LOB_SPLIT_STATS
// instrumented variant only: the side-split build's wait counters, then reset
int lob_split_stats_read(uint64_t *h) {
    cudaError_t e = cudaMemcpyFromSymbol(h, g_split_stats, sizeof(g_split_stats));
    static const unsigned long long z[4][3] = {};
    if (e == cudaSuccess) e = cudaMemcpyToSymbol(g_split_stats, z, sizeof(z));
    return e == cudaSuccess ? LOB_OK : cuda_fail(e, "split stats read");
}
int lob_split_trace_read(int64_t *h) {
    cudaError_t e = cudaMemcpyFromSymbol(h, g_split_trace, sizeof(g_split_trace));
    return e == cudaSuccess ? LOB_OK : cuda_fail(e, "split trace read");
}
#endif

const char *lob_strerror(int code) {
    switch (code) {
        case LOB_OK: return "ok";
        case LOB_EINVAL: return "invalid argument";
        case LOB_ECUDA: return "CUDA error";
        case LOB_ENOMEM: return "out of memory";
        case LOB_EUNSUPPORTED: return "unsupported configuration";
        default: return "unknown error";
    }
}

const char *lob_last_error(void) { return g_err; }

}  // extern "C"
