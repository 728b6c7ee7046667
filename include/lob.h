/*
 * include/lob.h -- C ABI of the B200 batched limit-order-book engine.
 *
 * The engine runs the data-parallel hot path of JAX-LOB (arXiv 2308.13289,
 * PAPER.md Section 4): K independent books, each two fixed-capacity unsorted
 * order arrays, step through message streams; every message is an add, a
 * cancel/delete or a match with trade logging; an L2 snapshot is taken after
 * every step.  Citations "P:Lnnn" are lines of PAPER.md; "Gnn" are the
 * readings listed in DESIGN.md (ambiguity ledger).
 *
 * Conventions (all entry points):
 *  - Memory: every device buffer is allocated by the CALLER (e.g. torch CUDA
 *    tensors) and passed as a raw pointer; the library never allocates or
 *    frees device memory.  The state buffer (lob_state_bytes) must outlive the
 *    context and be 256-byte aligned.
 *  - Streams: every call enqueues asynchronously on the given cudaStream_t
 *    (pass torch's current stream; NULL = legacy default stream); nothing
 *    synchronises implicitly except lob_process_messages_host, which does not
 *    synchronise either (the caller waits on the stream).
 *  - Errors: return codes report caller mistakes only (bad dimensions, NULL
 *    required pointer, wrong device, size overflow, unsupported capacity) and
 *    CUDA launch failures (LOB_ECUDA, detail in lob_last_error()).
 *    Data-dependent conditions are never errors: they are per-book counters
 *    (add overflow, trade-log overflow, unknown cancel, malformed message).
 *  - Threads: a context is used by one host thread at a time; one context per
 *    device and process.  Calls on one context must be stream-ordered (one
 *    stream, or streams joined by events): they share the state buffer and
 *    the step kernel's two scheduler words, which every launch leaves zeroed.
 *    Independent contexts (separate state buffers) may run concurrently.
 *  - Layouts: all records are int32 in the paper's field order; counters int64.
 */
#ifndef LOB_H
#define LOB_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LOB_MSG_FIELDS 8    /* Eq.6  m = [T, S, Q, P, OID, TID, Ts, Tns] */
#define LOB_ORDER_FIELDS 6  /* Eq.2  o = [P, Q, OID, TID, Ts, Tns] */
#define LOB_TRADE_FIELDS 6  /* Eq.3  t = [P, Q, OID_aggr, OID_stand, Ts, Tns] P:L187 */
#define LOB_L2_FIELDS 4     /* [ask_p, ask_q, bid_p, bid_q] per level (G23)           */
#define LOB_MAX_CAPACITY 2048
#define LOB_MAX_L2_LEVELS 32

enum { LOB_LIMIT = 1, LOB_CANCEL = 2, LOB_DELETE = 3, LOB_MARKET = 4 };
enum { LOB_BID = 1, LOB_ASK = -1 };
enum { LOB_OK = 0, LOB_EINVAL = -1, LOB_ECUDA = -2, LOB_ENOMEM = -3, LOB_EUNSUPPORTED = -4 };

/* per-book counters, cumulative since lob_init */
enum {
    LOB_ST_MSGS = 0,             /* every message, including padding (T=0) and malformed   */
    LOB_ST_BAD,                  /* malformed: T not in 1..4, S not +-1, limit P<=0,
                                    cancel/delete Q<=0 (G22)                                */
    LOB_ST_TRADES,               /* fills executed (logged or not)                          */
    LOB_ST_TRADES_DROPPED,       /* fills whose record did not fit the trade log (G8)       */
    LOB_ST_TRADED_QTY,           /* sum of fill quantities                                  */
    LOB_ST_CANCELLED_QTY,        /* sum of min(Q_cancel, Q_resting) (G14)                   */
    LOB_ST_UNKNOWN_CANCELS,      /* cancels/deletes that found no order (G15)               */
    LOB_ST_ADD_OVERFLOW,         /* limit remainders dropped because the side was full (G6) */
    LOB_ST_OVERFLOW_QTY,         /* their quantity                                          */
    LOB_ST_MARKET_DISCARDED_QTY, /* unmatched market quantity, disregarded         */
    LOB_NSTATS
};

typedef struct {
    int32_t n_books;    /* K >= 0: independent books                          */
    int32_t capacity;   /* N in 1..LOB_MAX_CAPACITY: orders per side (Eq.1)    */
    int32_t trades_cap; /* rows of the trade log per book per call (Eq.4, G7), >= 0    */
    int32_t l2_levels;  /* L in 1..LOB_MAX_L2_LEVELS: levels per L2 snapshot (G23)     */
    int32_t device;     /* CUDA device ordinal the state lives on (must be current)    */
} lob_config;

typedef struct lob_ctx lob_ctx; /* opaque host-side handle: dims, pointers, launch config */

/* Bytes of device state for `cfg` (books in an internal padded SoA layout, the
 * trade logs, trade counts and counters).  0 if cfg is invalid. */
size_t lob_state_bytes(const lob_config *cfg);

/* Create a host handle over caller-allocated device state (no GPU work).
 * Returns LOB_EINVAL for a bad config / NULL / misaligned state,
 * LOB_EUNSUPPORTED for capacity > LOB_MAX_CAPACITY, LOB_ECUDA if the device
 * cannot be queried. */
int lob_create(lob_ctx **out, const lob_config *cfg, void *d_state);
/* Test hooks, read from the environment by lob_create (results never change, only
 * the launch shape): LOB_FORCE_WIDE=1 launches the many-wave build of the step
 * kernel for every 4-row batch; LOB_GRID_CAP=n caps the persistent grid at n CTAs,
 * so small batches run through the dynamic book scheduler; LOB_SPLIT_BPS=n and
 * LOB_SPLIT_MIN_MSGS=m move the bounds of the side-split build (one warp per book
 * side, capacity <= 512, lob_process_messages only; default: at most 8 books per SM
 * with at least 4096 messages per book -- the latency-bound RL shape; n = 0: never). */
void lob_destroy(lob_ctx *ctx); /* frees the host handle only */

/* a0: book init.  Both sides and the trade log become -1
 * (P:L168), counters zero.  If d_init_l2 is non-NULL it is a
 * [K][init_levels][4] int32 Level-2 snapshot [ask_p, ask_q, bid_p, bid_q] per
 * level: one synthetic order per populated level (P>0 and Q>0, G24),
 * OIDs -9000, -9001, ... over asks best->worst then bids, TID -9000, time
 * (init_ts, init_tns).  init_levels must be <= capacity. */
int lob_init(lob_ctx *ctx, const int32_t *d_init_l2, int32_t init_levels, int32_t init_ts,
             int32_t init_tns, void *cuda_stream);

/* a1..a11: process n_steps*msgs_per_step messages per book.
 *  d_msgs:   [K][n_steps*msgs_per_step][8] int32, Eq.6 order (G19); book k's
 *            stream is processed serially in order, books in parallel.
 *            Message rules: P:L287-292; T=0 is padding (G21).
 *  d_l2_out: NULL or [K][n_steps][L][4] int32, the L2 snapshot after the last
 *            message of every step (absent levels (-1, 0), G23).
 * The trade log is cleared at the start of the call (G9); counters accumulate.
 * n_steps*msgs_per_step == 0 is allowed (clears the trade log only). */
int lob_process_messages(lob_ctx *ctx, const int32_t *d_msgs, int32_t n_steps,
                         int32_t msgs_per_step, int32_t *d_l2_out, void *cuda_stream);

/* NEXT row N1: lob_process_messages plus the Level-1 trace --
 * after EVERY message, [best ask P, total Q at it, best bid P, total Q at it]
 * (the exec-env state of P:L435-441; absent side (-1, 0)) into d_l1_out, a
 * [K][n_steps*msgs_per_step][4] int32 buffer (required, 16-byte aligned).
 * Everything else is identical to lob_process_messages. */
int lob_process_messages_l1(lob_ctx *ctx, const int32_t *d_msgs, int32_t n_steps, int32_t msgs_per_step,
                            int32_t *d_l2_out, int32_t *d_l1_out, void *cuda_stream);

/* Same call with HOST buffers (the end-to-end path: every output of the method comes
 * back to the host).  Copies h_msgs (pinned host, [K][n_steps*msgs_per_step][8]) into
 * the caller's device buffer d_msgs_buf, processes it, and returns to the host:
 *  h_l2_out          NULL or [K][n_steps][L][4] int32 L2 snapshots (device staging in
 *                    d_l2_buf, same shape);
 *  h_stats_out       NULL or [K][LOB_NSTATS] int64 counters;
 *  h_trades_out      NULL or pinned (page-locked, mapped) host memory of capacity
 *                    K*trades_cap rows of [6] int32: the call's LOGGED trade rows
 *                    (Eq.3), book 0's first, then book 1's, ... packed
 *                    without gaps (book k's rows start at sum of counts[0..k-1]); rows
 *                    past the total are not written.  Written by a device kernel
 *                    straight into the host buffer, so only logged rows cross PCIe;
 *  h_trade_counts_out  [K] int32 logged rows per book (required with h_trades_out).
 * Books are processed in `chunks` slices so that copies overlap kernels.  All work is
 * enqueued on cuda_stream and two copy streams the context owns (created on first use,
 * joined back to cuda_stream by events), so the call may be captured into a CUDA graph
 * from cuda_stream.  The caller synchronises the stream before reading host outputs.
 * Errors: LOB_EINVAL for null required buffers, misaligned device buffers (16 B) or
 * trade output (8 B), or an h_trades_out that is not pinned mapped memory. */
int lob_process_messages_host(lob_ctx *ctx, const int32_t *h_msgs, int32_t n_steps,
                              int32_t msgs_per_step, int32_t *h_l2_out, int64_t *h_stats_out,
                              int32_t *h_trades_out, int32_t *h_trade_counts_out,
                              int32_t *d_msgs_buf, int32_t *d_l2_buf, int32_t chunks,
                              void *cuda_stream);

/* NEXT row N2: step reward epilogue over the trade log of the
 * last lob_process_messages call (= one env step when called once per step,
 * G9).  Per book k, over the logged trades i and the agent's trades j:
 *   P_VWAP = sum_i Q_i P_i / sum_i Q_i                         (eq:vwap)
 *   R      = sum_j Q_j (P_j - P_VWAP) + lambda sum_j Q_j (P_VWAP - P_init)
 *                                                             (eq:rewardfunc)
 *  d_agent_oids: [K][2] int32 inclusive OID range of the agent's orders; a trade is
 *                the agent's if its aggressor or standing OID lies in it (G29).
 *  d_p_init:     [K] f64 initial mid price of the episode.
 *  d_task_side:  [K] int32, -1 sell task (the paper's form), +1 buy task (R negated, G30).
 *  Outputs (each nullable): d_reward [K] f64, d_vwap [K] f64, d_agent_qty [K] int64
 *  (executed agent quantity).  A step without trades gives R = 0, P_VWAP = 0 (G31).
 *  Double precision; P_VWAP is exact up to one rounding, R agrees with the serial
 *  definition to 1e-12 of the magnitude of its terms. */
int lob_step_reward(lob_ctx *ctx, const int32_t *d_agent_oids, const double *d_p_init,
                    const int32_t *d_task_side, double lambda, double *d_reward, double *d_vwap,
                    int64_t *d_agent_qty, void *cuda_stream);

/* NEXT row N3: the execution-environment step on the device, one
 * env per book (Sec.5.1.3 and 5.2; readings E1-E8 in DESIGN.md). */
typedef struct {
    int32_t task_side;      /* -1 sell task, +1 buy task                               */
    int32_t task_size;      /* shares to execute (> 0)                                 */
    int32_t n_passive;      /* passive price = near touch -/+ n ticks      */
    int32_t tick;           /* price tick (> 0)                                        */
    int32_t episode_s;      /* episode length in seconds; forced market order
                               for the remaining task 60 s before the end      */
    int32_t agent_tid;      /* TID stamped on the agent's orders                        */
    int32_t agent_oid_base; /* the agent's OIDs are base, base+1, ... (G29); > 0       */
    int32_t reserved;
    double lambda;          /* drift weight of eq:rewardfunc               */
} lob_env_config;

/* Bytes of env state for n_envs envs (caller-allocated device memory, 16-byte aligned). */
size_t lob_env_state_bytes(int32_t n_envs);

/* After lob_init: start an episode in every book: P_init = (best ask + best bid)/2
 * of the current book, time = (init_ts, init_tns), executed = 0.
 * lob_env_reset and lob_env_step return LOB_EINVAL for an invalid cfg (task_side not
 * +-1, task_size/tick/episode_s <= 0, n_passive < 0, agent_oid_base <= 0). */
int lob_env_reset(lob_ctx *ctx, void *d_env, const lob_env_config *cfg, int32_t init_ts,
                  int32_t init_tns, void *cuda_stream);

/* One env step in every book, ONE kernel launch on cuda_stream (the agent's messages,
 * then the step's data, then reward / time / termination, fused per book):
 *  d_actions [K][4] f32: sizes at the far-touch, mid, near-touch and passive prices
 *  (P:L476-493), rounded half-even, negative/NaN -> 0, capped far-touch first by the
 *  remaining task; d_data [K][msgs_per_step][8]: the step's data messages (zero rows
 *  are padding, G21); d_work [K][8][8] int32 receives the agent's messages of the step
 *  (zero-padded; processed before the data); outputs (nullable):
 *  d_reward [K] f64 (eq:rewardfunc), d_done [K] int32, d_executed [K] int64, and the
 *  post-step L2 d_l2_out [K][1][L][4].  A finished env receives padding only (its
 *  counters still count 8 + msgs_per_step messages). */
int lob_env_step(lob_ctx *ctx, void *d_env, const lob_env_config *cfg, const float *d_actions,
                 const int32_t *d_data, int32_t msgs_per_step, int32_t *d_work, double *d_reward,
                 int32_t *d_done, int64_t *d_executed, int32_t *d_l2_out, void *cuda_stream);

/* NEXT row N3, residency ("a persistent kernel ... for K <~ 7k";
 * PAPER.md P:L414-423): a RESIDENT env session.  lob_session_begin launches ONE
 * persistent kernel (on a stream owned by the context, forked from cuda_stream) that
 * loads every book once and keeps it on chip for a whole episode; each
 * lob_session_step(ctx, s) then runs exactly what one lob_env_step call runs (agent
 * messages from d_actions, the step's data, the post-step L2, reward / done / executed)
 * without reloading or storing any book, and lob_session_end writes the books and
 * counters back.  Results are identical to calling lob_env_step once per step.
 *  d_data [K][n_steps][msgs_per_step][8]: the whole episode's data messages, read-only
 *    for the session's lifetime (streamed ahead of the steps);
 *  d_actions [K][4] f32: READ AT EACH STEP -- the caller writes step s's actions into it
 *    on cuda_stream before lob_session_step;
 *  d_work, d_reward, d_done, d_executed, d_l2_out ([K][L][4], nullable): the same
 *    outputs as lob_env_step, overwritten by every step, complete on cuda_stream after
 *    lob_session_step returns (stream order).
 * lob_session_step enqueues ONE 32-thread kernel on cuda_stream that releases the next
 * step (a release store to a device flag) and spins until every CTA of the session has
 * finished it; the host does not block, and the call can be captured into a CUDA graph
 * (with capture started on a side stream: see the synchronisation rule below).
 * Between begin and end the trade log and its count are per step (as after a
 * lob_env_step); the book (lob_get_book) and the counters are updated at end.
 * Requirements: one session per context; msgs_per_step >= 1; every book resident at
 * once (ceil(K / books per CTA) CTAs in one wave of the GPU, else LOB_EUNSUPPORTED);
 * at most n_steps steps (then LOB_EINVAL).  (Test hook LOB_SESSION_MEMOPS=1: release and
 * wait by the driver's stream memory operations instead; LOB_EUNSUPPORTED if absent.)
 * Rules while a session runs: calls on the context other than lob_session_* are
 * undefined; a DEVICE-wide synchronisation (cudaDeviceSynchronize, torch.cuda.graph's
 * entry) deadlocks -- it waits for the resident kernel, which waits for the next step --
 * so synchronise streams instead; under lazy module loading, launch every kernel the
 * step loop uses once before lob_session_begin (a first launch loads its module, and
 * the load waits for the device).  lob_destroy stops a running session. */
int lob_session_begin(lob_ctx *ctx, void *d_env, const lob_env_config *cfg, const float *d_actions,
                      const int32_t *d_data, int32_t n_steps, int32_t msgs_per_step, int32_t *d_work,
                      double *d_reward, int32_t *d_done, int64_t *d_executed, int32_t *d_l2_out,
                      void *cuda_stream);
int lob_session_step(lob_ctx *ctx, void *cuda_stream);
int lob_session_end(lob_ctx *ctx, void *cuda_stream);

/* Current L2 snapshot of every book: d_out [K][L][4] int32. */
int lob_get_l2(lob_ctx *ctx, int32_t *d_out, void *cuda_stream);

/* Trade log of the last call: d_out [K][trades_cap][6] int32 (rows >=
 * count are -1), d_counts [K] int32 (nullable). */
int lob_get_trades(lob_ctx *ctx, int32_t *d_out, int32_t *d_counts, void *cuda_stream);

/* Full book state for parity/checkpointing: d_out [K][2][N][6] int32,
 * side 0 = asks (A), side 1 = bids (B); empty slots all -1. */
int lob_get_book(lob_ctx *ctx, int32_t *d_out, void *cuda_stream);

/* Counters: d_out [K][LOB_NSTATS] int64. */
int lob_get_stats(lob_ctx *ctx, int64_t *d_out, void *cuda_stream);

/* Per-book state digest (the full-state fingerprint that lets ranks and
 * world sizes be compared without moving the state).  d_out [K] uint64: FNV-1a-64
 * (offset basis 0xcbf29ce484222325, prime 0x100000001b3) over the little-endian bytes of,
 * in order, the book as lob_get_book exports it ([2][N][6] int32, empty slots -1), the
 * trade log as lob_get_trades exports it ([trades_cap][6] int32, -1 tail), n_trades
 * (int32) and the counters ([LOB_NSTATS] int64).  Equal digests <=> (up to hash
 * collisions) identical observable state.  Off the hot path: one thread per book.
 * Errors: LOB_EINVAL for a null d_out with K > 0. */
int lob_digest(lob_ctx *ctx, uint64_t *d_out, void *cuda_stream);

/* Number of kernels this process has launched through the library (all contexts). */
int64_t lob_launch_count(void);

/* Build provenance: a hash of the sources and build flags the library was compiled
 * from (Makefile LOB_BUILD_ID), so measurements can be tied to the binary that made them. */
const char *lob_build_id(void);

const char *lob_strerror(int code);
const char *lob_last_error(void); /* thread-local detail for the last failure */

#ifdef __cplusplus
}
#endif
#endif /* LOB_H */
