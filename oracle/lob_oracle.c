/*
 * oracle/lob_oracle.c -- CPU ORACLE. TEST INFRASTRUCTURE ONLY.
 *
 * This file is the plain, slow, single-threaded reference for the JAX-LOB
 * hot path (arXiv 2308.13289, "JAX-LOB", Section 4).  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
 * may load it.  It shares NO code, header or constant with the CUDA path in
 * paper_2308_13289_b200/csrc (field indices below are restated from the paper,
 * not included from include/lob.h).
 *
 * Citations: "P:Lnnn" = line of PAPER.md, "Gnn" = reading in DESIGN.md's
 * ambiguity ledger (taken from SURVEY.md section 8(c)).
 *
 * The algorithm is written in the paper's order and notation:
 *   book sides A (asks) and B (bids), arrays of N orders   Eq.1
 *   order o_i = [P, Q, OID, TID, Ts, Tns]                   Eq.2
 *   empty slot = all features -1
 *   add / cancel / match
 *   trade t_j = [P_j, Q_j, OID_a, OID_s, Ts_j, Tns_j]       Eq.3
 *   trades array T of fixed size                            Eq.4
 *   sweep Q <= 0 -> -1
 *   best standing order (price, then time)                  Eq.5
 *   matching while-loop condition
 *   message m = [T, S, Q, P, OID, TID, Ts, Tns]             Eq.6
 *   per-type processing rules
 *   synthetic initial book, OIDs from -9000 descending
 *
 * Parity pins: tests/test_oracle_*.py (golden hand traces in tests/golden/,
 * an independent sorted-map FIFO engine, exhaustive tiny-input brute force,
 * closed forms, inline invariants).  Every function below is pinned; none is
 * "parity unpinned".
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* Eq.2: order features */
#define O_P 0
#define O_Q 1
#define O_OID 2
#define O_TID 3
#define O_TS 4
#define O_TNS 5
#define O_NF 6
/* Eq.6: message fields, in Eq.6 order (G19) */
#define M_T 0
#define M_S 1
#define M_Q 2
#define M_P 3
#define M_OID 4
#define M_TID 5
#define M_TS 6
#define M_TNS 7
#define M_NF 8
/* Eq.3: trade fields */
#define T_NF 6
/* counters */
#define C_MSGS 0
#define C_BAD 1
#define C_TRADES 2
#define C_TRADES_DROPPED 3
#define C_TRADED_QTY 4
#define C_CANCELLED_QTY 5
#define C_UNKNOWN_CANCELS 6
#define C_ADD_OVERFLOW 7
#define C_OVERFLOW_QTY 8
#define C_MARKET_DISCARDED_QTY 9
#define C_N 10

#define INT32_MAX_ 2147483647  /* "max_int" for a market buy, G18 */

typedef struct {
    int32_t *A;        /* asks  [N][6] */
    int32_t *B;        /* bids  [N][6]  */
    int32_t *trades;   /* T     [T_cap][6] (Eq.4) */
    int32_t n_trades;
    int64_t c[C_N];
    /* bookkeeping used only by the invariant checker (check mode) */
    int64_t limit_in, limit_aggr_traded, limit_rested, market_in, market_aggr_traded;
    int64_t resting_init;
    int64_t call_trades0, call_dropped0;   /* counters at the start of the current call */
    int64_t violations;
} obook;

typedef struct {
    int32_t K, N, T_cap, L;
    int32_t check;
    obook *books;
} oracle_ctx;

/* ---------------------------------------------------------------- basics */

/* G5: a slot is occupied iff its quantity is positive. */
static int occupied(const int32_t *o) { return o[O_Q] > 0; }

/* empty positions have all features -1. */
static void set_empty(int32_t *o) {
    for (int f = 0; f < O_NF; f++) o[f] = -1;
}

/* Eq.5 + G1/G2/G4: is standing order x strictly better than y?
 * Asks: lower price first; bids: higher price first (Eq.5 prints min for both,
 * G1 reads max for bids).  Then earlier (Ts, Tns).  The caller scans
 * slots in increasing index and only replaces on strictly better, so equal
 * keys resolve to the lowest slot (G4). */
static int better(const int32_t *x, const int32_t *y, int is_ask) {
    if (x[O_P] != y[O_P]) return is_ask ? (x[O_P] < y[O_P]) : (x[O_P] > y[O_P]);
    if (x[O_TS] != y[O_TS]) return x[O_TS] < y[O_TS];
    return x[O_TNS] < y[O_TNS];
}

/* Best(o_s): index of the best occupied order on a side, or -1. */
static int best_standing(const int32_t *side, int N, int is_ask) {
    int best = -1;
    for (int i = 0; i < N; i++) {
        const int32_t *o = side + (size_t)i * O_NF;
        if (!occupied(o)) continue;
        if (best < 0 || better(o, side + (size_t)best * O_NF, is_ask)) best = i;
    }
    return best;
}

/* ------------------------------------------------------ invariant checks */

static int64_t side_resting(const int32_t *side, int N) {
    int64_t s = 0;
    for (int i = 0; i < N; i++)
        if (occupied(side + (size_t)i * O_NF)) s += side[(size_t)i * O_NF + O_Q];
    return s;
}

/* Sentinel discipline: every slot is either all -1 or occupied with a
 * positive price; never crossed: best ask > best bid. */
static void check_book(oracle_ctx *X, obook *b) {
    int N = X->N;
    for (int s = 0; s < 2; s++) {
        const int32_t *side = s ? b->B : b->A;
        for (int i = 0; i < N; i++) {
            const int32_t *o = side + (size_t)i * O_NF;
            if (occupied(o)) {
                if (o[O_P] < 1) b->violations++;
            } else {
                for (int f = 0; f < O_NF; f++)
                    if (o[f] != -1) { b->violations++; break; }
            }
        }
    }
    int ia = best_standing(b->A, N, 1), ib = best_standing(b->B, N, 0);
    if (ia >= 0 && ib >= 0 && !(b->A[(size_t)ia * O_NF + O_P] > b->B[(size_t)ib * O_NF + O_P]))
        b->violations++;
    /* quantity conservation per book:
     * resting = init + rested limit remainders - traded(standing) - cancelled */
    int64_t r = side_resting(b->A, N) + side_resting(b->B, N);
    int64_t expect = b->resting_init + b->limit_rested - b->c[C_TRADED_QTY] - b->c[C_CANCELLED_QTY];
    if (r != expect) b->violations++;
    /* limit qty in = traded as aggressor + rested + overflow */
    if (b->limit_in != b->limit_aggr_traded + b->limit_rested + b->c[C_OVERFLOW_QTY]) b->violations++;
    /* market qty in = traded as aggressor + discarded */
    if (b->market_in != b->market_aggr_traded + b->c[C_MARKET_DISCARDED_QTY]) b->violations++;
    /* every fill of this call is logged or counted as dropped (Eq.4, G8) */
    if (b->c[C_TRADES] - b->call_trades0 != b->n_trades + (b->c[C_TRADES_DROPPED] - b->call_dropped0))
        b->violations++;
    if (b->n_trades > X->T_cap) b->violations++;
}

/* Priority check: no occupied slot on the standing side has a strictly
 * better key than the one selected.  Written as a pairwise comparison over all
 * slots so that it does not reuse best_standing's scan. */
static void check_priority(oracle_ctx *X, obook *b, const int32_t *side, int j, int is_ask) {
    const int32_t *s = side + (size_t)j * O_NF;
    for (int i = 0; i < X->N; i++) {
        const int32_t *o = side + (size_t)i * O_NF;
        if (!occupied(o) || i == j) continue;
        int64_t po = is_ask ? o[O_P] : -(int64_t)o[O_P];
        int64_t ps = is_ask ? s[O_P] : -(int64_t)s[O_P];
        if (po < ps) { b->violations++; continue; }
        if (po > ps) continue;
        if (o[O_TS] < s[O_TS] || (o[O_TS] == s[O_TS] && o[O_TNS] < s[O_TNS]) ||
            (o[O_TS] == s[O_TS] && o[O_TNS] == s[O_TNS] && i < j))
            b->violations++;
    }
}

/* -------------------------------------------------------- the operations */

/* Cancellation: locate the order by OID on the message's side (G16)
 * and remove the quantity; delete is identical (G13).  Synthetic
 * initial orders are also matched by price, read as OID <= -9000
 * (G12); an exact OID match wins (G12).  Lowest slot on ties. */
static void cancel(oracle_ctx *X, obook *b, int32_t *side, int32_t P, int32_t OID, int32_t Q) {
    int N = X->N;
    if (Q <= 0) { b->c[C_BAD]++; return; }                       /* G22 */
    int i = -1;
    for (int k = 0; k < N; k++) {
        const int32_t *o = side + (size_t)k * O_NF;
        if (occupied(o) && o[O_OID] == OID) { i = k; break; }
    }
    if (i < 0) {
        for (int k = 0; k < N; k++) {
            const int32_t *o = side + (size_t)k * O_NF;
            if (occupied(o) && o[O_OID] <= -9000 && o[O_P] == P) { i = k; break; }
        }
    }
    if (i < 0) { b->c[C_UNKNOWN_CANCELS]++; return; }            /* G15 */
    int32_t *o = side + (size_t)i * O_NF;
    b->c[C_CANCELLED_QTY] += (Q < o[O_Q]) ? Q : o[O_Q];           /* G14 */
    o[O_Q] -= Q;
    if (o[O_Q] <= 0) set_empty(o);
}

/* One message, dispatched on (T, S). */
static void process(oracle_ctx *X, obook *b, const int32_t *m) {
    int N = X->N;
    b->c[C_MSGS]++;
    int32_t T = m[M_T], S = m[M_S];
    if (T == 0) return;                                           /* zero padding, G21 */
    if (T < 1 || T > 4 || (S != 1 && S != -1)) { b->c[C_BAD]++; return; }   /* G22 */
    int32_t *own = (S == 1) ? b->B : b->A;                        /* S=1 bid, S=-1 ask */
    int32_t *opp = (S == 1) ? b->A : b->B;
    int opp_is_ask = (S == 1);
    if (T == 2 || T == 3) {                                       /* cancel == delete */
        int32_t *snap = NULL;
        int64_t unk0 = b->c[C_UNKNOWN_CANCELS];
        if (X->check) {
            snap = (int32_t *)malloc(sizeof(int32_t) * (size_t)N * O_NF);
            memcpy(snap, own, sizeof(int32_t) * (size_t)N * O_NF);
        }
        cancel(X, b, own, m[M_P], m[M_OID], m[M_Q]);
        if (X->check) {
            /* idempotent unknown cancel: book bit-identical */
            if (b->c[C_UNKNOWN_CANCELS] != unk0 &&
                memcmp(snap, own, sizeof(int32_t) * (size_t)N * O_NF) != 0)
                b->violations++;
            free(snap);
        }
        return;
    }
    if (T == 1 && m[M_P] <= 0) { b->c[C_BAD]++; return; }         /* G22 */
    /* a market order uses P_m = 0 (sell) or max_int (buy) */
    int32_t Pa = (T == 4) ? (S == 1 ? INT32_MAX_ : 0) : m[M_P];
    int32_t Qa = m[M_Q];
    if (X->check) {
        if (T == 1) b->limit_in += (Qa > 0 ? Qa : 0);
        else b->market_in += (Qa > 0 ? Qa : 0);
    }
    /* matching while-loop */
    while (Qa > 0) {
        int j = best_standing(opp, N, opp_is_ask);
        if (j < 0) break;                                         /* book side empty */
        int32_t *os = opp + (size_t)j * O_NF;
        int32_t Ps = os[O_P];
        if ((S == 1 && Pa < Ps) || (S == -1 && Pa > Ps)) break;   /* no overlap */
        if (X->check) check_priority(X, b, opp, j, opp_is_ask);
        int32_t Qs = os[O_Q];
        int32_t Qs2 = (Qs - Qa > 0) ? (Qs - Qa) : 0;              /* Q_s' = max(0, Q_s - Q_a) */
        int32_t q = Qs - Qs2;                                     /* Q_j = Q_s - Q_s' */
        Qa = Qa - Qs;                                             /* Q_a' = Q_a - Q_s */
        if (b->n_trades < X->T_cap) {                             /* "up to N trades", G8 */
            int32_t *t = b->trades + (size_t)b->n_trades * T_NF;
            t[0] = Ps;                                            /* P_j = P_s */
            t[1] = q;                                             /* Q_j */
            t[2] = m[M_OID];                                      /* OID_a */
            t[3] = os[O_OID];                                     /* OID_s */
            t[4] = m[M_TS];                                       /* Ts_j = Ts_a */
            t[5] = m[M_TNS];                                      /* Tns_j = Tns_a */
            b->n_trades++;
        } else {
            b->c[C_TRADES_DROPPED]++;
        }
        b->c[C_TRADES]++;
        b->c[C_TRADED_QTY] += q;
        if (X->check) {
            if (T == 1) b->limit_aggr_traded += q; else b->market_aggr_traded += q;
        }
        os[O_Q] = Qs2;
        if (Qs2 <= 0) set_empty(os);                              /* removal, G10 */
    }
    if (T == 1 && Qa > 0) {                                       /* remainder added */
        int i = -1;
        for (int k = 0; k < N; k++)                               /* lowest empty slot, G3 */
            if (!occupied(own + (size_t)k * O_NF)) { i = k; break; }
        if (i < 0) {                                              /* saturated side, G6 */
            b->c[C_ADD_OVERFLOW]++;
            b->c[C_OVERFLOW_QTY] += Qa;
        } else {
            int32_t *o = own + (size_t)i * O_NF;                  /* G27: limit price, msg ids/time */
            o[O_P] = m[M_P]; o[O_Q] = Qa; o[O_OID] = m[M_OID];
            o[O_TID] = m[M_TID]; o[O_TS] = m[M_TS]; o[O_TNS] = m[M_TNS];
            if (X->check) b->limit_rested += Qa;
        }
    }
    if (T == 4 && Qa > 0) b->c[C_MARKET_DISCARDED_QTY] += Qa;    /* remainder disregarded */
    if (X->check) check_book(X, b);
}

/* L2 top-L (G23): k-th best distinct price per side with its summed quantity;
 * absent levels are (-1, 0).  The sum is taken in int64; the record's fields are
 * 32-bit, so a level volume above INT32_MAX is reported as INT32_MAX
 * (saturated: "at least 2^31 - 1"; reading G20).  Generator profiles keep sums < 2^31. */
static void l2_levels(oracle_ctx *X, const obook *b, int32_t *out /*[L][4]*/, int L) {
    int N = X->N;
    for (int s = 0; s < 2; s++) {
        const int32_t *side = s ? b->B : b->A;
        int is_ask = (s == 0);
        int have_prev = 0;
        int32_t prev = 0;
        for (int k = 0; k < L; k++) {
            /* next distinct price strictly worse than prev */
            int found = 0;
            int32_t best = 0;
            for (int i = 0; i < N; i++) {
                const int32_t *o = side + (size_t)i * O_NF;
                if (!occupied(o)) continue;
                int32_t p = o[O_P];
                if (have_prev && (is_ask ? !(p > prev) : !(p < prev))) continue;
                if (!found || (is_ask ? p < best : p > best)) { best = p; found = 1; }
            }
            int32_t price = -1, qty = 0;
            if (found) {
                int64_t sum = 0;
                for (int i = 0; i < N; i++) {
                    const int32_t *o = side + (size_t)i * O_NF;
                    if (occupied(o) && o[O_P] == best) sum += o[O_Q];
                }
                price = best;
                qty = sum > INT32_MAX_ ? INT32_MAX_ : (int32_t)sum;
                prev = best;
                have_prev = 1;
            }
            out[(size_t)k * 4 + (is_ask ? 0 : 2)] = price;
            out[(size_t)k * 4 + (is_ask ? 1 : 3)] = qty;
        }
    }
}

static void l2_snapshot(oracle_ctx *X, const obook *b, int32_t *out /*[L][4]*/) { l2_levels(X, b, out, X->L); }

/* NEXT row N1: Level-1 data after every processed message:
 * [best ask P, volume at it, best bid P, volume at it] = level 1 of the L2
 * definition (G23), absent side (-1, 0). */
static void l1_snapshot(oracle_ctx *X, const obook *b, int32_t *out /*[4]*/) { l2_levels(X, b, out, 1); }

/* ------------------------------------------------------------ public API */

oracle_ctx *oracle_create(int32_t K, int32_t N, int32_t T_cap, int32_t L, int32_t check) {
    if (K < 0 || N < 1 || T_cap < 0 || L < 0) return NULL;
    oracle_ctx *X = (oracle_ctx *)calloc(1, sizeof(oracle_ctx));
    X->K = K; X->N = N; X->T_cap = T_cap; X->L = L; X->check = check;
    X->books = (obook *)calloc((size_t)(K > 0 ? K : 1), sizeof(obook));
    for (int k = 0; k < K; k++) {
        obook *b = &X->books[k];
        b->A = (int32_t *)malloc(sizeof(int32_t) * (size_t)N * O_NF);
        b->B = (int32_t *)malloc(sizeof(int32_t) * (size_t)N * O_NF);
        b->trades = (int32_t *)malloc(sizeof(int32_t) * (size_t)(T_cap > 0 ? T_cap : 1) * T_NF);
    }
    return X;
}

void oracle_destroy(oracle_ctx *X) {
    if (!X) return;
    for (int k = 0; k < X->K; k++) {
        free(X->books[k].A); free(X->books[k].B); free(X->books[k].trades);
    }
    free(X->books);
    free(X);
}

/* Book init: both sides -1, trade log -1,
 * counters zero; then one synthetic order per populated L2 level:
 * OIDs -9000, -9001, ... over asks best->worst then bids (G24), TID -9000,
 * time = the caller's init time.  init_l2 rows are [ask_p, ask_q, bid_p, bid_q]. */
static void init_book(oracle_ctx *X, obook *b, const int32_t *l2 /*[L0][4] or NULL*/, int32_t L0,
                      int32_t ts, int32_t tns) {
    int N = X->N;
    for (int i = 0; i < N; i++) { set_empty(b->A + (size_t)i * O_NF); set_empty(b->B + (size_t)i * O_NF); }
    for (int i = 0; i < X->T_cap; i++) for (int f = 0; f < T_NF; f++) b->trades[(size_t)i * T_NF + f] = -1;
    b->n_trades = 0;
    memset(b->c, 0, sizeof(b->c));
    b->call_trades0 = b->call_dropped0 = 0;
    b->limit_in = b->limit_aggr_traded = b->limit_rested = b->market_in = b->market_aggr_traded = 0;
    b->violations = 0;
    int32_t oid = -9000;
    if (l2) {
        for (int s = 0; s < 2; s++) {
            int32_t *side = s ? b->B : b->A;
            int next = 0;
            for (int k = 0; k < L0; k++) {
                int32_t p = l2[(size_t)k * 4 + 2 * s], q = l2[(size_t)k * 4 + 2 * s + 1];
                if (p <= 0 || q <= 0) continue;                   /* G24 */
                if (next >= N) break;                             /* cannot happen: L0 <= N is enforced */
                int32_t *o = side + (size_t)next * O_NF;
                o[O_P] = p; o[O_Q] = q; o[O_OID] = oid--; o[O_TID] = -9000; o[O_TS] = ts; o[O_TNS] = tns;
                next++;
            }
        }
    }
    b->resting_init = side_resting(b->A, N) + side_resting(b->B, N);
}

/* init_l2: [K][L0][4] or NULL */
int oracle_init(oracle_ctx *X, int32_t k0, int32_t k1, const int32_t *init_l2, int32_t L0,
                int32_t ts, int32_t tns) {
    if (L0 < 0 || L0 > X->N) return -1;
    for (int k = k0; k < k1; k++)
        init_book(X, &X->books[k], init_l2 ? init_l2 + (size_t)k * L0 * 4 : NULL, L0, ts, tns);
    return 0;
}

/* One call over books [k0, k1): the trade log is cleared at the start of the
 * call (G9); counters accumulate; L2 after the last message of each step.
 * msgs: [K][n_steps*M][8]; l2_out: [K][n_steps][L][4] or NULL. */
int oracle_process_ex(oracle_ctx *X, int32_t k0, int32_t k1, const int32_t *msgs, int32_t n_steps,
                      int32_t M, int32_t *l2_out, int32_t *l1_out /* [K][n_steps*M][4] or NULL */) {
    int64_t per_book = (int64_t)n_steps * M;
    for (int k = k0; k < k1; k++) {
        obook *b = &X->books[k];
        for (int i = 0; i < X->T_cap; i++) for (int f = 0; f < T_NF; f++) b->trades[(size_t)i * T_NF + f] = -1;
        b->n_trades = 0;
        b->call_trades0 = b->c[C_TRADES];
        b->call_dropped0 = b->c[C_TRADES_DROPPED];
        const int32_t *mk = msgs + (size_t)k * per_book * M_NF;
        for (int s = 0; s < n_steps; s++) {
            for (int i = 0; i < M; i++) {
                process(X, b, mk + ((size_t)s * M + i) * M_NF);
                if (l1_out) l1_snapshot(X, b, l1_out + ((size_t)k * per_book + (size_t)s * M + i) * 4);
            }
            if (l2_out) l2_snapshot(X, b, l2_out + (((size_t)k * n_steps + s) * X->L) * 4);
        }
    }
    return 0;
}

int oracle_process(oracle_ctx *X, int32_t k0, int32_t k1, const int32_t *msgs, int32_t n_steps,
                   int32_t M, int32_t *l2_out) {
    return oracle_process_ex(X, k0, k1, msgs, n_steps, M, l2_out, NULL);
}

/* NEXT row N2: step reward over the trade log of the last call (one env step).
 *   P_VWAP = sum_i Q_i P_i / sum_i Q_i over every logged trade i     (eq:vwap)
 *   R      = sum_j Q_j (P_j - P_VWAP) + lambda sum_j Q_j (P_VWAP - P_init)
 *                                                                  (eq:rewardfunc)
 * j = the agent's trades: aggressor or standing OID in [agent_lo, agent_hi] (reading G29);
 * side -1 = sell task (the paper's form), +1 = buy task: both terms negated (G30);
 * no trades in the step: P_VWAP = 0 and R = 0 (G31).  Double precision, trade-log order. */
void oracle_step_reward(oracle_ctx *X, const int32_t *agent /*[K][2]*/, const double *p_init /*[K]*/,
                        const int32_t *side /*[K]*/, double lambda, double *reward, double *vwap,
                        int64_t *agent_qty) {
    for (int k = 0; k < X->K; k++) {
        const obook *b = &X->books[k];
        double sqp = 0.0, sq = 0.0;
        for (int i = 0; i < b->n_trades; i++) {
            const int32_t *t = b->trades + (size_t)i * T_NF;
            sqp += (double)t[1] * (double)t[0];
            sq += (double)t[1];
        }
        double v = (sq > 0.0) ? sqp / sq : 0.0;
        double adv = 0.0, drift = 0.0;
        int64_t qa = 0;
        int32_t lo = agent[2 * k], hi = agent[2 * k + 1];
        for (int i = 0; i < b->n_trades && sq > 0.0; i++) {
            const int32_t *t = b->trades + (size_t)i * T_NF;
            int mine = (t[2] >= lo && t[2] <= hi) || (t[3] >= lo && t[3] <= hi);
            if (!mine) continue;
            adv += (double)t[1] * ((double)t[0] - v);
            drift += (double)t[1] * (v - p_init[k]);
            qa += t[1];
        }
        double r = adv + lambda * drift;
        if (side[k] == 1) r = -r;
        if (reward) reward[k] = r;
        if (vwap) vwap[k] = v;
        if (agent_qty) agent_qty[k] = qa;
    }
}

/* exports: book [K][2][N][6] (side 0 = asks), trades [K][T_cap][6] + counts,
 * current L2 [K][L][4], counters [K][10], invariant violations [K] */
void oracle_get_book(oracle_ctx *X, int32_t *out) {
    size_t sz = (size_t)X->N * O_NF;
    for (int k = 0; k < X->K; k++) {
        memcpy(out + (size_t)k * 2 * sz, X->books[k].A, sz * sizeof(int32_t));
        memcpy(out + (size_t)k * 2 * sz + sz, X->books[k].B, sz * sizeof(int32_t));
    }
}
void oracle_get_trades(oracle_ctx *X, int32_t *out, int32_t *counts) {
    size_t sz = (size_t)X->T_cap * T_NF;
    for (int k = 0; k < X->K; k++) {
        if (sz) memcpy(out + (size_t)k * sz, X->books[k].trades, sz * sizeof(int32_t));
        counts[k] = X->books[k].n_trades;
    }
}
void oracle_get_l2(oracle_ctx *X, int32_t *out) {
    for (int k = 0; k < X->K; k++) l2_snapshot(X, &X->books[k], out + (size_t)k * X->L * 4);
}
void oracle_get_stats(oracle_ctx *X, int64_t *out) {
    for (int k = 0; k < X->K; k++) memcpy(out + (size_t)k * C_N, X->books[k].c, sizeof(int64_t) * C_N);
}
void oracle_get_violations(oracle_ctx *X, int64_t *out) {
    for (int k = 0; k < X->K; k++) out[k] = X->books[k].violations;
}

/* ===================================================================== */
/* NEXT row N3: the execution-environment step (Sec.5.1.3 and 5.2), one env
 * per book.  Written in the order of the paper's step:
 *   1. the agent's action becomes messages: cancel the agent's orders of
 *      the previous step, then either the forced market order for the remaining
 *      task one minute before the episode ends or one limit order per
 *      positive size at the far-touch, mid, near-touch and passive prices
 *      (P:L476-493);
 *   2. the step's data messages follow -- one trade log for the step (G9);
 *   3. the current time becomes the last data message's time;
 *   4. reward (eq:rewardfunc, N2) and the executed quantity from the agent's trades;
 *   5. done when the task is complete or the episode time is over
 *      (P:L423).  Readings E1-E8 are listed in DESIGN.md. */
typedef struct {
    int32_t task_side;   /* -1 sell, +1 buy */
    int32_t task_size;
    int32_t n_passive;   /* ticks behind the near touch for the passive price */
    int32_t tick;
    int32_t episode_s;
    int32_t agent_tid;
    int32_t oid_base;    /* agent OIDs are oid_base, oid_base+1, ... (E4) */
    int32_t pad;
    double lambda;
} env_cfg;

typedef struct {
    int64_t executed;
    int32_t init_ts, init_tns, cur_ts, cur_tns, next_oid, done, last_ask, last_bid;
    int32_t live[4];
    double p_init;
} oenv;

static int32_t best_price_of(oracle_ctx *X, const obook *b, int ask) {
    int32_t o[4];
    l2_levels(X, b, o, 1);
    return ask ? o[0] : o[2];
}

void *oracle_env_create(int32_t K) { return calloc((size_t)(K > 0 ? K : 1), sizeof(oenv)); }
void oracle_env_destroy(void *e) { free(e); }

/* after oracle_init: P_init = the mid price (P_ask + P_bid)/2 of the initial book */
void oracle_env_reset(oracle_ctx *X, void *envp, const env_cfg *c, int32_t init_ts, int32_t init_tns) {
    oenv *E = (oenv *)envp;
    for (int k = 0; k < X->K; k++) {
        oenv *e = &E[k];
        memset(e, 0, sizeof *e);
        e->init_ts = e->cur_ts = init_ts;
        e->init_tns = e->cur_tns = init_tns;
        e->next_oid = c->oid_base;
        e->last_ask = best_price_of(X, &X->books[k], 1);
        e->last_bid = best_price_of(X, &X->books[k], 0);
        /* E7: a one-sided initial book takes the price of the side that exists */
        int32_t a = e->last_ask > 0 ? e->last_ask : e->last_bid, bq = e->last_bid > 0 ? e->last_bid : e->last_ask;
        e->p_init = (a > 0) ? ((double)a + (double)bq) / 2.0 : 0.0;
    }
}

static int64_t elapsed_ns(const oenv *e) {
    return ((int64_t)e->cur_ts - e->init_ts) * 1000000000LL + ((int64_t)e->cur_tns - e->init_tns);
}

/* The agent's messages of one step for one env (at most 8; unused rows stay zero):
 * exposed so tests can check the action mapping on its own. */
static void env_agent_msgs(oracle_ctx *X, const obook *b, oenv *e, const env_cfg *c, const float *a,
                           int32_t *m /*[8][8]*/) {
    memset(m, 0, 8 * 8 * sizeof(int32_t));
    if (e->done) return;
    int n = 0;
    int32_t S = c->task_side;
    for (int i = 0; i < 4; i++)                                   /* E1: cancel the previous orders */
        if (e->live[i] != 0) {
            int32_t *r = m + 8 * n++;
            r[0] = 3; r[1] = S; r[2] = 2147483647; r[3] = 0; r[4] = e->live[i]; r[5] = c->agent_tid;
            r[6] = e->cur_ts; r[7] = e->cur_tns;
            e->live[i] = 0;
        }
    int64_t remaining = (int64_t)c->task_size - e->executed;
    if (remaining <= 0) return;
    if (elapsed_ns(e) >= ((int64_t)c->episode_s - 60) * 1000000000LL) {   /* forced market order */
        int32_t *r = m + 8 * n++;
        r[0] = 4; r[1] = S; r[2] = (int32_t)(remaining > 2147483647 ? 2147483647 : remaining); r[3] = 0;
        r[4] = e->next_oid++; r[5] = c->agent_tid; r[6] = e->cur_ts; r[7] = e->cur_tns;
        return;
    }
    /* prices from the current book; an empty side keeps its last valid price (E6) */
    int32_t ask = best_price_of(X, b, 1), bid = best_price_of(X, b, 0);
    if (ask > 0) e->last_ask = ask; else ask = e->last_ask;
    if (bid > 0) e->last_bid = bid; else bid = e->last_bid;
    int32_t far = (S == -1) ? bid : ask;
    int32_t near = (S == -1) ? ask : bid;
    int32_t passive = (near > 0) ? near - S * c->n_passive * c->tick : 0;
    int32_t mid = 0;                                                      /* P:L449, E5 */
    if (ask > 0 && bid > 0) {
        int64_t twice = (int64_t)ask + bid, t2 = 2LL * c->tick;
        int64_t q = twice / t2, rmd = twice % t2;
        mid = (int32_t)((S == -1 && rmd) ? (q + 1) * c->tick : q * c->tick);
    }
    int32_t price[4] = {far, mid, near, passive};
    int li = 0;
    for (int k = 0; k < 4; k++) {
        float x = a[k];
        int64_t q = 0;                                                    /* E2: rint, NaN/negative -> 0 */
        if (x == x && x > 0.0f) q = (x >= 2147483647.0f) ? 2147483647LL : (int64_t)rintf(x);
        if (q > remaining) q = remaining;                                 /* E3: far touch first */
        if (q <= 0 || price[k] <= 0) continue;
        remaining -= q;
        int32_t *r = m + 8 * n++;
        r[0] = 1; r[1] = S; r[2] = (int32_t)q; r[3] = price[k]; r[4] = e->next_oid; r[5] = c->agent_tid;
        r[6] = e->cur_ts; r[7] = e->cur_tns;
        e->live[li++] = e->next_oid++;
    }
}

void oracle_env_step(oracle_ctx *X, void *envp, const env_cfg *c, const float *actions /*[K][4]*/,
                     const int32_t *data /*[K][M][8]*/, int32_t M, double *reward, int32_t *done,
                     int64_t *executed, int32_t *agent_out /*[K][8][8] or NULL*/) {
    oenv *E = (oenv *)envp;
    int32_t *stream = (int32_t *)malloc(sizeof(int32_t) * (size_t)(8 + M) * 8);
    for (int k = 0; k < X->K; k++) {
        oenv *e = &E[k];
        obook *b = &X->books[k];
        int was_done = e->done;
        env_agent_msgs(X, b, e, c, actions + 4 * k, stream);
        if (agent_out) memcpy(agent_out + (size_t)k * 64, stream, 64 * sizeof(int32_t));
        /* E8: a finished env receives only padding (T = 0) messages: its book does not
         * change; the padding is counted and the trade log cleared like any call */
        if (was_done) memset(stream + 64, 0, sizeof(int32_t) * (size_t)M * 8);
        else memcpy(stream + 64, data + (size_t)k * M * 8, sizeof(int32_t) * (size_t)M * 8);
        /* one call of 8 + M messages: the trade log is the step's (G9) */
        for (int i = 0; i < X->T_cap; i++) for (int f = 0; f < T_NF; f++) b->trades[(size_t)i * T_NF + f] = -1;
        b->n_trades = 0;
        b->call_trades0 = b->c[C_TRADES];
        b->call_dropped0 = b->c[C_TRADES_DROPPED];
        for (int i = 0; i < 8 + M; i++) process(X, b, stream + (size_t)i * M_NF);
        if (was_done) { reward[k] = 0.0; done[k] = 1; executed[k] = e->executed; continue; }
        int32_t agent[2] = {c->oid_base, e->next_oid - 1};
        double r, v;
        int64_t qa;
        oracle_ctx one = *X;                                              /* reward over this book only */
        one.K = 1;
        one.books = b;
        oracle_step_reward(&one, agent, &e->p_init, &c->task_side, c->lambda, &r, &v, &qa);
        e->executed += qa;
        for (int i = M - 1; i >= 0; i--) {
            const int32_t *d = data + ((size_t)k * M + i) * 8;
            if (d[0] != 0) { e->cur_ts = d[6]; e->cur_tns = d[7]; break; }
        }
        e->done = (e->executed >= c->task_size) || (elapsed_ns(e) > (int64_t)c->episode_s * 1000000000LL);
        reward[k] = r; done[k] = e->done; executed[k] = e->executed;
    }
    free(stream);
}

/* env state export: [K][16] int64 = executed, init ts/tns, cur ts/tns, next_oid, done,
 * last_ask, last_bid, live[4], p_init bits, 0 */
void oracle_env_get(oracle_ctx *X, void *envp, int64_t *out) {
    oenv *E = (oenv *)envp;
    for (int k = 0; k < X->K; k++) {
        oenv *e = &E[k];
        int64_t *o = out + (size_t)k * 16;
        o[0] = e->executed; o[1] = e->init_ts; o[2] = e->init_tns; o[3] = e->cur_ts; o[4] = e->cur_tns;
        o[5] = e->next_oid; o[6] = e->done; o[7] = e->last_ask; o[8] = e->last_bid;
        for (int i = 0; i < 4; i++) o[9 + i] = e->live[i];
        memcpy(&o[13], &e->p_init, sizeof(double));
        o[14] = o[15] = 0;
    }
}
