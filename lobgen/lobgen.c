/*
 * lobgen/lobgen.c -- seeded synthetic LOBSTER-shaped message streams.
 *
 * This module is shared input plumbing for the oracle, the CUDA path, the
 * tests and bench.py.  It holds none of the method's arithmetic: it never
 * matches, never looks at a book, and only keeps its own list of the orders it
 * has issued (to aim cancels/deletes at plausible targets and to bound
 * occupancy).  Integer-only, so the bytes are identical on every host.
 *
 * Determinism: book b's stream depends only on (seed, global book id b), via
 * splitmix64(seed ^ phi*(b+1)) seeding xoshiro256**; it is invariant under the
 * number of books generated, the book range, the GPU count and thread count.
 *
 * Record layouts follow the paper: message m = [T, S, Q, P, OID, TID, Ts, Tns]
 * (Eq.6); initial L2 rows [ask_p, ask_q, bid_p, bid_q].
 * Recipe (units, mixes, profiles): DESIGN.md "Input recipe".
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>

#define TICK 100           /* LOBSTER prices are $1e-4; one cent tick */
#define REF0 1000000       /* $100.00 */
#define T0_S 34200         /* 09:30:00, LOBSTER seconds after midnight */
#define LOT 100

enum { P_LOBSTER = 0, P_HEAVY_MARKET = 1, P_CANCEL_HEAVY = 2, P_TIES = 3, P_OVERFLOW = 4,
       P_SYNTHETIC = 5, P_GARBAGE = 6, P_SATURATE = 7, P_NPROFILES = 8 };

typedef struct {
    int limit, cancel, del, market;  /* mix, percent (sums to 100) */
    int mkt_limit_pct;               /* share of limits priced through the reference */
    int unknown_pct;                 /* share of cancels/deletes with an unknown OID */
    int heavy_market_q;              /* market Q log-uniform over [1, 10^4] */
    int ties_pct;                    /* share of zero time gaps */
    int garbage_pct;                 /* share of malformed messages */
    int occ_control;                 /* keep issued-live orders within [low, cap] */
    int synth_pct;                   /* share of cancels aimed at init prices */
} profile_t;

static const profile_t PROFILES[P_NPROFILES] = {
    /* lobster      */ {50, 10, 35,  5, 10,  5, 0,  0, 0, 1,  0},
    /* heavy_market */ {75,  5, 10, 10, 15,  5, 1,  0, 0, 1,  0},
    /* cancel_heavy */ {40, 15, 43,  2,  5, 10, 0,  0, 0, 1,  5},
    /* ties         */ {50, 10, 35,  5, 10,  5, 0, 30, 0, 1,  0},
    /* overflow     */ {70,  5, 20,  5, 10,  5, 0,  0, 0, 0,  0},
    /* synthetic    */ {40, 25, 30,  5, 10,  5, 0,  0, 0, 1, 50},
    /* garbage      */ {50, 10, 35,  5, 10,  5, 0,  0, 5, 1,  0},
    /* saturate     */ {95,  3,  2,  0,  0,  5, 0,  0, 0, 0,  0},  /* passive limits fill both sides past N */
};

/* ---------------------------------------------------------------- RNG */
static uint64_t splitmix64(uint64_t *x) {
    uint64_t z = (*x += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
typedef struct { uint64_t s[4]; } rng_t;
static inline uint64_t rotl(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }
static uint64_t next64(rng_t *r) {
    uint64_t *s = r->s;
    uint64_t res = rotl(s[1] * 5, 7) * 9, t = s[1] << 17;
    s[2] ^= s[0]; s[3] ^= s[1]; s[1] ^= s[2]; s[0] ^= s[3]; s[2] ^= t; s[3] = rotl(s[3], 45);
    return res;
}
static void rng_seed(rng_t *r, uint64_t seed, int64_t book) {
    uint64_t x = seed ^ (0x9E3779B97F4A7C15ull * (uint64_t)(book + 1));
    for (int i = 0; i < 4; i++) r->s[i] = splitmix64(&x);
}
/* uniform in [0, n) (n >= 1), multiply-shift */
static inline int64_t uni(rng_t *r, int64_t n) {
    return (int64_t)(((__uint128_t)next64(r) * (uint64_t)n) >> 64);
}
static inline int64_t uni_ab(rng_t *r, int64_t a, int64_t b) { return a + uni(r, b - a + 1); }
static inline int pct(rng_t *r, int p) { return uni(r, 100) < p; }
/* geometric number of failures before success with success prob num/den, capped */
static int geom(rng_t *r, int num, int den, int cap) {
    int k = 0;
    while (k < cap && uni(r, den) >= num) k++;
    return k;
}

/* ------------------------------------------------ issued-live order list */
typedef struct { int32_t oid, p, q, synth; } live_t;
typedef struct { live_t *v; int n; } livelist;

static void live_push(livelist *l, int32_t oid, int32_t p, int32_t q, int synth) {
    l->v[l->n].oid = oid; l->v[l->n].p = p; l->v[l->n].q = q; l->v[l->n].synth = synth; l->n++;
}
static void live_del(livelist *l, int i) { l->v[i] = l->v[--l->n]; }

static int32_t limit_q(rng_t *r) {
    if (pct(r, 80)) { int q = LOT * (1 + geom(r, 1, 2, 30)); return q > 1000 ? 1000 : q; }
    return (int32_t)uni_ab(r, 1, 99);                             /* odd lot */
}
static int32_t market_q(rng_t *r, const profile_t *pf) {
    if (pf->heavy_market_q) {                                     /* log-uniform over [1, 1e4] */
        static const int32_t dec[5] = {1, 10, 100, 1000, 10000};
        int e = (int)uni(r, 4);
        return (int32_t)uni_ab(r, dec[e], dec[e + 1]);
    }
    return (int32_t)uni_ab(r, 1, 3) * LOT;
}

typedef struct {
    uint64_t seed;
    int64_t book_begin;
    int32_t n_books, N, n_msgs, L0, profile, occ_cap_pct;
    int32_t *msgs, *init_l2;
} job_t;

static void gen_book(const job_t *J, int64_t k, livelist *live) {
    const profile_t *pf = &PROFILES[J->profile];
    rng_t r;
    rng_seed(&r, J->seed, J->book_begin + k);
    int32_t ref = REF0;
    int32_t ts = T0_S, tns = 0;
    int32_t next_oid = 1;
    live[0].n = live[1].n = 0;                                    /* 0 = asks, 1 = bids */
    /* initial L2 snapshot: one level per tick away from the reference */
    for (int lv = 0; lv < J->L0; lv++) {
        int32_t ap = ref + (lv + 1) * TICK, bp = ref - (lv + 1) * TICK;
        int32_t aq = LOT * (int32_t)uni_ab(&r, 1, 5), bq = LOT * (int32_t)uni_ab(&r, 1, 5);
        if (J->init_l2) {
            int32_t *row = J->init_l2 + ((size_t)k * J->L0 + lv) * 4;
            row[0] = ap; row[1] = aq; row[2] = bp; row[3] = bq;
        }
        live_push(&live[0], 0, ap, aq, 1);
        live_push(&live[1], 0, bp, bq, 1);
    }
    int cap = (int)((int64_t)J->N * J->occ_cap_pct / 100);
    if (cap < 1) cap = 1;
    int low = J->N / 5;
    int32_t *out = J->msgs + (size_t)k * J->n_msgs * 8;
    for (int i = 0; i < J->n_msgs; i++) {
        int32_t *m = out + (size_t)i * 8;
        /* time: strictly increasing unless a tie is drawn */
        int32_t gap = (pf->ties_pct && pct(&r, pf->ties_pct)) ? 0 : (int32_t)uni_ab(&r, 1, 2000000);
        tns += gap;
        if (tns >= 1000000000) { tns -= 1000000000; ts++; }
        if (pct(&r, 5)) ref += pct(&r, 50) ? TICK : -TICK;        /* reference random walk */
        if (ref - (J->L0 + 25) * TICK < TICK) ref += TICK;          /* keep every price positive */
        if (pf->garbage_pct && pct(&r, pf->garbage_pct)) {
            m[0] = (int32_t)uni_ab(&r, -1, 6); m[1] = (int32_t)uni_ab(&r, -2, 2);
            m[2] = (int32_t)uni_ab(&r, -5, 100000); m[3] = (int32_t)uni_ab(&r, -5, 2 * REF0);
            m[4] = (int32_t)uni_ab(&r, -9005, next_oid + 5); m[5] = (int32_t)uni(&r, 1000);
            m[6] = ts; m[7] = tns;
            continue;
        }
        int sd = (int)uni(&r, 2);                                 /* 0 ask (S=-1), 1 bid (S=+1) */
        int32_t S = sd ? 1 : -1;
        int64_t u = uni(&r, 100);
        int type = u < pf->limit ? 1 : u < pf->limit + pf->cancel ? 2
                 : u < pf->limit + pf->cancel + pf->del ? 3 : 4;
        if (pf->occ_control) {
            if (type == 1 && live[sd].n >= cap) type = 3;         /* keep occupancy below N */
            else if ((type == 2 || type == 3) && live[sd].n < low) type = 1;
        }
        m[1] = S; m[5] = (int32_t)uni(&r, 1000); m[6] = ts; m[7] = tns;
        if (type == 1) {
            int32_t p;
            if (pct(&r, pf->mkt_limit_pct)) p = ref + S * (int32_t)(1 + uni(&r, 4)) * TICK;
            else p = ref - S * (int32_t)(1 + geom(&r, 35, 100, 19)) * TICK;
            int32_t q = limit_q(&r);
            m[0] = 1; m[2] = q; m[3] = p; m[4] = next_oid;
            if (live[sd].n < J->n_msgs + J->L0) live_push(&live[sd], next_oid, p, q, 0);
            next_oid++;
        } else if (type == 4) {
            m[0] = 4; m[2] = market_q(&r, pf); m[3] = 0; m[4] = next_oid++;
        } else {
            m[0] = type;
            int unknown = live[sd].n == 0 || pct(&r, pf->unknown_pct);
            int idx = -1;
            if (!unknown) {
                if (pf->synth_pct && pct(&r, pf->synth_pct)) {    /* aim at an init price */
                    for (int t = 0; t < 4 && idx < 0; t++) {
                        int c = (int)uni(&r, live[sd].n);
                        if (live[sd].v[c].synth) idx = c;
                    }
                }
                if (idx < 0) idx = (int)uni(&r, live[sd].n);
            }
            if (idx < 0) {
                m[2] = (int32_t)uni_ab(&r, 1, 500);
                m[3] = ref - S * (int32_t)(1 + uni(&r, 10)) * TICK;
                m[4] = (int32_t)uni_ab(&r, 1900000000, 1999999999);
            } else {
                live_t *o = &live[sd].v[idx];
                int32_t q;
                if (type == 2 && o->q >= 2) q = (int32_t)uni_ab(&r, 1, o->q - 1);
                else q = o->q;
                m[2] = q; m[3] = o->p;
                /* a synthetic order carries no real OID: the cancel hits it by price */
                m[4] = o->synth ? (int32_t)uni_ab(&r, 1900000000, 1999999999) : o->oid;
                o->q -= q;
                if (o->q <= 0) live_del(&live[sd], idx);
            }
        }
    }
}

typedef struct { const job_t *J; int64_t k0, k1; } slice_t;

static void *worker(void *arg) {
    slice_t *s = (slice_t *)arg;
    livelist live[2];
    int cap = s->J->n_msgs + s->J->L0 + 1;
    live[0].v = (live_t *)malloc(sizeof(live_t) * (size_t)cap);
    live[1].v = (live_t *)malloc(sizeof(live_t) * (size_t)cap);
    for (int64_t k = s->k0; k < s->k1; k++) gen_book(s->J, k, live);
    free(live[0].v); free(live[1].v);
    return NULL;
}

/* msgs_out: [n_books][n_msgs][8]; init_l2_out: [n_books][init_levels][4] or NULL.
 * Returns 0, or -1 on bad arguments. */
int lobgen_generate(uint64_t seed, int64_t book_begin, int32_t n_books, int32_t capacity,
                    int32_t n_msgs, int32_t init_levels, int32_t profile, int32_t occ_cap_pct,
                    int32_t n_threads, int32_t *msgs_out, int32_t *init_l2_out) {
    if (n_books < 0 || capacity < 1 || n_msgs < 0 || init_levels < 0 || profile < 0 ||
        profile >= P_NPROFILES || (n_books > 0 && n_msgs > 0 && !msgs_out) || occ_cap_pct < 1)
        return -1;
    job_t J = {seed, book_begin, n_books, capacity, n_msgs, init_levels, profile, occ_cap_pct,
               msgs_out, init_l2_out};
    if (n_threads < 1) n_threads = 1;
    if (n_threads > n_books) n_threads = n_books > 0 ? n_books : 1;
    pthread_t th[256];
    slice_t sl[256];
    if (n_threads > 256) n_threads = 256;
    int64_t per = (n_books + n_threads - 1) / n_threads;
    for (int t = 0; t < n_threads; t++) {
        sl[t].J = &J; sl[t].k0 = t * per; sl[t].k1 = (t + 1) * per < n_books ? (t + 1) * per : n_books;
        if (sl[t].k0 > sl[t].k1) sl[t].k0 = sl[t].k1;
    }
    for (int t = 1; t < n_threads; t++) pthread_create(&th[t], NULL, worker, &sl[t]);
    worker(&sl[0]);
    for (int t = 1; t < n_threads; t++) pthread_join(th[t], NULL);
    return 0;
}
