/*
 * lobster_io.c -- NEXT row N4: LOBSTER ingestion, host side.
 *
 * Parses LOBSTER message files ("Time,Type,OrderID,Size,Price,Direction", one
 * row per event, time in decimal seconds after midnight, price in $1e-4) and
 * orderbook files (per level: AskPrice,AskSize,BidPrice,BidSize) into fixed
 * int32 records for the engine:
 *   message -> Eq.6 m = [T, S, Q, P, OID, TID, Ts, Tns]
 *   type 1 -> limit (T=1), 2 -> cancel (T=2), 3 -> delete (T=3)
 *   types 4/5 (executions), 6 (cross), 7 (halt) are skipped and counted (S:L238,
 *   reading G33), unless exec_as_market = 1, which replays a visible execution
 *   (type 4) as a market order of the same size on the opposite side.
 *   Ts = whole seconds, Tns = fractional part in ns, rounded half-even.
 *   TID = 0 for replayed data.
 * Windowing and the initial book per window are done by the
 * Python layer (paper_2308_13289_b200/lobster.py) on the parsed arrays.
 *
 * Errors: a malformed row aborts with its 1-based row number.
 */
#include <errno.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static char g_err[256];
const char *lobster_last_error(void) { return g_err; }

/* decimal "S.FFFFFFFFF..." -> (seconds, nanoseconds) with round-half-even at 1e-9 */
static int parse_time(const char *s, const char *e, int32_t *ts, int32_t *tns) {
    int64_t sec = 0;
    const char *p = s;
    if (p == e) return -1;
    while (p < e && *p >= '0' && *p <= '9') { sec = sec * 10 + (*p - '0'); p++; if (sec > 2147483647) return -1; }
    int64_t ns = 0;
    int digits = 0, round_digit = -1, sticky = 0;
    if (p < e && *p == '.') {
        p++;
        while (p < e && *p >= '0' && *p <= '9') {
            if (digits < 9) { ns = ns * 10 + (*p - '0'); digits++; }
            else if (round_digit < 0) round_digit = *p - '0';
            else if (*p != '0') sticky = 1;
            p++;
        }
    }
    if (p != e) return -1;
    while (digits < 9) { ns *= 10; digits++; }
    if (round_digit > 5 || (round_digit == 5 && (sticky || (ns & 1)))) ns++;
    if (ns >= 1000000000) { ns -= 1000000000; sec++; }
    *ts = (int32_t)sec;
    *tns = (int32_t)ns;
    return 0;
}

static int parse_int64(const char *s, const char *e, int64_t *out) {
    const char *p = s;
    int neg = 0;
    if (p < e && (*p == '-' || *p == '+')) { neg = *p == '-'; p++; }
    if (p == e) return -1;
    int64_t v = 0;
    while (p < e) {
        if (*p < '0' || *p > '9') return -1;
        v = v * 10 + (*p - '0');
        if (v > (int64_t)1e17) return -1;
        p++;
    }
    *out = neg ? -v : v;
    return 0;
}

/* split one line into fields; returns the field count */
static int split(char *line, const char **fs, const char **fe, int maxf) {
    int n = 0;
    char *p = line;
    size_t len = strlen(line);
    while (len && (line[len - 1] == '\n' || line[len - 1] == '\r')) line[--len] = 0;
    if (len == 0) return 0;
    for (;;) {
        char *c = strchr(p, ',');
        if (n < maxf) { fs[n] = p; fe[n] = c ? c : p + strlen(p); }
        n++;
        if (!c) break;
        p = c + 1;
    }
    return n;
}

/* Parse a message file.  out: [cap][8] int32 or NULL (count only); row_of: [cap]
 * int64 source row (0-based) of every kept message or NULL; skipped[8]: per LOBSTER
 * type counts of dropped rows.  Returns the number of kept messages, or -1 on error
 * (lobster_last_error()).  exec_as_market: see the header comment. */
int64_t lobster_parse_messages(const char *path, int32_t *out, int64_t cap, int32_t exec_as_market,
                               int64_t *row_of, int64_t *skipped) {
    FILE *f = fopen(path, "r");
    if (!f) { snprintf(g_err, sizeof g_err, "%s: %s", path, strerror(errno)); return -1; }
    char line[512];
    const char *fs[8], *fe[8];
    int64_t kept = 0, row = 0;
    if (skipped) memset(skipped, 0, 8 * sizeof(int64_t));
    while (fgets(line, sizeof line, f)) {
        row++;
        int nf = split(line, fs, fe, 8);
        if (nf == 0) continue;
        int64_t type, oid, size, price, dir;
        int32_t ts, tns;
        if (nf != 6 || parse_time(fs[0], fe[0], &ts, &tns) || parse_int64(fs[1], fe[1], &type) ||
            parse_int64(fs[2], fe[2], &oid) || parse_int64(fs[3], fe[3], &size) ||
            parse_int64(fs[4], fe[4], &price) || parse_int64(fs[5], fe[5], &dir) || type < 1 || type > 7 ||
            (dir != 1 && dir != -1) || oid < INT32_MIN || oid > INT32_MAX || size < INT32_MIN ||
            size > INT32_MAX || price < INT32_MIN || price > INT32_MAX) {
            snprintf(g_err, sizeof g_err, "%s: malformed row %lld", path, (long long)row);
            fclose(f);
            return -1;
        }
        int32_t T, S = (int32_t)dir;
        if (type <= 3) T = (int32_t)type;
        else if (type == 4 && exec_as_market) { T = 4; S = -S; }  /* the aggressor sat on the other side */
        else { if (skipped) skipped[type]++; continue; }
        if (out) {
            if (kept >= cap) { snprintf(g_err, sizeof g_err, "capacity %lld exceeded", (long long)cap); fclose(f); return -1; }
            int32_t *m = out + kept * 8;
            m[0] = T; m[1] = S; m[2] = (int32_t)size; m[3] = (int32_t)price;
            m[4] = (int32_t)oid; m[5] = 0; m[6] = ts; m[7] = tns;
            if (row_of) row_of[kept] = row - 1;
        }
        kept++;
    }
    fclose(f);
    return kept;
}

/* Parse an orderbook file with `levels` levels into out [rows][levels][4] int32
 * [ask_p, ask_q, bid_p, bid_q]; LOBSTER's empty-level sentinels (ask 9999999999,
 * bid -9999999999, size <= 0) become absent levels (0, 0).
 * out NULL counts rows.  Returns the row count or -1. */
int64_t lobster_parse_orderbook(const char *path, int32_t levels, int32_t *out, int64_t cap) {
    FILE *f = fopen(path, "r");
    if (!f) { snprintf(g_err, sizeof g_err, "%s: %s", path, strerror(errno)); return -1; }
    static char line[1 << 16];
    const char *fs[4 * 64], *fe[4 * 64];
    if (levels < 1 || levels > 64) { fclose(f); snprintf(g_err, sizeof g_err, "levels must be 1..64"); return -1; }
    int64_t rows = 0, lineno = 0;
    while (fgets(line, sizeof line, f)) {
        lineno++;
        int nf = split(line, fs, fe, 4 * 64);
        if (nf == 0) continue;
        if (nf != 4 * levels) {
            snprintf(g_err, sizeof g_err, "%s: row %lld has %d columns, expected %d", path, (long long)lineno, nf,
                     4 * levels);
            fclose(f);
            return -1;
        }
        if (out) {
            if (rows >= cap) { snprintf(g_err, sizeof g_err, "capacity exceeded"); fclose(f); return -1; }
            for (int l = 0; l < levels; l++) {
                int64_t v[4];
                for (int c = 0; c < 4; c++)
                    if (parse_int64(fs[4 * l + c], fe[4 * l + c], &v[c])) {
                        snprintf(g_err, sizeof g_err, "%s: malformed row %lld", path, (long long)lineno);
                        fclose(f);
                        return -1;
                    }
                int32_t *o = out + (rows * levels + l) * 4;
                int ask_ok = v[0] > 0 && v[0] < 9999999999LL && v[1] > 0 && v[0] <= INT32_MAX && v[1] <= INT32_MAX;
                int bid_ok = v[2] > 0 && v[3] > 0 && v[2] <= INT32_MAX && v[3] <= INT32_MAX;
                o[0] = ask_ok ? (int32_t)v[0] : 0; o[1] = ask_ok ? (int32_t)v[1] : 0;
                o[2] = bid_ok ? (int32_t)v[2] : 0; o[3] = bid_ok ? (int32_t)v[3] : 0;
            }
        }
        rows++;
    }
    fclose(f);
    return rows;
}
