/*
 * pmh_oracle.c -- CPU ORACLE (test infrastructure only).
 *
 * A plain-C restatement of the reference ProbMinHash kernels
 *   /root/reference/pkg/src/probminhash/_kernels.py   (cited below as K:<line>)
 * used ONLY by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference leg, as the checker and as the CPU baseline.  The product
 * path (paper_1911_00675_b200 + libpmh.so) never links or calls this file.
 *
 * Arithmetic contract: every floating-point operation is
 * one IEEE double rounding, evaluated in the reference's order, no FMA
 * contraction (compile with -ffp-contract=off), and every transcendental is the
 * host glibc libm call the reference reaches through numba (log1p, expm1, log,
 * exp).  Parity of this restatement is pinned against the live numba reference
 * by tests/golden/make_golden.py (fixtures committed under tests/golden/).
 *
 * Extra instrumentation (not in the reference): `pin` -- when finite, every
 * stop-limit read nodes[root] is replaced by the constant `pin` (the
 * schedule-free points_min of SURVEY.md §8d); `hfinal` returns nodes[root].
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef uint64_t u64;
typedef int64_t i64;

#define GOLDEN 0x9E3779B97F4A7C15ULL /* K:20 */
#define MIX1 0xBF58476D1CE4E5B9ULL   /* K:21 */
#define MIX2 0x94D049BB133111EBULL   /* K:22 */
#define INV53 1.1102230246251565e-16 /* K:30, 2**-53 */
#define BBIT_SALT 0xD1B54A32D192ED03ULL
#define OPH_SALT 0xA24BAED4963EE407ULL /* K:33 */
#define REJECT_CAP 4096                /* K:37 */

/* error codes (mirrored by oracle/oracle.py) */
#define ORC_OK 0
#define ORC_RANDOMNESS_FAILURE 3
#define ORC_NOMEM 4
#define ORC_BAD_ALGO 5

/* algorithm ids, K:866-881 */
enum {
    ALG_PMINHASH = 0, ALG_PMH1 = 1, ALG_PMH1A = 2, ALG_PMH2 = 3, ALG_PMH3 = 4,
    ALG_PMH3A = 5, ALG_PMH4 = 6, ALG_MINHASH = 10, ALG_SUPERMINHASH = 11,
    ALG_OPH = 12, ALG_UW1 = 13, ALG_UW1A = 14, ALG_UW2 = 15, ALG_UW3 = 16,
    ALG_UW3A = 17, ALG_UW4 = 18
};

/* ---- stream: K:40-78 ---------------------------------------------------- */
typedef struct { u64 s, buf, nb, words; } stream_t;

static inline u64 mix64(u64 x) { /* K:40-44 */
    u64 z = (x ^ (x >> 30)) * MIX1;
    z = (z ^ (z >> 27)) * MIX2;
    return z ^ (z >> 31);
}
static inline void rng_seed(stream_t *st, u64 seed) { /* K:47-52 */
    st->s = seed; st->buf = 0; st->nb = 0; st->words = 0;
}
static inline u64 next_u64(stream_t *st) { /* K:55-60 */
    st->s += GOLDEN;
    st->words += 1;
    return mix64(st->s);
}
static inline u64 next_bits(stream_t *st, u64 k) { /* K:63-78 */
    u64 nb = st->nb;
    if (nb >= k) {
        u64 out = st->buf & ((1ULL << k) - 1ULL);
        st->buf = st->buf >> k;
        st->nb = nb - k;
        return out;
    }
    u64 out = st->buf;
    u64 w = next_u64(st);
    u64 need = k - nb;
    out = out | ((w & ((1ULL << need) - 1ULL)) << nb);
    /* numba: w >> need with need in 1..63 */
    st->buf = w >> need;
    st->nb = 64 - need;
    return out;
}
static inline double uniform01(stream_t *st) { /* K:81-83 */
    return (double)next_bits(st, 53) * INV53;
}
static inline u64 bits_for(i64 n) { /* K:86-94 */
    u64 k = 0;
    i64 v = n - 1;
    while (v > 0) { v >>= 1; k++; }
    return k;
}
/* K:97-110; returns -1 on cap overflow */
static inline i64 uniform_int_masked(stream_t *st, u64 n_u, u64 kbits) {
    if (n_u <= 1) return 0;
    int rounds = 0;
    for (;;) {
        u64 r = next_bits(st, kbits);
        if (r < n_u) return (i64)r;
        rounds++;
        if (rounds > REJECT_CAP) return -1;
    }
}
static inline i64 uniform_int(stream_t *st, i64 n) { /* K:113-117 */
    if (n <= 1) return 0;
    return uniform_int_masked(st, (u64)n, bits_for(n));
}
static inline double exp1(stream_t *st) { /* K:120-122 */
    return -log1p(-uniform01(st));
}
/* K:125-151; *fail set on cap overflow */
static inline double trunc_exp(stream_t *st, double lam, double c1, double c2,
                               double c3, int *fail) {
    double x = c1 * uniform01(st);
    if (x < 1.0) return x;
    int rounds = 0;
    for (;;) {
        x = uniform01(st);
        if (x < c2) return x;
        double y = 0.5 * uniform01(st);
        if (y > 1.0 - x) { x = 1.0 - x; y = 1.0 - y; }
        if (x <= c3 * (1.0 - y)) return x;
        if (y * c1 <= 1.0 - x) return x;
        if (y * c1 * lam <= expm1(lam * (1.0 - x))) return x;
        rounds++;
        if (rounds > REJECT_CAP) { *fail = 1; return 0.0; }
    }
}
static inline void trunc_exp_consts(double lam, double *c1, double *c2,
                                    double *c3) { /* K:186-191 */
    *c1 = expm1(lam) / lam;
    *c2 = log(2.0 / (1.0 + exp(-lam))) / lam;
    *c3 = -expm1(-lam) / lam;
}

/* ---- stop-limit tree, K:198-215 ----------------------------------------- */
static inline i64 tree_update(double *nodes, i64 m, i64 k, double h) {
    i64 writes = 0;
    while (h < nodes[k]) {
        nodes[k] = h;
        writes++;
        i64 i = m + ((k + 1) >> 1);
        if (i >= 2 * m) break;
        i64 j = ((k - 1) ^ 1) + 1;
        if (nodes[j] >= nodes[i]) break;
        if (h < nodes[j]) h = nodes[j];
        k = i;
    }
    return writes;
}

/* ---- lazy Fisher-Yates, K:222-235; returns -1 on cap overflow ----------- */
static inline i64 perm_next(stream_t *st, i64 *perm, u64 *vers, u64 counter,
                            i64 i, i64 m) {
    i64 r = uniform_int(st, m - i + 1);
    if (r < 0) return -1;
    i64 j = i + r;
    i64 k = (vers[j] == counter) ? perm[j] : j;
    perm[j] = (vers[i] == counter) ? perm[i] : i;
    vers[j] = counter;
    return k;
}

static inline i64 coupon_cap(i64 m) { /* K:279-281 */
    return (i64)(64.0 * (double)m * (1.0 + log((double)m)) + 64.0);
}

/* thresholds: the reference reads nodes[root]; `pin` replaces it if finite */
#define THR() (pinned ? pin : nodes[root])

/* common output: sig[m], stats[3], hfinal */
typedef struct {
    u64 *sig; i64 *stats; double *hfinal; double pin;
} out_t;

static double *alloc_nodes(i64 m) {
    double *nodes = (double *)malloc(sizeof(double) * 2 * m);
    if (!nodes) return NULL;
    for (i64 i = 0; i < 2 * m; i++) nodes[i] = INFINITY;
    return nodes;
}

/* K:284-300 */
static int k_pminhash(const u64 *ids, const double *w, i64 n, i64 m, out_t o) {
    double *hmin = (double *)malloc(sizeof(double) * m);
    if (!hmin) return ORC_NOMEM;
    for (i64 k = 0; k < m; k++) { hmin[k] = INFINITY; o.sig[k] = 0; }
    stream_t st;
    for (i64 e = 0; e < n; e++) {
        rng_seed(&st, ids[e]);
        double winv = 1.0 / w[e];
        for (i64 k = 0; k < m; k++) {
            double h = winv * exp1(&st);
            if (h < hmin[k]) { hmin[k] = h; o.sig[k] = ids[e]; }
        }
    }
    double hm = -INFINITY;
    for (i64 k = 0; k < m; k++) if (hmin[k] > hm) hm = hmin[k];
    if (o.hfinal) *o.hfinal = hm;
    o.stats[0] = n * m; o.stats[1] = 0; o.stats[2] = 0;
    free(hmin);
    return ORC_OK;
}

/* K:303-337 */
static int k_pmh1(const u64 *ids, const double *w, i64 n, i64 m, out_t o) {
    double *nodes = alloc_nodes(m);
    if (!nodes) return ORC_NOMEM;
    const double pin = o.pin; const int pinned = !isnan(pin);
    for (i64 k = 0; k < m; k++) o.sig[k] = 0;
    i64 root = 2 * m - 1;
    u64 m_u = (u64)m, kbits = bits_for(m);
    i64 cap = coupon_cap(m), points = 0, tw = 0;
    stream_t st;
    int rc = ORC_OK;
    for (i64 e = 0; e < n && rc == ORC_OK; e++) {
        rng_seed(&st, ids[e]);
        double winv = 1.0 / w[e];
        double x = winv * exp1(&st);
        points++;
        i64 cnt = 1;
        while (x < THR()) {
            i64 r = uniform_int_masked(&st, m_u, kbits);
            if (r < 0) { rc = ORC_RANDOMNESS_FAILURE; break; }
            i64 k = 1 + r;
            if (x < nodes[k]) {
                o.sig[k - 1] = ids[e];
                tw += tree_update(nodes, m, k, x);
                if (x >= THR()) break;
            }
            x += winv * exp1(&st);
            points++;
            cnt++;
            if (cnt > cap) { rc = ORC_RANDOMNESS_FAILURE; break; }
        }
    }
    if (o.hfinal) *o.hfinal = nodes[root];
    o.stats[0] = points; o.stats[1] = 0; o.stats[2] = tw;
    free(nodes);
    return rc;
}

/* K:340-405 */
static int k_pmh1a(const u64 *ids, const double *w, i64 n, i64 m, out_t o) {
    double *nodes = alloc_nodes(m);
    u64 *bid = (u64 *)malloc(sizeof(u64) * (n ? n : 1));
    double *bwinv = (double *)malloc(sizeof(double) * (n ? n : 1));
    double *bx = (double *)malloc(sizeof(double) * (n ? n : 1));
    stream_t *bst = (stream_t *)malloc(sizeof(stream_t) * (n ? n : 1));
    int rc = ORC_OK;
    if (!nodes || !bid || !bwinv || !bx || !bst) { rc = ORC_NOMEM; goto done; }
    const double pin = o.pin; const int pinned = !isnan(pin);
    for (i64 k = 0; k < m; k++) o.sig[k] = 0;
    i64 root = 2 * m - 1;
    u64 m_u = (u64)m, kbits = bits_for(m);
    i64 cap = coupon_cap(m), points = 0, tw = 0;
    stream_t st;
    i64 b = 0;
    for (i64 e = 0; e < n; e++) {
        rng_seed(&st, ids[e]);
        double winv = 1.0 / w[e];
        double x = winv * exp1(&st);
        points++;
        if (x >= THR()) continue;
        i64 r = uniform_int_masked(&st, m_u, kbits);
        if (r < 0) { rc = ORC_RANDOMNESS_FAILURE; goto done; }
        i64 k = 1 + r;
        if (x < nodes[k]) {
            o.sig[k - 1] = ids[e];
            tw += tree_update(nodes, m, k, x);
            if (x >= THR()) continue;
        }
        bid[b] = ids[e]; bwinv[b] = winv; bx[b] = x; bst[b] = st;
        b++;
    }
    i64 maxbuf = b, passes = 0;
    while (b > 0) {
        i64 b2 = 0;
        for (i64 j = 0; j < b; j++) {
            if (bx[j] >= THR()) continue;
            double x = bx[j] + bwinv[j] * exp1(&bst[j]);
            points++;
            if (x >= THR()) continue;
            i64 r = uniform_int_masked(&bst[j], m_u, kbits);
            if (r < 0) { rc = ORC_RANDOMNESS_FAILURE; goto done; }
            i64 k = 1 + r;
            if (x < nodes[k]) {
                o.sig[k - 1] = bid[j];
                tw += tree_update(nodes, m, k, x);
                if (x >= THR()) continue;
            }
            bid[b2] = bid[j]; bwinv[b2] = bwinv[j]; bx[b2] = x; bst[b2] = bst[j];
            b2++;
        }
        b = b2;
        passes++;
        if (passes > cap) { rc = ORC_RANDOMNESS_FAILURE; goto done; }
    }
    if (o.hfinal) *o.hfinal = nodes[root];
    o.stats[0] = points; o.stats[1] = maxbuf; o.stats[2] = tw;
done:
    free(nodes); free(bid); free(bwinv); free(bx); free(bst);
    return rc;
}

/* K:408-445 */
static int k_pmh2(const u64 *ids, const double *w, i64 n, i64 m, out_t o) {
    double *nodes = alloc_nodes(m);
    i64 *perm = (i64 *)calloc(m + 1, sizeof(i64));
    u64 *vers = (u64 *)calloc(m + 1, sizeof(u64));
    double *beta = (double *)malloc(sizeof(double) * (m + 1));
    int rc = ORC_OK;
    if (!nodes || !perm || !vers || !beta) { rc = ORC_NOMEM; goto done; }
    const double pin = o.pin; const int pinned = !isnan(pin);
    for (i64 k = 0; k < m; k++) o.sig[k] = 0;
    i64 root = 2 * m - 1;
    u64 counter = 0;
    for (i64 i = 2; i <= m; i++) beta[i] = (double)m / ((double)(m - i) + 1.0);
    i64 points = 0, tw = 0;
    stream_t st;
    for (i64 e = 0; e < n; e++) {
        rng_seed(&st, ids[e]);
        double winv = 1.0 / w[e];
        counter += 1;
        i64 i = 1;
        double x = winv * exp1(&st);
        points++;
        while (x < THR()) {
            i64 k = perm_next(&st, perm, vers, counter, i, m);
            if (k < 0) { rc = ORC_RANDOMNESS_FAILURE; goto done; }
            if (x < nodes[k]) {
                o.sig[k - 1] = ids[e];
                tw += tree_update(nodes, m, k, x);
                if (x >= THR()) break;
            }
            i++;
            if (i > m) break;
            x += winv * beta[i] * exp1(&st);
            points++;
        }
    }
    if (o.hfinal) *o.hfinal = nodes[root];
    o.stats[0] = points; o.stats[1] = 0; o.stats[2] = tw;
done:
    free(nodes); free(perm); free(vers); free(beta);
    return rc;
}

/* K:448-485 */
static int k_pmh3(const u64 *ids, const double *w, i64 n, i64 m, out_t o) {
    double *nodes = alloc_nodes(m);
    if (!nodes) return ORC_NOMEM;
    const double pin = o.pin; const int pinned = !isnan(pin);
    for (i64 k = 0; k < m; k++) o.sig[k] = 0;
    i64 root = 2 * m - 1;
    u64 m_u = (u64)m, kbits = bits_for(m);
    i64 cap = coupon_cap(m), points = 0, tw = 0;
    double lam = log1p(1.0 / ((double)m - 1.0)), c1, c2, c3;
    trunc_exp_consts(lam, &c1, &c2, &c3);
    stream_t st;
    int rc = ORC_OK, fail = 0;
    for (i64 e = 0; e < n && rc == ORC_OK; e++) {
        rng_seed(&st, ids[e]);
        double winv = 1.0 / w[e];
        double x = winv * trunc_exp(&st, lam, c1, c2, c3, &fail);
        if (fail) { rc = ORC_RANDOMNESS_FAILURE; break; }
        points++;
        i64 i = 1;
        while (x < THR()) {
            i64 r = uniform_int_masked(&st, m_u, kbits);
            if (r < 0) { rc = ORC_RANDOMNESS_FAILURE; break; }
            i64 k = 1 + r;
            if (x < nodes[k]) {
                o.sig[k - 1] = ids[e];
                tw += tree_update(nodes, m, k, x);
            }
            i++;
            if (i > cap) { rc = ORC_RANDOMNESS_FAILURE; break; }
            x = winv * ((double)i - 1.0);
            if (x >= THR()) break;
            x += winv * trunc_exp(&st, lam, c1, c2, c3, &fail);
            if (fail) { rc = ORC_RANDOMNESS_FAILURE; break; }
            points++;
        }
    }
    if (o.hfinal) *o.hfinal = nodes[root];
    o.stats[0] = points; o.stats[1] = 0; o.stats[2] = tw;
    free(nodes);
    return rc;
}

/* K:488-554 */
static int k_pmh3a(const u64 *ids, const double *w, i64 n, i64 m, out_t o) {
    double *nodes = alloc_nodes(m);
    u64 *bid = (u64 *)malloc(sizeof(u64) * (n ? n : 1));
    double *bwinv = (double *)malloc(sizeof(double) * (n ? n : 1));
    stream_t *bst = (stream_t *)malloc(sizeof(stream_t) * (n ? n : 1));
    int rc = ORC_OK, fail = 0;
    if (!nodes || !bid || !bwinv || !bst) { rc = ORC_NOMEM; goto done; }
    const double pin = o.pin; const int pinned = !isnan(pin);
    for (i64 k = 0; k < m; k++) o.sig[k] = 0;
    i64 root = 2 * m - 1;
    u64 m_u = (u64)m, kbits = bits_for(m);
    i64 cap = coupon_cap(m), points = 0, tw = 0;
    double lam = log1p(1.0 / ((double)m - 1.0)), c1, c2, c3;
    trunc_exp_consts(lam, &c1, &c2, &c3);
    stream_t st;
    i64 b = 0;
    for (i64 e = 0; e < n; e++) {
        rng_seed(&st, ids[e]);
        double winv = 1.0 / w[e];
        double x = winv * trunc_exp(&st, lam, c1, c2, c3, &fail);
        if (fail) { rc = ORC_RANDOMNESS_FAILURE; goto done; }
        points++;
        if (x >= THR()) continue;
        i64 r = uniform_int_masked(&st, m_u, kbits);
        if (r < 0) { rc = ORC_RANDOMNESS_FAILURE; goto done; }
        i64 k = 1 + r;
        if (x < nodes[k]) {
            o.sig[k - 1] = ids[e];
            tw += tree_update(nodes, m, k, x);
        }
        if (winv >= THR()) continue;
        bid[b] = ids[e]; bwinv[b] = winv; bst[b] = st;
        b++;
    }
    i64 maxbuf = b;
    i64 i = 2;
    while (b > 0) {
        i64 b2 = 0;
        for (i64 j = 0; j < b; j++) {
            double winv = bwinv[j];
            double x = winv * ((double)i - 1.0);
            if (x >= THR()) continue;
            x += winv * trunc_exp(&bst[j], lam, c1, c2, c3, &fail);
            if (fail) { rc = ORC_RANDOMNESS_FAILURE; goto done; }
            points++;
            if (x >= THR()) continue;
            i64 r = uniform_int_masked(&bst[j], m_u, kbits);
            if (r < 0) { rc = ORC_RANDOMNESS_FAILURE; goto done; }
            i64 k = 1 + r;
            if (x < nodes[k]) {
                o.sig[k - 1] = bid[j];
                tw += tree_update(nodes, m, k, x);
            }
            if (winv * (double)i >= THR()) continue;
            bid[b2] = bid[j]; bwinv[b2] = bwinv[j]; bst[b2] = bst[j];
            b2++;
        }
        b = b2;
        i++;
        if (i > cap) { rc = ORC_RANDOMNESS_FAILURE; goto done; }
    }
    if (o.hfinal) *o.hfinal = nodes[root];
    o.stats[0] = points; o.stats[1] = maxbuf; o.stats[2] = tw;
done:
    free(nodes); free(bid); free(bwinv); free(bst);
    return rc;
}

/* K:557-614 */
static int k_pmh4(const u64 *ids, const double *w, i64 n, i64 m, out_t o) {
    double *nodes = alloc_nodes(m);
    i64 *perm = (i64 *)calloc(m + 1, sizeof(i64));
    u64 *vers = (u64 *)calloc(m + 1, sizeof(u64));
    double *lam = (double *)malloc(sizeof(double) * m);
    double *tc1 = (double *)malloc(sizeof(double) * m);
    double *tc2 = (double *)malloc(sizeof(double) * m);
    double *tc3 = (double *)malloc(sizeof(double) * m);
    double *gam = (double *)malloc(sizeof(double) * m);
    int rc = ORC_OK, fail = 0;
    if (!nodes || !perm || !vers || !lam || !tc1 || !tc2 || !tc3 || !gam) {
        rc = ORC_NOMEM; goto done;
    }
    const double pin = o.pin; const int pinned = !isnan(pin);
    for (i64 k = 0; k < m; k++) o.sig[k] = 0;
    i64 root = 2 * m - 1;
    u64 counter = 0;
    gam[0] = 0.0;
    double lam1 = log1p(1.0 / ((double)m - 1.0));
    for (i64 i = 1; i < m; i++) {
        lam[i] = log1p(1.0 / (double)(m - i));
        trunc_exp_consts(lam[i], &tc1[i], &tc2[i], &tc3[i]);
        gam[i] = log1p((double)i / (double)(m - i)) / lam1;
    }
    double delta = 1.0 / lam1;
    i64 points = 0, tw = 0;
    stream_t st;
    for (i64 e = 0; e < n; e++) {
        rng_seed(&st, ids[e]);
        double winv = 1.0 / w[e];
        counter += 1;
        double x = winv * trunc_exp(&st, lam[1], tc1[1], tc2[1], tc3[1], &fail);
        if (fail) { rc = ORC_RANDOMNESS_FAILURE; goto done; }
        points++;
        i64 i = 1;
        while (x < THR()) {
            i64 k = perm_next(&st, perm, vers, counter, i, m);
            if (k < 0) { rc = ORC_RANDOMNESS_FAILURE; goto done; }
            if (x < nodes[k]) {
                o.sig[k - 1] = ids[e];
                tw += tree_update(nodes, m, k, x);
            }
            i++;
            if (winv * gam[i - 1] >= THR()) break;
            if (i < m) {
                double t = trunc_exp(&st, lam[i], tc1[i], tc2[i], tc3[i], &fail);
                if (fail) { rc = ORC_RANDOMNESS_FAILURE; goto done; }
                x = winv * (gam[i - 1] + (gam[i] - gam[i - 1]) * t);
                points++;
            } else {
                x = winv * (gam[m - 1] + delta * exp1(&st));
                points++;
                if (x < THR()) {
                    k = perm_next(&st, perm, vers, counter, m, m);
                    if (k < 0) { rc = ORC_RANDOMNESS_FAILURE; goto done; }
                    if (x < nodes[k]) {
                        o.sig[k - 1] = ids[e];
                        tw += tree_update(nodes, m, k, x);
                    }
                }
                break;
            }
        }
    }
    if (o.hfinal) *o.hfinal = nodes[root];
    o.stats[0] = points; o.stats[1] = 0; o.stats[2] = tw;
done:
    free(nodes); free(perm); free(vers); free(lam); free(tc1); free(tc2);
    free(tc3); free(gam);
    return rc;
}

/* K:619-653 */
static int k_uw3(const u64 *ids, i64 n, i64 m, out_t o) {
    double *nodes = alloc_nodes(m);
    if (!nodes) return ORC_NOMEM;
    const double pin = o.pin; const int pinned = !isnan(pin);
    for (i64 k = 0; k < m; k++) o.sig[k] = 0;
    i64 root = 2 * m - 1;
    u64 m_u = (u64)m, kbits = bits_for(m);
    i64 cap = coupon_cap(m), points = 0, tw = 0;
    stream_t st;
    int rc = ORC_OK;
    for (i64 e = 0; e < n && rc == ORC_OK; e++) {
        rng_seed(&st, ids[e]);
        double x = uniform01(&st);
        points++;
        i64 i = 1;
        while (x < THR()) {
            i64 r = uniform_int_masked(&st, m_u, kbits);
            if (r < 0) { rc = ORC_RANDOMNESS_FAILURE; break; }
            i64 k = 1 + r;
            if (x < nodes[k]) {
                o.sig[k - 1] = ids[e];
                tw += tree_update(nodes, m, k, x);
            }
            i++;
            if (i > cap) { rc = ORC_RANDOMNESS_FAILURE; break; }
            x = (double)i - 1.0;
            if (x >= THR()) break;
            x += uniform01(&st);
            points++;
        }
    }
    if (o.hfinal) *o.hfinal = nodes[root];
    o.stats[0] = points; o.stats[1] = 0; o.stats[2] = tw;
    free(nodes);
    return rc;
}

/* K:656-718 */
static int k_uw3a(const u64 *ids, i64 n, i64 m, out_t o) {
    double *nodes = alloc_nodes(m);
    u64 *bid = (u64 *)malloc(sizeof(u64) * (n ? n : 1));
    stream_t *bst = (stream_t *)malloc(sizeof(stream_t) * (n ? n : 1));
    int rc = ORC_OK;
    if (!nodes || !bid || !bst) { rc = ORC_NOMEM; goto done; }
    const double pin = o.pin; const int pinned = !isnan(pin);
    for (i64 k = 0; k < m; k++) o.sig[k] = 0;
    i64 root = 2 * m - 1;
    u64 m_u = (u64)m, kbits = bits_for(m);
    i64 cap = coupon_cap(m), points = 0, tw = 0;
    stream_t st;
    i64 b = 0;
    for (i64 e = 0; e < n; e++) {
        rng_seed(&st, ids[e]);
        double x = uniform01(&st);
        points++;
        if (x >= THR()) continue;
        i64 r = uniform_int_masked(&st, m_u, kbits);
        if (r < 0) { rc = ORC_RANDOMNESS_FAILURE; goto done; }
        i64 k = 1 + r;
        if (x < nodes[k]) {
            o.sig[k - 1] = ids[e];
            tw += tree_update(nodes, m, k, x);
        }
        if (1.0 >= THR()) continue;
        bid[b] = ids[e]; bst[b] = st;
        b++;
    }
    i64 maxbuf = b;
    i64 i = 2;
    while (b > 0) {
        i64 b2 = 0;
        for (i64 j = 0; j < b; j++) {
            double x = (double)i - 1.0;
            if (x >= THR()) continue;
            x += uniform01(&bst[j]);
            points++;
            if (x >= THR()) continue;
            i64 r = uniform_int_masked(&bst[j], m_u, kbits);
            if (r < 0) { rc = ORC_RANDOMNESS_FAILURE; goto done; }
            i64 k = 1 + r;
            if (x < nodes[k]) {
                o.sig[k - 1] = bid[j];
                tw += tree_update(nodes, m, k, x);
            }
            if ((double)i >= THR()) continue;
            bid[b2] = bid[j]; bst[b2] = bst[j];
            b2++;
        }
        b = b2;
        i++;
        if (i > cap) { rc = ORC_RANDOMNESS_FAILURE; goto done; }
    }
    if (o.hfinal) *o.hfinal = nodes[root];
    o.stats[0] = points; o.stats[1] = maxbuf; o.stats[2] = tw;
done:
    free(nodes); free(bid); free(bst);
    return rc;
}

/* K:721-763 */
static int k_uw4(const u64 *ids, i64 n, i64 m, out_t o) {
    double *nodes = alloc_nodes(m);
    i64 *perm = (i64 *)calloc(m + 1, sizeof(i64));
    u64 *vers = (u64 *)calloc(m + 1, sizeof(u64));
    int rc = ORC_OK;
    if (!nodes || !perm || !vers) { rc = ORC_NOMEM; goto done; }
    const double pin = o.pin; const int pinned = !isnan(pin);
    for (i64 k = 0; k < m; k++) o.sig[k] = 0;
    i64 root = 2 * m - 1;
    u64 counter = 0;
    i64 points = 0, tw = 0;
    stream_t st;
    for (i64 e = 0; e < n; e++) {
        rng_seed(&st, ids[e]);
        counter += 1;
        double x = uniform01(&st);
        points++;
        i64 i = 1;
        while (x < THR()) {
            i64 k = perm_next(&st, perm, vers, counter, i, m);
            if (k < 0) { rc = ORC_RANDOMNESS_FAILURE; goto done; }
            if (x < nodes[k]) {
                o.sig[k - 1] = ids[e];
                tw += tree_update(nodes, m, k, x);
            }
            i++;
            if ((double)i - 1.0 >= THR()) break;
            if (i < m) {
                x = ((double)i - 1.0) + uniform01(&st);
                points++;
            } else {
                x = ((double)m - 1.0) + uniform01(&st);
                points++;
                if (x < THR()) {
                    k = perm_next(&st, perm, vers, counter, m, m);
                    if (k < 0) { rc = ORC_RANDOMNESS_FAILURE; goto done; }
                    if (x < nodes[k]) {
                        o.sig[k - 1] = ids[e];
                        tw += tree_update(nodes, m, k, x);
                    }
                }
                break;
            }
        }
    }
    if (o.hfinal) *o.hfinal = nodes[root];
    o.stats[0] = points; o.stats[1] = 0; o.stats[2] = tw;
done:
    free(nodes); free(perm); free(vers);
    return rc;
}

/* ---- baselines K:768-846 ------------------------------------------------ */
static int k_minhash(const u64 *ids, i64 n, i64 m, u64 *sig) {
    double *hmin = (double *)malloc(sizeof(double) * m);
    if (!hmin) return ORC_NOMEM;
    for (i64 k = 0; k < m; k++) { hmin[k] = INFINITY; sig[k] = 0; }
    stream_t st;
    for (i64 e = 0; e < n; e++) {
        rng_seed(&st, ids[e]);
        for (i64 k = 0; k < m; k++) {
            double h = uniform01(&st);
            if (h < hmin[k]) { hmin[k] = h; sig[k] = ids[e]; }
        }
    }
    free(hmin);
    return ORC_OK;
}

static int k_superminhash(const u64 *ids, i64 n, i64 m, u64 *sig) {
    double *hmin = (double *)malloc(sizeof(double) * m);
    i64 *p = (i64 *)malloc(sizeof(i64) * m);
    int rc = ORC_OK;
    if (!hmin || !p) { rc = ORC_NOMEM; goto done; }
    for (i64 k = 0; k < m; k++) { hmin[k] = INFINITY; sig[k] = 0; }
    stream_t st;
    for (i64 e = 0; e < n; e++) {
        rng_seed(&st, ids[e]);
        for (i64 k = 0; k < m; k++) p[k] = k;
        for (i64 k = 0; k < m; k++) {
            double u = uniform01(&st);
            i64 r0 = uniform_int(&st, m - k);
            if (r0 < 0) { rc = ORC_RANDOMNESS_FAILURE; goto done; }
            i64 r = k + r0;
            i64 tmp = p[k]; p[k] = p[r]; p[r] = tmp;
            double h = u + (double)p[k];
            if (h < hmin[k]) { hmin[k] = h; sig[k] = ids[e]; }
        }
    }
done:
    free(hmin); free(p);
    return rc;
}

static int k_oph(const u64 *ids, i64 n, i64 m, u64 *sig) {
    double *hmin = (double *)malloc(sizeof(double) * m);
    unsigned char *filled = (unsigned char *)calloc(m, 1);
    int rc = ORC_OK;
    if (!hmin || !filled) { rc = ORC_NOMEM; goto done; }
    for (i64 k = 0; k < m; k++) { hmin[k] = INFINITY; sig[k] = 0; }
    u64 m_u = (u64)m, kbits = bits_for(m);
    i64 cap = coupon_cap(m);
    stream_t st;
    for (i64 e = 0; e < n; e++) {
        rng_seed(&st, ids[e]);
        i64 b = uniform_int_masked(&st, m_u, kbits);
        if (b < 0) { rc = ORC_RANDOMNESS_FAILURE; goto done; }
        double v = uniform01(&st);
        if (v < hmin[b]) { hmin[b] = v; sig[b] = ids[e]; filled[b] = 1; }
    }
    for (i64 k = 0; k < m; k++) {
        if (filled[k]) continue;
        rng_seed(&st, OPH_SALT + (u64)k * GOLDEN);
        i64 attempts = 0;
        for (;;) {
            i64 j = uniform_int_masked(&st, m_u, kbits);
            if (j < 0) { rc = ORC_RANDOMNESS_FAILURE; goto done; }
            if (filled[j]) { sig[k] = sig[j]; hmin[k] = hmin[j]; break; }
            attempts++;
            if (attempts > cap) { rc = ORC_RANDOMNESS_FAILURE; goto done; }
        }
    }
done:
    free(hmin); free(filled);
    return rc;
}

/* ---- public entry points ------------------------------------------------ */

/* One set.  weights may be NULL only for the unweighted-only algorithms
 * (uw3/3a/4 and the baselines); UW1/1A/2 use unit weights (sketch.py:200-207).
 * stats[3] = [points, max buffer, tree writes]; hfinal may be NULL.
 * pin = NAN for the reference behaviour.                                    */
int orc_sketch(int algo, const u64 *ids, const double *w, i64 n, i64 m,
               u64 *sig, i64 *stats, double *hfinal, double pin) {
    i64 dummy[3];
    out_t o = {sig, stats ? stats : dummy, hfinal, pin};
    double *ones = NULL;
    int rc;
    if ((algo == ALG_UW1 || algo == ALG_UW1A || algo == ALG_UW2) || !w) {
        if (algo <= ALG_PMH4 || algo == ALG_UW1 || algo == ALG_UW1A ||
            algo == ALG_UW2) {
            ones = (double *)malloc(sizeof(double) * (n ? n : 1));
            if (!ones) return ORC_NOMEM;
            for (i64 i = 0; i < n; i++) ones[i] = 1.0;
            w = ones;
        }
    }
    switch (algo) {
    case ALG_PMINHASH: rc = k_pminhash(ids, w, n, m, o); break;
    case ALG_PMH1: case ALG_UW1: rc = k_pmh1(ids, w, n, m, o); break;
    case ALG_PMH1A: case ALG_UW1A: rc = k_pmh1a(ids, w, n, m, o); break;
    case ALG_PMH2: case ALG_UW2: rc = k_pmh2(ids, w, n, m, o); break;
    case ALG_PMH3: rc = k_pmh3(ids, w, n, m, o); break;
    case ALG_PMH3A: rc = k_pmh3a(ids, w, n, m, o); break;
    case ALG_PMH4: rc = k_pmh4(ids, w, n, m, o); break;
    case ALG_UW3: rc = k_uw3(ids, n, m, o); break;
    case ALG_UW3A: rc = k_uw3a(ids, n, m, o); break;
    case ALG_UW4: rc = k_uw4(ids, n, m, o); break;
    case ALG_MINHASH: rc = k_minhash(ids, n, m, sig); memset(o.stats, 0, 24); break;
    case ALG_SUPERMINHASH: rc = k_superminhash(ids, n, m, sig); memset(o.stats, 0, 24); break;
    case ALG_OPH: rc = k_oph(ids, n, m, sig); memset(o.stats, 0, 24); break;
    default: rc = ORC_BAD_ALGO;
    }
    free(ones);
    return rc;
}

/* CSR batch over sets [s0, s1), single-threaded (the reference is
 * single-threaded; oracle.py fans disjoint set ranges out over host cores with
 * threads -- ctypes releases the GIL -- SURVEY.md §8d).  stats may be NULL.
 * Returns the first non-zero error code, or 0.                               */
int orc_sketch_csr(int algo, i64 m, const u64 *ids, const double *w,
                   const i64 *offsets, i64 s0, i64 s1, u64 *sig, i64 *stats) {
    for (i64 s = s0; s < s1; s++) {
        i64 a = offsets[s], b = offsets[s + 1];
        int rc = orc_sketch(algo, ids + a, w ? w + a : NULL, b - a, m,
                            sig + (s - s0) * m, stats ? stats + (s - s0) * 3 : NULL,
                            NULL, NAN);
        if (rc) return rc;
    }
    return 0;
}

/* P-MinHash (K:284-300) over one element range of a set, for the balanced
 * CPU baseline: folds elements [0, n) (global in-set indices e0 + e) into the
 * caller's running minima hmin[m] / idx[m] (init +inf / -1).  P-MinHash is
 * order-independent: the reference's strict `<` in element order keeps the
 * lexicographic minimum of (h, index), so parts merged on (h, index) give
 * exactly the sequential signature.                                          */
void orc_pminhash_part(const u64 *ids, const double *w, i64 n, i64 m, i64 e0,
                       double *hmin, i64 *idx) {
    stream_t st;
    for (i64 e = 0; e < n; e++) {
        rng_seed(&st, ids[e]);
        double winv = 1.0 / w[e];
        for (i64 k = 0; k < m; k++) {
            double h = winv * exp1(&st);
            if (h < hmin[k]) { hmin[k] = h; idx[k] = e0 + e; }
        }
    }
}

/* b-bit reduction K:851-861 */
void orc_bbit(const u64 *sig, i64 m, int b, i64 *out) {
    u64 mask = (1ULL << (u64)b) - 1ULL;
    for (i64 i = 0; i < m; i++)
        out[i] = (i64)(mix64(sig[i] + GOLDEN * (u64)(i + 1)) & mask);
}

/* equal-component counts (estimate.py:91-95 numerator) */
void orc_count_equal(const u64 *a, const u64 *b, i64 npairs, i64 m, int32_t *cnt) {
    for (i64 p = 0; p < npairs; p++) {
        int32_t c = 0;
        for (i64 k = 0; k < m; k++) c += a[p * m + k] == b[p * m + k];
        cnt[p] = c;
    }
}

/* all-pairs upper triangle counts for rows [r0,r1) x cols (row, n) */
void orc_allpairs(const u64 *sigs, i64 n, i64 m, i64 r0, i64 r1, int32_t *out) {
    /* out is (r1-r0) x n dense, lower part untouched */
    for (i64 i = r0; i < r1; i++)
        for (i64 j = i + 1; j < n; j++) {
            int32_t c = 0;
            for (i64 k = 0; k < m; k++) c += sigs[i * m + k] == sigs[j * m + k];
            out[(i - r0) * n + j] = c;
        }
}

/* raw stream primitives for unit tests of the restatement */
void orc_stream_words(u64 seed, i64 count, u64 *out) {
    stream_t st; rng_seed(&st, seed);
    for (i64 i = 0; i < count; i++) out[i] = next_u64(&st);
}
void orc_stream_uniform01(u64 seed, i64 count, double *out) {
    stream_t st; rng_seed(&st, seed);
    for (i64 i = 0; i < count; i++) out[i] = uniform01(&st);
}
void orc_stream_exp1(u64 seed, i64 count, double *out) {
    stream_t st; rng_seed(&st, seed);
    for (i64 i = 0; i < count; i++) out[i] = exp1(&st);
}
int orc_stream_trunc_exp(u64 seed, double lam, i64 count, double *out) {
    stream_t st; rng_seed(&st, seed);
    double c1, c2, c3; int fail = 0;
    trunc_exp_consts(lam, &c1, &c2, &c3);
    for (i64 i = 0; i < count; i++) {
        out[i] = trunc_exp(&st, lam, c1, c2, c3, &fail);
        if (fail) return ORC_RANDOMNESS_FAILURE;
    }
    return 0;
}
/* Fill a stream-generated synthetic batch helper: u64 words (u64_batch) */
void orc_trunc_exp_consts(double lam, double *c) { trunc_exp_consts(lam, c, c + 1, c + 2); }
