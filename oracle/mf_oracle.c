/*
 * mf_oracle.c -- CPU restatement of the reference decimation / pooling path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product package links or calls
 * this file; it is loaded by tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg (as the checker / the CPU timing arm), never as a fallback.
 *
 * It restates, with explicit scalar loops, the numpy algorithm of the
 * reference package `meshforge` (/root/reference/pkg/src/meshforge):
 *
 *   facet geometry            mesh.py:72-88
 *   facet / vertex quadrics   quadrics.py:36-45, 61-77
 *   unique edge list          mesh.py:125-134
 *   pair costs                quadrics.py:53-58, 117-132
 *   sorted pair order         decimate.py:181-191 (incl. PCG64 shuffle keys)
 *   greedy pairing            decimate.py:248-263
 *   leftover absorption       decimate.py:194-226
 *   output order              decimate.py:130-137
 *   contraction + output      decimate.py:140-169, 275-291
 *   round chain               decimate.py:294-316
 *   pool / unpool             pooling.py:36-77
 *   'inverse' placement       quadrics.py:89-114, decimate.py:284-286 (mf_inverse.h;
 *                             tolerance-only vs LAPACK, see that header)
 *
 * Floating-point order follows the numpy calls bit for bit:
 * products and sums are separately rounded (compile with -ffp-contract=off),
 * `np.add.at` is a sequential fold in index order, and the two einsum
 * reductions use the order selected by `einsum_order`:
 *   0 = SIMD lane-split order numpy 2.3 uses on AVX-512 hosts:
 *       dot3(u,v) = (u0*v0 + u2*v2) + u1*v1
 *   1 = plain sequential order ((u0*v0 + u1*v1) + u2*v2)
 * The 9-term quadratic form of Quadric.evaluate is a row-major sequential
 * fold on both.
 *
 * Parity of this restatement against the reference is pinned by
 * tests/test_oracle_golden.py against fixtures produced by
 * tests/golden/make_golden.py from the real reference.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "mf_oracle.h"
#include "mf_inverse.h"

/* ------------------------------------------------------------------ */
/* small helpers                                                        */

static void *xmalloc(size_t n) {
    void *p = malloc(n ? n : 1);
    if (!p) abort();
    return p;
}
static void *xcalloc(size_t n, size_t s) {
    void *p = calloc(n ? n : 1, s ? s : 1);
    if (!p) abort();
    return p;
}

static double dot3(const double *u, const double *v, int order) {
    if (order == 0) return (u[0] * v[0] + u[2] * v[2]) + u[1] * v[1];
    return (u[0] * v[0] + u[1] * v[1]) + u[2] * v[2];
}

/* numpy comparison of float64 inside lexsort: NaN sorts last. */
static int cmp_f64(double a, double b) {
    int na = isnan(a), nb = isnan(b);
    if (na || nb) return na - nb;
    return (a < b) ? -1 : (a > b) ? 1 : 0;
}
static int cmp_i64(int64_t a, int64_t b) { return (a < b) ? -1 : (a > b) ? 1 : 0; }

/* generic stable merge sort of int64 indices with a context comparator */
typedef int (*cmp_fn)(const void *ctx, int64_t a, int64_t b);

static void msort_rec(int64_t *a, int64_t *tmp, int64_t n, cmp_fn cmp, const void *ctx) {
    if (n < 2) return;
    if (n <= 16) {
        for (int64_t i = 1; i < n; i++) {
            int64_t x = a[i], j = i - 1;
            while (j >= 0 && cmp(ctx, a[j], x) > 0) { a[j + 1] = a[j]; j--; }
            a[j + 1] = x;
        }
        return;
    }
    int64_t h = n / 2;
    msort_rec(a, tmp, h, cmp, ctx);
    msort_rec(a + h, tmp, n - h, cmp, ctx);
    int64_t i = 0, j = h, k = 0;
    while (i < h && j < n) tmp[k++] = (cmp(ctx, a[j], a[i]) < 0) ? a[j++] : a[i++];
    while (i < h) tmp[k++] = a[i++];
    while (j < n) tmp[k++] = a[j++];
    memcpy(a, tmp, (size_t)n * sizeof(int64_t));
}
static void stable_sort_idx(int64_t *idx, int64_t n, cmp_fn cmp, const void *ctx) {
    int64_t *tmp = (int64_t *)xmalloc((size_t)n * sizeof(int64_t));
    msort_rec(idx, tmp, n, cmp, ctx);
    free(tmp);
}

/* ------------------------------------------------------------------ */
/* PCG64 (numpy default_rng bit generator), XSL-RR 128/64               */

typedef struct { uint64_t hi, lo; } u128;

static u128 mul128(u128 a, u128 b) {
    unsigned __int128 x = ((unsigned __int128)a.hi << 64) | a.lo;
    unsigned __int128 y = ((unsigned __int128)b.hi << 64) | b.lo;
    unsigned __int128 z = x * y;
    u128 r = {(uint64_t)(z >> 64), (uint64_t)z};
    return r;
}
static u128 add128(u128 a, u128 b) {
    unsigned __int128 x = ((unsigned __int128)a.hi << 64) | a.lo;
    unsigned __int128 y = ((unsigned __int128)b.hi << 64) | b.lo;
    unsigned __int128 z = x + y;
    u128 r = {(uint64_t)(z >> 64), (uint64_t)z};
    return r;
}
static const u128 PCG_MULT = {0x2360ED051FC65DA4ULL, 0x4385DF649FCCF645ULL};

/* rng.random(n): key k = (out_{k} >> 11) * 2^-53, out_k = XSL-RR of the
 * state after k+1 LCG steps (numpy pcg64 next64 / next_double). */
static void pcg64_random(const uint64_t pcg[4], int64_t n, double *out) {
    u128 s = {pcg[0], pcg[1]}, inc = {pcg[2], pcg[3]};
    for (int64_t k = 0; k < n; k++) {
        s = add128(mul128(s, PCG_MULT), inc);
        uint64_t x = s.hi ^ s.lo;
        unsigned rot = (unsigned)(s.hi >> 58);
        uint64_t r = (x >> rot) | (x << ((64 - rot) & 63));
        out[k] = (double)(r >> 11) * (1.0 / 9007199254740992.0);
    }
}

/* ------------------------------------------------------------------ */
/* round chain -- decimate.py:294-316                                  */

int64_t mfo_round_targets(int64_t n_in, int64_t target, int64_t rounds, int64_t *chain, int64_t cap) {
    int64_t len = 0;
    if (rounds < 0) { /* 'auto' */
        int64_t cur = n_in;
        while ((cur + 1) / 2 > target) {
            cur = (cur + 1) / 2;
            if (len < cap) chain[len] = cur;
            len++;
        }
        if (len < cap) chain[len] = target;
        return len + 1;
    }
    if (rounds == 1) {
        if (cap > 0) chain[0] = target;
        return 1;
    }
    double ratio = pow((double)target / (double)n_in, 1.0 / (double)rounds);
    int64_t cur = n_in;
    for (int64_t r = 1; r < rounds; r++) {
        double v = (double)n_in * pow(ratio, (double)r);
        int64_t step = (int64_t)ceil(v);
        if (step < target) step = target;
        if (step > cur) step = cur;
        if (len < cap) chain[len] = step;
        len++;
        cur = step;
    }
    if (len < cap) chain[len] = target;
    return len + 1;
}

/* ------------------------------------------------------------------ */
/* one mesh                                                             */

typedef struct {
    int64_t n, m, c;
    double *P;  /* n*3 */
    int64_t *F; /* m*3 */
    double *X;  /* n*c */
} omesh;

static void omesh_free(omesh *a) {
    free(a->P); free(a->F); free(a->X);
    a->P = NULL; a->F = NULL; a->X = NULL;
}

/* ---- vertex quadrics: quadrics.py:36-45, 61-77 + mesh.py:72-88 ---- */
/* Q layout per vertex: a[9] row-major, b[3], c  (13 doubles) */
#define QW 13

static void facet_planes(const omesh *g, int order, double *plane /* m*4: n0 n1 n2 d */, uint8_t *degen) {
    for (int64_t f = 0; f < g->m; f++) {
        const double *v0 = g->P + 3 * g->F[3 * f + 0];
        const double *v1 = g->P + 3 * g->F[3 * f + 1];
        const double *v2 = g->P + 3 * g->F[3 * f + 2];
        double a[3] = {v1[0] - v0[0], v1[1] - v0[1], v1[2] - v0[2]};
        double b[3] = {v2[0] - v0[0], v2[1] - v0[1], v2[2] - v0[2]};
        double cr[3];
        cr[0] = a[1] * b[2] - a[2] * b[1];
        cr[1] = a[2] * b[0] - a[0] * b[2];
        cr[2] = a[0] * b[1] - a[1] * b[0];
        double nrm = sqrt((cr[0] * cr[0] + cr[1] * cr[1]) + cr[2] * cr[2]);
        double nn[3] = {0.0, 0.0, 0.0};
        int dg = (nrm == 0.0);
        if (!dg) { nn[0] = cr[0] / nrm; nn[1] = cr[1] / nrm; nn[2] = cr[2] / nrm; }
        double d = -dot3(nn, v0, order);
        plane[4 * f + 0] = nn[0]; plane[4 * f + 1] = nn[1]; plane[4 * f + 2] = nn[2];
        plane[4 * f + 3] = d;
        degen[f] = (uint8_t)dg;
    }
}

static void vertex_quadrics(const omesh *g, int order, double *Q /* n*QW */) {
    double *plane = (double *)xmalloc((size_t)g->m * 4 * sizeof(double));
    uint8_t *degen = (uint8_t *)xmalloc((size_t)g->m);
    facet_planes(g, order, plane, degen);
    memset(Q, 0, (size_t)g->n * QW * sizeof(double));
    for (int corner = 0; corner < 3; corner++) {
        for (int64_t f = 0; f < g->m; f++) {
            double *q = Q + QW * g->F[3 * f + corner];
            const double *p = plane + 4 * f;
            double d = p[3];
            for (int r = 0; r < 3; r++)
                for (int c = 0; c < 3; c++) q[3 * r + c] += p[r] * p[c];
            for (int r = 0; r < 3; r++) q[9 + r] += d * p[r];
            q[12] += degen[f] ? 0.0 : d * d;
        }
    }
    free(plane); free(degen);
}

static void q13_a6(const double *q, double a6[6]) {
    a6[0] = q[0]; a6[1] = q[1]; a6[2] = q[2]; a6[3] = q[4]; a6[4] = q[5]; a6[5] = q[8];
}

/* Quadric.evaluate (quadrics.py:53-58) of Q at x */
static double q_evaluate(const double *a, const double *b, double c, const double *x, int order) {
    double quad = 0.0;
    for (int r = 0; r < 3; r++)
        for (int k = 0; k < 3; k++) quad = quad + (x[r] * a[3 * r + k]) * x[k];
    double lin = 2.0 * dot3(b, x, order);
    return (quad + lin) + c;
}

/* ---- edge_list: mesh.py:125-134 ---- */
static int cmp_pair(const void *pa, const void *pb) {
    const int64_t *a = (const int64_t *)pa, *b = (const int64_t *)pb;
    int r = cmp_i64(a[0], b[0]);
    return r ? r : cmp_i64(a[1], b[1]);
}
static int64_t edge_list(const omesh *g, int64_t **out) {
    int64_t *raw = (int64_t *)xmalloc((size_t)g->m * 6 * sizeof(int64_t));
    static const int pr[3][2] = {{0, 1}, {1, 2}, {2, 0}};
    for (int s = 0; s < 3; s++)
        for (int64_t f = 0; f < g->m; f++) {
            int64_t i = g->F[3 * f + pr[s][0]], j = g->F[3 * f + pr[s][1]];
            int64_t *e = raw + 2 * (s * g->m + f);
            e[0] = i < j ? i : j;
            e[1] = i < j ? j : i;
        }
    int64_t total = 3 * g->m;
    qsort(raw, (size_t)total, 2 * sizeof(int64_t), cmp_pair);
    int64_t e = 0;
    for (int64_t k = 0; k < total; k++) {
        if (e > 0 && raw[2 * k] == raw[2 * (e - 1)] && raw[2 * k + 1] == raw[2 * (e - 1) + 1]) continue;
        raw[2 * e] = raw[2 * k]; raw[2 * e + 1] = raw[2 * k + 1];
        e++;
    }
    *out = raw;
    return e;
}

/* ---- sort contexts ---- */
typedef struct { const double *cost; const int64_t *E; } ctx_plain;
static int cmp_plain(const void *c, int64_t a, int64_t b) {
    const ctx_plain *x = (const ctx_plain *)c;
    int r = cmp_f64(x->cost[a], x->cost[b]);
    if (r) return r;
    r = cmp_i64(x->E[2 * a], x->E[2 * b]);
    if (r) return r;
    return cmp_i64(x->E[2 * a + 1], x->E[2 * b + 1]);
}
typedef struct { const int64_t *bucket; const double *key; } ctx_seed;
static int cmp_seed(const void *c, int64_t a, int64_t b) {
    const ctx_seed *x = (const ctx_seed *)c;
    int r = cmp_i64(x->bucket[a], x->bucket[b]);
    if (r) return r;
    return cmp_f64(x->key[a], x->key[b]);
}
/* absorb grouping: lexsort((target_rep, edge_cost, loose)) */
typedef struct { const int64_t *loose, *rep; const double *cost; } ctx_abs;
static int cmp_abs_group(const void *c, int64_t a, int64_t b) {
    const ctx_abs *x = (const ctx_abs *)c;
    int r = cmp_i64(x->loose[a], x->loose[b]);
    if (r) return r;
    r = cmp_f64(x->cost[a], x->cost[b]);
    if (r) return r;
    return cmp_i64(x->rep[a], x->rep[b]);
}
/* lexsort((loose, target_rep, edge_cost)) */
static int cmp_abs_order(const void *c, int64_t a, int64_t b) {
    const ctx_abs *x = (const ctx_abs *)c;
    int r = cmp_f64(x->cost[a], x->cost[b]);
    if (r) return r;
    r = cmp_i64(x->rep[a], x->rep[b]);
    if (r) return r;
    return cmp_i64(x->loose[a], x->loose[b]);
}
/* dedupe: lexicographic on sorted triple */
typedef struct { const int64_t *key; } ctx_tri;
static int cmp_tri(const void *c, int64_t a, int64_t b) {
    const ctx_tri *x = (const ctx_tri *)c;
    for (int k = 0; k < 3; k++) {
        int r = cmp_i64(x->key[3 * a + k], x->key[3 * b + k]);
        if (r) return r;
    }
    return 0;
}

/* ---- _absorb_leftovers: decimate.py:194-226 ---- */
static int64_t absorb_leftovers(int64_t *cluster, int64_t n, int64_t seeded_count, const int64_t *E, int64_t ne,
                                const double *cost, int64_t budget, int64_t removed) {
    int64_t *rep = (int64_t *)xmalloc((size_t)seeded_count * sizeof(int64_t));
    for (int64_t k = 0; k < seeded_count; k++) rep[k] = n;
    for (int64_t v = 0; v < n; v++)
        if (cluster[v] >= 0 && v < rep[cluster[v]]) rep[cluster[v]] = v;
    int64_t *loose = (int64_t *)xmalloc((size_t)ne * sizeof(int64_t));
    int64_t *target = (int64_t *)xmalloc((size_t)ne * sizeof(int64_t));
    int64_t *trep = (int64_t *)xmalloc((size_t)ne * sizeof(int64_t));
    double *ecost = (double *)xmalloc((size_t)ne * sizeof(double));
    int64_t *grp = (int64_t *)xmalloc((size_t)ne * sizeof(int64_t));
    int64_t *best = (int64_t *)xmalloc((size_t)ne * sizeof(int64_t));
    while (removed < budget) {
        int64_t h = 0;
        for (int64_t e = 0; e < ne; e++) {
            int64_t c0 = cluster[E[2 * e]], c1 = cluster[E[2 * e + 1]];
            if ((c0 < 0) == (c1 < 0)) continue;
            loose[h] = c0 < 0 ? E[2 * e] : E[2 * e + 1];
            target[h] = c0 < 0 ? c1 : c0;
            ecost[h] = cost[e];
            trep[h] = rep[target[h]];
            h++;
        }
        if (h == 0) break;
        for (int64_t k = 0; k < h; k++) grp[k] = k;
        ctx_abs cx = {loose, trep, ecost};
        stable_sort_idx(grp, h, cmp_abs_group, &cx);
        int64_t nb = 0;
        for (int64_t k = 0; k < h; k++)
            if (k == 0 || loose[grp[k]] != loose[grp[k - 1]]) best[nb++] = grp[k];
        stable_sort_idx(best, nb, cmp_abs_order, &cx);
        int64_t take = budget - removed;
        if (take > nb) take = nb;
        for (int64_t k = 0; k < take; k++) cluster[loose[best[k]]] = target[best[k]];
        for (int64_t k = 0; k < take; k++) {
            int64_t t = target[best[k]], l = loose[best[k]];
            if (l < rep[t]) rep[t] = l;
        }
        removed += take;
    }
    free(rep); free(loose); free(target); free(trep); free(ecost); free(grp); free(best);
    return removed;
}

/* ---- _output_order: decimate.py:130-137 ---- */
static void output_order(const int64_t *cluster_ids, int64_t n, int64_t n_clusters, int64_t *replace) {
    int64_t *rep = (int64_t *)xmalloc((size_t)n_clusters * sizeof(int64_t));
    for (int64_t k = 0; k < n_clusters; k++) rep[k] = n;
    for (int64_t v = 0; v < n; v++)
        if (v < rep[cluster_ids[v]]) rep[cluster_ids[v]] = v;
    /* reps are distinct vertex ids: the rank of rep[k] among reps is the
     * output index; a vertex v is a rep iff rep[cluster(v)] == v */
    int64_t *out_of_vertex = (int64_t *)xmalloc((size_t)(n + 1) * sizeof(int64_t));
    int64_t r = 0;
    for (int64_t v = 0; v < n; v++) {
        out_of_vertex[v] = r;
        if (rep[cluster_ids[v]] == v) r++;
    }
    for (int64_t v = 0; v < n; v++) replace[v] = out_of_vertex[rep[cluster_ids[v]]];
    free(rep); free(out_of_vertex);
}

/* ---- _build_output: decimate.py:140-169 ---- */
static void build_output(const omesh *g, const int64_t *replace, int64_t n_out, double *Pout, omesh *out,
                         int64_t *mapping) {
    int64_t c = g->c;
    int64_t *counts = (int64_t *)xcalloc((size_t)n_out, sizeof(int64_t));
    for (int64_t v = 0; v < g->n; v++) counts[replace[v]]++;
    double *X = (double *)xcalloc((size_t)(n_out * c), sizeof(double));
    for (int64_t v = 0; v < g->n; v++)
        for (int64_t k = 0; k < c; k++) X[replace[v] * c + k] += g->X[v * c + k];
    for (int64_t r = 0; r < n_out; r++)
        for (int64_t k = 0; k < c; k++) X[r * c + k] /= (double)counts[r];

    int64_t m = g->m;
    int64_t *mapped = (int64_t *)xmalloc((size_t)m * 3 * sizeof(int64_t));
    uint8_t *degen = (uint8_t *)xmalloc((size_t)m);
    int64_t nlive = 0;
    for (int64_t f = 0; f < m; f++) {
        int64_t a = replace[g->F[3 * f]], b = replace[g->F[3 * f + 1]], d = replace[g->F[3 * f + 2]];
        degen[f] = (a == b) || (b == d) || (a == d);
        if (!degen[f]) {
            mapped[3 * nlive] = a; mapped[3 * nlive + 1] = b; mapped[3 * nlive + 2] = d;
            nlive++;
        }
    }
    int64_t *Fout = (int64_t *)xmalloc((size_t)(nlive * 3) * sizeof(int64_t));
    int64_t mout = 0;
    if (nlive) {
        int64_t *key = (int64_t *)xmalloc((size_t)nlive * 3 * sizeof(int64_t));
        for (int64_t f = 0; f < nlive; f++) {
            int64_t a = mapped[3 * f], b = mapped[3 * f + 1], d = mapped[3 * f + 2], t;
            if (a > b) { t = a; a = b; b = t; }
            if (b > d) { t = b; b = d; d = t; }
            if (a > b) { t = a; a = b; b = t; }
            key[3 * f] = a; key[3 * f + 1] = b; key[3 * f + 2] = d;
        }
        int64_t *idx = (int64_t *)xmalloc((size_t)nlive * sizeof(int64_t));
        for (int64_t f = 0; f < nlive; f++) idx[f] = f;
        ctx_tri cx = {key};
        stable_sort_idx(idx, nlive, cmp_tri, &cx);
        uint8_t *keep = (uint8_t *)xcalloc((size_t)nlive, 1);
        for (int64_t k = 0; k < nlive; k++)
            if (k == 0 || cmp_tri(&cx, idx[k], idx[k - 1]) != 0) keep[idx[k]] = 1;
        for (int64_t f = 0; f < nlive; f++)
            if (keep[f]) {
                Fout[3 * mout] = mapped[3 * f]; Fout[3 * mout + 1] = mapped[3 * f + 1];
                Fout[3 * mout + 2] = mapped[3 * f + 2];
                mout++;
            }
        free(key); free(idx); free(keep);
    }
    uint8_t *had = (uint8_t *)xcalloc((size_t)g->n, 1), *live = (uint8_t *)xcalloc((size_t)g->n, 1);
    for (int64_t f = 0; f < m; f++)
        for (int k = 0; k < 3; k++) {
            had[g->F[3 * f + k]] = 1;
            if (!degen[f]) live[g->F[3 * f + k]] = 1;
        }
    for (int64_t v = 0; v < g->n; v++) mapping[v] = (had[v] && !live[v]) ? -1 : replace[v];
    out->n = n_out; out->m = mout; out->c = c;
    out->P = Pout; out->F = Fout; out->X = X;
    free(counts); free(mapped); free(degen); free(had); free(live);
}

/* ---- _decimate_round: decimate.py:229-291 ('average' placement) ---- */
static int decimate_round(const omesh *g, int64_t target, int seeded, const uint64_t pcg[4], int order,
                          int placement, omesh *out, int64_t *replace, int64_t *mapping, int64_t *achievable) {
    int64_t n = g->n;
    if (target == n) { /* _identity_result */
        out->n = n; out->m = g->m; out->c = g->c;
        out->P = (double *)xmalloc((size_t)n * 3 * sizeof(double));
        out->F = (int64_t *)xmalloc((size_t)g->m * 3 * sizeof(int64_t));
        out->X = (double *)xmalloc((size_t)(n * g->c) * sizeof(double));
        memcpy(out->P, g->P, (size_t)n * 3 * sizeof(double));
        memcpy(out->F, g->F, (size_t)g->m * 3 * sizeof(int64_t));
        memcpy(out->X, g->X, (size_t)(n * g->c) * sizeof(double));
        for (int64_t v = 0; v < n; v++) replace[v] = mapping[v] = v;
        return 0;
    }
    int64_t budget = n - target;
    double *Q = (double *)xmalloc((size_t)n * QW * sizeof(double));
    vertex_quadrics(g, order, Q);
    int64_t *E = NULL;
    int64_t ne = edge_list(g, &E);
    if (ne == 0) {
        free(Q); free(E);
        *achievable = n;
        return MFO_INFEASIBLE;
    }
    double *cost = (double *)xmalloc((size_t)ne * sizeof(double));
    for (int64_t e = 0; e < ne; e++) {
        const double *qi = Q + QW * E[2 * e], *qj = Q + QW * E[2 * e + 1];
        double q[QW];
        for (int k = 0; k < QW; k++) q[k] = qi[k] + qj[k];
        const double *pi = g->P + 3 * E[2 * e], *pj = g->P + 3 * E[2 * e + 1];
        double x[3] = {0.5 * (pi[0] + pj[0]), 0.5 * (pi[1] + pj[1]), 0.5 * (pi[2] + pj[2])};
        if (placement) { /* optimal_positions(q, midpoints, 'inverse'), quadrics.py:131 */
            double a6[6], t[3];
            q13_a6(q, a6);
            mf_optimal_position(a6, q + 9, x, t);
            x[0] = t[0]; x[1] = t[1]; x[2] = t[2];
        }
        cost[e] = q_evaluate(q, q + 9, q[12], x, order);
    }
    int64_t *ord = (int64_t *)xmalloc((size_t)ne * sizeof(int64_t));
    for (int64_t e = 0; e < ne; e++) ord[e] = e;
    if (!seeded) {
        ctx_plain cx = {cost, E};
        stable_sort_idx(ord, ne, cmp_plain, &cx);
    } else {
        double lo = cost[0], hi = cost[0];
        for (int64_t e = 1; e < ne; e++) {
            /* np.min / np.max propagate NaN */
            if (isnan(cost[e]) || cost[e] < lo) lo = isnan(lo) ? lo : cost[e];
            if (isnan(cost[e]) || cost[e] > hi) hi = isnan(hi) ? hi : cost[e];
        }
        double width = 1e-12 * (hi - lo);
        int64_t *bucket = (int64_t *)xmalloc((size_t)ne * sizeof(int64_t));
        for (int64_t e = 0; e < ne; e++) bucket[e] = (width > 0.0) ? (int64_t)floor((cost[e] - lo) / width) : 0;
        double *key = (double *)xmalloc((size_t)ne * sizeof(double));
        pcg64_random(pcg, ne, key);
        ctx_seed cx = {bucket, key};
        stable_sort_idx(ord, ne, cmp_seed, &cx);
        free(bucket); free(key);
    }
    /* greedy scan: decimate.py:251-263 */
    int64_t *cluster = (int64_t *)xmalloc((size_t)n * sizeof(int64_t));
    for (int64_t v = 0; v < n; v++) cluster[v] = -1;
    int64_t next_id = 0, removed = 0;
    for (int64_t k = 0; k < ne; k++) {
        if (removed == budget) break;
        int64_t i = E[2 * ord[k]], j = E[2 * ord[k] + 1];
        if (cluster[i] < 0 && cluster[j] < 0) {
            cluster[i] = cluster[j] = next_id++;
            removed++;
        }
    }
    if (removed < budget && next_id > 0)
        removed = absorb_leftovers(cluster, n, next_id, E, ne, cost, budget, removed);
    free(ord);
    if (removed < budget) {
        free(Q); free(E); free(cost); free(cluster);
        *achievable = n - removed;
        return MFO_INFEASIBLE;
    }
    int64_t nc = next_id;
    for (int64_t v = 0; v < n; v++)
        if (cluster[v] < 0) cluster[v] = nc++;
    output_order(cluster, n, nc, replace);
    /* contraction by member mean: decimate.py:280-283 */
    int64_t *counts = (int64_t *)xcalloc((size_t)nc, sizeof(int64_t));
    double *Pout = (double *)xcalloc((size_t)nc * 3, sizeof(double));
    for (int64_t v = 0; v < n; v++) {
        counts[replace[v]]++;
        for (int k = 0; k < 3; k++) Pout[3 * replace[v] + k] += g->P[3 * v + k];
    }
    for (int64_t r = 0; r < nc; r++)
        for (int k = 0; k < 3; k++) Pout[3 * r + k] = Pout[3 * r + k] / (double)counts[r];
    if (placement) { /* accumulate_quadrics + optimal_positions(..., 'inverse'), decimate.py:284-286 */
        double *Qc = (double *)xcalloc((size_t)nc * QW, sizeof(double));
        for (int64_t v = 0; v < n; v++)
            for (int k = 0; k < QW; k++) Qc[QW * replace[v] + k] += Q[QW * v + k];
        for (int64_t r = 0; r < nc; r++) {
            double a6[6], t[3];
            q13_a6(Qc + QW * r, a6);
            mf_optimal_position(a6, Qc + QW * r + 9, Pout + 3 * r, t);
            Pout[3 * r] = t[0]; Pout[3 * r + 1] = t[1]; Pout[3 * r + 2] = t[2];
        }
        free(Qc);
    }
    build_output(g, replace, nc, Pout, out, mapping);
    free(counts); free(Q); free(E); free(cost); free(cluster);
    return 0;
}

/* ---- decimate_parallel for one mesh: decimate.py:363-382 ---- */
int mfo_decimate_mesh(const double *P, int64_t n, const int64_t *F, int64_t m, const double *X, int64_t c,
                      const int64_t *chain, int64_t nchain, int seeded, const uint64_t pcg[4], int order,
                      int placement, mfo_result **res_out, int64_t *achievable) {
    omesh cur;
    cur.n = n; cur.m = m; cur.c = c;
    cur.P = (double *)xmalloc((size_t)n * 3 * sizeof(double));
    cur.F = (int64_t *)xmalloc((size_t)m * 3 * sizeof(int64_t));
    cur.X = (double *)xmalloc((size_t)(n * c) * sizeof(double));
    memcpy(cur.P, P, (size_t)n * 3 * sizeof(double));
    memcpy(cur.F, F, (size_t)m * 3 * sizeof(int64_t));
    memcpy(cur.X, X, (size_t)(n * c) * sizeof(double));
    int64_t *replace = (int64_t *)xmalloc((size_t)n * sizeof(int64_t));
    int64_t *mapping = (int64_t *)xmalloc((size_t)n * sizeof(int64_t));
    for (int64_t v = 0; v < n; v++) replace[v] = mapping[v] = v;
    int64_t *sr = (int64_t *)xmalloc((size_t)n * sizeof(int64_t));
    int64_t *sm = (int64_t *)xmalloc((size_t)n * sizeof(int64_t));
    for (int64_t r = 0; r < nchain; r++) {
        omesh nxt;
        int st = decimate_round(&cur, chain[r], seeded, pcg, order, placement, &nxt, sr, sm, achievable);
        if (st) {
            omesh_free(&cur); free(replace); free(mapping); free(sr); free(sm);
            return st;
        }
        for (int64_t v = 0; v < n; v++) {
            replace[v] = sr[replace[v]];
            mapping[v] = mapping[v] < 0 ? -1 : sm[mapping[v]];
        }
        omesh_free(&cur);
        cur = nxt;
    }
    mfo_result *res = (mfo_result *)xcalloc(1, sizeof(mfo_result));
    res->n_in = n; res->n_out = cur.n; res->m_out = cur.m; res->c = c;
    res->positions = cur.P; res->facets = cur.F; res->features = cur.X;
    res->replace = replace; res->mapping = mapping;
    free(sr); free(sm);
    *res_out = res;
    return 0;
}

void mfo_result_sizes(const mfo_result *r, int64_t *n_in, int64_t *n_out, int64_t *m_out, int64_t *c) {
    *n_in = r->n_in; *n_out = r->n_out; *m_out = r->m_out; *c = r->c;
}
void mfo_result_copy(const mfo_result *r, double *positions, int64_t *facets, double *features, int64_t *replace,
                     int64_t *mapping) {
    memcpy(positions, r->positions, (size_t)r->n_out * 3 * sizeof(double));
    memcpy(facets, r->facets, (size_t)r->m_out * 3 * sizeof(int64_t));
    memcpy(features, r->features, (size_t)(r->n_out * r->c) * sizeof(double));
    memcpy(replace, r->replace, (size_t)r->n_in * sizeof(int64_t));
    memcpy(mapping, r->mapping, (size_t)r->n_in * sizeof(int64_t));
}
void mfo_result_free(mfo_result *r) {
    if (!r) return;
    free(r->positions); free(r->facets); free(r->features); free(r->replace); free(r->mapping);
    free(r);
}

/* exposed pieces for unit-level parity checks */
void mfo_vertex_quadrics(const double *P, int64_t n, const int64_t *F, int64_t m, int order, double *Q13) {
    omesh g = {n, m, 0, (double *)P, (int64_t *)F, NULL};
    vertex_quadrics(&g, order, Q13);
}
/* quality_report (decimate.py:580-602) up to the numpy reductions: the original
 * vertex quadrics (quadrics.py:69-77) summed per cluster in vertex order from +0.0
 * (accumulate_quadrics, quadrics.py:80-86), evaluated at the output positions
 * (Quadric.evaluate, quadrics.py:53-58). */
int mfo_quality_errors(const double *P, int64_t n, const int64_t *F, int64_t m, const int64_t *replace,
                       int64_t n_out, const double *Pout, int order, double *errors) {
    double *Q = (double *)xmalloc((size_t)(n ? n : 1) * QW * sizeof(double));
    double *acc = (double *)xcalloc((size_t)(n_out ? n_out : 1) * QW, sizeof(double));
    omesh g = {n, m, 0, (double *)P, (int64_t *)F, NULL};
    vertex_quadrics(&g, order, Q);
    for (int64_t v = 0; v < n; v++) {
        int64_t r = replace[v];
        if (r < 0 || r >= n_out) { free(Q); free(acc); return 2; }
        for (int k = 0; k < QW; k++) acc[QW * r + k] += Q[QW * v + k];
    }
    for (int64_t r = 0; r < n_out; r++) {
        const double *q = acc + QW * r;
        errors[r] = q_evaluate(q, q + 9, q[12], Pout + 3 * r, order);
    }
    free(Q); free(acc);
    return 0;
}

int64_t mfo_edge_costs(const double *P, int64_t n, const int64_t *F, int64_t m, int order, int64_t *edges_out,
                       double *cost_out) {
    omesh g = {n, m, 0, (double *)P, (int64_t *)F, NULL};
    double *Q = (double *)xmalloc((size_t)n * QW * sizeof(double));
    vertex_quadrics(&g, order, Q);
    int64_t *E = NULL;
    int64_t ne = edge_list(&g, &E);
    for (int64_t e = 0; e < ne; e++) {
        const double *qi = Q + QW * E[2 * e], *qj = Q + QW * E[2 * e + 1];
        double q[QW];
        for (int k = 0; k < QW; k++) q[k] = qi[k] + qj[k];
        const double *pi = P + 3 * E[2 * e], *pj = P + 3 * E[2 * e + 1];
        double x[3] = {0.5 * (pi[0] + pj[0]), 0.5 * (pi[1] + pj[1]), 0.5 * (pi[2] + pj[2])};
        if (cost_out) cost_out[e] = q_evaluate(q, q + 9, q[12], x, order);
        if (edges_out) { edges_out[2 * e] = E[2 * e]; edges_out[2 * e + 1] = E[2 * e + 1]; }
    }
    free(Q); free(E);
    return ne;
}
void mfo_pcg64_random(const uint64_t pcg[4], int64_t n, double *out) { pcg64_random(pcg, n, out); }

/* ------------------------------------------------------------------ */
/* pooling.py:36-77                                                     */

/* mode: 0 average, 1 max, 2 weighted, 3 sum.  Returns 0, or 1 when a
 * weighted cluster has zero total weight (pooling.py:64-66). */
int mfo_pool_f64(const double *X, int64_t n, int64_t c, const int64_t *replace, int64_t n_out, int mode,
                 const double *w, double *out) {
    if (mode == 1) {
        for (int64_t k = 0; k < n_out * c; k++) out[k] = -INFINITY;
        for (int64_t v = 0; v < n; v++)
            for (int64_t k = 0; k < c; k++) {
                double a = out[replace[v] * c + k], b = X[v * c + k];
                out[replace[v] * c + k] = (isnan(a) || a > b) ? a : b;
            }
        return 0;
    }
    memset(out, 0, (size_t)(n_out * c) * sizeof(double));
    if (mode == 2) {
        double *den = (double *)xcalloc((size_t)n_out, sizeof(double));
        for (int64_t v = 0; v < n; v++) {
            for (int64_t k = 0; k < c; k++) out[replace[v] * c + k] += X[v * c + k] * w[v];
            den[replace[v]] += w[v];
        }
        int bad = 0;
        for (int64_t r = 0; r < n_out; r++) bad |= (den[r] == 0.0);
        if (bad) { free(den); return 1; }
        for (int64_t r = 0; r < n_out; r++)
            for (int64_t k = 0; k < c; k++) out[r * c + k] = out[r * c + k] / den[r];
        free(den);
        return 0;
    }
    int64_t *cnt = (int64_t *)xcalloc((size_t)n_out, sizeof(int64_t));
    for (int64_t v = 0; v < n; v++) {
        cnt[replace[v]]++;
        for (int64_t k = 0; k < c; k++) out[replace[v] * c + k] += X[v * c + k];
    }
    if (mode == 0)
        for (int64_t r = 0; r < n_out; r++)
            for (int64_t k = 0; k < c; k++) out[r * c + k] = out[r * c + k] / (double)cnt[r];
    free(cnt);
    return 0;
}

int mfo_pool_f32(const float *X, int64_t n, int64_t c, const int64_t *replace, int64_t n_out, int mode,
                 const float *w, float *out) {
    if (mode == 1) {
        for (int64_t k = 0; k < n_out * c; k++) out[k] = -INFINITY;
        for (int64_t v = 0; v < n; v++)
            for (int64_t k = 0; k < c; k++) {
                float a = out[replace[v] * c + k], b = X[v * c + k];
                out[replace[v] * c + k] = (isnan(a) || a > b) ? a : b;
            }
        return 0;
    }
    memset(out, 0, (size_t)(n_out * c) * sizeof(float));
    if (mode == 2) {
        float *den = (float *)xcalloc((size_t)n_out, sizeof(float));
        for (int64_t v = 0; v < n; v++) {
            for (int64_t k = 0; k < c; k++) out[replace[v] * c + k] += X[v * c + k] * w[v];
            den[replace[v]] += w[v];
        }
        int bad = 0;
        for (int64_t r = 0; r < n_out; r++) bad |= (den[r] == 0.0f);
        if (bad) { free(den); return 1; }
        for (int64_t r = 0; r < n_out; r++)
            for (int64_t k = 0; k < c; k++) out[r * c + k] = out[r * c + k] / den[r];
        free(den);
        return 0;
    }
    int64_t *cnt = (int64_t *)xcalloc((size_t)n_out, sizeof(int64_t));
    for (int64_t v = 0; v < n; v++) {
        cnt[replace[v]]++;
        for (int64_t k = 0; k < c; k++) out[replace[v] * c + k] += X[v * c + k];
    }
    /* in-place `out /= counts` on float32: true_divide runs in float64 and
     * the result is cast back to float32 (pooling.py:69-70) */
    if (mode == 0)
        for (int64_t r = 0; r < n_out; r++)
            for (int64_t k = 0; k < c; k++) out[r * c + k] = (float)((double)out[r * c + k] / (double)cnt[r]);
    free(cnt);
    return 0;
}
