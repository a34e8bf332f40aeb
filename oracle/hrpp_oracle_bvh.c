/*
 * hrpp_oracle_bvh.c -- TEST INFRASTRUCTURE ONLY (part of the C oracle).
 *
 * The reference's BVH builder restated in plain C: hrpp/bvh.py:184-357
 * (build_bvh_from_arrays + _find_split).  It exists so that bench.py's
 * reference arm builds the scene's BVH without the product library (the
 * reference's own Python builder needs ~0.36 ms per triangle, hours at
 * BASELINE config c5).  Pinned against the reference-built golden BVHs by
 * tests/test_oracle_golden.py (bit-identical arrays).
 *
 * Structure (not the reference's): the triangles of a node occupy a
 * contiguous range of one permutation array, partitioned stably in place,
 * with the per-triangle centroid and bounds permuted alongside so every
 * pass over a node streams memory.  Nodes are emitted in the reference's
 * pop order (DFS preorder, left child first), so the leaves' ranges come in
 * increasing position order and the final permutation IS the reference's
 * triangle order (np.concatenate(order_chunks), bvh.py:259).
 *
 * median_split = 1: no SAH; every node with more than max_leaf_size
 * triangles takes the reference's forced split (stable median on the widest
 * centroid axis, bvh.py:351-357) -- the "binary median-split" tree of
 * BASELINE config c1, the same definition as the product builder's option.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define SAH_BINS 16                 /* hrpp/bvh.py:31 */
#define MAX_SUPPORTED_DEPTH 254     /* hrpp/bvh.py:34: MAX_STACK // 2 - 2 */
#define DEGENERATE_AREA_EPS 1e-12   /* hrpp/geom.py:36 */

typedef struct {
    int64_t n;         /* kept triangles */
    int64_t *perm;     /* position -> kept triangle */
    double *cent;      /* (n,3) by position */
    float *lo, *hi;    /* (n,3) triangle bounds by position */
    int64_t *tmp_i;    /* scratch for the stable partition */
    double *tmp_c;
    float *tmp_lo, *tmp_hi;
    uint8_t *side;     /* per position: 1 = right child */
} bld;

/* hrpp/bvh.py:285-287 */
static double half_area(const double lo[3], const double hi[3]) {
    double d0 = hi[0] - lo[0], d1 = hi[1] - lo[1], d2 = hi[2] - lo[2];
    d0 = d0 > 0.0 ? d0 : 0.0;
    d1 = d1 > 0.0 ? d1 : 0.0;
    d2 = d2 > 0.0 ? d2 : 0.0;
    return d0 * d1 + d1 * d2 + d2 * d0;
}

/* Stable partition of [b, e) by side[] (0 first), moving every permuted
 * array; returns the size of the left part. */
static int64_t partition(bld *B, int64_t b, int64_t e) {
    int64_t w = b, r = 0;
    for (int64_t p = b; p < e; p++) {
        if (!B->side[p]) {
            B->perm[w] = B->perm[p];
            memmove(B->cent + 3 * w, B->cent + 3 * p, 3 * sizeof(double));
            memmove(B->lo + 3 * w, B->lo + 3 * p, 3 * sizeof(float));
            memmove(B->hi + 3 * w, B->hi + 3 * p, 3 * sizeof(float));
            w++;
        } else {
            B->tmp_i[r] = B->perm[p];
            memcpy(B->tmp_c + 3 * r, B->cent + 3 * p, 3 * sizeof(double));
            memcpy(B->tmp_lo + 3 * r, B->lo + 3 * p, 3 * sizeof(float));
            memcpy(B->tmp_hi + 3 * r, B->hi + 3 * p, 3 * sizeof(float));
            r++;
        }
    }
    memcpy(B->perm + w, B->tmp_i, r * sizeof(int64_t));
    memcpy(B->cent + 3 * w, B->tmp_c, 3 * r * sizeof(double));
    memcpy(B->lo + 3 * w, B->tmp_lo, 3 * r * sizeof(float));
    memcpy(B->hi + 3 * w, B->tmp_hi, 3 * r * sizeof(float));
    return w - b;
}

static const double *g_sort_c;   /* qsort context: centroid column */
static int g_sort_ax;

static int cmp_median(const void *x, const void *y) {
    int64_t a = *(const int64_t *)x, b = *(const int64_t *)y;
    double ca = g_sort_c[3 * a + g_sort_ax], cb = g_sort_c[3 * b + g_sort_ax];
    if (ca < cb) return -1;
    if (ca > cb) return 1;
    return a < b ? -1 : (a > b ? 1 : 0);   /* np.argsort(kind="stable") */
}

/* hrpp/bvh.py:290-357 on positions [b, e).  Returns -1 for "no split"
 * (leaf), else the axis, with side[] marking the right child. */
static int find_split(bld *B, int64_t b, int64_t e, int max_leaf, int median) {
    const int64_t n = e - b;
    double cmin[3] = {INFINITY, INFINITY, INFINITY}, cmax[3] = {-INFINITY, -INFINITY, -INFINITY};
    double plo[3] = {INFINITY, INFINITY, INFINITY}, phi[3] = {-INFINITY, -INFINITY, -INFINITY};
    for (int64_t p = b; p < e; p++)
        for (int a = 0; a < 3; a++) {
            const double c = B->cent[3 * p + a];
            if (c < cmin[a]) cmin[a] = c;
            if (c > cmax[a]) cmax[a] = c;
            if (B->lo[3 * p + a] < plo[a]) plo[a] = B->lo[3 * p + a];
            if (B->hi[3 * p + a] > phi[a]) phi[a] = B->hi[3 * p + a];
        }
    double ext[3];
    for (int a = 0; a < 3; a++) ext[a] = cmax[a] - cmin[a];
    double best_cost = INFINITY;
    int best_ax = -1, best_k = -1;
    for (int ax = 0; ax < 3 && !median; ax++) {
        if (ext[ax] <= 0.0) continue;
        const double scale = SAH_BINS / ext[ax];
        int64_t cnt[SAH_BINS] = {0};
        double blo[SAH_BINS][3], bhi[SAH_BINS][3];
        for (int k = 0; k < SAH_BINS; k++)
            for (int a = 0; a < 3; a++) { blo[k][a] = INFINITY; bhi[k][a] = -INFINITY; }
        for (int64_t p = b; p < e; p++) {
            int64_t k = (int64_t)((B->cent[3 * p + ax] - cmin[ax]) * scale);
            if (k > SAH_BINS - 1) k = SAH_BINS - 1;
            cnt[k]++;
            for (int a = 0; a < 3; a++) {
                if (B->lo[3 * p + a] < blo[k][a]) blo[k][a] = B->lo[3 * p + a];
                if (B->hi[3 * p + a] > bhi[k][a]) bhi[k][a] = B->hi[3 * p + a];
            }
        }
        /* suffix boxes (right of each boundary), then the left sweep */
        double rlo[SAH_BINS][3], rhi[SAH_BINS][3];
        for (int a = 0; a < 3; a++) { rlo[SAH_BINS - 1][a] = blo[SAH_BINS - 1][a];
                                      rhi[SAH_BINS - 1][a] = bhi[SAH_BINS - 1][a]; }
        for (int k = SAH_BINS - 2; k >= 0; k--)
            for (int a = 0; a < 3; a++) {
                rlo[k][a] = blo[k][a] < rlo[k + 1][a] ? blo[k][a] : rlo[k + 1][a];
                rhi[k][a] = bhi[k][a] > rhi[k + 1][a] ? bhi[k][a] : rhi[k + 1][a];
            }
        double llo[3] = {INFINITY, INFINITY, INFINITY}, lhi[3] = {-INFINITY, -INFINITY, -INFINITY};
        int64_t nl = 0;
        for (int k = 0; k < SAH_BINS - 1; k++) {
            for (int a = 0; a < 3; a++) {
                if (blo[k][a] < llo[a]) llo[a] = blo[k][a];
                if (bhi[k][a] > lhi[a]) lhi[a] = bhi[k][a];
            }
            nl += cnt[k];
            const int64_t nr = n - nl;
            if (nl == 0 || nr == 0) continue;
            const double cost = half_area(llo, lhi) * (double)nl +
                                half_area(rlo[k + 1], rhi[k + 1]) * (double)nr;
            if (cost < best_cost) { best_cost = cost; best_ax = ax; best_k = k; }
        }
    }
    if (ext[0] <= 0.0 && ext[1] <= 0.0 && ext[2] <= 0.0) return -1;   /* bvh.py:337-338 */
    const double parent_area = half_area(plo, phi);
    if (best_ax >= 0 && parent_area > 0.0 && 1.0 + best_cost / parent_area < (double)n) {
        const double scale = SAH_BINS / ext[best_ax];
        for (int64_t p = b; p < e; p++) {
            int64_t k = (int64_t)((B->cent[3 * p + best_ax] - cmin[best_ax]) * scale);
            if (k > SAH_BINS - 1) k = SAH_BINS - 1;
            B->side[p] = k > best_k;
        }
        return best_ax;
    }
    if (n <= max_leaf) return -1;
    /* forced split: stable median on the widest centroid axis (np.argmax
     * takes the first maximum) */
    int ax = 0;
    for (int a = 1; a < 3; a++) if (ext[a] > ext[ax]) ax = a;
    int64_t *ord = (int64_t *)malloc(sizeof(int64_t) * n);
    for (int64_t j = 0; j < n; j++) ord[j] = j;
    g_sort_c = B->cent + 3 * b;
    g_sort_ax = ax;
    qsort(ord, n, sizeof(int64_t), cmp_median);
    for (int64_t j = 0; j < n; j++) B->side[b + ord[j]] = j >= n / 2;
    /* The reference lists the left half in sorted order, not range order:
     * reorder the range by the sort so partition() keeps that order. */
    int64_t *pp = (int64_t *)malloc(sizeof(int64_t) * n);
    double *cc = (double *)malloc(sizeof(double) * 3 * n);
    float *ll = (float *)malloc(sizeof(float) * 3 * n), *hh = (float *)malloc(sizeof(float) * 3 * n);
    uint8_t *ss = (uint8_t *)malloc(n);
    for (int64_t j = 0; j < n; j++) {
        const int64_t s = b + ord[j];
        pp[j] = B->perm[s];
        ss[j] = B->side[s];
        memcpy(cc + 3 * j, B->cent + 3 * s, 3 * sizeof(double));
        memcpy(ll + 3 * j, B->lo + 3 * s, 3 * sizeof(float));
        memcpy(hh + 3 * j, B->hi + 3 * s, 3 * sizeof(float));
    }
    memcpy(B->perm + b, pp, n * sizeof(int64_t));
    memcpy(B->side + b, ss, n);
    memcpy(B->cent + 3 * b, cc, 3 * n * sizeof(double));
    memcpy(B->lo + 3 * b, ll, 3 * n * sizeof(float));
    memcpy(B->hi + 3 * b, hh, 3 * n * sizeof(float));
    free(pp); free(cc); free(ll); free(hh); free(ss); free(ord);
    return ax;
}

typedef struct { int64_t b, e; int32_t parent; int32_t is_left; int32_t depth; } item;

/* hrpp/bvh.py:184-276.  Output arrays sized for 2*n_tris - 1 nodes and
 * n_tris triangles.  Returns 0, 3 (EmptyScene: nothing left after the
 * degenerate filter) or 4 (depth above the supported maximum). */
int or_build_bvh(const float *v0, const float *v1, const float *v2, const int32_t *ids,
                 int64_t m_in, int max_leaf, int median,
                 float *bmin, float *bmax, int32_t *left, int32_t *right, int8_t *axis,
                 int32_t *first, int32_t *count, int32_t *parent, int32_t *depth,
                 float *tv0, float *tv1, float *tv2, int32_t *tri_ids,
                 int64_t *n_nodes_out, int64_t *n_tris_out, int32_t *max_depth_out) {
    if (max_leaf < 1 || m_in < 0) return 3;
    bld B;
    memset(&B, 0, sizeof(B));
    B.perm = (int64_t *)malloc(sizeof(int64_t) * (m_in + 1));
    /* degenerate filter: |(v1-v0) x (v2-v0)| in float64 > 2e-12 (bvh.py:195,279-282) */
    int64_t m = 0;
    for (int64_t i = 0; i < m_in; i++) {
        const double ax_ = (double)v1[3 * i] - v0[3 * i], ay = (double)v1[3 * i + 1] - v0[3 * i + 1],
                     az = (double)v1[3 * i + 2] - v0[3 * i + 2];
        const double bx = (double)v2[3 * i] - v0[3 * i], by = (double)v2[3 * i + 1] - v0[3 * i + 1],
                     bz = (double)v2[3 * i + 2] - v0[3 * i + 2];
        const double cx = ay * bz - az * by, cy = az * bx - ax_ * bz, cz = ax_ * by - ay * bx;
        if (sqrt(cx * cx + cy * cy + cz * cz) > 2.0 * DEGENERATE_AREA_EPS) B.perm[m++] = i;
    }
    *n_tris_out = m;
    if (m == 0) { free(B.perm); return 3; }
    B.n = m;
    B.cent = (double *)malloc(sizeof(double) * 3 * m);
    B.lo = (float *)malloc(sizeof(float) * 3 * m);
    B.hi = (float *)malloc(sizeof(float) * 3 * m);
    B.tmp_i = (int64_t *)malloc(sizeof(int64_t) * m);
    B.tmp_c = (double *)malloc(sizeof(double) * 3 * m);
    B.tmp_lo = (float *)malloc(sizeof(float) * 3 * m);
    B.tmp_hi = (float *)malloc(sizeof(float) * 3 * m);
    B.side = (uint8_t *)malloc(m);
    for (int64_t p = 0; p < m; p++) {
        const int64_t i = B.perm[p];
        for (int a = 0; a < 3; a++) {
            float x = v0[3 * i + a], y = v1[3 * i + a], z = v2[3 * i + a];
            float lo = x < y ? x : y, hi = x > y ? x : y;   /* np.minimum / np.maximum */
            lo = lo < z ? lo : z;
            hi = hi > z ? hi : z;
            B.lo[3 * p + a] = lo;
            B.hi[3 * p + a] = hi;
            B.cent[3 * p + a] = ((double)lo + (double)hi) * 0.5;   /* bvh.py:203 */
        }
    }
    int64_t cap = 64, top = 0, nn = 0;
    item *stk = (item *)malloc(sizeof(item) * cap);
    stk[top++] = (item){0, m, -1, 0, 0};
    int32_t maxd = 0;
    int rc = 0;
    while (top > 0) {
        const item it = stk[--top];
        const int64_t me = nn++;
        float lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
        for (int64_t p = it.b; p < it.e; p++)
            for (int a = 0; a < 3; a++) {
                if (B.lo[3 * p + a] < lo[a]) lo[a] = B.lo[3 * p + a];
                if (B.hi[3 * p + a] > hi[a]) hi[a] = B.hi[3 * p + a];
            }
        memcpy(bmin + 3 * me, lo, sizeof(lo));
        memcpy(bmax + 3 * me, hi, sizeof(hi));
        left[me] = -1; right[me] = -1; axis[me] = 0; first[me] = -1; count[me] = 0;
        parent[me] = it.parent;
        depth[me] = it.depth;
        if (it.parent >= 0) (it.is_left ? left : right)[it.parent] = (int32_t)me;
        const int64_t n = it.e - it.b;
        const int ax = n > 1 ? find_split(&B, it.b, it.e, max_leaf, median) : -1;
        if (ax < 0) {   /* leaf: its triangles are the range, in order */
            first[me] = (int32_t)it.b;
            count[me] = (int32_t)n;
            if (it.depth > maxd) maxd = it.depth;
            continue;
        }
        axis[me] = (int8_t)ax;
        if (it.depth + 1 > MAX_SUPPORTED_DEPTH) { rc = 4; break; }
        const int64_t nl = partition(&B, it.b, it.e);
        if (top + 2 > cap) { cap *= 2; stk = (item *)realloc(stk, sizeof(item) * cap); }
        stk[top++] = (item){it.b + nl, it.e, (int32_t)me, 0, it.depth + 1};   /* right first */
        stk[top++] = (item){it.b, it.b + nl, (int32_t)me, 1, it.depth + 1};
    }
    if (rc == 0) {
        for (int64_t p = 0; p < m; p++) {
            const int64_t i = B.perm[p];
            memcpy(tv0 + 3 * p, v0 + 3 * i, 3 * sizeof(float));
            memcpy(tv1 + 3 * p, v1 + 3 * i, 3 * sizeof(float));
            memcpy(tv2 + 3 * p, v2 + 3 * i, 3 * sizeof(float));
            tri_ids[p] = ids ? ids[i] : (int32_t)i;
        }
        *n_nodes_out = nn;
        *max_depth_out = maxd;
    }
    free(stk); free(B.perm); free(B.cent); free(B.lo); free(B.hi); free(B.tmp_i);
    free(B.tmp_c); free(B.tmp_lo); free(B.tmp_hi); free(B.side);
    return rc;
}
