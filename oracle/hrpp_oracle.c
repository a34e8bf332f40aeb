/*
 * hrpp_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C restatement of the reference HRPP hot path (arXiv 1910.01304
 * limit-study workbench, package `hrpp` 0.1.0).  It is the checker for the
 * CUDA product path and the CPU baseline arm of bench.py.  Nothing in the
 * product package (paper_1910_01304_b200/) links, imports or executes this
 * file; only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs do.
 *
 * Parity is PINNED: tests/test_oracle_golden.py checks every entry point
 * below against golden vectors produced by the real reference package
 * (tests/golden/make_golden.py imports /root/reference/pkg/src/hrpp).
 *
 * Arithmetic follows the reference exactly: float64, no FMA contraction
 * (build with -ffp-contract=off), operation order of hrpp/kernels.py.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define OR_OK 0
#define OR_NONFINITE 1
#define OR_CAPACITY 2
#define OR_INVALID 3

#define MAX_STACK 512           /* hrpp/kernels.py:18 */
#define DET_EPS 1e-9            /* hrpp/kernels.py:20 */
#define WRONG_CLOSEST_EPS 1e-9  /* hrpp/tracer.py:52 */

/* ------------------------------------------------------------------------ */
/* Ray hash: hrpp/rayhash.py:67-78 (map_float_to_hash), :99-122 (hash_rays) */
/* ------------------------------------------------------------------------ */

static inline uint32_t lane_hash(uint32_t bits, int p) {
    /* hrpp/rayhash.py:118-122 */
    uint32_t sign = bits >> 31;
    uint32_t exp_top = ((bits >> 23) & 0xFFu) >> (8 - p);
    uint32_t man_top = (bits & 0x7FFFFFu) >> (23 - p);
    return (sign << (2 * p)) | (exp_top << p) | man_top;
}

/* hrpp/rayhash.py:99-115.  Returns OR_NONFINITE (no keys written) if any
 * component has an all-ones exponent, like the reference's up-front check. */
int or_hash_rays(const float *O, const float *D, int64_t n, int p, uint64_t *keys) {
    if (p < 1 || p > 7) return OR_INVALID;
    const uint32_t *bo = (const uint32_t *)O;
    const uint32_t *bd = (const uint32_t *)D;
    for (int64_t i = 0; i < 3 * n; i++) {
        if (((bo[i] >> 23) & 0xFFu) == 0xFFu) return OR_NONFINITE;
        if (((bd[i] >> 23) & 0xFFu) == 0xFFu) return OR_NONFINITE;
    }
    /* LANE_PAIRS = ((0,2),(1,1),(2,0)), LANE_SHIFTS = (0,16,32): rayhash.py:37-39 */
    for (int64_t i = 0; i < n; i++) {
        uint64_t k = 0;
        k |= (uint64_t)(lane_hash(bo[3 * i + 0], p) ^ lane_hash(bd[3 * i + 2], p)) << 0;
        k |= (uint64_t)(lane_hash(bo[3 * i + 1], p) ^ lane_hash(bd[3 * i + 1], p)) << 16;
        k |= (uint64_t)(lane_hash(bo[3 * i + 2], p) ^ lane_hash(bd[3 * i + 0], p)) << 32;
        keys[i] = k;
    }
    return OR_OK;
}

/* ------------------------------------------------------------------------ */
/* BVH view (the 10-array kernel ABI of hrpp/bvh.py:126-128 + depth/parent)  */
/* ------------------------------------------------------------------------ */

typedef struct {
    const float *bmin, *bmax;   /* (N,3) f32 */
    const int32_t *left, *right;
    const int8_t *axis;
    const int32_t *first, *count;
    const float *tv0, *tv1, *tv2; /* (M,3) f32 */
    const int32_t *depth;       /* (N,) used by the predictor */
    const int32_t *anc;         /* go-up ancestor LUT (N,) or NULL */
    int64_t n_nodes, n_tris;
} or_bvh;

typedef struct {
    int found;
    double t;
    int32_t slot, leaf;
    double u, v;
    int64_t boxes, tris, visited;
} or_hit;

/* hrpp/kernels.py:23-51 */
static inline int box_hit(const or_bvh *b, int32_t nd, double ox, double oy, double oz,
                          double ivx, double ivy, double ivz, double t0, double t1) {
    double bnx = (double)b->bmin[3 * nd + 0], bny = (double)b->bmin[3 * nd + 1],
           bnz = (double)b->bmin[3 * nd + 2];
    double bxx = (double)b->bmax[3 * nd + 0], bxy = (double)b->bmax[3 * nd + 1],
           bxz = (double)b->bmax[3 * nd + 2];
    double tn = t0, tf = t1, a, c, s;
    a = (bnx - ox) * ivx; c = (bxx - ox) * ivx;
    if (ivx < 0.0) { s = a; a = c; c = s; }
    if (a > tn) tn = a;
    if (c < tf) tf = c;
    a = (bny - oy) * ivy; c = (bxy - oy) * ivy;
    if (ivy < 0.0) { s = a; a = c; c = s; }
    if (a > tn) tn = a;
    if (c < tf) tf = c;
    a = (bnz - oz) * ivz; c = (bxz - oz) * ivz;
    if (ivz < 0.0) { s = a; a = c; c = s; }
    if (a > tn) tn = a;
    if (c < tf) tf = c;
    return tn <= tf;
}

/* hrpp/kernels.py:54-86 */
static inline int tri_test(const or_bvh *b, int32_t k, double ox, double oy, double oz,
                           double dx, double dy, double dz, double *t, double *u, double *v) {
    double ax = (double)b->tv0[3 * k + 0], ay = (double)b->tv0[3 * k + 1],
           az = (double)b->tv0[3 * k + 2];
    double e1x = (double)b->tv1[3 * k + 0] - ax, e1y = (double)b->tv1[3 * k + 1] - ay,
           e1z = (double)b->tv1[3 * k + 2] - az;
    double e2x = (double)b->tv2[3 * k + 0] - ax, e2y = (double)b->tv2[3 * k + 1] - ay,
           e2z = (double)b->tv2[3 * k + 2] - az;
    double px = dy * e2z - dz * e2y;
    double py = dz * e2x - dx * e2z;
    double pz = dx * e2y - dy * e2x;
    double det = e1x * px + e1y * py + e1z * pz;
    if (fabs(det) <= DET_EPS) return 0;
    double inv_det = 1.0 / det;
    double tx = ox - ax, ty = oy - ay, tz = oz - az;
    double uu = (tx * px + ty * py + tz * pz) * inv_det;
    if (uu < 0.0 || uu > 1.0) return 0;
    double qx = ty * e1z - tz * e1y;
    double qy = tz * e1x - tx * e1z;
    double qz = tx * e1y - ty * e1x;
    double vv = (dx * qx + dy * qy + dz * qz) * inv_det;
    if (vv < 0.0 || uu + vv > 1.0) return 0;
    *t = (e2x * qx + e2y * qy + e2z * qz) * inv_det;
    *u = uu;
    *v = vv;
    return 1;
}

static inline double recip(double d) { return d != 0.0 ? 1.0 / d : copysign(INFINITY, d); }

/* hrpp/kernels.py:89-154 (closest) and :157-206 (any) */
static or_hit trace_one(const or_bvh *b, int closest, double ox, double oy, double oz,
                        double dx, double dy, double dz, double rtmin, double rtmax, int32_t start) {
    double ivx = recip(dx), ivy = recip(dy), ivz = recip(dz);
    int32_t stack[MAX_STACK];
    int top = 1;
    stack[0] = start;
    or_hit h;
    h.found = 0; h.t = closest ? rtmax : 0.0; h.slot = -1; h.leaf = -1; h.u = 0.0; h.v = 0.0;
    h.boxes = 0; h.tris = 0; h.visited = 0;
    while (top > 0) {
        int32_t nd = stack[--top];
        h.visited++;
        h.boxes++;
        if (!box_hit(b, nd, ox, oy, oz, ivx, ivy, ivz, rtmin, closest ? h.t : rtmax)) continue;
        int32_t l = b->left[nd];
        if (l < 0) {
            int32_t f = b->first[nd], e = f + b->count[nd];
            for (int32_t k = f; k < e; k++) {
                double t, u, v;
                h.tris++;
                if (tri_test(b, k, ox, oy, oz, dx, dy, dz, &t, &u, &v) && t >= rtmin && t <= rtmax) {
                    if (!closest) {
                        h.found = 1; h.t = t; h.slot = k; h.leaf = nd; h.u = u; h.v = v;
                        return h;
                    }
                    if (!h.found || t < h.t) {
                        h.found = 1; h.t = t; h.slot = k; h.leaf = nd; h.u = u; h.v = v;
                    }
                }
            }
        } else {
            int ax = b->axis[nd];
            double dval = ax == 1 ? dy : (ax == 2 ? dz : dx);
            int32_t nearc, farc;
            if (dval >= 0.0) { nearc = l; farc = b->right[nd]; }
            else { nearc = b->right[nd]; farc = l; }
            stack[top++] = farc;
            stack[top++] = nearc;
        }
    }
    return h;
}

/* hrpp/kernels.py:251-278 (closest) and :281-297 (any) */
static or_hit eval_entry(const or_bvh *b, int closest, const int32_t *nodes, int64_t n_nodes,
                         double ox, double oy, double oz, double dx, double dy, double dz,
                         double rtmin, double rtmax) {
    or_hit acc;
    acc.found = 0; acc.t = closest ? INFINITY : 0.0; acc.slot = -1; acc.leaf = -1;
    acc.u = 0.0; acc.v = 0.0; acc.boxes = 0; acc.tris = 0; acc.visited = 0;
    for (int64_t j = 0; j < n_nodes; j++) {
        or_hit r = trace_one(b, closest, ox, oy, oz, dx, dy, dz, rtmin, rtmax, nodes[j]);
        acc.boxes += r.boxes; acc.tris += r.tris; acc.visited += r.visited;
        if (closest) {
            if (r.found && (!acc.found || r.t < acc.t)) {
                acc.found = 1; acc.t = r.t; acc.slot = r.slot; acc.leaf = r.leaf;
                acc.u = r.u; acc.v = r.v;
            }
        } else if (r.found) {
            acc.found = 1; acc.t = r.t; acc.slot = r.slot; acc.leaf = r.leaf;
            acc.u = r.u; acc.v = r.v;
            return acc;
        }
    }
    return acc;
}

#define BVH_ARGS const float *bmin, const float *bmax, const int32_t *left, \
    const int32_t *right, const int8_t *axis, const int32_t *first, const int32_t *count, \
    const float *tv0, const float *tv1, const float *tv2, const int32_t *depth, int64_t n_nodes, \
    int64_t n_tris
#define BVH_INIT(bv) or_bvh bv = {bmin, bmax, left, right, axis, first, count, tv0, tv1, tv2, \
    depth, NULL, n_nodes, n_tris}

/* hrpp/kernels.py:209-248 via hrpp/bvh.py:398-442.  O/D f32 (widened exactly
 * to f64 as bvh.py:401-402 does); u/v may be NULL (the any-hit batch has none). */
int or_trace_batch(BVH_ARGS, int closest, const float *O, const float *D,
                   const double *tmins, const double *tmaxs, int32_t start, int64_t n,
                   uint8_t *found, double *t, int32_t *slot, int32_t *leaf, double *u, double *v,
                   int64_t *box, int64_t *tri, int64_t *vis, int nthreads) {
    BVH_INIT(bv);
    if (start < 0 || start >= n_nodes) return OR_INVALID;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel for schedule(dynamic, 256)
#endif
    for (int64_t i = 0; i < n; i++) {
        or_hit h = trace_one(&bv, closest, O[3 * i], O[3 * i + 1], O[3 * i + 2], D[3 * i],
                             D[3 * i + 1], D[3 * i + 2], tmins[i], tmaxs[i], start);
        found[i] = (uint8_t)h.found; t[i] = h.t; slot[i] = h.slot; leaf[i] = h.leaf;
        if (u) u[i] = h.u;
        if (v) v[i] = h.v;
        box[i] = h.boxes; tri[i] = h.tris; vis[i] = h.visited;
    }
    return OR_OK;
}

/* ------------------------------------------------------------------------ */
/* Predictor table: hrpp/predictor.py:70-211                                */
/* ------------------------------------------------------------------------ */

typedef struct {
    uint64_t key;
    int32_t *nodes;
    int64_t len, cap;
} or_entry;

typedef struct {
    int64_t max_entries;
    int64_t n_entries, stored;
    or_entry *entries;       /* insertion order */
    int64_t ent_cap;
    int64_t *slots;          /* open addressing: entry index or -1 */
    int64_t slot_cap;        /* power of two */
} or_table;

static inline uint64_t mix64(uint64_t x) {
    x ^= x >> 33; x *= 0xff51afd7ed558ccdULL; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ULL;
    x ^= x >> 33; return x;
}

or_table *or_table_create(int64_t max_entries) {
    or_table *t = (or_table *)calloc(1, sizeof(or_table));
    t->max_entries = max_entries;
    t->slot_cap = 1024;
    t->slots = (int64_t *)malloc(sizeof(int64_t) * t->slot_cap);
    for (int64_t i = 0; i < t->slot_cap; i++) t->slots[i] = -1;
    t->ent_cap = 256;
    t->entries = (or_entry *)malloc(sizeof(or_entry) * t->ent_cap);
    return t;
}

void or_table_destroy(or_table *t) {
    if (!t) return;
    for (int64_t i = 0; i < t->n_entries; i++) free(t->entries[i].nodes);
    free(t->entries); free(t->slots); free(t);
}

static int64_t find_slot(const or_table *t, uint64_t key) {
    uint64_t m = (uint64_t)t->slot_cap - 1, h = mix64(key) & m;
    for (;;) {
        int64_t e = t->slots[h];
        if (e < 0 || t->entries[e].key == key) return (int64_t)h;
        h = (h + 1) & m;
    }
}

/* predictor.py:143-145: entry index or -1 */
static inline int64_t t_lookup(const or_table *t, uint64_t key) {
    return t->slots[find_slot(t, key)];
}

/* predictor.py:147-160 (PredictorEntry.add :84-94).  Returns 1 if grew, 0 if
 * duplicate, -1 (CapacityExceeded) if a NEW key would exceed the cap. */
static int t_record(or_table *t, uint64_t key, int32_t node) {
    int64_t s = find_slot(t, key);
    int64_t e = t->slots[s];
    if (e < 0) {
        if (t->n_entries >= t->max_entries) return -1;
        if (t->n_entries == t->ent_cap) {
            t->ent_cap *= 2;
            t->entries = (or_entry *)realloc(t->entries, sizeof(or_entry) * t->ent_cap);
        }
        e = t->n_entries++;
        or_entry *en = &t->entries[e];
        en->key = key; en->len = 0; en->cap = 4;
        en->nodes = (int32_t *)malloc(sizeof(int32_t) * 4);
        t->slots[s] = e;
        if (2 * t->n_entries > t->slot_cap) { /* grow + rehash */
            int64_t nc = t->slot_cap * 2;
            free(t->slots);
            t->slots = (int64_t *)malloc(sizeof(int64_t) * nc);
            for (int64_t i = 0; i < nc; i++) t->slots[i] = -1;
            t->slot_cap = nc;
            for (int64_t i = 0; i < t->n_entries; i++) t->slots[find_slot(t, t->entries[i].key)] = i;
        }
    }
    or_entry *en = &t->entries[e];
    for (int64_t j = 0; j < en->len; j++)
        if (en->nodes[j] == node) return 0;
    if (en->len == en->cap) {
        en->cap *= 2;
        en->nodes = (int32_t *)realloc(en->nodes, sizeof(int32_t) * en->cap);
    }
    en->nodes[en->len++] = node;
    t->stored++;
    return 1;
}

/* Batched sequential record (in order).  inserted[i] = 0/1.  Returns
 * OR_CAPACITY at the first failing record (earlier records stay applied,
 * exactly as a Python loop over PredictorTable.record would leave them). */
int or_table_record(or_table *t, const uint64_t *keys, const int32_t *nodes, int64_t n,
                    uint8_t *inserted) {
    for (int64_t i = 0; i < n; i++) {
        int r = t_record(t, keys[i], nodes[i]);
        if (r < 0) return OR_CAPACITY;
        if (inserted) inserted[i] = (uint8_t)r;
    }
    return OR_OK;
}

/* Lookup: returns entry length (0 = absent) per key; if nodes_out != NULL and
 * cap >= len for a single key query, copies the node list. */
int64_t or_table_lookup(const or_table *t, uint64_t key, int32_t *nodes_out, int64_t cap) {
    int64_t e = t_lookup(t, key);
    if (e < 0) return 0;
    const or_entry *en = &t->entries[e];
    if (nodes_out) for (int64_t j = 0; j < en->len && j < cap; j++) nodes_out[j] = en->nodes[j];
    return en->len;
}

void or_table_info(const or_table *t, int64_t *entries, int64_t *stored, int64_t *max_len) {
    int64_t m = 0;
    for (int64_t i = 0; i < t->n_entries; i++) if (t->entries[i].len > m) m = t->entries[i].len;
    *entries = t->n_entries; *stored = t->stored; *max_len = m;
}

static int cmp_entry_key(const void *a, const void *b) {
    uint64_t x = (*(const or_entry *const *)a)->key, y = (*(const or_entry *const *)b)->key;
    return x < y ? -1 : (x > y ? 1 : 0);
}

/* Export sorted by key (dump_lines order, predictor.py:207-211):
 * keys[n_entries], offsets[n_entries+1], nodes[stored]. */
void or_table_export(const or_table *t, uint64_t *keys, int64_t *offsets, int32_t *nodes) {
    const or_entry **ptr = (const or_entry **)malloc(sizeof(void *) * (t->n_entries + 1));
    for (int64_t i = 0; i < t->n_entries; i++) ptr[i] = &t->entries[i];
    qsort(ptr, t->n_entries, sizeof(void *), cmp_entry_key);
    int64_t off = 0;
    for (int64_t i = 0; i < t->n_entries; i++) {
        keys[i] = ptr[i]->key;
        offsets[i] = off;
        memcpy(nodes + off, ptr[i]->nodes, sizeof(int32_t) * ptr[i]->len);
        off += ptr[i]->len;
    }
    offsets[t->n_entries] = off;
    free(ptr);
}

/* ------------------------------------------------------------------------ */
/* Consult loops and the wave: hrpp/tracer.py:217-371                        */
/* ------------------------------------------------------------------------ */

/* stats layout = RayKindStats field order (hrpp/metrics.py:38-51) */
enum { S_RAYS, S_TP, S_FP, S_NEG, S_BB, S_BT, S_OB, S_OT, S_SK, S_EST, S_WRONG, S_N };

/* hrpp/tracer.py:217-275.  log_* may be NULL.  With owner != NULL only the
 * rays whose owner[i] == me are consulted (in ray order): the key-sharded
 * multi-threaded wave below gives each thread the keys it owns. */
static int consult_limit(or_table *t, const or_bvh *b, int closest, const uint64_t *keys,
                         const float *O, const float *D, const double *tmins,
                         const double *tmaxs, const uint8_t *bfound, const double *bt,
                         const int32_t *bleaf, const int64_t *bbox, int64_t n, int64_t *stats,
                         int8_t *log_cls, int64_t *log_eval_box, double *log_pred_t,
                         int64_t *log_pred_slot, const uint16_t *owner, uint16_t me) {
    int64_t tp = 0, fp = 0, neg = 0, ob = 0, ot = 0, sk = 0, est = 0, wrong = 0;
    for (int64_t i = 0; i < n; i++) {
        if (owner && owner[i] != me) continue;
        uint64_t key = keys[i];
        int64_t e = t_lookup(t, key);
        if (e < 0) {
            neg++;
            if (log_cls) { log_cls[i] = 2; log_eval_box[i] = 0; log_pred_t[i] = INFINITY; log_pred_slot[i] = -1; }
            if (bfound[i] && t_record(t, key, b->anc[bleaf[i]]) < 0) return OR_CAPACITY;
            continue;
        }
        /* copy-free: entry pointer stays valid (no record happens before eval) */
        or_hit r = eval_entry(b, closest, t->entries[e].nodes, t->entries[e].len,
                              O[3 * i], O[3 * i + 1], O[3 * i + 2], D[3 * i], D[3 * i + 1],
                              D[3 * i + 2], tmins[i], tmaxs[i]);
        ob += r.boxes; ot += r.tris;
        if (r.found) {
            tp++;
            sk += bbox[i] - r.boxes;
            int64_t x = (int64_t)b->depth[r.leaf] + 1 - r.boxes;
            est += x > 0 ? x : 0;
            if (closest && r.t > bt[i] + WRONG_CLOSEST_EPS) wrong++;
        } else {
            fp++;
            if (bfound[i] && t_record(t, key, b->anc[bleaf[i]]) < 0) return OR_CAPACITY;
        }
        if (log_cls) {
            log_cls[i] = r.found ? 0 : 1;
            log_eval_box[i] = r.boxes;
            log_pred_t[i] = r.found ? r.t : INFINITY;
            log_pred_slot[i] = r.found ? r.slot : -1;
        }
    }
    stats[S_TP] += tp; stats[S_FP] += fp; stats[S_NEG] += neg;
    stats[S_OB] += ob; stats[S_OT] += ot; stats[S_SK] += sk; stats[S_EST] += est;
    stats[S_WRONG] += wrong;
    return OR_OK;
}

/* hrpp/tracer.py:278-340 */
static int consult_live(or_table *t, const or_bvh *b, int closest, const uint64_t *keys,
                        const float *O, const float *D, const double *tmins, const double *tmaxs,
                        int64_t n, int64_t *stats, uint8_t *ofound, double *ot_, int32_t *oslot,
                        int32_t *oleaf, const uint16_t *owner, uint16_t me) {
    int64_t tp = 0, fp = 0, neg = 0, ob = 0, ot = 0, est = 0, bb = 0, bt = 0;
    for (int64_t i = 0; i < n; i++) {
        if (owner && owner[i] != me) continue;
        ofound[i] = 0; ot_[i] = 0.0; oslot[i] = -1; oleaf[i] = -1;
    }
    for (int64_t i = 0; i < n; i++) {
        if (owner && owner[i] != me) continue;
        uint64_t key = keys[i];
        int64_t e = t_lookup(t, key);
        int predicted = 0;
        double ox = O[3 * i], oy = O[3 * i + 1], oz = O[3 * i + 2];
        double dx = D[3 * i], dy = D[3 * i + 1], dz = D[3 * i + 2];
        if (e >= 0) {
            or_hit r = eval_entry(b, closest, t->entries[e].nodes, t->entries[e].len, ox, oy, oz,
                                  dx, dy, dz, tmins[i], tmaxs[i]);
            ob += r.boxes; ot += r.tris;
            if (r.found) {
                tp++;
                int64_t x = (int64_t)b->depth[r.leaf] + 1 - r.boxes;
                est += x > 0 ? x : 0;
                ofound[i] = 1; ot_[i] = r.t; oslot[i] = r.slot; oleaf[i] = r.leaf;
                predicted = 1;
            } else {
                fp++;
            }
        } else {
            neg++;
        }
        if (!predicted) {
            or_hit h = trace_one(b, closest, ox, oy, oz, dx, dy, dz, tmins[i], tmaxs[i], 0);
            bb += h.boxes; bt += h.tris;
            if (h.found) {
                ofound[i] = 1; ot_[i] = h.t; oslot[i] = h.slot; oleaf[i] = h.leaf;
                if (t_record(t, key, b->anc[h.leaf]) < 0) return OR_CAPACITY;
            }
        }
    }
    stats[S_TP] += tp; stats[S_FP] += fp; stats[S_NEG] += neg;
    stats[S_OB] += ob; stats[S_OT] += ot; stats[S_EST] += est;
    stats[S_BB] += bb; stats[S_BT] += bt;
    return OR_OK;
}

/* Fast mode (mode 3): the product's sort-free live mode (DESIGN.md "Fast
 * mode"), restated sequentially so the GPU can be checked bit for bit.  It
 * runs the reference's live loop (hrpp/tracer.py:295-331) as rounds of
 * key-parallel speculation instead of one ray at a time:
 *  round 0  every ray evaluates its entry as it stood at the start of the
 *           wave; a hit is a TP (final);
 *  round k  (1 <= k <= R) among the rays still unresolved, the first of each
 *           key in ray order is the key's round-k leader: NEG (no entry at
 *           its turn) or FP, traced from the root (final).  If it hit and
 *           its node anc[leaf] is new to the entry, every later unresolved
 *           ray of the key evaluates that node: a hit makes it a TP;
 *  final    the rays still unresolved after R rounds are traced (NEG or FP);
 *           the rounds also end early, before round k >= 2, when round k-1
 *           resolved fewer than n / stop_div rays (deterministic counts).
 * Records (key, anc[leaf]) of every traced ray with a hit are applied after
 * the wave in ray order with set semantics (hrpp/predictor.py:147-160).
 * Every ray's decision sees exactly the nodes earlier rays appended, as in
 * the reference, EXCEPT the rays resolved in the final pass, which do not see
 * each other's appends: with R at least the number of appends any key needs
 * in the wave the statistics, hits and table are the reference's; with
 * fewer rounds some of those rays are traced instead of predicted (fewer
 * TPs; DESIGN.md states the measured tolerance).  Counters: overhead = every
 * entry/node evaluation, baseline = the traced rays' traversals, est over
 * TPs with the ray's total evaluation boxes. */
static int g_fast_rounds = 8, g_fast_stop_div = 32;
void or_set_fast_rounds(int r, int stop_div) {
    g_fast_rounds = r < 0 ? 0 : r;
    g_fast_stop_div = stop_div < 0 ? 0 : stop_div;
}

typedef struct { int64_t cap; int64_t *ray; } key_map;   /* key -> ray (first/last seen) */

static int64_t *km_slot(key_map *m, const uint64_t *keys, uint64_t key) {
    uint64_t h = mix64(key) & (uint64_t)(m->cap - 1);
    while (m->ray[h] >= 0 && keys[m->ray[h]] != key) h = (h + 1) & (uint64_t)(m->cap - 1);
    return &m->ray[h];
}

static int fast_wave(or_table *t, const or_bvh *b, int closest, const uint64_t *keys,
                     const float *O, const float *D, const double *tmins, const double *tmaxs,
                     int64_t n, int64_t *stats, uint8_t *ofound, double *ot_, int32_t *oslot,
                     int32_t *oleaf) {
    int64_t tp = 0, fp = 0, neg = 0, ob = 0, ovt = 0, est = 0, bb = 0, bt = 0;
    const int64_t nn = n > 0 ? n : 1;
    int64_t *eid = (int64_t *)malloc(sizeof(int64_t) * nn);
    int64_t *evbox = (int64_t *)malloc(sizeof(int64_t) * nn);  /* evaluation boxes so far */
    uint8_t *traced = (uint8_t *)calloc(nn, 1);
    int64_t *unres = (int64_t *)malloc(sizeof(int64_t) * nn), nu = 0;
    key_map lead = {1024, NULL}, hit = {1024, NULL}, added = {1024, NULL};
    while (lead.cap < 2 * nn) lead.cap <<= 1;
    hit.cap = added.cap = lead.cap;
    lead.ray = (int64_t *)malloc(sizeof(int64_t) * lead.cap);
    hit.ray = (int64_t *)malloc(sizeof(int64_t) * lead.cap);    /* key's traced rays hit */
    for (int64_t h = 0; h < lead.cap; h++) hit.ray[h] = -1;
    /* appended nodes per key so far: a linked list through `nxt` by ray */
    int64_t *nxt = (int64_t *)malloc(sizeof(int64_t) * nn);
    added.ray = (int64_t *)malloc(sizeof(int64_t) * lead.cap);  /* head: last appending ray */
    for (int64_t h = 0; h < lead.cap; h++) added.ray[h] = -1;
    /* round 0 */
    for (int64_t i = 0; i < n; i++) {
        ofound[i] = 0; ot_[i] = 0.0; oslot[i] = -1; oleaf[i] = -1;
        eid[i] = t_lookup(t, keys[i]);
        evbox[i] = 0;
        if (eid[i] >= 0) {
            const or_entry *en = &t->entries[eid[i]];
            or_hit r = eval_entry(b, closest, en->nodes, en->len, O[3 * i], O[3 * i + 1],
                                  O[3 * i + 2], D[3 * i], D[3 * i + 1], D[3 * i + 2], tmins[i],
                                  tmaxs[i]);
            ob += r.boxes; ovt += r.tris;
            evbox[i] = r.boxes;
            if (r.found) {
                tp++;
                int64_t x = (int64_t)b->depth[r.leaf] + 1 - r.boxes;
                est += x > 0 ? x : 0;
                ofound[i] = 1; ot_[i] = r.t; oslot[i] = (int32_t)r.slot; oleaf[i] = (int32_t)r.leaf;
                continue;
            }
        }
        unres[nu++] = i;
    }
    int64_t resolved = 0;
    int stopped = 0;
    for (int round = 0; round <= g_fast_rounds && nu > 0; round++) {
        if (round >= 1 && g_fast_stop_div > 0 && resolved * g_fast_stop_div < n) stopped = 1;
        resolved = 0;
        const int last = round == g_fast_rounds || stopped;
        for (int64_t h = 0; h < lead.cap; h++) lead.ray[h] = -1;
        int64_t keep = 0;
        for (int64_t u = 0; u < nu; u++) {
            const int64_t i = unres[u];
            int64_t *ls = km_slot(&lead, keys, keys[i]);
            const int is_leader = last || *ls < 0;
            if (*ls < 0) *ls = i;
            const double ox = O[3 * i], oy = O[3 * i + 1], oz = O[3 * i + 2];
            const double dx = D[3 * i], dy = D[3 * i + 1], dz = D[3 * i + 2];
            int64_t *hs = km_slot(&hit, keys, keys[i]);
            if (is_leader) {   /* traced: its entry exists iff listed or an earlier trace hit */
                if (eid[i] >= 0 || *hs >= 0) fp++;
                else neg++;
                or_hit h = trace_one(b, closest, ox, oy, oz, dx, dy, dz, tmins[i], tmaxs[i], 0);
                bb += h.boxes; bt += h.tris;
                traced[i] = 1;
                if (h.found) {
                    ofound[i] = 1; ot_[i] = h.t; oslot[i] = (int32_t)h.slot; oleaf[i] = (int32_t)h.leaf;
                    if (*hs < 0) *hs = i;
                    /* a node new to the entry becomes visible to later rays */
                    const int32_t node = b->anc[h.leaf];
                    int listed = 0;
                    if (eid[i] >= 0) {
                        const or_entry *en = &t->entries[eid[i]];
                        for (int64_t k = 0; k < en->len && !listed; k++) listed = en->nodes[k] == node;
                    }
                    int64_t *as = km_slot(&added, keys, keys[i]);
                    for (int64_t r = *as; r >= 0 && !listed; r = nxt[r])
                        listed = b->anc[oleaf[r]] == node;
                    if (!listed) { nxt[i] = *as; *as = i; }
                }
                continue;
            }
            /* follower of this round's leader L: L's node, if L appended one */
            const int64_t L = *ls;
            int64_t *as = km_slot(&added, keys, keys[i]);
            if (*as == L) {
                const int32_t node = b->anc[oleaf[L]];
                or_hit r = trace_one(b, closest, ox, oy, oz, dx, dy, dz, tmins[i], tmaxs[i], node);
                ob += r.boxes; ovt += r.tris;
                evbox[i] += r.boxes;
                if (r.found) {
                    tp++;
                    resolved++;
                    int64_t x = (int64_t)b->depth[r.leaf] + 1 - evbox[i];
                    est += x > 0 ? x : 0;
                    ofound[i] = 1; ot_[i] = r.t; oslot[i] = (int32_t)r.slot; oleaf[i] = (int32_t)r.leaf;
                    continue;
                }
            }
            unres[keep++] = i;
        }
        nu = keep;
        if (last) break;
    }
    int rc = OR_OK;
    for (int64_t i = 0; i < n && rc == OR_OK; i++)
        if (traced[i] && ofound[i] && t_record(t, keys[i], b->anc[oleaf[i]]) < 0) rc = OR_CAPACITY;
    free(eid); free(evbox); free(traced); free(unres); free(lead.ray); free(hit.ray);
    free(added.ray); free(nxt);
    stats[S_TP] += tp; stats[S_FP] += fp; stats[S_NEG] += neg;
    stats[S_OB] += ob; stats[S_OT] += ovt; stats[S_EST] += est;
    stats[S_BB] += bb; stats[S_BT] += bt;
    return rc;
}

/* hrpp/tracer.py:343-371.  mode: 0 baseline, 1 limit, 2 live, 3 fast.
 * Outputs (found,t,slot,leaf) are the rays shading would use (base for
 * baseline/limit, live hits for live).  base_* (u,v,box,tri,vis) optional.
 * keys_out optional.  anc = go-up LUT of the table's level (NULL in baseline). */
int or_trace_wave(BVH_ARGS, const int32_t *anc, or_table *table, int p, int mode, int closest,
                  const float *O, const float *D, const double *tmins, const double *tmaxs,
                  int64_t n, uint8_t *found, double *t, int32_t *slot, int32_t *leaf,
                  double *u, double *v, int64_t *box, int64_t *tri, int64_t *vis,
                  uint64_t *keys_out, int64_t *stats, int8_t *log_cls, int64_t *log_eval_box,
                  double *log_pred_t, int64_t *log_pred_slot, int nthreads) {
    BVH_INIT(bv);
    bv.anc = anc;
    stats[S_RAYS] += n;                    /* tracer.py:350 (before hashing) */
    uint64_t *keys = NULL;
    int rc = OR_OK;
    if (mode != 0) {
        keys = keys_out ? keys_out : (uint64_t *)malloc(sizeof(uint64_t) * (n > 0 ? n : 1));
        rc = or_hash_rays(O, D, n, p, keys);
        if (rc != OR_OK) goto done;
    }
    if (mode == 2) {
        rc = consult_live(table, &bv, closest, keys, O, D, tmins, tmaxs, n, stats, found, t, slot,
                          leaf, NULL, 0);
        goto done;
    }
    if (mode == 3) {
        rc = fast_wave(table, &bv, closest, keys, O, D, tmins, tmaxs, n, stats, found, t, slot,
                       leaf);
        goto done;
    }
    {
        int64_t *bx = box ? box : (int64_t *)malloc(sizeof(int64_t) * (n > 0 ? n : 1));
        int64_t *tr = tri ? tri : (int64_t *)malloc(sizeof(int64_t) * (n > 0 ? n : 1));
        int64_t *vs = vis ? vis : (int64_t *)malloc(sizeof(int64_t) * (n > 0 ? n : 1));
        or_trace_batch(bmin, bmax, left, right, axis, first, count, tv0, tv1, tv2, depth, n_nodes,
                       n_tris, closest, O, D, tmins, tmaxs, 0, n, found, t, slot, leaf,
                       closest ? u : NULL, closest ? v : NULL, bx, tr, vs, nthreads);
        int64_t sb = 0, st = 0;
        for (int64_t i = 0; i < n; i++) { sb += bx[i]; st += tr[i]; }
        stats[S_BB] += sb; stats[S_BT] += st;
        if (mode == 1)
            rc = consult_limit(table, &bv, closest, keys, O, D, tmins, tmaxs, found, t, leaf, bx, n,
                               stats, log_cls, log_eval_box, log_pred_t, log_pred_slot, NULL, 0);
        if (!box) free(bx);
        if (!tri) free(tr);
        if (!vis) free(vs);
    }
done:
    if (keys && keys != keys_out) free(keys);
    return rc;
}

/* The same wave with the consult spread over `shards` host threads by key:
 * thread s owns the keys with (mix64(key) >> 32) % shards == s and runs the
 * reference's sequential loop over its rays, in ray order, against its own
 * table tables[s].  A key's entry is read and written only by rays with
 * that key (hrpp/tracer.py:233-267, :295-331), so hits and statistics are
 * those of one table and the union of the shards' tables is that table
 * (the entry cap applies per shard).  Used as the CPU baseline: the
 * reference's consult is single-threaded by design; this is its result
 * computed with all host cores. */
int or_trace_wave_sharded(BVH_ARGS, const int32_t *anc, or_table **tables, int shards, int p,
                          int mode, int closest, const float *O, const float *D,
                          const double *tmins, const double *tmaxs, int64_t n, uint8_t *found,
                          double *t, int32_t *slot, int32_t *leaf, double *u, double *v,
                          int64_t *box, int64_t *tri, int64_t *vis, uint64_t *keys_out,
                          int64_t *stats) {
    if (mode < 1 || mode > 2 || shards < 1 || shards > 65535) return OR_INVALID;
    BVH_INIT(bv);
    bv.anc = anc;
    stats[S_RAYS] += n;
    const int64_t nn = n > 0 ? n : 1;
    uint64_t *keys = keys_out ? keys_out : (uint64_t *)malloc(sizeof(uint64_t) * nn);
    uint16_t *owner = (uint16_t *)malloc(sizeof(uint16_t) * nn);
    int64_t *bx = NULL, *tr = NULL, *vs = NULL;
    int rc = or_hash_rays(O, D, n, p, keys);
    if (rc != OR_OK) goto done;
    for (int64_t i = 0; i < n; i++) owner[i] = (uint16_t)((mix64(keys[i]) >> 32) % (uint64_t)shards);
    if (mode == 1) {
        bx = box ? box : (int64_t *)malloc(sizeof(int64_t) * nn);
        tr = tri ? tri : (int64_t *)malloc(sizeof(int64_t) * nn);
        vs = vis ? vis : (int64_t *)malloc(sizeof(int64_t) * nn);
        or_trace_batch(bmin, bmax, left, right, axis, first, count, tv0, tv1, tv2, depth, n_nodes,
                       n_tris, closest, O, D, tmins, tmaxs, 0, n, found, t, slot, leaf,
                       closest ? u : NULL, closest ? v : NULL, bx, tr, vs, shards);
        int64_t sb = 0, st = 0;
        for (int64_t i = 0; i < n; i++) { sb += bx[i]; st += tr[i]; }
        stats[S_BB] += sb; stats[S_BT] += st;
    }
    int64_t *part = (int64_t *)calloc((size_t)shards * S_N, sizeof(int64_t));
    int *rcs = (int *)calloc((size_t)shards, sizeof(int));
#ifdef _OPENMP
#pragma omp parallel for schedule(dynamic, 1) num_threads(shards)
#endif
    for (int s = 0; s < shards; s++) {
        if (mode == 2)
            rcs[s] = consult_live(tables[s], &bv, closest, keys, O, D, tmins, tmaxs, n,
                                  part + (size_t)s * S_N, found, t, slot, leaf, owner, (uint16_t)s);
        else
            rcs[s] = consult_limit(tables[s], &bv, closest, keys, O, D, tmins, tmaxs, found, t,
                                   leaf, bx, n, part + (size_t)s * S_N, NULL, NULL, NULL, NULL,
                                   owner, (uint16_t)s);
    }
    for (int s = 0; s < shards; s++) {
        for (int k = 1; k < S_N; k++) stats[k] += part[(size_t)s * S_N + k];
        if (rcs[s] != OR_OK) rc = rcs[s];
    }
    free(part);
    free(rcs);
done:
    if (bx && bx != box) free(bx);
    if (tr && tr != tri) free(tr);
    if (vs && vs != vis) free(vs);
    if (keys != keys_out) free(keys);
    free(owner);
    return rc;
}

/* PredictorTable.predict (hrpp/predictor.py:167-192) for a batch of rays
 * against a FROZEN table.  cls: 0 TP, 1 FP, 2 NEG. */
int or_predict_batch(BVH_ARGS, or_table *table, int closest, const uint64_t *keys,
                     const float *O, const float *D, const double *tmins, const double *tmaxs,
                     int64_t n, int8_t *cls, double *t, int32_t *slot, int32_t *leaf, double *u,
                     double *v, int64_t *box, int64_t *tri, int64_t *vis, int64_t *est) {
    BVH_INIT(bv);
    for (int64_t i = 0; i < n; i++) {
        int64_t e = t_lookup(table, keys[i]);
        if (e < 0) {
            cls[i] = 2; t[i] = INFINITY; slot[i] = -1; leaf[i] = -1; u[i] = 0; v[i] = 0;
            box[i] = 0; tri[i] = 0; vis[i] = 0; est[i] = 0;
            continue;
        }
        or_hit r = eval_entry(&bv, closest, table->entries[e].nodes, table->entries[e].len,
                              O[3 * i], O[3 * i + 1], O[3 * i + 2], D[3 * i], D[3 * i + 1],
                              D[3 * i + 2], tmins[i], tmaxs[i]);
        cls[i] = r.found ? 0 : 1;
        t[i] = r.t; slot[i] = r.slot; leaf[i] = r.leaf; u[i] = r.u; v[i] = r.v;
        box[i] = r.boxes; tri[i] = r.tris; vis[i] = r.visited;
        if (r.found) {
            int64_t x = (int64_t)depth[r.leaf] + 1 - r.boxes;
            est[i] = x > 0 ? x : 0;
        } else {
            est[i] = 0;
        }
    }
    return OR_OK;
}

int or_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
