/*
 * hrpp_b200.h -- C ABI of the B200-native HRPP hot path (sm_100a).
 *
 * Drop-in boundary for the reference package `hrpp` 0.1.0 (arXiv 1910.01304
 * limit-study workbench).  The reference's native seam is the set of numba
 * kernels in hrpp/kernels.py plus the Python wave driver _trace_wave in
 * hrpp/tracer.py; each entry point below cites the reference interface it
 * replaces.  The Python package paper_1910_01304_b200 binds this library with
 * ctypes and mirrors the reference's public names.
 *
 * Conventions
 *  - Plain pointers and sizes; no torch or CUDA types in the signatures.
 *    `stream` is a cudaStream_t passed as void* (NULL = legacy default).
 *  - Ray and output arrays may be DEVICE pointers (zero-copy) or HOST
 *    pointers (pageable or pinned); the library detects which and stages
 *    host arrays through its own device workspace.  All arrays of one call
 *    must be of one kind.  Calls return once results are in place.
 *  - Ray arrays: O and D are (n,3) float32 row-major, tmin/tmax float64 --
 *    exactly the arrays _trace_wave receives (hrpp/tracer.py:429-430,463).
 *  - Status codes map to the reference's exceptions (hrpp/errors.py):
 *      HRPP_OK 0, HRPP_NONFINITE 1 -> NonFiniteInput, HRPP_CAPACITY 2 ->
 *      CapacityExceeded, HRPP_INVALID_ARG 3 -> ValueError, HRPP_CUDA 4 ->
 *      RuntimeError.  hrpp_last_error() gives the message.
 *  - Ownership: the library owns BVH and table device memory behind the
 *    opaque handles; outputs are caller-allocated.
 *  - Threading: a handle must not be used from two host threads at once
 *    (the reference predictor is single-writer).
 */
#ifndef HRPP_B200_H
#define HRPP_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HRPP_OK 0
#define HRPP_NONFINITE 1
#define HRPP_CAPACITY 2
#define HRPP_INVALID_ARG 3
#define HRPP_CUDA 4

#define HRPP_HIT_ANY 0
#define HRPP_CLOSEST_HIT 1

#define HRPP_MODE_BASELINE 0
#define HRPP_MODE_LIMIT 1
#define HRPP_MODE_LIVE 2
/* Sort-free live mode: the live loop of
 * hrpp/tracer.py:295-331 as key-parallel speculation rounds; exact up to the
 * round limit (hrpp_set_fast_rounds), statistics within the tolerance
 * DESIGN.md states beyond it.  Deterministic. */
#define HRPP_MODE_FAST 3

typedef struct hrpp_bvh_s *hrpp_bvh_t;
typedef struct hrpp_table_s *hrpp_table_t;

/* Stats vector: int64[11] in RayKindStats field order (hrpp/metrics.py:38-51):
 * rays, tp, fp, neg, baseline_box_tests, baseline_tri_tests,
 * overhead_box_tests, overhead_tri_tests, skipped_box_tests,
 * skipped_box_tests_estimated, wrong_closest.  Calls ADD into it. */
#define HRPP_STATS_LEN 11

/* Per-wave outputs (all optional = NULL).  found/t/slot/leaf are the hits
 * shading would use: the full-traversal result in baseline and limit mode,
 * the live (predicted-or-full) result in live mode (hrpp/tracer.py:340,371).
 * u, v, box, tri, visited are the baseline arrays (limit/baseline only). */
typedef struct {
  uint8_t *found;
  double *t;
  int32_t *slot;
  int32_t *leaf;
  double *u, *v;
  int64_t *box, *tri, *visited;
  uint64_t *keys;            /* hash keys (limit/live) */
} hrpp_wave_out;

/* Limit-mode OutcomeLog (hrpp/tracer.py:144-153), per ray in wave order.
 * cls 0 = TP, 1 = FP, 2 = NEG; pred_t = inf and pred_slot = -1 unless TP. */
typedef struct {
  int8_t *cls;
  int64_t *eval_box;
  double *pred_t;
  int64_t *pred_slot;
} hrpp_outcome_log;

/* ---- library ------------------------------------------------------------ */
const char *hrpp_last_error(void);
int hrpp_version(void);
/* Number of the library's own kernel launches since load (evidence for
 * bench.py's gpu_launches). */
int64_t hrpp_launch_count(void);
int hrpp_device_count(int *count);

/* ---- ray hash: hrpp/rayhash.py:99-122 (hash_rays, _lane_hash) ----------- */
/* keys[n] <- 48-bit keys at precision p in [1,7].  HRPP_NONFINITE if any
 * component of O or D has an all-ones exponent (rayhash.py:106-108). */
int hrpp_hash_rays(const float *O, const float *D, int64_t n, int p, uint64_t *keys,
                   void *stream);
/* hrpp/rayhash.py:67-78 map_float_to_hash over a float32 array. */
int hrpp_hash_floats(const float *f, int64_t n, int p, uint32_t *out, void *stream);
/* hrpp/rayhash.py:125-147 coarsen_key: 48-bit keys at precision p -> the
 * keys of the same rays at p - 1 (p in [2, 7]), computed per lane on the
 * device (host or device arrays). */
int hrpp_coarsen_keys(const uint64_t *keys, int64_t n, int p, uint64_t *out, void *stream);

/* ---- BVH: hrpp/bvh.py:75-92 (Bvh(...)) and the 10-array kernel ABI of
 * hrpp/bvh.py:126-128, plus parent/depth (predictor) and tri_ids.  Host
 * arrays; copied into the device layout of DESIGN.md. ----------------------- */
int hrpp_bvh_create(const float *bmin, const float *bmax, const int32_t *left,
                    const int32_t *right, const int8_t *axis, const int32_t *first,
                    const int32_t *count, const int32_t *parent, const int32_t *depth,
                    const float *tv0, const float *tv1, const float *tv2,
                    const int32_t *tri_ids, int64_t n_nodes, int64_t n_tris, int device,
                    hrpp_bvh_t *out);
int hrpp_bvh_destroy(hrpp_bvh_t bvh);
/* hrpp/bvh.py:140-151 ancestor_lut -> host int32[n_nodes]. */
int hrpp_bvh_ancestor_lut(hrpp_bvh_t bvh, int go_up_level, int32_t *lut_host);
/* Native binned-SAH builder restating hrpp/bvh.py:184-357 (16 bins, stable
 * median fallback, oversized leaf for coincident centroids).  median_split=1
 * selects the plain median-split builder (BASELINE c1).  Outputs are host
 * arrays sized n_tris (tris) / 2*n_tris (nodes); *n_nodes_out and
 * *max_depth_out receive the sizes.  Returns HRPP_INVALID_ARG for an empty
 * scene (EmptyScene) after degenerate filtering. */
int hrpp_build_bvh(const float *v0, const float *v1, const float *v2, const int32_t *ids,
                   int64_t n_tris, int max_leaf_size, int median_split, float *bmin,
                   float *bmax, int32_t *left, int32_t *right, int8_t *axis, int32_t *first,
                   int32_t *count, int32_t *parent, int32_t *depth, float *tv0, float *tv1,
                   float *tv2, int32_t *tri_ids, int64_t *n_nodes_out, int64_t *n_tris_out,
                   int32_t *max_depth_out);

/* ---- ray generation and spawning on the device (waves stay in HBM) ----- */
/* generate_primary_rays (hrpp/tracer.py:173-211) with unit_floats
 * (hrpp/rng.py:23-31): O, D device (width*height*spp, 3) float32, pixel-major /
 * sample-minor; basis9 = camera (forward, right, up) float64 from
 * Camera.basis (hrpp/tracer.py:84-97); sx, sy = the stratum grid. */
int hrpp_gen_primary(const float *cam_pos, const double *basis9, double tan_half, double aspect,
                     int64_t width, int64_t height, int64_t spp, int64_t sx, int64_t sy,
                     uint64_t seed, int jitter, float *O, float *D, void *stream);
/* Secondary waves from a closest-hit wave's hits (device arrays): hit points
 * offset 1e-4 along the facing geometric normal (hrpp/tracer.py:442-453).
 * shadow_kind 1 = point light light3 (hrpp/tracer.py:456-464), 2 = y-facing
 * square area light centred at light3 with half extent `half` (uniform
 * samples); bounce_kind 1 = mirror (hrpp/tracer.py:488-492), 2 =
 * cosine-weighted diffuse.  Outputs sized n (hits are compacted in ray
 * order); *count_out = number of hits. */
int hrpp_spawn(hrpp_bvh_t bvh, const float *O, const float *D, const uint8_t *found,
               const double *t, const int32_t *slot, int64_t n, int shadow_kind,
               const double *light3, double half, int bounce_kind, uint64_t seed, float *so,
               float *sd, double *s0, double *s1, float *bo, float *bd, double *b0, double *b1,
               int64_t *count_out, void *stream);

/* ---- traversal batch: hrpp/kernels.py:209-248 via hrpp/bvh.py:398-442 --- */
/* kind = HRPP_CLOSEST_HIT or HRPP_HIT_ANY; start = subtree root (0 = root).
 * out->u/v ignored for hit-any (the reference batch has none). */
int hrpp_trace_batch(hrpp_bvh_t bvh, int kind, const float *O, const float *D,
                     const double *tmin, const double *tmax, int32_t start, int64_t n,
                     hrpp_wave_out *out, void *stream);

/* ---- predictor table: hrpp/predictor.py:117-211 ------------------------ */
int hrpp_table_create(int precision, int go_up_level, int kind, int64_t max_entries,
                      int device, hrpp_table_t *out);
int hrpp_table_destroy(hrpp_table_t table);
int hrpp_table_clear(hrpp_table_t table);
/* the same, stream-ordered on `stream` (host returns at once) */
int hrpp_table_clear_async(hrpp_table_t table, void *stream);
/* entries, stored nodes, max nodes per entry (predictor.py:135-141). */
int hrpp_table_info(hrpp_table_t table, int64_t *entries, int64_t *stored, int64_t *max_len);
/* predictor.py:147-160 record, batched with sequential semantics (ray order):
 * inserted[i] = whether record i grew its entry.  HRPP_CAPACITY if the new
 * keys would exceed max_entries (the table is then left unchanged). */
int hrpp_table_record(hrpp_table_t table, const uint64_t *keys, const int32_t *nodes,
                      int64_t n, uint8_t *inserted, void *stream);
/* predictor.py:143-145 lookup: *len_out = entry length (0 = absent); up to
 * cap node ids copied to nodes_host in insertion order. */
int hrpp_table_lookup(hrpp_table_t table, uint64_t key, int32_t *nodes_host, int64_t cap,
                      int64_t *len_out);
/* dump order (predictor.py:207-211): keys sorted ascending, CSR node lists.
 * Host arrays: keys[entries], offsets[entries+1], nodes[stored]. */
int hrpp_table_export(hrpp_table_t table, uint64_t *keys, int64_t *offsets, int32_t *nodes);

/* Multi-GPU support: in deferred mode a wave does
 * not modify the table; its append records (key, node, triggering ray index
 * within the wave) are kept, sorted by ray index, and read with
 * hrpp_table_pending (host or device pointers).  The caller all-gathers the
 * records of every rank's contiguous ray block and applies them in global
 * ray order with hrpp_table_record, which leaves every rank's table
 * identical.  With one rank this equals the direct commit. */
int hrpp_table_set_deferred(hrpp_table_t table, int on);
int hrpp_table_pending(hrpp_table_t table, uint64_t *keys, int32_t *nodes, int32_t *rays,
                       int64_t cap, int64_t *count);
/* Exact multi-GPU mode (key sharding): owner of key k among
 * `world` ranks = (mix64(k) >> 32) % world.  perm (device int32[n]) receives
 * the local rays grouped by owner, ray order kept within each owner (stable);
 * counts (int64[world], host or device) the rays per owner -- with a device
 * array the call does not wait for the device.  After an all-to-all of the
 * permuted rays every owner holds all rays of its keys in global ray order
 * and its consult is the single-GPU consult restricted to those keys, so
 * hits, statistics and the union of the tables equal one GPU's at any world
 * size.  keys: device uint64[n] from hrpp_hash_rays. */
int hrpp_partition_by_owner(const uint64_t *keys, int64_t n, int world, int32_t *perm,
                            int64_t *counts, void *stream);
/* Key-sharding exchange rows (device arrays; one all-to-all each way):
 * a ray row is 40 B {O.xyz f32, D.xyz f32, tmin f64, tmax f64}, gathered in
 * `perm` order; a hit row is 24 B {t f64, slot i32, leaf i32, found u8, pad},
 * scattered back to positions perm[k]. */
int hrpp_pack_rays(const int32_t *perm, int64_t n, const float *O, const float *D,
                   const double *tmin, const double *tmax, void *rows, void *stream);
int hrpp_unpack_rays(const void *rows, int64_t n, float *O, float *D, double *tmin,
                     double *tmax, void *stream);
int hrpp_pack_hits(int64_t n, const uint8_t *found, const double *t, const int32_t *slot,
                   const int32_t *leaf, void *rows, void *stream);
int hrpp_unpack_hits(const void *rows, const int32_t *perm, int64_t n, uint8_t *found,
                     double *t, int32_t *slot, int32_t *leaf, void *stream);

/* ---- predict: hrpp/predictor.py:167-192 over a batch, frozen table ------ */
/* cls 0 TP / 1 FP / 2 NEG; t/slot/leaf/u/v of the entry result (t = inf for
 * NEG, the any-hit miss convention otherwise); box/tri/visited = overhead
 * counters; est = skipped_box_tests (live lower bound). */
int hrpp_predict_batch(hrpp_bvh_t bvh, hrpp_table_t table, const uint64_t *keys,
                       const float *O, const float *D, const double *tmin, const double *tmax,
                       int64_t n, int8_t *cls, double *t, int32_t *slot, int32_t *leaf,
                       double *u, double *v, int64_t *box, int64_t *tri, int64_t *visited,
                       int64_t *est, void *stream);

/* ---- the wave: hrpp/tracer.py:343-371 (_trace_wave) with _consult_limit
 * (:217-275) and _consult_live (:278-340) ---------------------------------
 * mode = HRPP_MODE_{BASELINE,LIMIT,LIVE}; closest = 1 for hit-all rays.
 * table may be NULL in baseline mode and must match `closest` otherwise.
 * Deterministic ray-ordered semantics: identical tables, stats, outputs and
 * outcome log to the reference's sequential loop.  log may be NULL. */
int hrpp_trace_wave(hrpp_bvh_t bvh, hrpp_table_t table, int mode, int closest,
                    const float *O, const float *D, const double *tmin, const double *tmax,
                    int64_t n, hrpp_wave_out *out, hrpp_outcome_log *log, int64_t *stats,
                    void *stream);

/* Per-stage CUDA-event profiler: when enabled, each stage the library
 * launches is bracketed by events on its own stream.  Stages (index):
 * 0 hash, 1 full traversal batch, 2 live fallback traversal (queue),
 * 3 grouping (radix sort by key + segment heads), 4 consult, 5 table commit,
 * 6 other.  hrpp_profile_read synchronizes the device and returns the
 * accumulated milliseconds and stage counts (number of stages = 7). */
int hrpp_profile_enable(int on);
/* Record only the stages whose bit is set in `mask` (bit = stage index);
 * 0 disables.  Fewer events keep the profiler out of the timed path. */
int hrpp_profile_stages(unsigned mask);
int hrpp_profile_read(double *ms, int64_t *counts, int n, int reset);

/* Live-mode speculation policy (rounds of exact per-key scan before the
 * speculative round).  Default 0.  Affects speed only, never results. */
int hrpp_set_live_rounds(int rounds);
/* Fast mode's speculation policy: at most `rounds` rounds (default 8), and
 * no further round once one resolved fewer than n / stop_div of the wave's
 * n rays (default 32; 0 = never stop early).  Every ray decided within the
 * rounds sees exactly the appends of the rays before it; the rest are
 * traced.  Affects statistics within the stated tolerance, never found
 * flags or table_entries. */
int hrpp_set_fast_rounds(int rounds, int stop_div);
/* Key segments with at most `len` rays are replayed by one lane, longer ones
 * by a whole warp (default 32).  Affects speed only, never results. */
int hrpp_set_consult_short(int len);

#ifdef __cplusplus
}
#endif
#endif /* HRPP_B200_H */
