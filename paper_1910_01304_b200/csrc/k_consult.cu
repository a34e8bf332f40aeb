// k_consult.cu -- the predictor consult of one wave, exact in ray order.
//
// The reference consults and trains the table one ray at a time in wave
// order (hrpp/tracer.py:233-267 limit, :295-331 live).  A table entry is
// read and written only by rays carrying its key, so the loop is
// independent per key; after a stable sort by key the wave is a set of key
// segments, each replayed in ray order.  The work splits in two:
//
//  1. k_eval0 -- ray-parallel, one thread per sorted position: evaluate the
//     entry as it stood at the start of the wave (hrpp/kernels.py:251-297)
//     for every ray.  A ray that hits here is a true positive whatever the
//     wave appends later (entries only grow and every node is evaluated).
//  2. k_replay -- per key segment, in ray order: fold the nodes appended
//     earlier in this wave into each ray's running result, classify
//     TP / FP / NEG, and append anc[leaf] (de-duplicated) after each non-TP
//     ray with a hit.  Short segments run one lane each, long ones on a
//     whole warp whose lanes hold 32 consecutive rays (a ballot finds the
//     next non-TP ray).
//
// Limit mode knows every full-traversal result up front.  Live mode needs
// the full result of each non-TP ray: by default (g_live_rounds = 0) every
// ray that is not a TP against the wave-start entry is traced (one dense,
// ray-ordered traversal launch) before a single replay.  With rounds > 0 the
// replay suspends at the first ray of a segment whose full result is
// unknown, the queue is traced and the replay resumes; after `rounds` exact
// rounds one speculative round traces every unresolved ray.  Either way the
// results are exact: speculation only costs traversals.
#include <cub/cub.cuh>
#include <cstring>

#include "../../include/hrpp_b200.h"
#include "hrpp_internal.h"

namespace hrpp {

#ifndef HRPP_EARLY_TRACE
#define HRPP_EARLY_TRACE 1
#endif

#ifndef HRPP_SORT_PRIO
#define HRPP_SORT_PRIO 0
#endif
#ifndef HRPP_LEADER_FIRST
#define HRPP_LEADER_FIRST 0
#endif

int g_live_rounds = 0;
int g_consult_short = 32;  // segments up to this many rays are replayed by one lane

enum { S_RAYS, S_TP, S_FP, S_NEG, S_BB, S_BT, S_OB, S_OT, S_SK, S_EST, S_WRONG };
constexpr int S_START_TP = 14;  // (library-internal) TPs against the wave-start table

// Running eval_entry result of one ray (by ray index): 32 bytes, two 16-B
// accesses.  `applied` = number of entry nodes already folded.
struct __align__(16) RayState {
  double t;
  int32_t slot, leaf;
  int32_t boxes, tris;
  int32_t applied;
  int32_t found;
};

struct ConsultArgs {
  const DNode* nodes;
  const DTri* tris;
  const int32_t* depth;
  const int32_t* anc;
  const float* O;
  const float* D;
  const double* tmin;
  const double* tmax;
  const unsigned long long* skeys;
  const int32_t* sidx;
  const int32_t* seg_start;
  const int32_t* seg_id;
  const int* nsegs;
  const Bucket* idx;
  uint64_t mask;
  const int64_t* e_off;
  const int32_t* e_len;
  const int32_t* arena;
  // per segment
  int32_t* seg_eid;
  int64_t* seg_exoff;
  int32_t* seg_exlen;
  int32_t* seg_napp;
  int32_t* seg_cursor;
  int32_t* app;      // appended nodes of segment s live at app[seg_start[s] ...]
  int32_t* app_ray;  // ray index that triggered each append (deferred mode)
  RayState* state;   // per ray index
  int32_t* seg_of_ray;  // per ray index: key segment
  // full-traversal results by ray index (baseline in limit mode)
  const uint8_t* f_found;
  const double* f_t;
  const int32_t* f_slot;
  const int32_t* f_leaf;
  const int64_t* f_box;
  const int64_t* f_tri;
  const int32_t* f_box32;  // live: the fallback traversal's counts
  const int32_t* f_tri32;
  const uint8_t* f_known;  // live only
  uint8_t* f_known_clear;  // live: eval0 zeroes it (one pass fewer)
  // outputs by ray index
  uint8_t* o_found;
  double* o_t;
  int32_t* o_slot;
  int32_t* o_leaf;
  int8_t* log_cls;
  int64_t* log_eval_box;
  double* log_pred_t;
  int64_t* log_pred_slot;
  unsigned long long* stats;
  uint8_t* need;  // live: rays (by index) whose full traversal is needed next
  int32_t* seg_f1;  // first sorted position of the segment that appends (or INT_MAX)
  int spec;       // live replay: 0 mark the first unknown ray, 2 mark every unresolved ray
  int sparse_state;  // 1: eval0 stores no state for rays whose key had no entry
  const int* err;
};

constexpr unsigned kFull = 0xffffffffu;

__device__ __forceinline__ void load_state(const ConsultArgs& a, int32_t pos, Hit& acc,
                                           int32_t& applied) {
  const RayState s = a.state[pos];
  acc.found = s.found != 0;
  acc.t = s.t;
  acc.slot = s.slot;
  acc.leaf = s.leaf;
  acc.boxes = s.boxes;
  acc.tris = s.tris;
  applied = s.applied;
}

__device__ __forceinline__ void store_state(const ConsultArgs& a, int32_t pos, const Hit& acc,
                                            int32_t applied) {
  RayState s;
  s.t = acc.t;
  s.slot = acc.slot;
  s.leaf = acc.leaf;
  s.boxes = acc.boxes;
  s.tris = acc.tris;
  s.applied = applied;
  s.found = acc.found;
  a.state[pos] = s;
}

// The state of a ray whose key had no entry at the wave start is the empty
// entry result; with sparse_state it is never materialised.
template <bool CLOSEST>
__device__ __forceinline__ void get_state(const ConsultArgs& a, int32_t idx, int32_t ex_len,
                                          Hit& acc, int32_t& applied) {
  if (a.sparse_state && ex_len == 0) {
    acc = empty_entry_result(CLOSEST);
    applied = 0;
  } else {
    load_state(a, idx, acc, applied);
  }
}

struct Tally {
  long long tp = 0, fp = 0, neg = 0, ob = 0, ot = 0, sk = 0, est = 0, wr = 0, bb = 0, bt = 0;
};

// Add a warp's tallies into the wave counters (for kernels whose warps
// finish at very different times: no block barrier holds finished warps).
__device__ __forceinline__ void flush_tally_warp(const Tally& c, unsigned long long* stats) {
  const long long v[10] = {c.tp, c.fp, c.neg, c.bb, c.bt, c.ob, c.ot, c.sk, c.est, c.wr};
  const int slot[10] = {S_TP, S_FP, S_NEG, S_BB, S_BT, S_OB, S_OT, S_SK, S_EST, S_WRONG};
#pragma unroll
  for (int k = 0; k < 10; k++) {
    const long long w = warp_sum(v[k]);
    if ((threadIdx.x & 31) == 0 && w) atomicAdd(stats + slot[k], (unsigned long long)w);
  }
}

// Add a block's tallies into the wave counters: warp sums, then one atomic
// per counter per block (per-warp atomics on 10 shared addresses serialised
// in L2).  Every thread of the block must call it.
__device__ __forceinline__ void flush_tally(const Tally& c, unsigned long long* stats) {
  __shared__ long long part[10][8];  // <= 8 warps per block (callers: 128 / 256 threads)
  const long long v[10] = {c.tp, c.fp, c.neg, c.bb, c.bt, c.ob, c.ot, c.sk, c.est, c.wr};
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
#pragma unroll
  for (int k = 0; k < 10; k++) {
    const long long w = warp_sum(v[k]);
    if (lane == 0) part[k][warp] = w;
  }
  __syncthreads();
  if (threadIdx.x < 10) {
    const int slot[10] = {S_TP, S_FP, S_NEG, S_BB, S_BT, S_OB, S_OT, S_SK, S_EST, S_WRONG};
    long long sum = 0;
    for (int w = 0; w < nw; w++) sum += part[threadIdx.x][w];
    if (sum) atomicAdd(stats + slot[threadIdx.x], (unsigned long long)sum);
  }
}

// The entry's j-th node: stored list first, then this wave's appends.
__device__ __forceinline__ int32_t entry_node(const ConsultArgs& a, int64_t ex_off,
                                              int32_t ex_len, const int32_t* app, int32_t j) {
  return j < ex_len ? a.arena[ex_off + j] : app[j - ex_len];
}

// Fold entry nodes [from, L) into acc: eval_entry_{closest,any}, resumable.
template <bool CLOSEST, int STACK>
__device__ __forceinline__ void catch_up(const ConsultArgs& a, const Ray& r, Hit& acc, int32_t from,
                                      int32_t L, int64_t ex_off, int32_t ex_len,
                                      const int32_t* app) {
  for (int32_t j = from; j < L; j++) {
    if (!CLOSEST && acc.found) break;  // eval_entry_any stops at the first hit
    fold_entry<CLOSEST>(acc, trace_from<CLOSEST, STACK>(a.nodes, a.tris, r,
                                                        entry_node(a, ex_off, ex_len, app, j)));
  }
}

template <bool CLOSEST, bool LIVE>
__device__ __forceinline__ void commit_tp(const ConsultArgs& a, Tally& c, int32_t idx,
                                          const Hit& acc) {
  c.tp++;
  c.ob += acc.boxes;
  c.ot += acc.tris;
  const int64_t x = (int64_t)a.depth[acc.leaf] + 1 - acc.boxes;
  c.est += x > 0 ? x : 0;
  if (LIVE) {
    a.o_found[idx] = 1;
    a.o_t[idx] = acc.t;
    a.o_slot[idx] = acc.slot;
    a.o_leaf[idx] = acc.leaf;
  } else {
    c.sk += a.f_box[idx] - acc.boxes;
    if (CLOSEST && acc.t > a.f_t[idx] + kWrongClosestEps) c.wr++;
    if (a.log_cls) {
      a.log_cls[idx] = 0;
      a.log_eval_box[idx] = acc.boxes;
      a.log_pred_t[idx] = acc.t;
      a.log_pred_slot[idx] = acc.slot;
    }
  }
}

template <bool LIVE>
__device__ __forceinline__ void commit_miss(const ConsultArgs& a, Tally& c, int32_t idx,
                                            const Hit& acc, bool neg) {
  if (neg) c.neg++;
  else c.fp++;
  c.ob += acc.boxes;
  c.ot += acc.tris;
  if (LIVE) {  // the outputs already hold the full traversal (written by it)
    c.bb += a.f_box32[idx];
    c.bt += a.f_tri32[idx];
  } else if (a.log_cls) {
    a.log_cls[idx] = neg ? 2 : 1;
    a.log_eval_box[idx] = acc.boxes;
    a.log_pred_t[idx] = __longlong_as_double(0x7ff0000000000000LL);
    a.log_pred_slot[idx] = -1;
  }
}

// ---------------------------------------------------------------------------
// stage 1: per segment entry lookup, then per ray wave-start evaluation
// ---------------------------------------------------------------------------

// Minimum resident 128-thread blocks per SM (register caps) per kernel family.
#ifndef HRPP_EVAL_MINB
#define HRPP_EVAL_MINB 6  // measured: consult -30 us per frame vs uncapped
#endif
#ifndef HRPP_FIN_MINB
#define HRPP_FIN_MINB 12  // 40 registers: a fuller SM for this latency-bound walk
#endif
#ifndef HRPP_FIN_GRID
#define HRPP_FIN_GRID 12  // k_finalize blocks per SM (grid-stride over rays)
#endif
#ifndef HRPP_REPLAY_MINB
#define HRPP_REPLAY_MINB 6  // 80 registers (measured: consult 4.66 -> 4.11 ms on c2)
#endif
#ifndef HRPP_FIN_BS
#define HRPP_FIN_BS 128  // k_finalize block size
#endif
// flush_tally keeps one partial per warp of the block in part[10][8]
static_assert(HRPP_FIN_BS % 32 == 0 && HRPP_FIN_BS <= 256, "k_finalize: at most 8 warps");
#ifndef HRPP_FA_BS
#define HRPP_FA_BS 256  // k_first_append block size
#endif
#ifndef HRPP_EVAL_BS
#define HRPP_EVAL_BS 128  // k_eval0 block size (32 measured slower)
#endif
#ifndef HRPP_REPLAY_BS
#define HRPP_REPLAY_BS 32  // k_replay_group block size (warps take tickets on their own)
#endif

__global__ void k_seg_lookup(ConsultArgs a, int64_t n) {
  const int ns = *a.nsegs;
  for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < ns;
       s += (int64_t)gridDim.x * blockDim.x) {
    const int32_t beg = a.seg_start[s];
    const int32_t eid = index_lookup(a.idx, a.mask, a.skeys[beg]);
    a.seg_eid[s] = eid;
    a.seg_exoff[s] = eid >= 0 ? a.e_off[eid] : 0;
    a.seg_exlen[s] = eid >= 0 ? a.e_len[eid] : 0;
    a.seg_napp[s] = 0;
    a.seg_cursor[s] = beg;
    a.seg_f1[s] = 0x7fffffff;
  }
}

// ---------------------------------------------------------------------------
// stage 1b (all full results known): rays up to and including the first ray
// of their segment that appends see exactly the wave-start entry, so they
// are classified ray-parallel; only the rest of each segment is replayed.
// ---------------------------------------------------------------------------

__device__ __forceinline__ bool in_list(const ConsultArgs& a, int64_t off, int32_t len,
                                        int32_t node) {
  for (int32_t k = 0; k < len; k++)
    if (a.arena[off + k] == node) return true;
  return false;
}

// The stable sort keeps rays of one key in ray order, so within a segment
// "first in the replay" is "smallest ray index".
__global__ void k_first_append(ConsultArgs a, int64_t n) {
  if (*a.err) return;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t s = a.seg_of_ray[i];
    const int32_t ex_len = a.seg_exlen[s];
    if (ex_len > 0 && a.state[i].found) continue;  // TP against the wave-start entry
    if (a.f_known && !a.f_known[i]) continue;  // (live) no full result: never a first append
    // a full result's leaf is -1 exactly when nothing was found (k_trace), so
    // the found flags need no read of their own
    const int32_t lf = a.f_leaf[i];
    if (lf < 0) continue;
    // (no entry: every hit appends -- skip the ancestor read)
    if (ex_len == 0 || !in_list(a, a.seg_exoff[s], ex_len, a.anc[lf]))
      atomicMin(a.seg_f1 + s, (int32_t)i);
  }
}

template <bool CLOSEST, bool LIVE>
__global__ void __launch_bounds__(HRPP_FIN_BS, HRPP_FIN_MINB * 128 / HRPP_FIN_BS)
    k_finalize(ConsultArgs a, int64_t n) {
  if (*a.err) return;
  Tally c;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t s = a.seg_of_ray[i];
    const int32_t f1 = a.seg_f1[s];
    if (i > f1) continue;  // after the first append: replayed
    const int32_t ex_len = a.seg_exlen[s];
    Hit acc;
    int32_t applied;
    get_state<CLOSEST>(a, (int32_t)i, ex_len, acc, applied);
    if (ex_len > 0 && acc.found) commit_tp<CLOSEST, LIVE>(a, c, (int32_t)i, acc);
    else commit_miss<LIVE>(a, c, (int32_t)i, acc, ex_len == 0);
    if (i == f1) {  // the first record(key, anc[leaf]) of this segment
      const int32_t beg = a.seg_start[s];
      a.app[beg] = a.anc[a.f_leaf[i]];
      a.app_ray[beg] = (int32_t)i;
    }
  }
  flush_tally(c, a.stats);
}



// Every ray against the entry as it stood at the start of the wave, fused
// with the ray -> segment scatter: threads walk sorted positions (segment
// data coalesced, one random 4-B store per ray); only rays whose key already
// had an entry read their ray and evaluate it.
template <bool CLOSEST, int STACK>
__global__ void __launch_bounds__(HRPP_EVAL_BS, HRPP_EVAL_MINB * 128 / HRPP_EVAL_BS)
    k_eval0(ConsultArgs a, int64_t n, int mark_need) {
  if (*a.err) return;
  unsigned long long tps = 0;  // wave-start TPs (the early-traversal policy)
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n;
       p += (int64_t)gridDim.x * blockDim.x) {
    const int32_t i = a.sidx[p];
    const int32_t s = a.seg_id[p] - 1;
    a.seg_of_ray[i] = s;
    if (a.f_known_clear) a.f_known_clear[i] = 0;
    const int32_t ex_len = a.seg_exlen[s];
    Hit acc = empty_entry_result(CLOSEST);
    if (ex_len > 0) {
      const Ray r = make_ray(a.O, a.D, a.tmin, a.tmax, i);
      catch_up<CLOSEST, STACK>(a, r, acc, 0, ex_len, a.seg_exoff[s], ex_len, nullptr);
    }
    if (ex_len > 0 || !a.sparse_state) store_state(a, i, acc, ex_len);
    // need[] is preset to 1 (coalesced memset): only the wave-start TPs,
    // rare, are cleared here with a scattered store
    if (mark_need && ex_len > 0 && acc.found) a.need[i] = 0;
    tps += ex_len > 0 && acc.found;
  }
  tps = warp_sum(tps);
  if ((threadIdx.x & 31) == 0 && tps) atomicAdd(a.stats + S_START_TP, tps);
}

// ---------------------------------------------------------------------------
// stage 2: per segment replay in ray order
// ---------------------------------------------------------------------------

// Speculative round: every not-yet-TP ray of the rest of the segment gets its
// full traversal (TP status only grows with the entry, so after this round
// every ray that can still need a full result has one).
template <bool CLOSEST, int STACK>
__device__ void speculate_rest(const ConsultArgs& a, int32_t from, int32_t end, int32_t L,
                               int64_t ex_off, int32_t ex_len, const int32_t* app) {
  for (int32_t j = from; j < end; j++) {
    const int32_t idx = a.sidx[j];
    Hit acc;
    int32_t applied;
    load_state(a, idx, acc, applied);
    if (applied < L && (CLOSEST || !acc.found)) {
      const Ray r = make_ray(a.O, a.D, a.tmin, a.tmax, idx);
      catch_up<CLOSEST, STACK>(a, r, acc, applied, L, ex_off, ex_len, app);
      store_state(a, idx, acc, L);
    }
    if (!(L > 0 && acc.found) && !a.f_known[idx]) a.need[idx] = 1;
  }
}

// One short key segment, replayed by one lane.
template <bool CLOSEST, bool LIVE, int STACK>
__device__ void seg_thread(const ConsultArgs& a, Tally& c, int s, int32_t beg, int32_t end,
                           int32_t cur) {
  const int64_t ex_off = a.seg_exoff[s];
  const int32_t ex_len = a.seg_exlen[s];
  int32_t* app = a.app + beg;
  int32_t napp = a.seg_napp[s];
  int32_t j = cur;
  for (; j < end; j++) {
    const int32_t idx = a.sidx[j];
    Hit acc;
    int32_t applied;
    get_state<CLOSEST>(a, idx, ex_len, acc, applied);
    const int32_t L = ex_len + napp;
    if (applied < L && (CLOSEST || !acc.found)) {
      const Ray r = make_ray(a.O, a.D, a.tmin, a.tmax, idx);
      catch_up<CLOSEST, STACK>(a, r, acc, applied, L, ex_off, ex_len, app);
    }
    if (L > 0 && acc.found) {
      commit_tp<CLOSEST, LIVE>(a, c, idx, acc);
      continue;
    }
    if (LIVE && !a.f_known[idx]) {  // suspend until its full traversal is known
      a.need[idx] = 1;
      store_state(a, idx, acc, L);
      if (a.spec >= 2) speculate_rest<CLOSEST, STACK>(a, j + 1, end, L, ex_off, ex_len, app);
      break;
    }
    commit_miss<LIVE>(a, c, idx, acc, L == 0);
    if (a.f_found[idx]) {  // record(key, anc[leaf]), de-duplicated
      const int32_t node = a.anc[a.f_leaf[idx]];
      bool dup = false;
      for (int32_t k = 0; k < L && !dup; k++) dup = entry_node(a, ex_off, ex_len, app, k) == node;
      if (!dup) {
        app[napp] = node;
        a.app_ray[beg + napp] = idx;
        napp++;
      }
    }
  }
  a.seg_cursor[s] = j;
  a.seg_napp[s] = napp;
}

// One long key segment, replayed by the whole warp: lanes hold 32
// consecutive rays; a ballot finds the next non-TP ray.
template <bool CLOSEST, bool LIVE, int STACK>
__device__ void seg_warp(const ConsultArgs& a, Tally& c, int s, int lane) {
  const int32_t beg = a.seg_start[s], end = a.seg_start[s + 1];
  int32_t tb = a.seg_cursor[s];
  int32_t napp = a.seg_napp[s];
  const int64_t ex_off = a.seg_exoff[s];
  const int32_t ex_len = a.seg_exlen[s];
  int32_t* app = a.app + beg;
  bool suspended = false;
  while (tb < end) {
    const int32_t pos = tb + lane;
    const bool valid = pos < end;
    const int32_t idx = valid ? a.sidx[pos] : 0;
    Hit acc = empty_entry_result(CLOSEST);
    int32_t applied = 0;
    if (valid) get_state<CLOSEST>(a, idx, ex_len, acc, applied);
    int32_t L = ex_len + napp;
    const bool fknown = valid && (!LIVE || a.f_known[idx]);
    int32_t cnode = -1;
    if (fknown && a.f_found[idx]) cnode = a.anc[a.f_leaf[idx]];
    bool inL = false;
    for (int32_t j = 0; j < L; j++) inL |= entry_node(a, ex_off, ex_len, app, j) == cnode;
    Ray r{};
    if (valid) r = make_ray(a.O, a.D, a.tmin, a.tmax, idx);
    if (valid && applied < L && (CLOSEST || !acc.found))
      catch_up<CLOSEST, STACK>(a, r, acc, applied, L, ex_off, ex_len, app);
    applied = L;
    int cursor = 0;
    for (;;) {
      const bool need = valid && lane >= cursor && (L == 0 || !acc.found);
      const unsigned m = __ballot_sync(kFull, need);
      const int f = m ? __ffs(m) - 1 : 32;
      if (valid && lane >= cursor && lane < f) commit_tp<CLOSEST, LIVE>(a, c, idx, acc);
      if (f == 32) break;
      if (LIVE && !__shfl_sync(kFull, fknown, f)) {  // suspend at ray f
        if (lane == f || (a.spec >= 1 && need && !fknown)) a.need[idx] = 1;
        if (valid && lane >= f) store_state(a, idx, acc, applied);
        if (a.spec >= 2) {
          for (int32_t t2 = tb + 32 + lane; t2 < end; t2 += 32) {
            const int32_t i2 = a.sidx[t2];
            Hit a2;
            int32_t ap2;
            load_state(a, i2, a2, ap2);
            if (ap2 < L && (CLOSEST || !a2.found)) {
              const Ray r2 = make_ray(a.O, a.D, a.tmin, a.tmax, i2);
              catch_up<CLOSEST, STACK>(a, r2, a2, ap2, L, ex_off, ex_len, app);
              store_state(a, i2, a2, L);
            }
            if (!(L > 0 && a2.found) && !a.f_known[i2]) a.need[i2] = 1;
          }
        }
        if (lane == 0) {
          a.seg_cursor[s] = tb + f;
          a.seg_napp[s] = napp;
        }
        suspended = true;
        break;
      }
      if (lane == f) commit_miss<LIVE>(a, c, idx, acc, L == 0);
      const int32_t cf = __shfl_sync(kFull, cnode, f);
      const bool inLf = __shfl_sync(kFull, inL, f);
      if (cf >= 0 && !inLf) {  // record(key, anc[leaf]) grows the entry
        const int32_t rf = __shfl_sync(kFull, idx, f);
        if (lane == 0) {
          app[napp] = cf;
          a.app_ray[beg + napp] = rf;
        }
        __syncwarp();
        napp++;
        L++;
        inL |= cnode == cf;
        if (valid && lane > f && (CLOSEST || !acc.found))
          catch_up<CLOSEST, STACK>(a, r, acc, L - 1, L, ex_off, ex_len, app);
        applied = L;
      }
      cursor = f + 1;
    }
    if (suspended) break;
    tb += 32;
  }
  if (lane == 0 && !suspended) {
    a.seg_napp[s] = napp;
    a.seg_cursor[s] = end;
  }
}

// Short segments: thread t owns key segment t.
template <bool CLOSEST, bool LIVE, int STACK>
__global__ void __launch_bounds__(128, HRPP_REPLAY_MINB) k_replay_short(ConsultArgs a, int short_len) {
  if (*a.err) return;
  const int ns = *a.nsegs;
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  Tally c;
  if (s < ns) {
    const int32_t beg = a.seg_start[s], end = a.seg_start[s + 1];
    const int32_t cur = a.seg_cursor[s];
    if (cur < end && end - beg <= short_len) seg_thread<CLOSEST, LIVE, STACK>(a, c, s, beg, end, cur);
  }
  flush_tally_warp(c, a.stats);
}

// Long segments: one warp per segment of the compacted list.
template <bool CLOSEST, bool LIVE, int STACK>
__global__ void __launch_bounds__(128, HRPP_REPLAY_MINB) k_replay_long(ConsultArgs a, const int32_t* list,
                                                     const int* count) {
  if (*a.err) return;
  const int lane = threadIdx.x & 31;
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  const int m = *count;
  Tally c;
  for (int k = w; k < m; k += nw) seg_warp<CLOSEST, LIVE, STACK>(a, c, list[k], lane);
  flush_tally_warp(c, a.stats);
}

// Grouped single-tile replay: a group of G lanes replays one key segment
// with at most G rays left (the rays after its first append), 32/G segments
// per warp.  Within a group this is seg_warp's ballot loop.
template <bool CLOSEST, bool LIVE, int STACK, int G>
__global__ void __launch_bounds__(HRPP_REPLAY_BS, HRPP_REPLAY_MINB * 128 / HRPP_REPLAY_BS)
    k_replay_group(ConsultArgs a, const int32_t* ids, const int* counts, int64_t cap, int K,
                   int* ticket) {
  if (*a.err) return;
  // Persistent warps take 32 / G segments at a time from the class's ticket
  // (each warp on its own: no warp waits for a slower one in its block); the
  // class (list, count) is read on the device, so the host launches without
  // waiting for the class bounds.
  const int32_t* list = ids + (int64_t)K * cap;
  const int count = counts[K];
  const int lane = threadIdx.x & 31;
  const int gl = lane % G, gbase = lane - gl;
  const unsigned gmask = G == 32 ? 0xffffffffu : (((1u << G) - 1u) << gbase);
  Tally c;
  for (;;) {
  int wbase = 0;
  if (lane == 0) wbase = atomicAdd(ticket, 32 / G);
  wbase = __shfl_sync(kFull, wbase, 0);
  if (wbase >= count) break;
  const int gid = wbase + lane / G;
  const bool gvalid = gid < count;
  int s = 0;
  int32_t beg = 0, end = 0, tb = 0, napp = 0, ex_len = 0;
  int64_t ex_off = 0;
  if (gvalid) {
    s = list[gid];
    beg = a.seg_start[s];
    end = a.seg_start[s + 1];
    tb = a.seg_cursor[s];
    napp = a.seg_napp[s];
    ex_off = a.seg_exoff[s];
    ex_len = a.seg_exlen[s];
  }
  int32_t* app = a.app + beg;
  const int32_t pos = tb + gl;
  const bool valid = gvalid && pos < end;
  const int32_t idx = valid ? a.sidx[pos] : 0;
  Hit acc = empty_entry_result(CLOSEST);
  int32_t applied = 0;
  if (valid) get_state<CLOSEST>(a, idx, ex_len, acc, applied);
  int32_t L = ex_len + napp;
  Ray r{};
  if (valid) {
    r = make_ray(a.O, a.D, a.tmin, a.tmax, idx);
    if (applied < L && (CLOSEST || !acc.found))
      catch_up<CLOSEST, STACK>(a, r, acc, applied, L, ex_off, ex_len, app);
  }
  // The record node (anc of the full-traversal leaf) matters only to a ray
  // that is not a TP now -- a TP stays one -- so only those lanes read it
  // (a TP's full result may never have been computed in live mode anyway).
  int32_t cnode = -1;
  bool inL = false;
  if (valid && (L == 0 || !acc.found) && (!LIVE || !a.f_known || a.f_known[idx])) {
    const int32_t lf = a.f_leaf[idx];  // -1: nothing found
    if (lf >= 0) cnode = a.anc[lf];
  }
  if (cnode >= 0) {
    for (int32_t j = 0; j < L; j++) inL |= entry_node(a, ex_off, ex_len, app, j) == cnode;
  }
  // Step from append to append: the rays before the next ray that grows the
  // entry see a constant list, so they are classified together (TP, or
  // FP/NEG without a new node); only an append changes the later rays.
  int cur_l = 0;
  for (;;) {
    const bool pend = valid && gl >= cur_l;
    const bool nontp = pend && (L == 0 || !acc.found);
    const bool grows = nontp && cnode >= 0 && !inL;
    const unsigned m = __ballot_sync(kFull, grows) & gmask;
    const int f = m ? __ffs(m) - 1 - gbase : G;
    if (pend && gl < f) {
      if (nontp) commit_miss<LIVE>(a, c, idx, acc, L == 0);
      else commit_tp<CLOSEST, LIVE>(a, c, idx, acc);
    }
    if (!__any_sync(kFull, f < G)) break;
    const int src = f < G ? gbase + f : lane;
    const int32_t cf = __shfl_sync(kFull, cnode, src);
    const int32_t rf = __shfl_sync(kFull, idx, src);
    if (f < G && gl == f) commit_miss<LIVE>(a, c, idx, acc, L == 0);
    if (f < G && gl == 0) {  // record(key, anc[leaf]) grows the entry
      app[napp] = cf;
      a.app_ray[beg + napp] = rf;
    }
    __syncwarp();
    if (f < G) {
      napp++;
      L++;
      inL |= cnode == cf;
      if (valid && gl > f && (CLOSEST || !acc.found))
        catch_up<CLOSEST, STACK>(a, r, acc, L - 1, L, ex_off, ex_len, app);
    }
    cur_l = f < G ? f + 1 : G;
  }
  if (gvalid && gl == 0) {
    a.seg_napp[s] = napp;
    a.seg_cursor[s] = end;
  }
  }
  flush_tally_warp(c, a.stats);
}

// Very long key segments (coarse hashes: ~10k rays per key at p = 3) would
// leave the GPU nearly idle with one warp each, so a block of kBlockReplay
// threads replays one of them in tiles of kBlockReplay consecutive rays:
// seg_warp's loop with a block-wide "first non-TP ray" (shared-memory
// atomicMin between barriers).  Same order, same appends, same results.
constexpr int kBlockReplay = 256;
#ifndef HRPP_BLOCK_REPLAY_MIN
#define HRPP_BLOCK_REPLAY_MIN 1024  // segments with more rays left get a 256-thread block
#endif
constexpr int kBlockReplayMin = HRPP_BLOCK_REPLAY_MIN;

#ifndef HRPP_BLOCK_MINB
#define HRPP_BLOCK_MINB 2
#endif
#ifndef HRPP_BLOCK32_MINB
#define HRPP_BLOCK32_MINB 32  // warp-per-segment replay: 32-thread blocks per SM
#endif

template <bool CLOSEST, bool LIVE, int STACK, int BS>
__global__ void __launch_bounds__(BS, BS == 32 ? HRPP_BLOCK32_MINB : HRPP_BLOCK_MINB)
    k_replay_block(ConsultArgs a, const int32_t* list, int count, const int* counts,
                   int64_t cap, int K, int* ticket) {
  if (*a.err) return;
  __shared__ int s_f;
  __shared__ int32_t s_cf, s_rf;
  __shared__ int s_k;
  const int tid = threadIdx.x;
  if (counts) {  // class read on the device; persistent blocks take tickets
    list += (int64_t)K * cap;
    count = counts[K];
  }
  Tally c;
  for (int k = blockIdx.x;;) {
    if (counts) {
      __syncthreads();
      if (tid == 0) s_k = atomicAdd(ticket, 1);
      __syncthreads();
      k = s_k;
    }
    if (k >= count) break;
    const int s = list[k];
    const int32_t beg = a.seg_start[s], end = a.seg_start[s + 1];
    int32_t tb = a.seg_cursor[s];
    int32_t napp = a.seg_napp[s];
    const int64_t ex_off = a.seg_exoff[s];
    const int32_t ex_len = a.seg_exlen[s];
    int32_t* app = a.app + beg;
    while (tb < end) {
      const int32_t pos = tb + tid;
      const bool valid = pos < end;
      const int32_t idx = valid ? a.sidx[pos] : 0;
      Hit acc = empty_entry_result(CLOSEST);
      int32_t applied = 0;
      if (valid) get_state<CLOSEST>(a, idx, ex_len, acc, applied);
      int32_t L = ex_len + napp;
      Ray r{};
      if (valid) {
        r = make_ray(a.O, a.D, a.tmin, a.tmax, idx);
        if (applied < L && (CLOSEST || !acc.found))
          catch_up<CLOSEST, STACK>(a, r, acc, applied, L, ex_off, ex_len, app);
      }
      int32_t cnode = -1;  // read only by rays that are not TPs now (see k_replay_group)
      bool inL = false;
      if (valid && (L == 0 || !acc.found) && (!LIVE || !a.f_known || a.f_known[idx])) {
        const int32_t lf = a.f_leaf[idx];  // -1: nothing found
        if (lf >= 0) cnode = a.anc[lf];
      }
      if (cnode >= 0) {
        for (int32_t j = 0; j < L; j++) inL |= entry_node(a, ex_off, ex_len, app, j) == cnode;
      }
      // append to append, as in k_replay_group
      int cursor = 0;
      for (;;) {
        const bool pend = valid && tid >= cursor;
        const bool nontp = pend && (L == 0 || !acc.found);
        const bool grows = nontp && cnode >= 0 && !inL;
        if (tid == 0) s_f = BS;
        __syncthreads();
        if (grows) atomicMin(&s_f, tid);
        __syncthreads();
        const int f = s_f;
        if (pend && tid < f) {
          if (nontp) commit_miss<LIVE>(a, c, idx, acc, L == 0);
          else commit_tp<CLOSEST, LIVE>(a, c, idx, acc);
        }
        if (f == BS) break;
        if (tid == f) {
          commit_miss<LIVE>(a, c, idx, acc, L == 0);
          s_cf = cnode;
          s_rf = idx;
        }
        __syncthreads();
        const int32_t cf = s_cf;
        if (tid == 0) {  // record(key, anc[leaf]) grows the entry
          app[napp] = cf;
          a.app_ray[beg + napp] = s_rf;
        }
        napp++;
        L++;
        inL |= cnode == cf;
        if (valid && tid > f && (CLOSEST || !acc.found))
          fold_entry<CLOSEST>(acc, trace_from<CLOSEST, STACK>(a.nodes, a.tris, r, cf));
        cursor = f + 1;
        __syncthreads();  // s_* reused by the next step
      }
      tb += BS;
      __syncthreads();  // app[] written by thread 0 is read by the next tile
    }
    if (tid == 0) {
      a.seg_napp[s] = napp;
      a.seg_cursor[s] = end;
    }
    if (!counts) k += gridDim.x;
  }
  flush_tally(c, a.stats);
}

// Rays left to replay in each listed segment (longest-first scheduling).
__global__ void k_seg_remaining(ConsultArgs a, const int32_t* list, int m, int32_t* rem) {
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < m; k += gridDim.x * blockDim.x) {
    const int s = list[k];
    rem[k] = a.seg_start[s + 1] - a.seg_cursor[s];
  }
}


// Start of every class in the class-sorted list (9 entries + end).
// Replay cursor and length class of every segment (rays left: 0 done,
// 1..6 for <= 1, 2, 4, 8, 16, 32 rays, 7 up to kBlockReplayMin, 8 longer),
// binning each segment straight into its class list (order within a class
// only affects scheduling): per-block shared counters, one global atomic
// per class per block.
__global__ void __launch_bounds__(256) k_replay_bin(ConsultArgs a, int64_t cap, int32_t* ids,
                                                    int* counts, int* counts_mapped) {
  __shared__ int s_cnt[9], s_base[9];
  if (threadIdx.x < 9) s_cnt[threadIdx.x] = 0;
  __syncthreads();
  const int ns = *a.nsegs;
  const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int k = 0, rank = 0;
  if (s < ns) {
    const int32_t f1 = a.seg_f1[s], end = a.seg_start[s + 1];
    int32_t cur = end;
    if (f1 != 0x7fffffff) {  // sidx ascends within a segment: f1's position
      int32_t lo = a.seg_start[s], hi = end;
      while (lo < hi) {
        const int32_t mid = (lo + hi) >> 1;
        if (a.sidx[mid] < f1) lo = mid + 1;
        else hi = mid;
      }
      cur = lo + 1;
    }
    a.seg_cursor[s] = cur;
    a.seg_napp[s] = f1 != 0x7fffffff ? 1 : 0;
    const int32_t rem = end - cur;
    k = rem <= 0 ? 0 : rem <= 1 ? 1 : rem <= 2 ? 2 : rem <= 4 ? 3 : rem <= 8 ? 4
      : rem <= 16 ? 5 : rem <= 32 ? 6 : rem <= kBlockReplayMin ? 7 : 8;
    if (k > 0) rank = atomicAdd(&s_cnt[k], 1);
  }
  __syncthreads();
  if (threadIdx.x < 9) s_base[threadIdx.x] = s_cnt[threadIdx.x] ? atomicAdd(counts + threadIdx.x,
                                                                             s_cnt[threadIdx.x])
                                                                 : 0;
  __syncthreads();
  if (k > 0) ids[(int64_t)k * cap + s_base[k] + rank] = (int32_t)s;
}

__global__ void k_counts_to_host(const int* counts, int* mapped) {
  if (threadIdx.x < 9) mapped[threadIdx.x] = counts[threadIdx.x];
}


// Flags of the active segments longer than short_len.
__global__ void k_long_flags(ConsultArgs a, int64_t n, int short_len, uint8_t* flags) {
  const int ns = *a.nsegs;
  for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < n;
       s += (int64_t)gridDim.x * blockDim.x) {
    bool f = false;
    if (s < ns) {
      const int32_t beg = a.seg_start[s], end = a.seg_start[s + 1];
      f = a.seg_cursor[s] < end && end - beg > short_len;
    }
    flags[s] = f;
  }
}

__global__ void k_check_done(const int* nsegs, const int32_t* seg_start,
                             const int32_t* seg_cursor, int* err) {
  const int ns = *nsegs;
  for (int s = blockIdx.x * blockDim.x + threadIdx.x; s < ns; s += gridDim.x * blockDim.x)
    if (seg_cursor[s] < seg_start[s + 1]) atomicCAS(err, 0, 4);
}

// ---------------------------------------------------------------------------
// host orchestration
// ---------------------------------------------------------------------------

struct LongList {
  uint8_t* flags;
  int32_t* list;
  int* count;
  int64_t nsegs_host;  // upper bound on the number of segments
};

template <bool CLOSEST, bool LIVE, int STACK>
static int replay_impl(cudaStream_t st, const ConsultArgs& a, Workspace& ws, const LongList& L,
                       int64_t n) {
  const int sl = g_consult_short;
  const int grid_s = (int)((L.nsegs_host + 127) / 128);
  k_replay_short<CLOSEST, LIVE, STACK><<<grid_s > 0 ? grid_s : 1, 128, 0, st>>>(a, sl);
  HRPP_LAUNCHED();
  k_long_flags<<<grid_for(L.nsegs_host, 256, num_sms() * 8), 256, 0, st>>>(a, L.nsegs_host, sl,
                                                                           L.flags);
  HRPP_LAUNCHED();
  int rc;
  if ((rc = compact_flags(ws, L.flags, L.nsegs_host, L.list, L.count, st))) return rc;
  // one warp per long segment (at most nsegs / (short_len + 1) of them)
  int64_t max_long = L.nsegs_host / (sl + 1) + 1;
  if (max_long > L.nsegs_host) max_long = L.nsegs_host;
  const int grid_l = (int)((max_long * 32 + 127) / 128);
  k_replay_long<CLOSEST, LIVE, STACK><<<grid_l > 0 ? grid_l : 1, 128, 0, st>>>(a, L.list, L.count);
  HRPP_LAUNCHED();
  return 0;
}

template <bool CLOSEST, bool LIVE>
static int dispatch_replay(int stack, cudaStream_t st, const ConsultArgs& a, Workspace& ws,
                           const LongList& L, int64_t n) {
  switch (stack) {
    case 64: return replay_impl<CLOSEST, LIVE, 64>(st, a, ws, L, n);
    case 256: return replay_impl<CLOSEST, LIVE, 256>(st, a, ws, L, n);
    default: return replay_impl<CLOSEST, LIVE, 512>(st, a, ws, L, n);
  }
}

static int launch_replay(bool closest, bool live, int stack, cudaStream_t st,
                         const ConsultArgs& a, Workspace& ws, const LongList& L, int64_t n) {
  ProfScope ps(P_CONSULT, st);
  if (closest)
    return live ? dispatch_replay<true, true>(stack, st, a, ws, L, n)
                : dispatch_replay<true, false>(stack, st, a, ws, L, n);
  return live ? dispatch_replay<false, true>(stack, st, a, ws, L, n)
              : dispatch_replay<false, false>(stack, st, a, ws, L, n);
}

// All full results known: replay every length class with its own group size.
#ifndef HRPP_REPLAY_STREAMS
#define HRPP_REPLAY_STREAMS 8
#endif

// Per host thread and device: side streams (and fork/join events) for the
// concurrent replay classes.
struct SidePool {
  cudaStream_t s[8];
  cudaEvent_t fork, join[8];
  cudaEvent_t seg_ready, cls_ready;  // segment count / class bounds written
  cudaEvent_t trace_done;            // early fallback traversal finished
  cudaStream_t hi;                   // highest priority: the grouping beside the early traversal
  cudaEvent_t group_done;
};

static SidePool& side_pool() {
  thread_local std::map<int, SidePool> pools;
  int dev = 0;
  cudaGetDevice(&dev);
  auto it = pools.find(dev);
  if (it == pools.end()) {
    SidePool p;
    for (int k = 0; k < 8; k++) {
      cudaStreamCreateWithFlags(&p.s[k], cudaStreamNonBlocking);
      cudaEventCreateWithFlags(&p.join[k], cudaEventDisableTiming);
    }
    cudaEventCreateWithFlags(&p.fork, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&p.seg_ready, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&p.cls_ready, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&p.trace_done, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&p.group_done, cudaEventDisableTiming);
    int lo_prio = 0, hi_prio = 0;
    cudaDeviceGetStreamPriorityRange(&lo_prio, &hi_prio);
    cudaStreamCreateWithPriority(&p.hi, cudaStreamNonBlocking, hi_prio);
    it = pools.emplace(dev, p).first;
  }
  return it->second;
}

template <bool CLOSEST, bool LIVE, int STACK>
static int grouped_impl(cudaStream_t st, const ConsultArgs& a, Workspace& ws, int64_t nseg_cap) {
  int32_t* ids;  // class k's segments at ids[k * m ...]
  int* ct;       // [0, 10) per-class counts, [10, 20) per-class tickets
  int rc;
  const int64_t m = nseg_cap > 0 ? nseg_cap : 1;
  if ((rc = ws.get("rg_idsbin", 9 * m, &ids)) || (rc = ws.get("rg_ct", 20, &ct))) return rc;
  int* counts = ct;
  int* tickets = ct + 10;
  HRPP_CK(cudaMemsetAsync(ct, 0, sizeof(int) * 20, st));
  long long* pin = pinned_scratch();
  if (!pin) return HRPP_CUDA;
  k_replay_bin<<<(int)((m + 255) / 256), 256, 0, st>>>(a, m, ids, counts, nullptr);
  HRPP_LAUNCHED();
  // the host needs only class 8's count, read through mapped memory behind
  // an event once classes 1-7 are queued
  k_counts_to_host<<<1, 32, 0, st>>>(counts, reinterpret_cast<int*>(pin + 40));
  HRPP_LAUNCHED();
  const cudaEvent_t ev_cls = side_pool().cls_ready;
  HRPP_CK(cudaEventRecord(ev_cls, st));
  // The classes hold disjoint segments, so their kernels run concurrently:
  // each is small and latency-bound (a few hundred blocks, or one long
  // chain per segment), and back to back each one's tail idled the GPU.
  SidePool& sp = side_pool();
  HRPP_CK(cudaEventRecord(sp.fork, st));
  int used = 0;
  auto side = [&](int k) -> cudaStream_t {
    if (HRPP_REPLAY_STREAMS <= 1) return st;
    cudaStream_t s2 = sp.s[k % HRPP_REPLAY_STREAMS];
    if (!(used & (1 << (k % HRPP_REPLAY_STREAMS)))) cudaStreamWaitEvent(s2, sp.fork, 0);
    used |= 1 << (k % HRPP_REPLAY_STREAMS);
    return s2;
  };
  // persistent grids: at most one resident wave of blocks, at most what the
  // segment count could need
  auto pgrid = [&](int64_t per_block, int64_t resident) -> int {
    const int64_t need = (m + per_block - 1) / per_block;
    const int64_t cap = (int64_t)num_sms() * resident;
    return (int)(need < cap ? (need > 0 ? need : 1) : cap);
  };
#define HRPP_GROUP(K, GS)                                                                     \
  k_replay_group<CLOSEST, LIVE, STACK, GS>                                                    \
      <<<pgrid(HRPP_REPLAY_BS / GS, 6 * 128 / HRPP_REPLAY_BS), HRPP_REPLAY_BS, 0, side(K)>>>( \
          a, ids, counts, m, K, tickets + K);                                                 \
  HRPP_LAUNCHED();
  HRPP_GROUP(1, 1)
  HRPP_GROUP(2, 2)
  HRPP_GROUP(3, 4)
  HRPP_GROUP(4, 8)
  HRPP_GROUP(5, 16)
  HRPP_GROUP(6, 32)
#undef HRPP_GROUP
  // long segments: a warp each, 32-ray tiles
  k_replay_block<CLOSEST, LIVE, STACK, 32><<<pgrid(1, HRPP_BLOCK32_MINB), 32, 0, side(7)>>>(
      a, ids, 0, counts, m, 7, tickets + 7);
  HRPP_LAUNCHED();
  HRPP_CK(cudaEventSynchronize(ev_cls));
  int hb[10];
  memcpy(hb, (const void*)(pin + 40), sizeof(int) * 9);
  auto cnt = [&](int k) { return hb[k]; };
  const int32_t* ids8_in = ids + 8 * m;
  // class 8 below runs on st after the join (it sorts by remaining length)
  for (int k = 0; k < HRPP_REPLAY_STREAMS; k++)
    if (used & (1 << k)) {
      HRPP_CK(cudaEventRecord(sp.join[k], sp.s[k]));
      HRPP_CK(cudaStreamWaitEvent(st, sp.join[k], 0));
    }
  if (cnt(8) > 0) {  // very long segments: a whole block each, longest first
    const int c8 = cnt(8);
    int32_t *rem, *rem2, *ids8;
    if ((rc = ws.get("rg_rem", c8, &rem)) || (rc = ws.get("rg_rem2", c8, &rem2)) ||
        (rc = ws.get("rg_ids8", c8, &ids8)))
      return rc;
    k_seg_remaining<<<grid_for(c8, 256, num_sms() * 4), 256, 0, st>>>(a, ids8_in, c8, rem);
    HRPP_LAUNCHED();
    size_t b8 = 0;
    cub::DeviceRadixSort::SortPairsDescending(nullptr, b8, rem, rem2, ids8_in, ids8, c8, 0, 32,
                                              st);
    void* tmp8;
    if ((rc = ws.get_raw("rg_tmp8", b8, &tmp8))) return rc;
    HRPP_CK(cub::DeviceRadixSort::SortPairsDescending(tmp8, b8, rem, rem2, ids8_in, ids8, c8, 0,
                                                      32, st));
    k_replay_block<CLOSEST, LIVE, STACK, kBlockReplay><<<c8, kBlockReplay, 0, st>>>(
        a, ids8, c8, nullptr, 0, 0, nullptr);
    HRPP_LAUNCHED();
  }
  return 0;
}

template <bool CLOSEST, bool LIVE>
static int dispatch_grouped(int stack, cudaStream_t st, const ConsultArgs& a, Workspace& ws,
                            int64_t nseg_cap) {
  switch (stack) {
    case 64: return grouped_impl<CLOSEST, LIVE, 64>(st, a, ws, nseg_cap);
    case 256: return grouped_impl<CLOSEST, LIVE, 256>(st, a, ws, nseg_cap);
    default: return grouped_impl<CLOSEST, LIVE, 512>(st, a, ws, nseg_cap);
  }
}

static int launch_grouped(bool closest, bool live, int stack, cudaStream_t st,
                          const ConsultArgs& a, Workspace& ws, int64_t nseg_cap) {
  ProfScope ps(P_CONSULT, st);
  if (closest)
    return live ? dispatch_grouped<true, true>(stack, st, a, ws, nseg_cap)
                : dispatch_grouped<true, false>(stack, st, a, ws, nseg_cap);
  return live ? dispatch_grouped<false, true>(stack, st, a, ws, nseg_cap)
              : dispatch_grouped<false, false>(stack, st, a, ws, nseg_cap);
}

// eval0 for a table without entries (the first wave of each ray kind in a
// frame): nothing to evaluate and no state to store, only the ray ->
// segment scatter -- without the traversal code's register footprint
// (94 registers held k_eval0 at a quarter occupancy on a pure scatter).
__global__ void __launch_bounds__(256) k_eval0_empty(const int32_t* __restrict__ sidx,
                                                     const int32_t* __restrict__ seg_id,
                                                     int64_t n, int32_t* __restrict__ seg_of_ray) {
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n;
       p += (int64_t)gridDim.x * blockDim.x)
    seg_of_ray[sidx[p]] = seg_id[p] - 1;
}

// ---------------------------------------------------------------------------
// Leader-first schedule of a live wave on an empty table (run_consult).
// Every key segment's first ray (its leader) is a NEG and needs its full
// traversal; if it hits, anc[leaf] is the entry's first node for every later
// ray of the key.  A later ray that hits that node is a TP at its turn
// whatever else the wave appends (entries only grow), so it never needs a
// full traversal; only the rays that miss it are traced.  The replay then
// runs as usual from the stored states (applied = 1).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_mark_leaders(ConsultArgs a) {
  const int ns = *a.nsegs;
  for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < ns;
       s += (int64_t)gridDim.x * blockDim.x)
    a.need[a.sidx[a.seg_start[s]]] = 1;
}

template <bool CLOSEST, int STACK>
__global__ void __launch_bounds__(HRPP_EVAL_BS, HRPP_EVAL_MINB * 128 / HRPP_EVAL_BS)
    k_follow(ConsultArgs a, int64_t n) {
  if (*a.err) return;
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n;
       p += (int64_t)gridDim.x * blockDim.x) {
    const int32_t i = a.sidx[p];
    const int32_t s = a.seg_id[p] - 1;
    const int32_t lead = a.sidx[a.seg_start[s]];
    Hit acc = empty_entry_result(CLOSEST);
    int32_t applied = 0;
    uint8_t need = 0;
    if (i != lead) {
      if (a.f_found[lead]) {
        const Ray r = make_ray(a.O, a.D, a.tmin, a.tmax, i);
        fold_entry<CLOSEST>(acc, trace_from<CLOSEST, STACK>(a.nodes, a.tris, r,
                                                            a.anc[a.f_leaf[lead]]));
        applied = 1;
        need = !acc.found;
      } else {
        need = 1;  // no entry yet at this ray's turn unless an earlier ray hits: trace
      }
    }
    store_state(a, i, acc, applied);
    a.need[i] = need;
  }
}

template <bool CLOSEST>
static void dispatch_follow(int stack, cudaStream_t st, const ConsultArgs& a, int64_t n) {
  const int egrid = (int)((n + HRPP_EVAL_BS - 1) / HRPP_EVAL_BS);
  switch (stack) {
    case 64: k_follow<CLOSEST, 64><<<egrid, HRPP_EVAL_BS, 0, st>>>(a, n); break;
    case 256: k_follow<CLOSEST, 256><<<egrid, HRPP_EVAL_BS, 0, st>>>(a, n); break;
    default: k_follow<CLOSEST, 512><<<egrid, HRPP_EVAL_BS, 0, st>>>(a, n); break;
  }
}

template <bool CLOSEST>
static void dispatch_eval0(int stack, int grid, cudaStream_t st, const ConsultArgs& a, int64_t n,
                           int mark, bool empty_table = false) {
  if (empty_table && a.sparse_state && !a.f_known_clear) {
    k_eval0_empty<<<grid_for(n, 256, num_sms() * 16), 256, 0, st>>>(a.sidx, a.seg_id, n,
                                                                    a.seg_of_ray);
    return;
  }
  (void)grid;
  const int egrid = (int)((n + HRPP_EVAL_BS - 1) / HRPP_EVAL_BS);
  switch (stack) {
    case 64: k_eval0<CLOSEST, 64><<<egrid, HRPP_EVAL_BS, 0, st>>>(a, n, mark); break;
    case 256: k_eval0<CLOSEST, 256><<<egrid, HRPP_EVAL_BS, 0, st>>>(a, n, mark); break;
    default: k_eval0<CLOSEST, 512><<<egrid, HRPP_EVAL_BS, 0, st>>>(a, n, mark); break;
  }
}

static int finalize_prefix(bool closest, bool live, int grid, cudaStream_t st,
                           const ConsultArgs& a, int64_t n, bool first_append_done = false) {
  ProfScope ps(P_CONSULT, st);
  if (!first_append_done) {
    k_first_append<<<grid_for(n, HRPP_FA_BS, num_sms() * 16 * 256 / HRPP_FA_BS), HRPP_FA_BS, 0,
                     st>>>(a, n);
    HRPP_LAUNCHED();
  }
  // about one resident wave of blocks: a thread walks several rays and each
  // block flushes its tallies once
  const int fgrid = grid_for(n, HRPP_FIN_BS, num_sms() * HRPP_FIN_GRID * 128 / HRPP_FIN_BS);
  (void)grid;
  if (closest) {
    if (live) k_finalize<true, true><<<fgrid, HRPP_FIN_BS, 0, st>>>(a, n);
    else k_finalize<true, false><<<fgrid, HRPP_FIN_BS, 0, st>>>(a, n);
  } else {
    if (live) k_finalize<false, true><<<fgrid, HRPP_FIN_BS, 0, st>>>(a, n);
    else k_finalize<false, false><<<fgrid, HRPP_FIN_BS, 0, st>>>(a, n);
  }
  HRPP_LAUNCHED();
  return 0;  // the replay cursors are set by k_replay_bin
}

int run_consult(const BvhDev& b, TableDev& t, const Consult& c, const uint64_t* keys,
                unsigned long long* stats_dev, int* err, cudaStream_t st, bool prepacked) {
  const int64_t n = c.n;
  if (n <= 0) return 0;
  int rc;
  const int32_t* anc;
  if ((rc = const_cast<BvhDev&>(b).ancestor_lut(t.go_up, &anc))) return rc;
  Segments seg;
  // new entries <= key segments: read the segment count once so the hash
  // index stays sized to the table (L2-resident for c1-c3 tables), not to the wave
  long long* pin = pinned_scratch();
  if (!pin) return HRPP_CUDA;
  // A live wave on an empty table needs every ray's full traversal (no
  // entry can make a ray a TP before its segment's first append), and that
  // traversal needs nothing from the grouping: it starts at once on a side
  // stream, overlapped with the sort and segment construction (memory-bound
  // against the issue-bound traversal), and joins before the first-append
  // bids and the replay.  The first wave of each ray kind in a frame.
  const int rounds0 = g_live_rounds < 0 ? 0 : g_live_rounds;
  // Also when the table is not empty but its last live wave had few
  // wave-start TPs (under 5 %): the early traversal then also traces those
  // few TPs (their outputs are overwritten by the entry result), a small
  // waste against the overlap won.
  // Leader-first (k_follow): on an empty table, when this table's last
  // empty-table live wave ended with enough TPs to pay for the extra pass
  // (no history: closest-hit tables only).  HRPP_LEADER_FIRST=0/1/2: never,
  // by history (default), always.  Only the schedule changes, never a result.
  static const int leader_mode = [] {
    const char* e = getenv("HRPP_LEADER_FIRST");
    return e ? atoi(e) : HRPP_LEADER_FIRST;
  }();
  const bool leader_first =
      c.live && rounds0 == 0 && t.n_entries == 0 &&
      (leader_mode == 2 ||
       (leader_mode == 1 && (t.empty_tp_frac < 0.0 ? t.closest : t.empty_tp_frac >= 0.25)));
  t.wave_started_empty = t.n_entries == 0;
  const bool early_trace =
      c.live && rounds0 == 0 && !leader_first &&
      (HRPP_EARLY_TRACE == 2 ||
       (HRPP_EARLY_TRACE == 1 && (t.n_entries == 0 || t.start_tp_frac < 0.05)));
  if (early_trace) {
    uint8_t* f_known;
    int32_t *f_box, *f_tri;
    if ((rc = t.ws.get("v_fknown", n, &f_known)) || (rc = t.ws.get("v_fbox32", n, &f_box)) ||
        (rc = t.ws.get("v_ftri32", n, &f_tri)))
      return rc;
    SidePool& sp = side_pool();
    HRPP_CK(cudaEventRecord(sp.fork, st));
    HRPP_CK(cudaStreamWaitEvent(sp.s[0], sp.fork, 0));
    TraceOut to;
    to.found = c.o_found;
    to.t = c.o_t;
    to.slot = c.o_slot;
    to.leaf = c.o_leaf;
    to.box32 = f_box;
    to.tri32 = f_tri;
    to.known = nullptr;  // every ray is traced: the consult reads no known flags (a.f_known = nullptr)
    (void)f_known;
    to.zero_miss_t = true;
    if ((rc = launch_trace(b, t.closest, c.O, c.D, c.tmin, c.tmax, 0, n, nullptr, nullptr, to,
                           err, sp.s[0], &t.ws, true)))
      return rc;
    HRPP_CK(cudaEventRecord(sp.trace_done, sp.s[0]));
  }
  static const int sort_prio = [] {
    const char* e = getenv("HRPP_SORT_PRIO");
    return e ? atoi(e) : HRPP_SORT_PRIO;
  }();
  if (early_trace && sort_prio) {
    // The traversal's one-warp blocks fill every SM, so a grouping queued at
    // the same priority only runs in the traversal's tail; at the highest
    // priority its blocks take the slots the traversal's blocks free.
    SidePool& sp = side_pool();
    HRPP_CK(cudaStreamWaitEvent(sp.hi, sp.fork, 0));
    if ((rc = group_by_key(t.ws, keys, n, 1 + 2 * t.precision, &seg, sp.hi,
                           reinterpret_cast<int*>(pin + 32), prepacked)))
      return rc;
    HRPP_CK(cudaEventRecord(sp.group_done, sp.hi));
    HRPP_CK(cudaStreamWaitEvent(st, sp.group_done, 0));
  } else if ((rc = group_by_key(t.ws, keys, n, 1 + 2 * t.precision, &seg, st,
                                reinterpret_cast<int*>(pin + 32), prepacked))) {
    return rc;
  }
  ConsultArgs a{};
  Workspace& ws = t.ws;
  if ((rc = ws.get("k_segofray", n, &a.seg_of_ray))) return rc;
  // The segment count (new entries <= segments) is read back through mapped
  // memory behind an event, and waited for only where the host needs it:
  // after the wave-start evaluation and the fallback traversal are queued,
  // so the GPU never idles for it.  The arena is reserved now for the
  // wave's upper bound of appends (one per ray): a compaction moves lists,
  // which is only safe before k_seg_lookup reads their offsets; the entry
  // arrays and the index grow later, copy-preserving.
  const cudaEvent_t ev_seg = side_pool().seg_ready;  // per host thread and device
  HRPP_CK(cudaEventRecord(ev_seg, st));
  if ((rc = t.reserve(0, n, st))) return rc;
  int nsegs_h = -1;
  LongList LL;
  auto resolve_nsegs = [&]() -> int {
    if (nsegs_h >= 0) return 0;
    HRPP_CK(cudaEventSynchronize(ev_seg));
    nsegs_h = *(volatile int*)(pin + 32);
    int r2;
    if ((r2 = t.reserve(nsegs_h, n, st))) return r2;
    a.idx = t.idx;
    a.mask = (uint64_t)t.idx_cap - 1;
    a.e_off = t.e_off;
    a.e_len = t.e_len;
    a.arena = t.arena;
    LL.nsegs_host = nsegs_h;
    if ((r2 = ws.get("k_lflags", nsegs_h + 1, &LL.flags)) ||
        (r2 = ws.get("k_llist", nsegs_h + 1, &LL.list)) || (r2 = ws.get("k_lcount", 1, &LL.count)))
      return r2;
    return 0;
  };
  a.nodes = b.nodes;
  a.tris = b.tris;
  a.depth = b.depth;
  a.anc = anc;
  a.O = c.O;
  a.D = c.D;
  a.tmin = c.tmin;
  a.tmax = c.tmax;
  a.skeys = seg.skeys;
  a.sidx = seg.sidx;
  a.seg_start = seg.seg_start;
  a.seg_id = seg.seg_id;
  a.nsegs = seg.nsegs;
  a.idx = t.idx;
  a.mask = (uint64_t)t.idx_cap - 1;
  a.e_off = t.e_off;
  a.e_len = t.e_len;
  a.arena = t.arena;
  a.stats = stats_dev;
  a.err = err;
  if ((rc = ws.get("k_eid", n, &a.seg_eid)) || (rc = ws.get("k_exoff", n, &a.seg_exoff)) ||
      (rc = ws.get("k_exlen", n, &a.seg_exlen)) || (rc = ws.get("k_napp", n, &a.seg_napp)) ||
      (rc = ws.get("k_cursor", n, &a.seg_cursor)) || (rc = ws.get("k_app", n, &a.app)) ||
      (rc = ws.get("k_appray", n, &a.app_ray)) || (rc = ws.get("k_state", n, &a.state)) ||
      (rc = ws.get("k_f1", n, &a.seg_f1)))
    return rc;
  const int grid = (int)((n + 127) / 128);
  {
    ProfScope ps(P_CONSULT, st);
    k_seg_lookup<<<grid_for(n, 256, num_sms() * 8), 256, 0, st>>>(a, n);
    HRPP_LAUNCHED();
  }
  const int rounds = g_live_rounds < 0 ? 0 : g_live_rounds;
  // suspend/resume rounds store states for every ray; the default path does not
  a.sparse_state = !(c.live && (rounds > 0 || leader_first));
  if (c.live) {
    // The fallback traversal writes the wave's outputs directly (a ray that
    // turns out a TP is overwritten by its entry result later; every other
    // ray's output is its full traversal), and its counts as int32.
    uint8_t* f_known;
    int32_t *queue, *f_box, *f_tri;
    int* qcount;
    if ((rc = ws.get("v_fknown", n, &f_known)) || (rc = ws.get("v_fbox32", n, &f_box)) ||
        (rc = ws.get("v_ftri32", n, &f_tri)) || (rc = ws.get("v_queue", n, &queue)) ||
        (rc = ws.get("v_qcount", 1, &qcount)) || (rc = ws.get("v_need", n, &a.need)))
      return rc;
    a.f_found = c.o_found;
    a.f_t = c.o_t;
    a.f_slot = c.o_slot;
    a.f_leaf = c.o_leaf;
    a.f_box32 = f_box;
    a.f_tri32 = f_tri;
    a.f_known = early_trace ? nullptr : f_known;  // early traversal: every full result is known
    a.o_found = c.o_found;
    a.o_t = c.o_t;
    a.o_slot = c.o_slot;
    a.o_leaf = c.o_leaf;
    // coalesced presets instead of two scattered byte stores per ray in eval0
    a.f_known_clear = nullptr;
    if (!early_trace) {  // (the early traversal writes known = 1 for every ray)
      HRPP_CK(cudaMemsetAsync(f_known, 0, n, st));
      // eval0 clears the TPs; leader-first marks the leaders
      HRPP_CK(cudaMemsetAsync(a.need, rounds > 0 || leader_first ? 0 : 1, n, st));
    }
    if (leader_first) {
      ProfScope ps(P_CONSULT, st);
      k_eval0_empty<<<grid_for(n, 256, num_sms() * 16), 256, 0, st>>>(a.sidx, a.seg_id, n,
                                                                      a.seg_of_ray);
      HRPP_LAUNCHED();
      k_mark_leaders<<<grid_for(n, 256, num_sms() * 8), 256, 0, st>>>(a);
      HRPP_LAUNCHED();
    } else {
      ProfScope ps(P_CONSULT, st);
      if (t.closest) dispatch_eval0<true>(b.stack, grid, st, a, n, rounds == 0, t.n_entries == 0);
      else dispatch_eval0<false>(b.stack, grid, st, a, n, rounds == 0, t.n_entries == 0);
      HRPP_LAUNCHED();
    }
    TraceOut to;
    to.found = c.o_found;
    to.t = c.o_t;
    to.slot = c.o_slot;
    to.leaf = c.o_leaf;
    to.box32 = f_box;
    to.tri32 = f_tri;
    to.known = f_known;
    to.zero_miss_t = true;  // hrpp/tracer.py:331-339: a live miss reports t = 0
    if (rounds == 0) {  // the queue is exactly k_first_append's candidate set
      to.fa_seg_of_ray = a.seg_of_ray;
      to.fa_exoff = a.seg_exoff;
      to.fa_exlen = a.seg_exlen;
      to.fa_arena = a.arena;
      to.fa_anc = a.anc;
      to.fa_f1 = a.seg_f1;
    }
    // rounds == 0: eval0 already marked every ray that is not a TP against the
    // wave-start entry; trace them, then one replay completes the wave.
    // rounds > 0: exact replay rounds, the last one speculative.
    if (rounds > 0 && (rc = resolve_nsegs())) return rc;  // the replay rounds use LL
    if (leader_first) {  // trace the leaders, then evaluate their node for the followers
      if ((rc = compact_flags(ws, a.need, n, queue, qcount, st))) return rc;
      if ((rc = launch_trace(b, t.closest, c.O, c.D, c.tmin, c.tmax, 0, n, queue, qcount, to,
                             err, st, &ws)))
        return rc;
      ProfScope ps(P_CONSULT, st);
      if (t.closest) dispatch_follow<true>(b.stack, st, a, n);
      else dispatch_follow<false>(b.stack, st, a, n);
      HRPP_LAUNCHED();
    }
    for (int r = rounds == 0 ? rounds : 0; r <= rounds && !early_trace; r++) {
      if (rounds > 0) {
        a.spec = r == rounds ? 2 : 0;
        HRPP_CK(cudaMemsetAsync(a.need, 0, n, st));
        if ((rc = launch_replay(t.closest, true, b.stack, st, a, ws, LL, n))) return rc;
      }
      // the rays whose full traversal is needed next, compacted in ray order:
      // neighbouring pixels share warps in the traversal kernel (key order
      // is worse: the xor-mixed key scatters unrelated rays into one warp)
      if ((rc = compact_flags(ws, a.need, n, queue, qcount, st))) return rc;
      if ((rc = launch_trace(b, t.closest, c.O, c.D, c.tmin, c.tmax, 0, n, queue, qcount, to,
                             err, st, &ws)))
        return rc;
    }
    a.spec = 0;
    if (early_trace) {  // join the early traversal; the first-append bids run here
      HRPP_CK(cudaStreamWaitEvent(st, side_pool().trace_done, 0));
      if ((rc = resolve_nsegs())) return rc;
      if ((rc = finalize_prefix(t.closest, true, grid, st, a, n, false))) return rc;
      if ((rc = launch_grouped(t.closest, true, b.stack, st, a, ws, nsegs_h))) return rc;
    } else if (rounds == 0) {
      if ((rc = finalize_prefix(t.closest, true, grid, st, a, n, true))) return rc;
      if ((rc = resolve_nsegs())) return rc;
      if ((rc = launch_grouped(t.closest, true, b.stack, st, a, ws, nsegs_h))) return rc;
    } else {
      if ((rc = launch_replay(t.closest, true, b.stack, st, a, ws, LL, n))) return rc;
    }
    // (every segment replayed to its end: checked by k_commit_count, or below
    // in deferred mode)
  } else {
    a.f_found = c.base_found;
    a.f_t = c.base_t;
    a.f_leaf = c.base_leaf;
    a.f_box = c.base_box;
    a.log_cls = c.log_cls;
    a.log_eval_box = c.log_eval_box;
    a.log_pred_t = c.log_pred_t;
    a.log_pred_slot = c.log_pred_slot;
    {
      ProfScope ps(P_CONSULT, st);
      if (t.closest) dispatch_eval0<true>(b.stack, grid, st, a, n, 0, t.n_entries == 0);
      else dispatch_eval0<false>(b.stack, grid, st, a, n, 0, t.n_entries == 0);
      HRPP_LAUNCHED();
    }
    if ((rc = finalize_prefix(t.closest, false, grid, st, a, n))) return rc;
    if ((rc = resolve_nsegs())) return rc;
    if ((rc = launch_grouped(t.closest, false, b.stack, st, a, ws, nsegs_h))) return rc;
  }
  if ((rc = resolve_nsegs())) return rc;
  if (t.deferred) {
    if (c.live) {
      k_check_done<<<grid_for(n, 256, num_sms() * 4), 256, 0, st>>>(seg.nsegs, seg.seg_start,
                                                                   a.seg_cursor, err);
      HRPP_LAUNCHED();
    }
    return table_collect_pending(t, seg, n, a.seg_napp, a.app, a.app_ray, err, st);
  }
  // one thread per key segment (nsegs_h of them), not per ray
  return table_commit(t, seg, nsegs_h, a.seg_eid, a.seg_napp, a.app, err, st,
                      c.live ? a.seg_cursor : nullptr);
}

}  // namespace hrpp
