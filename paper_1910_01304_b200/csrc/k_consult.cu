// k_consult.cu -- the predictor consult of one wave, exact in ray order.
//
// The reference consults and trains the table one ray at a time in wave
// order (hrpp/tracer.py:233-267 limit, :295-331 live).  A table entry is
// read and written only by rays carrying its key, so the loop is
// independent per key: after a stable sort by key, one warp replays each
// key segment in ray order.  Lanes hold 32 consecutive rays of the segment;
// each lane folds the entry's nodes into its running eval_entry result
// (hrpp/kernels.py:251-297) incrementally, so a node appended by ray f is
// evaluated only by the rays after f -- exactly the (ray, node) pairs the
// sequential loop evaluates.  A ballot finds the next ray that is not a
// true positive; the rays before it commit as TPs, it commits as NEG/FP
// and may append anc[leaf] (de-duplicated) to the entry.
//
// Live mode needs the full-traversal result of every non-TP ray, which the
// reference computes inline.  Here the warp suspends at the first such ray
// whose result is unknown and enqueues it; a dense traversal kernel traces
// the queue; the consult resumes.  After `g_live_rounds` exact rounds one
// speculative round enqueues every ray of the remaining segments that is
// not yet a TP (TP status is monotone in entry growth, so every ray that can
// still need a full result is then traced) and a final round completes all
// segments.  Speculation only costs extra traversals; results are exact.
#include "hrpp_internal.h"

namespace hrpp {

int g_live_rounds = 0;

enum { S_RAYS, S_TP, S_FP, S_NEG, S_BB, S_BT, S_OB, S_OT, S_SK, S_EST, S_WRONG };

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
  const int* nsegs;
  const unsigned long long* idx_keys;
  const int32_t* idx_vals;
  uint64_t mask;
  const int64_t* e_off;
  const int32_t* e_len;
  const int32_t* arena;
  int32_t* seg_eid;
  int32_t* seg_napp;
  int32_t* seg_cursor;
  int32_t* app;
  int32_t* app_ray;  // ray index that triggered each append (deferred mode)
  // full-traversal results by ray index (baseline in limit mode)
  const uint8_t* f_found;
  const double* f_t;
  const int32_t* f_slot;
  const int32_t* f_leaf;
  const int64_t* f_box;
  const int64_t* f_tri;
  const uint8_t* f_known;
  // live per-ray consult state by sorted position
  uint8_t* s_found;
  double* s_t;
  int32_t* s_slot;
  int32_t* s_leaf;
  int32_t* s_box;
  int32_t* s_tri;
  int32_t* s_applied;
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
  uint8_t* need;  // live: rays whose full traversal the consult needs next
  int32_t* queue;
  int* qcount;
  int spec;  // 0: enqueue the first unknown ray; 2: enqueue every unresolved ray
  const int* err;
};

constexpr unsigned kFull = 0xffffffffu;

int g_consult_short = 32;  // segments up to this many rays run one lane each

__device__ __forceinline__ Ray load_ray(const ConsultArgs& a, bool valid, int32_t idx) {
  if (valid) return make_ray(a.O, a.D, a.tmin, a.tmax, idx);
  Ray r{};
  return r;
}

__device__ __forceinline__ void load_state(const ConsultArgs& a, int32_t pos, Hit& acc,
                                           int32_t& applied) {
  applied = a.s_applied[pos];
  if (applied > 0) {
    acc.found = a.s_found[pos];
    acc.t = a.s_t[pos];
    acc.slot = a.s_slot[pos];
    acc.leaf = a.s_leaf[pos];
    acc.boxes = a.s_box[pos];
    acc.tris = a.s_tri[pos];
  }
}

__device__ __forceinline__ void store_state(const ConsultArgs& a, int32_t pos, const Hit& acc,
                                            int32_t applied) {
  a.s_applied[pos] = applied;
  a.s_found[pos] = acc.found;
  a.s_t[pos] = acc.t;
  a.s_slot[pos] = acc.slot;
  a.s_leaf[pos] = acc.leaf;
  a.s_box[pos] = acc.boxes;
  a.s_tri[pos] = acc.tris;
}

struct Tally {
  long long tp = 0, fp = 0, neg = 0, ob = 0, ot = 0, sk = 0, est = 0, wr = 0, bb = 0, bt = 0;
};

// The entry's j-th node: stored list first, then this wave's appends.
__device__ __forceinline__ int32_t entry_node(const ConsultArgs& a, int64_t ex_off,
                                              int32_t ex_len, const int32_t* app, int32_t j) {
  return j < ex_len ? a.arena[ex_off + j] : app[j - ex_len];
}

// Fold entry nodes [from, L) into acc: eval_entry_{closest,any}, resumable.
template <bool CLOSEST, int STACK>
__device__ __noinline__ void catch_up(const ConsultArgs& a, const Ray& r, Hit& acc, int32_t from,
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
  if (LIVE) {
    const bool ff = a.f_found[idx];
    c.bb += a.f_box[idx];
    c.bt += a.f_tri[idx];
    a.o_found[idx] = ff;
    a.o_t[idx] = ff ? a.f_t[idx] : 0.0;
    a.o_slot[idx] = ff ? a.f_slot[idx] : -1;
    a.o_leaf[idx] = ff ? a.f_leaf[idx] : -1;
  } else if (a.log_cls) {
    a.log_cls[idx] = neg ? 2 : 1;
    a.log_eval_box[idx] = acc.boxes;
    a.log_pred_t[idx] = __longlong_as_double(0x7ff0000000000000LL);
    a.log_pred_slot[idx] = -1;
  }
}

// Speculative round: every not-yet-TP ray of the rest of the segment gets its
// full traversal (TP status only grows with the entry, so after this round
// every ray that can still need a full result has one).
template <bool CLOSEST, int STACK>
__device__ void speculate_rest(const ConsultArgs& a, int32_t from, int32_t end, int32_t L,
                               int64_t ex_off, int32_t ex_len, const int32_t* app) {
  for (int32_t j = from; j < end; j++) {
    const int32_t idx = a.sidx[j];
    const Ray r = make_ray(a.O, a.D, a.tmin, a.tmax, idx);
    Hit acc = empty_entry_result(CLOSEST);
    int32_t applied = 0;
    load_state(a, j, acc, applied);
    catch_up<CLOSEST, STACK>(a, r, acc, applied, L, ex_off, ex_len, app);
    store_state(a, j, acc, L);
    if (!(L > 0 && acc.found) && !a.f_known[idx]) a.need[idx] = 1;
  }
}

// One short key segment, replayed by one lane (hrpp/tracer.py:233-267 or
// :295-331 restricted to one key).
template <bool CLOSEST, bool LIVE, int STACK>
__device__ void seg_thread(const ConsultArgs& a, Tally& c, int s, int32_t beg, int32_t end,
                           int32_t cur) {
  const int32_t eid = index_lookup(a.idx_keys, a.idx_vals, a.mask, a.skeys[beg]);
  const int64_t ex_off = eid >= 0 ? a.e_off[eid] : 0;
  const int32_t ex_len = eid >= 0 ? a.e_len[eid] : 0;
  int32_t* app = a.app + beg;
  int32_t napp = LIVE ? a.seg_napp[s] : 0;
  int32_t j = cur;
  for (; j < end; j++) {
    const int32_t idx = a.sidx[j];
    const Ray r = make_ray(a.O, a.D, a.tmin, a.tmax, idx);
    Hit acc = empty_entry_result(CLOSEST);
    int32_t applied = 0;
    if (LIVE) load_state(a, j, acc, applied);
    const int32_t L = ex_len + napp;
    catch_up<CLOSEST, STACK>(a, r, acc, applied, L, ex_off, ex_len, app);
    if (L > 0 && acc.found) {
      commit_tp<CLOSEST, LIVE>(a, c, idx, acc);
      continue;
    }
    if (LIVE && !a.f_known[idx]) {  // suspend until its full traversal is known
      a.need[idx] = 1;
      store_state(a, j, acc, L);
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
  if (LIVE) a.seg_cursor[s] = j;
  a.seg_napp[s] = napp;
  a.seg_eid[s] = eid;
}

// One long key segment, replayed by the whole warp: lanes hold 32
// consecutive rays; a ballot finds the next non-TP ray.
template <bool CLOSEST, bool LIVE, int STACK>
__device__ void seg_warp(const ConsultArgs& a, Tally& c, int s, int lane) {
  const int32_t beg = a.seg_start[s], end = a.seg_start[s + 1];
  int32_t tb = LIVE ? a.seg_cursor[s] : beg;
  int32_t napp = LIVE ? a.seg_napp[s] : 0;
  const int32_t eid = index_lookup(a.idx_keys, a.idx_vals, a.mask, a.skeys[beg]);
  const int64_t ex_off = eid >= 0 ? a.e_off[eid] : 0;
  const int32_t ex_len = eid >= 0 ? a.e_len[eid] : 0;
  int32_t* app = a.app + beg;
  bool suspended = false;
  while (tb < end) {
    const int32_t pos = tb + lane;
    const bool valid = pos < end;
    const int32_t idx = valid ? a.sidx[pos] : 0;
    const Ray r = load_ray(a, valid, idx);
    Hit acc = empty_entry_result(CLOSEST);
    int32_t applied = 0;
    if (LIVE && valid) load_state(a, pos, acc, applied);
    int32_t L = ex_len + napp;
    const bool fknown = valid && (!LIVE || a.f_known[idx]);
    int32_t cnode = -1;
    if (fknown && a.f_found[idx]) cnode = a.anc[a.f_leaf[idx]];
    bool inL = false;
    for (int32_t j = 0; j < L; j++) inL |= entry_node(a, ex_off, ex_len, app, j) == cnode;
    if (valid) catch_up<CLOSEST, STACK>(a, r, acc, applied, L, ex_off, ex_len, app);
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
        if (valid && lane >= f) store_state(a, pos, acc, applied);
        if (a.spec >= 2) {
          for (int32_t t2 = tb + 32 + lane; t2 < end; t2 += 32) {
            const int32_t i2 = a.sidx[t2];
            const Ray r2 = make_ray(a.O, a.D, a.tmin, a.tmax, i2);
            Hit a2 = empty_entry_result(CLOSEST);
            int32_t ap2 = 0;
            load_state(a, t2, a2, ap2);
            catch_up<CLOSEST, STACK>(a, r2, a2, ap2, L, ex_off, ex_len, app);
            store_state(a, t2, a2, L);
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
        if (valid && lane > f) catch_up<CLOSEST, STACK>(a, r, acc, L - 1, L, ex_off, ex_len, app);
        applied = L;
      }
      cursor = f + 1;
    }
    if (suspended) break;
    tb += 32;
  }
  if (lane == 0) {
    a.seg_eid[s] = eid;
    if (!suspended) {
      a.seg_napp[s] = napp;
      if (LIVE) a.seg_cursor[s] = end;
    }
  }
}

// Thread t owns key segment t; segments longer than `short_len` rays are
// replayed cooperatively by the owning warp.  No global work queue.
template <bool CLOSEST, bool LIVE, int STACK>
__global__ void __launch_bounds__(128) k_consult(ConsultArgs a, int short_len) {
  if (*a.err) return;
  const int lane = threadIdx.x & 31;
  const int ns = *a.nsegs;
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  Tally c;
  bool active = false, small = false;
  int32_t beg = 0, end = 0, cur = 0;
  if (s < ns) {
    beg = a.seg_start[s];
    end = a.seg_start[s + 1];
    cur = LIVE ? a.seg_cursor[s] : beg;
    active = cur < end;
    small = end - beg <= short_len;
  }
  if (active && small) seg_thread<CLOSEST, LIVE, STACK>(a, c, s, beg, end, cur);
  unsigned lm = __ballot_sync(kFull, active && !small);
  while (lm) {
    const int l = __ffs(lm) - 1;
    lm &= lm - 1;
    seg_warp<CLOSEST, LIVE, STACK>(a, c, __shfl_sync(kFull, s, l), lane);
  }
  long long v[10] = {c.tp, c.fp, c.neg, c.bb, c.bt, c.ob, c.ot, c.sk, c.est, c.wr};
  const int slot[10] = {S_TP, S_FP, S_NEG, S_BB, S_BT, S_OB, S_OT, S_SK, S_EST, S_WRONG};
#pragma unroll
  for (int k = 0; k < 10; k++) {
    long long w = warp_sum(v[k]);
    if (lane == 0 && w) atomicAdd(a.stats + slot[k], (unsigned long long)w);
  }
}

__global__ void k_seg_init(const int* nsegs, const int32_t* seg_start, int32_t* seg_cursor,
                           int32_t* seg_napp, int32_t* seg_eid, int64_t n) {
  const int ns = *nsegs;
  for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < ns;
       s += (int64_t)gridDim.x * blockDim.x) {
    seg_cursor[s] = seg_start[s];
    seg_napp[s] = 0;
    seg_eid[s] = -1;
  }
}

__global__ void k_check_done(const int* nsegs, const int32_t* seg_start,
                             const int32_t* seg_cursor, int* err) {
  const int ns = *nsegs;
  for (int s = blockIdx.x * blockDim.x + threadIdx.x; s < ns; s += gridDim.x * blockDim.x)
    if (seg_cursor[s] < seg_start[s + 1]) atomicCAS(err, 0, 4);
}

template <bool CLOSEST, bool LIVE>
static void dispatch_consult(int stack, int grid, cudaStream_t st, const ConsultArgs& a) {
  const int sl = g_consult_short;
  switch (stack) {
    case 64: k_consult<CLOSEST, LIVE, 64><<<grid, 128, 0, st>>>(a, sl); break;
    case 256: k_consult<CLOSEST, LIVE, 256><<<grid, 128, 0, st>>>(a, sl); break;
    default: k_consult<CLOSEST, LIVE, 512><<<grid, 128, 0, st>>>(a, sl); break;
  }
}

static void launch_consult(bool closest, bool live, int stack, int grid, cudaStream_t st,
                           const ConsultArgs& a) {
  ProfScope ps(P_CONSULT, st);
  if (closest) {
    if (live) dispatch_consult<true, true>(stack, grid, st, a);
    else dispatch_consult<true, false>(stack, grid, st, a);
  } else {
    if (live) dispatch_consult<false, true>(stack, grid, st, a);
    else dispatch_consult<false, false>(stack, grid, st, a);
  }
}

int run_consult(const BvhDev& b, TableDev& t, const Consult& c, const uint64_t* keys,
                unsigned long long* stats_dev, int* err, cudaStream_t st) {
  const int64_t n = c.n;
  if (n <= 0) return 0;
  int rc;
  if ((rc = t.reserve(n, st))) return rc;
  const int32_t* anc;
  if ((rc = const_cast<BvhDev&>(b).ancestor_lut(t.go_up, &anc))) return rc;
  Segments seg;
  if ((rc = group_by_key(t.ws, keys, n, &seg, st))) return rc;
  Workspace& ws = t.ws;
  ConsultArgs a{};
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
  a.nsegs = seg.nsegs;
  a.idx_keys = t.idx_keys;
  a.idx_vals = t.idx_vals;
  a.mask = (uint64_t)t.idx_cap - 1;
  a.e_off = t.e_off;
  a.e_len = t.e_len;
  a.arena = t.arena;
  a.stats = stats_dev;
  a.err = err;
  if ((rc = ws.get("k_eid", n, &a.seg_eid))) return rc;
  if ((rc = ws.get("k_napp", n, &a.seg_napp))) return rc;
  if ((rc = ws.get("k_cursor", n, &a.seg_cursor))) return rc;
  if ((rc = ws.get("k_app", n, &a.app))) return rc;
  if ((rc = ws.get("k_appray", n, &a.app_ray))) return rc;
  const int grid = (int)((n + 127) / 128);  // thread t owns segment t (nsegs <= n)
  if (!c.live) {
    a.f_found = c.base_found;
    a.f_t = c.base_t;
    a.f_leaf = c.base_leaf;
    a.f_box = c.base_box;
    a.log_cls = c.log_cls;
    a.log_eval_box = c.log_eval_box;
    a.log_pred_t = c.log_pred_t;
    a.log_pred_slot = c.log_pred_slot;
    launch_consult(t.closest, false, b.stack, grid, st, a);
    HRPP_LAUNCHED();
  } else {
    uint8_t *f_found, *f_known;
    double* f_t;
    int32_t *f_slot, *f_leaf;
    int64_t *f_box, *f_tri;
    if ((rc = ws.get("v_ffound", n, &f_found))) return rc;
    if ((rc = ws.get("v_fknown", n, &f_known))) return rc;
    if ((rc = ws.get("v_ft", n, &f_t))) return rc;
    if ((rc = ws.get("v_fslot", n, &f_slot))) return rc;
    if ((rc = ws.get("v_fleaf", n, &f_leaf))) return rc;
    if ((rc = ws.get("v_fbox", n, &f_box))) return rc;
    if ((rc = ws.get("v_ftri", n, &f_tri))) return rc;
    if ((rc = ws.get("v_sfound", n, &a.s_found))) return rc;
    if ((rc = ws.get("v_st", n, &a.s_t))) return rc;
    if ((rc = ws.get("v_sslot", n, &a.s_slot))) return rc;
    if ((rc = ws.get("v_sleaf", n, &a.s_leaf))) return rc;
    if ((rc = ws.get("v_sbox", n, &a.s_box))) return rc;
    if ((rc = ws.get("v_stri", n, &a.s_tri))) return rc;
    if ((rc = ws.get("v_sapplied", n, &a.s_applied))) return rc;
    if ((rc = ws.get("v_queue", n, &a.queue))) return rc;
    if ((rc = ws.get("v_qcount", 1, &a.qcount))) return rc;
    if ((rc = ws.get("v_need", n, &a.need))) return rc;
    a.f_found = f_found;
    a.f_t = f_t;
    a.f_slot = f_slot;
    a.f_leaf = f_leaf;
    a.f_box = f_box;
    a.f_tri = f_tri;
    a.f_known = f_known;
    a.o_found = c.o_found;
    a.o_t = c.o_t;
    a.o_slot = c.o_slot;
    a.o_leaf = c.o_leaf;
    HRPP_CK(cudaMemsetAsync(f_known, 0, n, st));
    HRPP_CK(cudaMemsetAsync(a.s_applied, 0, sizeof(int32_t) * n, st));
    k_seg_init<<<grid_for(n, 256, num_sms() * 8), 256, 0, st>>>(seg.nsegs, seg.seg_start,
                                                               a.seg_cursor, a.seg_napp,
                                                               a.seg_eid, n);
    HRPP_LAUNCHED();
    TraceOut to;
    to.found = f_found;
    to.t = f_t;
    to.slot = f_slot;
    to.leaf = f_leaf;
    to.box = f_box;
    to.tri = f_tri;
    to.known = f_known;
    const int rounds = g_live_rounds < 0 ? 0 : g_live_rounds;
    for (int r = 0; r <= rounds + 1; r++) {
      a.spec = r == rounds ? 2 : 0;
      HRPP_CK(cudaMemsetAsync(a.need, 0, n, st));
      launch_consult(t.closest, true, b.stack, grid, st, a);
      HRPP_LAUNCHED();
      if (r <= rounds) {
        // the rays whose full traversal is needed next, compacted in ray order
        // (coherent neighbouring rays share warps in the traversal kernel)
        if ((rc = compact_flags(ws, a.need, n, a.queue, a.qcount, st))) return rc;
        if ((rc = launch_trace(b, t.closest, c.O, c.D, c.tmin, c.tmax, 0, n, a.queue, a.qcount,
                               to, err, st)))
          return rc;
      }
    }
    k_check_done<<<grid_for(n, 256, num_sms() * 4), 256, 0, st>>>(seg.nsegs, seg.seg_start,
                                                                 a.seg_cursor, err);
    HRPP_LAUNCHED();
  }
  if (t.deferred)
    return table_collect_pending(t, seg, n, a.seg_napp, a.app, a.app_ray, err, st);
  return table_commit(t, seg, n, a.seg_eid, a.seg_napp, a.app, err, st);
}

}  // namespace hrpp
