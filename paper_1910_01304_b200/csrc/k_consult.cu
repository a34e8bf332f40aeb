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

int g_live_rounds = 3;

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
  int* work;
  int32_t* queue;
  int* qcount;
  int spec;  // 0: enqueue the first unknown ray; 2: enqueue every unresolved ray
  const int* err;
};

constexpr unsigned kFull = 0xffffffffu;

__device__ __forceinline__ void enqueue(const ConsultArgs& a, bool enq, int32_t idx, int lane) {
  unsigned em = __ballot_sync(kFull, enq);
  if (!em) return;
  int base = 0;
  if (lane == 0) base = atomicAdd(a.qcount, __popc(em));
  base = __shfl_sync(kFull, base, 0);
  if (enq) a.queue[base + __popc(em & ((1u << lane) - 1u))] = idx;
}

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

template <bool CLOSEST, bool LIVE, int STACK>
__global__ void __launch_bounds__(128) k_consult(ConsultArgs a) {
  if (*a.err) return;
  const int lane = threadIdx.x & 31;
  const int ns = *a.nsegs;
  long long c_tp = 0, c_fp = 0, c_neg = 0, c_ob = 0, c_ot = 0, c_sk = 0, c_est = 0, c_wr = 0,
            c_bb = 0, c_bt = 0;
  for (;;) {
    int s = 0;
    if (lane == 0) s = atomicAdd(a.work, 1);
    s = __shfl_sync(kFull, s, 0);
    if (s >= ns) break;
    const int32_t beg = a.seg_start[s], end = a.seg_start[s + 1];
    int32_t tb = beg, napp = 0;
    if (LIVE) {
      tb = a.seg_cursor[s];
      if (tb >= end) continue;
      napp = a.seg_napp[s];
    }
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
      int32_t c = -1;
      if (fknown && a.f_found[idx]) c = a.anc[a.f_leaf[idx]];
      bool inL = false;
      // bring every lane up to date with the current entry (and test
      // whether the lane's training node is already stored)
      for (int32_t j = 0; j < L; j++) {
        const int32_t nd = j < ex_len ? a.arena[ex_off + j] : app[j - ex_len];
        inL |= nd == c;
        if (valid && j >= applied && (CLOSEST || !acc.found))
          fold_entry<CLOSEST>(acc, trace_from<CLOSEST, STACK>(a.nodes, a.tris, r, nd));
      }
      applied = L;
      int cursor = 0;
      for (;;) {
        const bool need = valid && lane >= cursor && (L == 0 || !acc.found);
        const unsigned m = __ballot_sync(kFull, need);
        const int f = m ? __ffs(m) - 1 : 32;
        if (valid && lane >= cursor && lane < f) {  // true positives
          c_tp++;
          c_ob += acc.boxes;
          c_ot += acc.tris;
          const int64_t x = (int64_t)a.depth[acc.leaf] + 1 - acc.boxes;
          c_est += x > 0 ? x : 0;
          if (LIVE) {
            a.o_found[idx] = 1;
            a.o_t[idx] = acc.t;
            a.o_slot[idx] = acc.slot;
            a.o_leaf[idx] = acc.leaf;
          } else {
            c_sk += a.f_box[idx] - acc.boxes;
            if (CLOSEST && acc.t > a.f_t[idx] + kWrongClosestEps) c_wr++;
            if (a.log_cls) {
              a.log_cls[idx] = 0;
              a.log_eval_box[idx] = acc.boxes;
              a.log_pred_t[idx] = acc.t;
              a.log_pred_slot[idx] = acc.slot;
            }
          }
        }
        if (f == 32) break;
        if (LIVE && !__shfl_sync(kFull, fknown, f)) {
          // suspend: the full traversal of ray f is not known yet
          enqueue(a, (lane == f) || (a.spec >= 1 && need && !fknown), idx, lane);
          if (valid && lane >= f) store_state(a, pos, acc, applied);
          if (a.spec >= 2) {
            for (int32_t t2 = tb + 32; t2 < end; t2 += 32) {
              const int32_t p2 = t2 + lane;
              const bool v2 = p2 < end;
              const int32_t i2 = v2 ? a.sidx[p2] : 0;
              const Ray r2 = load_ray(a, v2, i2);
              Hit a2 = empty_entry_result(CLOSEST);
              int32_t ap2 = 0;
              if (v2) load_state(a, p2, a2, ap2);
              for (int32_t j = 0; j < L; j++) {
                const int32_t nd = j < ex_len ? a.arena[ex_off + j] : app[j - ex_len];
                if (v2 && j >= ap2 && (CLOSEST || !a2.found))
                  fold_entry<CLOSEST>(a2, trace_from<CLOSEST, STACK>(a.nodes, a.tris, r2, nd));
              }
              if (v2) store_state(a, p2, a2, L);
              enqueue(a, v2 && (L == 0 || !a2.found) && !a.f_known[i2], i2, lane);
            }
          }
          if (lane == 0) {
            a.seg_cursor[s] = tb + f;
            a.seg_napp[s] = napp;
          }
          suspended = true;
          break;
        }
        if (lane == f) {  // NEG (no entry yet) or FP
          if (L == 0) c_neg++;
          else c_fp++;
          c_ob += acc.boxes;
          c_ot += acc.tris;
          if (LIVE) {
            const bool ff = a.f_found[idx];
            c_bb += a.f_box[idx];
            c_bt += a.f_tri[idx];
            a.o_found[idx] = ff;
            a.o_t[idx] = ff ? a.f_t[idx] : 0.0;
            a.o_slot[idx] = ff ? a.f_slot[idx] : -1;
            a.o_leaf[idx] = ff ? a.f_leaf[idx] : -1;
          } else if (a.log_cls) {
            a.log_cls[idx] = L == 0 ? 2 : 1;
            a.log_eval_box[idx] = acc.boxes;
            a.log_pred_t[idx] = __longlong_as_double(0x7ff0000000000000LL);
            a.log_pred_slot[idx] = -1;
          }
        }
        const int32_t cf = __shfl_sync(kFull, c, f);
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
          inL |= c == cf;
          if (valid && lane > f && (CLOSEST || !acc.found))
            fold_entry<CLOSEST>(acc, trace_from<CLOSEST, STACK>(a.nodes, a.tris, r, cf));
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
  long long v[10] = {c_tp, c_fp, c_neg, c_bb, c_bt, c_ob, c_ot, c_sk, c_est, c_wr};
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
  switch (stack) {
    case 64: k_consult<CLOSEST, LIVE, 64><<<grid, 128, 0, st>>>(a); break;
    case 256: k_consult<CLOSEST, LIVE, 256><<<grid, 128, 0, st>>>(a); break;
    default: k_consult<CLOSEST, LIVE, 512><<<grid, 128, 0, st>>>(a); break;
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
  if ((rc = ws.get("k_work", 1, &a.work))) return rc;
  const int grid = num_sms() * 8;
  if (!c.live) {
    a.f_found = c.base_found;
    a.f_t = c.base_t;
    a.f_leaf = c.base_leaf;
    a.f_box = c.base_box;
    a.log_cls = c.log_cls;
    a.log_eval_box = c.log_eval_box;
    a.log_pred_t = c.log_pred_t;
    a.log_pred_slot = c.log_pred_slot;
    HRPP_CK(cudaMemsetAsync(a.work, 0, sizeof(int), st));
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
      HRPP_CK(cudaMemsetAsync(a.work, 0, sizeof(int), st));
      HRPP_CK(cudaMemsetAsync(a.qcount, 0, sizeof(int), st));
      launch_consult(t.closest, true, b.stack, grid, st, a);
      HRPP_LAUNCHED();
      if (r <= rounds) {
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
