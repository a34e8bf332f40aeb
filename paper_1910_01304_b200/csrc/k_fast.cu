// k_fast.cu -- fast mode: the live consult (hrpp/tracer.py:295-331) as
// key-parallel speculation rounds, without the grouping sort or the per-key
// replay of the exact path (k_consult.cu).
//
//   round 0  every ray hashes, looks its key up and evaluates the entry as it
//            stood at the start of the wave; a hit is a TP (final)
//   round k  among the rays still unresolved, the first of each key in ray
//            order (wave hash slot, atomicMin on the ray index) is its
//            round-k leader: NEG/FP, traced from the root; if it hit and its
//            node anc[leaf] is new to the entry, every other unresolved ray of
//            the key evaluates that node: a hit makes it a TP
//   final    the rays still unresolved after R rounds are traced (NEG/FP)
//   commit   (key, anc[leaf]) of every traced ray with a hit: entries claimed
//            in the table index with atomicCAS, (entry, node) pairs
//            de-duplicated in a wave hash set keeping the smallest ray, each
//            entry's new nodes ordered by that ray (= the reference's append
//            order, hrpp/predictor.py:147-160)
//
// Each ray's decision sees exactly the nodes the rays before it appended,
// except among the rays of the final pass; with R at least the appends any
// key needs in the wave the result is the reference's live mode (closest-hit
// TPs then skip only the evaluation of nodes appended between their round
// and their turn).  Deterministic: every choice is by ray index.  Checked
// bit for bit against oracle/hrpp_oracle.c fast_wave; DESIGN.md "Fast mode"
// states the measured distance to the exact mode.
#include <cub/cub.cuh>

#include "hrpp_internal.h"

namespace hrpp {

int g_fast_rounds = 8;
int g_fast_stop_div = 32;

namespace {

constexpr unsigned kFullMask = 0xffffffffu;
constexpr unsigned long long kEmptyWord = ~0ull;
constexpr uint32_t kNoRay = 0xffffffffu;

enum { S_RAYS, S_TP, S_FP, S_NEG, S_BB, S_BT, S_OB, S_OT, S_SK, S_EST, S_WRONG };
// device counters
enum { C_UIN, C_UOUT, C_F, C_TQ, C_BEG, C_TICKET, C_RES, C_STOP, C_NEWE, C_NREC, C_TOUCH,
       C_MULTI, C_N };

// Per key of the wave's unresolved rays: 32 B, one sector.
struct __align__(32) WSlot {
  unsigned long long key;  // kEmptyWord when free
  uint32_t first;          // this round's smallest unresolved ray
  uint32_t fhit;           // smallest final-pass ray with a hit
  long long cur;           // (round << 32) | node appended by this round's leader, or -1
  int32_t hit;             // a traced ray of the key hit
  int32_t head;            // last appending ray (chain through nxt), or -1
};
// (index bucket, node) pair of the commit with the smallest recording ray.
struct __align__(16) PSlot {
  unsigned long long pair;  // kEmptyWord when free
  uint32_t ray;
  uint32_t pad;
};

struct FastArgs {
  const DNode* nodes;
  const DTri* tris;
  const int32_t* depth;
  const int32_t* anc;
  const float* O;
  const float* D;
  const double* tmin;
  const double* tmax;
  int64_t n;
  int p;
  int stop_div;  // rounds stop once a round resolves fewer than n / stop_div rays
  // table (the wave-start entries; the commit appends)
  Bucket* idx;
  uint64_t mask;
  int64_t* e_off;
  int32_t* e_len;
  unsigned long long* e_key;
  int32_t* arena;
  long long* meta;
  int64_t n_entries0, max_entries;
  int empty;
  // outputs by ray
  uint8_t* o_found;
  double* o_t;
  int32_t* o_slot;
  int32_t* o_leaf;
  // per ray
  unsigned long long* keys;
  int32_t* eid;    // wave-start entry or -1
  int32_t* bkt;    // its index bucket
  int32_t* evbox;  // boxes of this ray's evaluations so far
  int32_t* wh;     // wave slot of the ray's key
  int32_t* nxt;    // appended-node chain per key, linked by ray
  // ray lists
  int32_t* U;  // unresolved rays (a round reads U[0, UIN), its followers refill it)
  int32_t* F;
  int32_t* TQ;
  // wave slots (one per key of an unresolved ray) and the commit's pair set
  WSlot* ws;
  uint64_t wmask;
  PSlot* ps;
  uint64_t pmask;
  int32_t* wbase;   // by index bucket: the key's range of the record buffer
  int32_t* multi;   // touched keys with more than one new node
  long long* lctr;  // [0] record-buffer fill, [1] entries created, [2] nodes stored
  int32_t* touched;
  int2* recs;
  unsigned long long* wrec;
  int* ctr;
  unsigned long long* stats;
  int* err;
};

struct FTally {
  long long tp = 0, fp = 0, neg = 0, ob = 0, ot = 0, est = 0, bb = 0, bt = 0;
};

__device__ __forceinline__ void flush(const FTally& c, unsigned long long* stats) {
  const long long v[8] = {c.tp, c.fp, c.neg, c.ob, c.ot, c.est, c.bb, c.bt};
  const int slot[8] = {S_TP, S_FP, S_NEG, S_OB, S_OT, S_EST, S_BB, S_BT};
#pragma unroll
  for (int k = 0; k < 8; k++) {
    const long long w = warp_sum(v[k]);
    if ((threadIdx.x & 31) == 0 && w) atomicAdd(stats + slot[k], (unsigned long long)w);
  }
}

constexpr int kBS = 256;  // block size of the list-building kernels

// Position of this thread's item in a list appended to by whole blocks (-1 if
// !pred): warp ballots, one atomic per block.  Every thread of the block must
// call it (block-uniform loops, FOR_BLOCK_CHUNKS).
__device__ __forceinline__ int block_append(int* counter, bool pred) {
  __shared__ int s_cnt[kBS / 32 + 1];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const unsigned m = __ballot_sync(kFullMask, pred);
  if (lane == 0) s_cnt[warp] = __popc(m);
  __syncthreads();
  if (threadIdx.x == 0) {
    int tot = 0;
    for (int w = 0; w < kBS / 32; w++) {
      const int c = s_cnt[w];
      s_cnt[w] = tot;
      tot += c;
    }
    s_cnt[kBS / 32] = tot ? atomicAdd(counter, tot) : 0;
  }
  __syncthreads();
  const int pos = s_cnt[kBS / 32] + s_cnt[warp] + __popc(m & ((1u << lane) - 1u));
  __syncthreads();  // s_cnt is reused by the next call
  return pred ? pos : -1;
}

// The same for a 64-bit total (arena offsets): returns this thread's offset.
__device__ __forceinline__ long long block_alloc(long long* counter, long long amount) {
  __shared__ long long s_part[kBS / 32 + 1];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  long long incl = amount;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const long long y = __shfl_up_sync(kFullMask, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) s_part[warp] = incl;
  __syncthreads();
  if (threadIdx.x == 0) {
    long long tot = 0;
    for (int w = 0; w < kBS / 32; w++) {
      const long long c = s_part[w];
      s_part[w] = tot;
      tot += c;
    }
    s_part[kBS / 32] =
        tot ? (long long)atomicAdd(reinterpret_cast<unsigned long long*>(counter),
                                   (unsigned long long)tot)
            : 0;
  }
  __syncthreads();
  const long long off = s_part[kBS / 32] + s_part[warp] + incl - amount;
  __syncthreads();
  return off;
}

__device__ __forceinline__ void write_hit(const FastArgs& a, int32_t i, const Hit& h) {
  a.o_found[i] = h.found;
  a.o_t[i] = h.found ? h.t : 0.0;  // hrpp/tracer.py:288-291: a live miss reports t = 0
  a.o_slot[i] = h.found ? h.slot : -1;
  a.o_leaf[i] = h.found ? h.leaf : -1;
}

__device__ __forceinline__ void tally_tp(const FastArgs& a, FTally& c, const Hit& h, int32_t boxes) {
  c.tp++;
  const long long x = (long long)a.depth[h.leaf] + 1 - boxes;
  c.est += x > 0 ? x : 0;
}

__device__ __forceinline__ bool in_entry(const FastArgs& a, int32_t e, int32_t node) {
  if (e < 0) return false;
  const int64_t off = a.e_off[e];
  const int32_t len = a.e_len[e];
  for (int32_t k = 0; k < len; k++)
    if (a.arena[off + k] == node) return true;
  return false;
}

// Block-uniform persistent loop over [0, count): every thread of a block
// runs the same iterations (block_append needs the whole block); item
// base_ + threadIdx.x.
#define FOR_BLOCK_CHUNKS(count_expr)                                                       \
  const int lane = threadIdx.x & 31;                                                       \
  (void)lane;                                                                              \
  const int64_t cnt_ = (count_expr);                                                       \
  for (int64_t base_ = (int64_t)blockIdx.x * blockDim.x; base_ < cnt_;                     \
       base_ += (int64_t)gridDim.x * blockDim.x)

__device__ __forceinline__ int32_t wave_claim(const FastArgs& a, unsigned long long key) {
  uint64_t h = mix64(key) & a.wmask;
  for (;;) {
    unsigned long long cur = a.ws[h].key;
    if (cur == key) return (int32_t)h;
    if (cur == kEmptyWord) {
      cur = atomicCAS(&a.ws[h].key, kEmptyWord, key);
      if (cur == kEmptyWord || cur == key) return (int32_t)h;
    }
    h = (h + 1) & a.wmask;
  }
}

// ---------------------------------------------------------------------------
// round 0: hash, wave-start lookup and evaluation
// ---------------------------------------------------------------------------

template <bool CLOSEST, int STACK>
__global__ void __launch_bounds__(kBS, 3) k_fast_probe(FastArgs a) {
  FTally c;
  bool bad = false;
  FOR_BLOCK_CHUNKS(a.n) {
    const int64_t i = base_ + threadIdx.x;
    const bool valid = i < a.n;
    bool tp = false;
    if (valid) {
      const uint32_t* ob = reinterpret_cast<const uint32_t*>(a.O) + 3 * i;
      const uint32_t* db = reinterpret_cast<const uint32_t*>(a.D) + 3 * i;
      const uint32_t o0 = ob[0], o1 = ob[1], o2 = ob[2], d0 = db[0], d1 = db[1], d2 = db[2];
      bad |= nonfinite(o0) | nonfinite(o1) | nonfinite(o2) | nonfinite(d0) | nonfinite(d1) |
             nonfinite(d2);
      const unsigned long long key = ray_key(o0, o1, o2, d0, d1, d2, a.p);
      a.keys[i] = key;
      int32_t e = -1, bk = -1;
      if (!a.empty) {  // index_lookup, keeping the bucket (the commit's key handle)
        uint64_t h = mix64(key) & a.mask;
        for (;;) {
          const ulonglong2 w = *reinterpret_cast<const ulonglong2*>(a.idx + h);
          if (w.x == key) {
            e = (int32_t)(w.y & 0xffffffffull);
            bk = (int32_t)h;
            break;
          }
          if (w.x == kEmptyKey) break;
          h = (h + 1) & a.mask;
        }
      }
      a.eid[i] = e;
      a.bkt[i] = bk;
      Hit acc = empty_entry_result(CLOSEST);
      if (e >= 0) {
        const Ray r = make_ray(a.O, a.D, a.tmin, a.tmax, i);
        const int64_t off = a.e_off[e];
        const int32_t len = a.e_len[e];
        for (int32_t j = 0; j < len; j++) {  // eval_entry_{closest,any}
          if (!CLOSEST && acc.found) break;
          fold_entry<CLOSEST>(acc, trace_from<CLOSEST, STACK>(a.nodes, a.tris, r, a.arena[off + j]));
        }
        c.ob += acc.boxes;
        c.ot += acc.tris;
        if (acc.found) {
          tp = true;
          tally_tp(a, c, acc, acc.boxes);
          write_hit(a, (int32_t)i, acc);
        }
      }
      a.evbox[i] = acc.boxes;
    }
    // round 1's leader election, fused: the key's wave slot and its
    // smallest unresolved ray (once per key and warp)
    const bool unres = valid && !tp;
    const unsigned long long gkey = unres ? a.keys[i] : (1ull << 63) | (unsigned)lane;
    const unsigned grp = __match_any_sync(kFullMask, gkey);
    const int gl = __ffs(grp) - 1;
    int32_t h = -1;
    if (unres && lane == gl) h = wave_claim(a, gkey);
    h = __shfl_sync(kFullMask, h, gl);
    const unsigned mn = __reduce_min_sync(grp, unres ? (unsigned)i : kNoRay);
    if (unres) {
      a.wh[i] = h;
      if (lane == gl) atomicMin(&a.ws[h].first, mn);
    }
    const int pos = block_append(a.ctr + C_UOUT, unres);
    if (pos >= 0) a.U[pos] = (int32_t)i;
  }
  flush(c, a.stats);
  if (__any_sync(kFullMask, bad) && (threadIdx.x & 31) == 0) atomicOr(a.err, 1);
}

// ---------------------------------------------------------------------------
// rounds
// ---------------------------------------------------------------------------

// Round bookkeeping (one thread, between rounds): the followers that
// survived the last round become this round's input; a round that resolved
// fewer than n / stop_div rays ends the rounds (the final pass takes the
// rest).  Deterministic: the counts are exact.
__global__ void k_fast_round(FastArgs a, int round, int final_pass) {
  int* c = a.ctr;
  if (!c[C_STOP]) {
    if (!final_pass && round >= 2 && a.stop_div > 0 &&
        (long long)c[C_RES] * a.stop_div < a.n) {
      c[C_STOP] = 1;
    }
    c[C_UIN] = c[C_UOUT];
    c[C_UOUT] = 0;
  }
  if (final_pass) c[C_STOP] = 0;
  c[C_RES] = 0;
  c[C_F] = 0;
  c[C_TICKET] = 0;
  c[C_BEG] = c[C_TQ];
}

// Rounds >= 2: the smallest unresolved ray of each key (slots were claimed
// by the probe).
__global__ void __launch_bounds__(kBS) k_fast_lead(FastArgs a) {
  if (*a.err || a.ctr[C_STOP]) return;
  FOR_BLOCK_CHUNKS(a.ctr[C_UIN]) {
    const int64_t q = base_ + threadIdx.x;
    const bool valid = q < cnt_;
    const int32_t i = valid ? a.U[q] : -1;
    const int32_t h = valid ? a.wh[i] : -1 - lane;
    const unsigned grp = __match_any_sync(kFullMask, h);
    const int gl = __ffs(grp) - 1;
    const unsigned mn = __reduce_min_sync(grp, valid ? (unsigned)i : kNoRay);
    if (valid && lane == gl) atomicMin(&a.ws[h].first, mn);
  }
}

// Leaders (or, in the final pass, every unresolved ray) go to the traced
// list, the other rays to the follower list.
__global__ void __launch_bounds__(kBS) k_fast_split(FastArgs a, int final_pass) {
  if (*a.err || a.ctr[C_STOP]) return;
  FTally c;
  FOR_BLOCK_CHUNKS(a.ctr[C_UIN]) {
    const int64_t q = base_ + threadIdx.x;
    const bool valid = q < cnt_;
    const int32_t i = valid ? a.U[q] : -1;
    bool lead = false;
    if (valid) {
      const int32_t h = a.wh[i];
      lead = final_pass || a.ws[h].first == (uint32_t)i;
      if (lead && !final_pass) {  // NEG iff no entry at its turn (hrpp/tracer.py:314-317)
        if (a.eid[i] >= 0 || a.ws[h].hit) c.fp++;
        else c.neg++;
      }
    }
    const int pt = block_append(a.ctr + C_TQ, lead);
    if (pt >= 0) a.TQ[pt] = i;
    const int pf = block_append(a.ctr + C_F, valid && !lead);
    if (pf >= 0) a.F[pf] = i;
  }
  flush(c, a.stats);
}

// Full traversal of TQ[beg, end) (persistent one-warp blocks taking
// kTicket-ray tickets).  Leaders then publish their node for this round's
// followers; in the final pass each key's first hitting ray is kept.
constexpr int kTicket = 32;  // one ray per lane: a round of few leaders has no serial tail

template <bool CLOSEST, int STACK, bool FINAL>
__device__ __forceinline__ void trace_listed(const FastArgs& a, FTally& c, int32_t i, int round) {
  const Ray r = make_ray(a.O, a.D, a.tmin, a.tmax, i);
  const Hit h = trace_from<CLOSEST, STACK>(a.nodes, a.tris, r, 0);
  write_hit(a, i, h);
  c.bb += h.boxes;
  c.bt += h.tris;
  WSlot& w = a.ws[a.wh[i]];
  if (FINAL) {
    if (h.found) atomicMin(&w.fhit, (uint32_t)i);
    return;
  }
  w.first = kNoRay;  // read by this round's split only
  if (!h.found) return;
  w.hit = 1;
  const int32_t node = a.anc[h.leaf];
  bool listed = in_entry(a, a.eid[i], node);
  for (int32_t x = w.head; x >= 0 && !listed; x = a.nxt[x]) listed = a.anc[a.o_leaf[x]] == node;
  if (!listed) {  // one leader per key and round: no race on the slot
    a.nxt[i] = w.head;
    w.head = i;
    w.cur = ((long long)round << 32) | (uint32_t)node;
  }
}

template <bool CLOSEST, int STACK, bool FINAL>
__global__ void __launch_bounds__(32, 32) k_fast_trace(FastArgs a, int round) {
  if (*a.err || a.ctr[C_STOP]) return;
  const int lane = threadIdx.x & 31;
  const int beg = a.ctr[C_BEG], end = a.ctr[C_TQ];
  FTally c;
  for (;;) {
    int t = 0;
    if (lane == 0) t = atomicAdd(a.ctr + C_TICKET, kTicket);
    t = __shfl_sync(kFullMask, t, 0);
    if (beg + t >= end) break;
    for (int sub = lane; sub < kTicket && beg + t + sub < end; sub += 32)
      trace_listed<CLOSEST, STACK, FINAL>(a, c, a.TQ[beg + t + sub], round);
  }
  flush(c, a.stats);
}

// Followers evaluate this round's new node of their key.
template <bool CLOSEST, int STACK>
__global__ void __launch_bounds__(kBS, 3) k_fast_follow(FastArgs a, int round) {
  if (*a.err || a.ctr[C_STOP]) return;
  FTally c;
  FOR_BLOCK_CHUNKS(a.ctr[C_F]) {
    const int64_t q = base_ + threadIdx.x;
    const bool valid = q < cnt_;
    bool keep = valid;
    if (valid) {
      const int32_t i = a.F[q];
      const long long w = a.ws[a.wh[i]].cur;
      if (w >= 0 && (int)(w >> 32) == round) {
        const Ray r = make_ray(a.O, a.D, a.tmin, a.tmax, i);
        const Hit h = trace_from<CLOSEST, STACK>(a.nodes, a.tris, r, (int32_t)(w & 0xffffffff));
        c.ob += h.boxes;
        c.ot += h.tris;
        const int32_t boxes = a.evbox[i] + h.boxes;
        a.evbox[i] = boxes;
        if (h.found) {
          keep = false;
          tally_tp(a, c, h, boxes);
          write_hit(a, i, h);
        }
      }
    }
    const int pos = block_append(a.ctr + C_UOUT, keep);
    if (pos >= 0) a.U[pos] = a.F[q];
  }
  const long long res = warp_sum(c.tp);
  if ((threadIdx.x & 31) == 0 && res) atomicAdd(a.ctr + C_RES, (int)res);
  flush(c, a.stats);
}

// Final pass: NEG/FP with the entry as it stood at each ray's turn (listed,
// or an earlier traced ray of the key hit).
__global__ void __launch_bounds__(kBS) k_fast_final_class(FastArgs a) {
  if (*a.err) return;
  FTally c;
  const int beg = a.ctr[C_BEG], end = a.ctr[C_TQ];
  for (int q = beg + blockIdx.x * blockDim.x + threadIdx.x; q < end;
       q += gridDim.x * blockDim.x) {
    const int32_t i = a.TQ[q];
    const WSlot& w = a.ws[a.wh[i]];
    if (a.eid[i] >= 0 || w.hit || w.fhit < (uint32_t)i) c.fp++;
    else c.neg++;
  }
  flush(c, a.stats);
}

// ---------------------------------------------------------------------------
// commit: (key, anc[leaf]) of every traced ray with a hit, set semantics,
// new nodes of an entry ordered by the first ray that recorded them.  Pairs
// and per-key counters are keyed by the key's index bucket (a new key's
// entry id is only assigned in k_fast_alloc): the count of a key's new nodes
// lives in its bucket's spare word (-1 = none), so a record touches the
// bucket's sector, one pair-set slot and no global counter.
// ---------------------------------------------------------------------------

__device__ __forceinline__ int32_t bucket_claim(const FastArgs& a, unsigned long long key) {
  uint64_t h = mix64(key) & a.mask;
  for (;;) {
    unsigned long long cur = a.idx[h].key;
    if (cur == key) return (int32_t)h;
    if (cur == kEmptyKey) {
      cur = atomicCAS(&a.idx[h].key, kEmptyKey, key);  // val stays -1 until k_fast_alloc
      if (cur == kEmptyKey || cur == key) return (int32_t)h;
    }
    h = (h + 1) & a.mask;
  }
}

__global__ void __launch_bounds__(kBS) k_fast_records(FastArgs a) {
  FOR_BLOCK_CHUNKS(a.ctr[C_TQ]) {
    const int64_t q = base_ + threadIdx.x;
    bool rec = false;
    int32_t b = -1, h2 = -1, rank = -1;
    if (q < cnt_) {
      const int32_t i = a.TQ[q];
      // the wave slot is done with (every slot has a round-1 leader here)
      const WSlot empty_slot{kEmptyWord, kNoRay, kNoRay, -1, 0, -1};
      a.ws[a.wh[i]] = empty_slot;
      if (a.o_found[i]) {
        const int32_t node = a.anc[a.o_leaf[i]];
        const int32_t e = a.eid[i];
        if (!in_entry(a, e, node)) {  // record() of a listed node is a no-op
          b = e >= 0 ? a.bkt[i] : bucket_claim(a, a.keys[i]);
          const unsigned long long pair = ((unsigned long long)(uint32_t)b << 32) | (uint32_t)node;
          uint64_t h = mix64(pair) & a.pmask;
          for (;;) {
            const unsigned long long cur = atomicCAS(&a.ps[h].pair, kEmptyWord, pair);
            if (cur == kEmptyWord || cur == pair) {
              atomicMin(&a.ps[h].ray, (uint32_t)i);
              if (cur == kEmptyWord) {
                rec = true;
                h2 = (int32_t)h;
                rank = atomicAdd(&a.idx[b].pad, 1) + 1;
              }
              break;
            }
            h = (h + 1) & a.pmask;
          }
        }
      }
    }
    const int pr = block_append(a.ctr + C_NREC, rec);
    if (pr >= 0) a.recs[pr] = make_int2(h2, rank);
    const int pt = block_append(a.ctr + C_TOUCH, rec && rank == 0);
    if (pt >= 0) a.touched[pt] = b;
  }
}

// Every touched key: a new entry id if it had none, then its list moves to
// the arena tail with room for the new nodes (lists stay contiguous, as in
// table_commit); keys with several new nodes get a range of the record
// buffer for ordering them.
//
// The commit kernels run even after an error so that the wave's scratch is
// left clean; a key whose new entry would pass the entry cap is not created
// (CapacityExceeded: its bucket keeps val -1, i.e. absent to every lookup).
__global__ void __launch_bounds__(kBS) k_fast_alloc(FastArgs a) {
  FOR_BLOCK_CHUNKS(a.ctr[C_TOUCH]) {
    const int64_t k = base_ + threadIdx.x;
    bool valid = k < cnt_;
    int32_t b = 0, add = 0, e = -1;
    if (valid) {
      b = a.touched[k];
      add = a.idx[b].pad + 1;
      e = a.idx[b].val;
    }
    const int pe = block_append(a.ctr + C_NEWE, valid && e < 0);
    if (pe >= 0) {
      if (a.n_entries0 + pe >= a.max_entries) {
        atomicCAS(a.err, 0, 2);  // CapacityExceeded
        a.idx[b].pad = -1;
        valid = false;
      } else {
        e = (int32_t)(a.n_entries0 + pe);
        a.e_key[e] = a.idx[b].key;
        a.e_len[e] = 0;
        a.e_off[e] = 0;
        a.idx[b].val = e;
      }
    }
    block_alloc(a.lctr + 1, pe >= 0 && valid ? 1 : 0);  // entries created
    block_alloc(a.lctr + 2, valid ? add : 0);          // nodes stored
    const int32_t old = valid ? a.e_len[e] : 0;
    const long long off = block_alloc(a.meta + 2, valid ? old + add : 0);
    const long long wb = block_alloc(a.lctr, valid && add > 1 ? add : 0);
    const int pm = block_append(a.ctr + C_MULTI, valid && add > 1);
    if (pm >= 0) a.multi[pm] = b;
    if (valid) {
      const int64_t src = a.e_off[e];
      for (int32_t j = 0; j < old; j++) a.arena[off + j] = a.arena[src + j];
      a.e_off[e] = off;
      a.e_len[e] = old + add;
      if (add > 1) a.wbase[b] = (int32_t)wb;
      else a.idx[b].pad = -1;  // single new node: placed by k_fast_scatter
    }
  }
}

// A single new node goes straight to its entry's last position; several go
// to the key's record range for k_fast_order.  The pair set is left empty.
__global__ void __launch_bounds__(kBS) k_fast_scatter(FastArgs a) {
  const int m = a.ctr[C_NREC];
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < m; k += gridDim.x * blockDim.x) {
    const int2 r = a.recs[k];
    const PSlot p = a.ps[r.x];
    const int32_t b = (int32_t)(p.pair >> 32);
    const int32_t node = (int32_t)(p.pair & 0xffffffffull);
    if (a.idx[b].val < 0) {
      // not created (entry cap)
    } else if (a.idx[b].pad < 0) {
      const int32_t e = a.idx[b].val;
      a.arena[a.e_off[e] + a.e_len[e] - 1] = node;
    } else {
      a.wrec[a.wbase[b] + r.y] = ((unsigned long long)p.ray << 32) | (uint32_t)node;
    }
    a.ps[r.x] = PSlot{kEmptyWord, kNoRay, 0};
  }
}

// One warp per key with several new nodes: in the order of the rays that
// first recorded them (rank = number of smaller (ray, node) words).
__global__ void __launch_bounds__(kBS) k_fast_order(FastArgs a) {
  const int lane = threadIdx.x & 31;
  const int m = a.ctr[C_MULTI];
  for (int k = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; k < m;
       k += (gridDim.x * blockDim.x) >> 5) {
    const int32_t b = a.multi[k];
    const int32_t add = a.idx[b].pad + 1;
    const int32_t e = a.idx[b].val;
    const unsigned long long* w = a.wrec + a.wbase[b];
    int32_t* dst = a.arena + a.e_off[e] + a.e_len[e] - add;
    for (int32_t j = lane; j < add; j += 32) {
      const unsigned long long x = w[j];
      int32_t rank = 0;
      for (int32_t q = 0; q < add; q++) rank += w[q] < x;
      dst[rank] = (int32_t)(x & 0xffffffffull);
    }
    __syncwarp();
    if (lane == 0) a.idx[b].pad = -1;
  }
}

__global__ void k_fast_meta(FastArgs a) {
  a.meta[0] += a.lctr[1];
  a.meta[1] += a.lctr[2];
}

__global__ void k_init_slots(WSlot* ws, PSlot* ps, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    ws[i] = WSlot{kEmptyWord, kNoRay, kNoRay, -1, 0, -1};
    ps[i] = PSlot{kEmptyWord, kNoRay, 0};
  }
}

template <bool CLOSEST, int STACK>
int fast_impl(const FastArgs& a, int rounds, cudaStream_t st) {
  const int sms = num_sms();
  const int gn = grid_for(a.n, kBS, sms * 8);
  k_fast_probe<CLOSEST, STACK><<<gn, kBS, 0, st>>>(a);
  HRPP_LAUNCHED();
  for (int k = 1; k <= rounds + 1; k++) {
    const bool fin = k == rounds + 1;
    k_fast_round<<<1, 1, 0, st>>>(a, k, fin ? 1 : 0);
    HRPP_LAUNCHED();
    if (k >= 2 && !fin) {
      k_fast_lead<<<gn, kBS, 0, st>>>(a);
      HRPP_LAUNCHED();
    }
    k_fast_split<<<gn, kBS, 0, st>>>(a, fin ? 1 : 0);
    HRPP_LAUNCHED();
    if (fin) {
      k_fast_trace<CLOSEST, STACK, true><<<sms * 32, 32, 0, st>>>(a, k);
      HRPP_LAUNCHED();
      k_fast_final_class<<<gn, kBS, 0, st>>>(a);
      HRPP_LAUNCHED();
    } else {
      k_fast_trace<CLOSEST, STACK, false><<<sms * 32, 32, 0, st>>>(a, k);
      HRPP_LAUNCHED();
      k_fast_follow<CLOSEST, STACK><<<gn, kBS, 0, st>>>(a, k);
      HRPP_LAUNCHED();
    }
  }
  k_fast_records<<<gn, kBS, 0, st>>>(a);
  HRPP_LAUNCHED();
  k_fast_alloc<<<gn, kBS, 0, st>>>(a);
  HRPP_LAUNCHED();
  k_fast_scatter<<<gn, kBS, 0, st>>>(a);
  HRPP_LAUNCHED();
  k_fast_order<<<gn, kBS, 0, st>>>(a);
  HRPP_LAUNCHED();
  k_fast_meta<<<1, 1, 0, st>>>(a);
  HRPP_LAUNCHED();
  return 0;
}

int64_t pow2_at_least(int64_t x) {
  int64_t p = 1024;
  while (p < x) p <<= 1;
  return p;
}

}  // namespace

int run_fast(const BvhDev& b, TableDev& t, const FastIO& io, unsigned long long* stats_dev,
             int* err, cudaStream_t st) {
  const int64_t n = io.n;
  if (n <= 0) return 0;
  int rc;
  const int32_t* anc;
  if ((rc = const_cast<BvhDev&>(b).ancestor_lut(t.go_up, &anc))) return rc;
  if ((rc = t.reserve(n, n, st))) return rc;  // new entries and nodes <= rays
  Workspace& ws = t.ws;
  FastArgs a{};
  a.nodes = b.nodes;
  a.tris = b.tris;
  a.depth = b.depth;
  a.anc = anc;
  a.O = io.O;
  a.D = io.D;
  a.tmin = io.tmin;
  a.tmax = io.tmax;
  a.n = n;
  a.p = t.precision;
  a.stop_div = g_fast_stop_div;
  a.idx = t.idx;
  a.mask = (uint64_t)t.idx_cap - 1;
  a.e_off = t.e_off;
  a.e_len = t.e_len;
  a.e_key = t.e_key;
  a.arena = t.arena;
  a.meta = t.meta;
  a.n_entries0 = t.n_entries;
  a.max_entries = t.max_entries;
  a.empty = t.n_entries == 0;
  a.o_found = io.found;
  a.o_t = io.t;
  a.o_slot = io.slot;
  a.o_leaf = io.leaf;
  a.keys = reinterpret_cast<unsigned long long*>(io.keys);
  a.stats = stats_dev;
  a.err = err;
  if ((rc = ws.get("f_eid", n, &a.eid)) || (rc = ws.get("f_evbox", n, &a.evbox)) ||
      (rc = ws.get("f_wh", n, &a.wh)) || (rc = ws.get("f_nxt", n, &a.nxt)) ||
      (rc = ws.get("f_u", n, &a.U)) ||
      (rc = ws.get("f_f", n, &a.F)) || (rc = ws.get("f_tq", n, &a.TQ)) ||
      (rc = ws.get("f_touched", n, &a.touched)) || (rc = ws.get("f_recs", n, &a.recs)) ||
      (rc = ws.get("f_wrec", n, &a.wrec)) || (rc = ws.get("f_ctr", C_N, &a.ctr)) ||
      (rc = ws.get("f_bkt", n, &a.bkt)) || (rc = ws.get("f_lctr", 3, &a.lctr)))
    return rc;
  // wave slots and the pair set: sized for 2n, initialised once, left empty
  // by every wave (k_fast_records, k_fast_scatter)
  const int64_t W = pow2_at_least(2 * n);
  if (W > t.fast_wcap) {
    if ((rc = ws.get("f_wslot", W, &a.ws)) || (rc = ws.get("f_pslot", W, &a.ps))) return rc;
    k_init_slots<<<grid_for(W, 256, num_sms() * 8), 256, 0, st>>>(a.ws, a.ps, W);
    HRPP_LAUNCHED();
    t.fast_wcap = W;
  }
  if ((rc = ws.get("f_wslot", t.fast_wcap, &a.ws)) || (rc = ws.get("f_pslot", t.fast_wcap, &a.ps)) ||
      (rc = ws.get("f_wbase", t.idx_cap, &a.wbase)) || (rc = ws.get("f_multi", n, &a.multi)))
    return rc;
  a.wmask = a.pmask = (uint64_t)t.fast_wcap - 1;
  HRPP_CK(cudaMemsetAsync(a.ctr, 0, sizeof(int) * C_N + 0, st));
  HRPP_CK(cudaMemsetAsync(a.lctr, 0, sizeof(long long) * 3, st));
  const int R = g_fast_rounds;
  switch (b.stack) {
    case 64:
      return t.closest ? fast_impl<true, 64>(a, R, st) : fast_impl<false, 64>(a, R, st);
    case 256:
      return t.closest ? fast_impl<true, 256>(a, R, st) : fast_impl<false, 256>(a, R, st);
    default:
      return t.closest ? fast_impl<true, 512>(a, R, st) : fast_impl<false, 512>(a, R, st);
  }
}

}  // namespace hrpp
