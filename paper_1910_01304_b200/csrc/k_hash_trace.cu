// k_hash_trace.cu -- ray hash kernel and full-traversal batch kernel.
#include <cstdlib>

#include <cub/cub.cuh>

#include "hrpp_internal.h"

namespace hrpp {

// ---------------------------------------------------------------------------
// Ray hash (hrpp/rayhash.py:99-122).  HBM-bound: 24 B in + 8 B out per ray.
// Each thread hashes 4 consecutive rays: 3 x 16-B streaming loads each of O
// and D (48 B = 4 rays x 3 floats), two 16-B key stores.
// ---------------------------------------------------------------------------

__device__ __forceinline__ uint32_t lane_hash(uint32_t bits, int p) {
  uint32_t sign = bits >> 31;
  uint32_t exp_top = ((bits >> 23) & 0xFFu) >> (8 - p);
  uint32_t man_top = (bits & 0x7FFFFFu) >> (23 - p);
  return (sign << (2 * p)) | (exp_top << p) | man_top;
}

__device__ __forceinline__ bool nonfinite(uint32_t b) { return ((b >> 23) & 0xFFu) == 0xFFu; }

// LANE_PAIRS ((0,2),(1,1),(2,0)) at shifts 0/16/32 (hrpp/rayhash.py:37-39)
__device__ __forceinline__ uint64_t ray_key(uint32_t ox, uint32_t oy, uint32_t oz, uint32_t dx,
                                            uint32_t dy, uint32_t dz, int p) {
  return (uint64_t)(lane_hash(ox, p) ^ lane_hash(dz, p)) |
         ((uint64_t)(lane_hash(oy, p) ^ lane_hash(dy, p)) << 16) |
         ((uint64_t)(lane_hash(oz, p) ^ lane_hash(dx, p)) << 32);
}

__global__ void __launch_bounds__(256) k_hash(const float* __restrict__ O,
                                              const float* __restrict__ D, int64_t n, int p,
                                              uint64_t* __restrict__ keys, int* err) {
  const int64_t nq = (n + 3) / 4;
  const bool vec = ((reinterpret_cast<uintptr_t>(O) | reinterpret_cast<uintptr_t>(D) |
                     reinterpret_cast<uintptr_t>(keys)) & 15) == 0;
  bool bad = false;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < nq;
       q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i0 = 4 * q;
    if (vec && i0 + 4 <= n) {
      const float4* o4 = reinterpret_cast<const float4*>(O + 3 * i0);
      const float4* d4 = reinterpret_cast<const float4*>(D + 3 * i0);
      float4 oa = __ldcs(o4), ob = __ldcs(o4 + 1), oc = __ldcs(o4 + 2);
      float4 da = __ldcs(d4), db = __ldcs(d4 + 1), dc = __ldcs(d4 + 2);
      uint32_t o[12] = {__float_as_uint(oa.x), __float_as_uint(oa.y), __float_as_uint(oa.z),
                        __float_as_uint(oa.w), __float_as_uint(ob.x), __float_as_uint(ob.y),
                        __float_as_uint(ob.z), __float_as_uint(ob.w), __float_as_uint(oc.x),
                        __float_as_uint(oc.y), __float_as_uint(oc.z), __float_as_uint(oc.w)};
      uint32_t d[12] = {__float_as_uint(da.x), __float_as_uint(da.y), __float_as_uint(da.z),
                        __float_as_uint(da.w), __float_as_uint(db.x), __float_as_uint(db.y),
                        __float_as_uint(db.z), __float_as_uint(db.w), __float_as_uint(dc.x),
                        __float_as_uint(dc.y), __float_as_uint(dc.z), __float_as_uint(dc.w)};
#pragma unroll
      for (int k = 0; k < 12; k++) bad |= nonfinite(o[k]) | nonfinite(d[k]);
      ulonglong2 k01, k23;
      k01.x = ray_key(o[0], o[1], o[2], d[0], d[1], d[2], p);
      k01.y = ray_key(o[3], o[4], o[5], d[3], d[4], d[5], p);
      k23.x = ray_key(o[6], o[7], o[8], d[6], d[7], d[8], p);
      k23.y = ray_key(o[9], o[10], o[11], d[9], d[10], d[11], p);
      ulonglong2* kp = reinterpret_cast<ulonglong2*>(keys + i0);
      __stcs(kp, k01);
      __stcs(kp + 1, k23);
    } else {
      const int64_t e = i0 + 4 < n ? i0 + 4 : n;
      for (int64_t i = i0; i < e; i++) {
        uint32_t o0 = __float_as_uint(O[3 * i]), o1 = __float_as_uint(O[3 * i + 1]),
                 o2 = __float_as_uint(O[3 * i + 2]);
        uint32_t d0 = __float_as_uint(D[3 * i]), d1 = __float_as_uint(D[3 * i + 1]),
                 d2 = __float_as_uint(D[3 * i + 2]);
        bad |= nonfinite(o0) | nonfinite(o1) | nonfinite(o2) | nonfinite(d0) | nonfinite(d1) |
               nonfinite(d2);
        keys[i] = ray_key(o0, o1, o2, d0, d1, d2, p);
      }
    }
  }
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(err, 1);
}

int launch_hash(const float* O, const float* D, int64_t n, int p, uint64_t* keys, int* err,
                cudaStream_t st) {
  if (n <= 0) return 0;
  int64_t nq = (n + 3) / 4;
  int grid = grid_for(nq, 256, num_sms() * 8);
  ProfScope ps(P_HASH, st);
  k_hash<<<grid, 256, 0, st>>>(O, D, n, p, keys, err);
  HRPP_LAUNCHED();
  return 0;
}

// hrpp/rayhash.py:67-78 map_float_to_hash over a float32 array
__global__ void k_hash_floats(const float* __restrict__ f, int64_t n, int p,
                              uint32_t* __restrict__ out, int* err) {
  bool bad = false;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    uint32_t b = __float_as_uint(f[i]);
    bad |= nonfinite(b);
    out[i] = lane_hash(b, p);
  }
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(err, 1);
}

int launch_hash_floats(const float* f, int64_t n, int p, uint32_t* out, int* err,
                       cudaStream_t st) {
  if (n <= 0) return 0;
  k_hash_floats<<<grid_for(n, 256, num_sms() * 8), 256, 0, st>>>(f, n, p, out, err);
  HRPP_LAUNCHED();
  return 0;
}

// ---------------------------------------------------------------------------
// Full traversal batch (hrpp/kernels.py:209-248): one ray per thread, f64,
// per-thread stack in local memory sized from the tree height.  Optional
// indirection (ray_idx / count_dev) traces a compacted queue of rays.
// ---------------------------------------------------------------------------

struct TraceArgs {
  const DNode* nodes;
  const DTri* tris;
  const float* O;
  const float* D;
  const double* tmin;
  const double* tmax;
  int32_t start;
  int64_t n;
  const int32_t* ray_idx;
  const int* count_dev;
  const int* err;
  TraceOut out;
};

// Register cap from the resident-block target: 7 x 128 threads -> 72
// registers (measured best of 1, 5, 6, 7, 8 on c2: +6 % primary, +8 %
// shadow, +13 % bounce over the uncapped 86).  A leaf-batched "while-while"
// loop (warp-synchronous box and triangle phases) measured 40 % slower.
#ifndef HRPP_TRACE_MINB
#define HRPP_TRACE_MINB 7
#endif

template <bool CLOSEST, int STACK>
__global__ void __launch_bounds__(128, HRPP_TRACE_MINB) k_trace(TraceArgs a) {
  if (a.err && *a.err) return;
  // one ray per thread; with a device-side count (fallback queue) the grid is
  // sized for the host-known upper bound and surplus threads exit at once
  const int64_t count = a.count_dev ? (int64_t)*a.count_dev : a.n;
  const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  unsigned long long sb = 0, stt = 0;
  if (q < count) {
    const int64_t i = a.ray_idx ? (int64_t)a.ray_idx[q] : q;
    Ray r = make_ray(a.O, a.D, a.tmin, a.tmax, i);
    Hit h = trace_from<CLOSEST, STACK>(a.nodes, a.tris, r, a.start);
    const TraceOut& o = a.out;
    if (o.found) o.found[i] = h.found;
    if (o.t) o.t[i] = h.t;
    if (o.slot) o.slot[i] = h.slot;
    if (o.leaf) o.leaf[i] = h.leaf;
    if (CLOSEST && (o.u || o.v)) {
      double u, v;
      hit_uv(a.tris, r, h, u, v);
      if (o.u) o.u[i] = u;
      if (o.v) o.v[i] = v;
    }
    if (o.box) o.box[i] = h.boxes;
    if (o.tri) o.tri[i] = h.tris;
    if (o.vis) o.vis[i] = h.boxes;  // visited == box_tests (kernels.py:115-116)
    if (o.known) o.known[i] = 1;
    sb = h.boxes;
    stt = h.tris;
  }
  if (a.out.sums) {  // one atomic pair per block (a.out.sums is uniform)
    __shared__ unsigned long long part[2][4];
    sb = warp_sum(sb);
    stt = warp_sum(stt);
    if ((threadIdx.x & 31) == 0) {
      part[0][threadIdx.x >> 5] = sb;
      part[1][threadIdx.x >> 5] = stt;
    }
    __syncthreads();
    if (threadIdx.x < 2) {
      const unsigned long long v = part[threadIdx.x][0] + part[threadIdx.x][1] +
                                   part[threadIdx.x][2] + part[threadIdx.x][3];
      if (v) atomicAdd(a.out.sums + threadIdx.x, v);
    }
  }
}

// Persistent traversal for divergent (secondary) waves: warps stay resident
// and refill finished lanes from a per-warp chunk of rays (one global atomic
// per 256 rays) whenever fewer than kRefillBelow lanes are busy.  Each ray's
// node-visit sequence is exactly trace_from's, so results are identical.
constexpr int kChunk = 256;
#ifndef HRPP_REFILL_BELOW
#define HRPP_REFILL_BELOW 24
#endif
#ifndef HRPP_PERSIST_STEPS
#define HRPP_PERSIST_STEPS 16
#endif
constexpr int kRefillBelow = HRPP_REFILL_BELOW;
int g_trace_persistent = 0;

template <bool CLOSEST>
__device__ __forceinline__ void store_hit(const TraceOut& o, const DTri* tris, const Ray& r,
                                          int64_t i, const Hit& h) {
  if (o.found) o.found[i] = h.found;
  if (o.t) o.t[i] = h.t;
  if (o.slot) o.slot[i] = h.slot;
  if (o.leaf) o.leaf[i] = h.leaf;
  if (CLOSEST && (o.u || o.v)) {
    double u, v;
    hit_uv(tris, r, h, u, v);
    if (o.u) o.u[i] = u;
    if (o.v) o.v[i] = v;
  }
  if (o.box) o.box[i] = h.boxes;
  if (o.tri) o.tri[i] = h.tris;
  if (o.vis) o.vis[i] = h.boxes;
  if (o.known) o.known[i] = 1;
}

#ifndef HRPP_PERSIST_MINB
#define HRPP_PERSIST_MINB 7
#endif

template <bool CLOSEST, int STACK>
__global__ void __launch_bounds__(128, HRPP_PERSIST_MINB) k_trace_persist(TraceArgs a,
                                                                          int* chunk_counter,
                                                                          int refill_below) {
  if (a.err && *a.err) return;
  const int64_t count = a.count_dev ? (int64_t)*a.count_dev : a.n;
  const int lane = threadIdx.x & 31;
  LocalStack<STACK> stack;
  int top = 0;
  int32_t nd = -1;  // next node to box-test; -1 = lane idle
  Hit h;
  h.found = false; h.t = 0.0; h.slot = -1; h.leaf = -1;
  h.boxes = 0; h.tris = 0;
  Ray r{};
  int64_t cur = -1;
  int64_t c_lo = 0, c_hi = 0;
  bool more = true;
  unsigned long long sb = 0, stt = 0;
  for (;;) {
    unsigned busy = __ballot_sync(0xffffffffu, cur >= 0);
    if (more && __popc(busy) < refill_below) {
      unsigned idle = ~busy;
      while (idle && more) {
        if (c_lo >= c_hi) {
          int base = 0;
          if (lane == 0) base = atomicAdd(chunk_counter, kChunk);
          base = __shfl_sync(0xffffffffu, base, 0);
          c_lo = base;
          c_hi = (int64_t)base + kChunk < count ? (int64_t)base + kChunk : count;
          if (c_lo >= count) {
            more = false;
            break;
          }
        }
        const int avail = (int)(c_hi - c_lo);
        const int rank = __popc(idle & ((1u << lane) - 1u));
        if (cur < 0 && rank < avail) {
          const int64_t q = c_lo + rank;
          cur = a.ray_idx ? (int64_t)a.ray_idx[q] : q;
          r = make_ray(a.O, a.D, a.tmin, a.tmax, cur);
          nd = a.start;
          top = 0;
          h.found = false;
          h.t = CLOSEST ? r.tmax : 0.0;
          h.slot = -1; h.leaf = -1; h.boxes = 0; h.tris = 0;
        }
        const int took = __popc(idle) < avail ? __popc(idle) : avail;
        c_lo += took;
        idle = __ballot_sync(0xffffffffu, cur < 0);
      }
      busy = __ballot_sync(0xffffffffu, cur >= 0);
    }
    if (!busy) break;
    if (cur >= 0) {
      // up to HRPP_PERSIST_STEPS node visits of trace_stk (hrpp/kernels.py:112-153)
      for (int it = 0; it < HRPP_PERSIST_STEPS && nd >= 0; it++) {
        h.boxes++;
        const NodeBox bx = load_node(a.nodes, nd);
        if (box_hit(bx, r.ox, r.oy, r.oz, r.ivx, r.ivy, r.ivz, r.tmin, CLOSEST ? h.t : r.tmax)) {
          if (bx.a >= 0) {
            const int axis = (uint32_t)bx.b >> 30;
            const int32_t right = bx.b & 0x3FFFFFFF;
            const double dval = axis == 1 ? r.dy : (axis == 2 ? r.dz : r.dx);
            stack[top++] = dval >= 0.0 ? right : bx.a;
            nd = dval >= 0.0 ? bx.a : right;
            continue;
          }
          const int32_t f = ~bx.a, e = f + bx.b;
          bool stop = false;
          for (int32_t k = f; k < e; k++) {
            double t, u, v;
            h.tris++;
            if (tri_test(a.tris, k, r.ox, r.oy, r.oz, r.dx, r.dy, r.dz, t, u, v) &&
                t >= r.tmin && t <= r.tmax) {
              if (!CLOSEST) {
                h.found = true; h.t = t; h.slot = k; h.leaf = nd;
                stop = true;
                break;
              }
              if (!h.found || t < h.t) {
                h.found = true; h.t = t; h.slot = k; h.leaf = nd;
              }
            }
          }
          if (stop) top = 0;
        }
        nd = top > 0 ? stack[--top] : -1;
      }
      if (nd < 0) {
        store_hit<CLOSEST>(a.out, a.tris, r, cur, h);
        sb += h.boxes;
        stt += h.tris;
        cur = -1;
      }
    }
  }
  if (a.out.sums) {
    sb = warp_sum(sb);
    stt = warp_sum(stt);
    if (lane == 0 && (sb | stt)) {
      atomicAdd(a.out.sums, sb);
      atomicAdd(a.out.sums + 1, stt);
    }
  }
}

template <bool CLOSEST, int STACK>
static void launch_persist(cudaStream_t st, const TraceArgs& a, int* counter) {
  static int refill = -1;
  if (refill < 0) {
    const char* e = getenv("HRPP_REFILL");
    refill = e ? atoi(e) : kRefillBelow;
  }
  static int per_sm = 0;  // resident blocks of this instantiation
  if (!per_sm &&
      (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_trace_persist<CLOSEST, STACK>,
                                                     128, 0) != cudaSuccess ||
       per_sm < 1))
    per_sm = 4;
  const int64_t need = (a.n + 127) / 128;
  const int64_t res = (int64_t)num_sms() * per_sm;
  const int grid = (int)(res < need ? res : (need > 0 ? need : 1));
  k_trace_persist<CLOSEST, STACK><<<grid, 128, 0, st>>>(a, counter, refill);
}

template <bool CLOSEST>
static void dispatch_persist(int stack, cudaStream_t st, const TraceArgs& a, int* counter) {
  switch (stack) {
    case 32: launch_persist<CLOSEST, 32>(st, a, counter); break;
    case 64: launch_persist<CLOSEST, 64>(st, a, counter); break;
    case 128: launch_persist<CLOSEST, 128>(st, a, counter); break;
    case 256: launch_persist<CLOSEST, 256>(st, a, counter); break;
    default: launch_persist<CLOSEST, 512>(st, a, counter); break;
  }
}

template <bool CLOSEST>
static void dispatch_trace(int stack, int grid, cudaStream_t st, const TraceArgs& a) {
  switch (stack) {
    case 32: k_trace<CLOSEST, 32><<<grid, 128, 0, st>>>(a); break;
    case 64: k_trace<CLOSEST, 64><<<grid, 128, 0, st>>>(a); break;
    case 128: k_trace<CLOSEST, 128><<<grid, 128, 0, st>>>(a); break;
    case 256: k_trace<CLOSEST, 256><<<grid, 128, 0, st>>>(a); break;
    default: k_trace<CLOSEST, 512><<<grid, 128, 0, st>>>(a); break;
  }
}

// ---------------------------------------------------------------------------
// Coherence order for traversal: 32-bit key = direction octant (3 bits) |
// Morton-interleaved direction (3 bits/axis) | Morton-interleaved origin in
// the scene box (6 bits/axis, 18 bits).  Sorting only permutes which lanes
// trace which rays.
// ---------------------------------------------------------------------------

int g_trace_coherent = 0;
static int coh_begin_bit() {  // radix passes = ceil((30 - begin) / 8)
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("HRPP_COH_BEGIN_BIT");
    v = e ? atoi(e) : 14;
    if (v < 0 || v > 29) v = 14;
  }
  return v;
}
constexpr int64_t kCoherentMin = 1 << 16;  // smaller batches trace in the given order

__device__ __forceinline__ uint32_t spread3(uint32_t x) {  // 10 bits -> every third bit
  x &= 0x3FF;
  x = (x | (x << 16)) & 0x30000FF;
  x = (x | (x << 8)) & 0x300F00F;
  x = (x | (x << 4)) & 0x30C30C3;
  x = (x | (x << 2)) & 0x9249249;
  return x;
}

__device__ __forceinline__ uint32_t quant(float v, float lo, float inv, uint32_t maxq) {
  float q = (v - lo) * inv;
  q = q < 0.f ? 0.f : q;
  uint32_t u = (uint32_t)q;
  return u > maxq ? maxq : u;
}

__global__ void k_coh_key(const float* __restrict__ O, const float* __restrict__ D,
                          const int32_t* __restrict__ ray_idx, const int* count_dev, int64_t n,
                          float3 lo, float3 inv, uint32_t* keys, int32_t* vals) {
  const int64_t count = count_dev ? (int64_t)*count_dev : n;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n;
       q += (int64_t)gridDim.x * blockDim.x) {
    if (q >= count) {  // padding sorts last and is never traced
      keys[q] = 0xFFFFFFFFu;
      vals[q] = 0;
      continue;
    }
    const int64_t i = ray_idx ? (int64_t)ray_idx[q] : q;
    const float dx = D[3 * i], dy = D[3 * i + 1], dz = D[3 * i + 2];
    const uint32_t oct = (dx < 0.f) | ((dz < 0.f) << 1) | ((dy < 0.f) << 2);
    const uint32_t dq = spread3(quant(dx, -1.f, 4.f, 7)) | (spread3(quant(dy, -1.f, 4.f, 7)) << 1) |
                        (spread3(quant(dz, -1.f, 4.f, 7)) << 2);
    const uint32_t oq = spread3(quant(O[3 * i], lo.x, inv.x, 63)) |
                        (spread3(quant(O[3 * i + 1], lo.y, inv.y, 63)) << 1) |
                        (spread3(quant(O[3 * i + 2], lo.z, inv.z, 63)) << 2);
    keys[q] = (oct << 27) | (dq << 18) | oq;
    vals[q] = (int32_t)i;
  }
}

int launch_trace(const BvhDev& b, bool closest, const float* O, const float* D,
                 const double* tmin, const double* tmax, int32_t start, int64_t n,
                 const int32_t* ray_idx, const int* count_dev, const TraceOut& out,
                 const int* err, cudaStream_t st, Workspace* ws) {
  if (n <= 0) return 0;
  if (g_trace_coherent && ws && n >= kCoherentMin) {
    uint32_t *keys, *keys2;
    int32_t *vals, *order;
    int rc;
    if ((rc = ws->get("coh_k", n, &keys)) || (rc = ws->get("coh_k2", n, &keys2)) ||
        (rc = ws->get("coh_v", n, &vals)) || (rc = ws->get("coh_o", n, &order)))
      return rc;
    float3 lo, inv;
    lo.x = b.root_lo[0];
    lo.y = b.root_lo[1];
    lo.z = b.root_lo[2];
    const float ex = b.root_hi[0] - b.root_lo[0], ey = b.root_hi[1] - b.root_lo[1],
                ez = b.root_hi[2] - b.root_lo[2];
    inv.x = ex > 0.f ? 64.f / ex : 0.f;
    inv.y = ey > 0.f ? 64.f / ey : 0.f;
    inv.z = ez > 0.f ? 64.f / ez : 0.f;
    size_t bytes = 0;
    const int bb = coh_begin_bit();
    cub::DeviceRadixSort::SortPairs(nullptr, bytes, keys, keys2, vals, order, (int)n, bb, 30, st);
    void* tmp;
    if ((rc = ws->get_raw("coh_tmp", bytes, &tmp))) return rc;
    {
      ProfScope ps(P_GROUP, st);
      k_coh_key<<<grid_for(n, 256, num_sms() * 16), 256, 0, st>>>(O, D, ray_idx, count_dev, n, lo,
                                                                  inv, keys, vals);
      HRPP_LAUNCHED();
      HRPP_CK(cub::DeviceRadixSort::SortPairs(tmp, bytes, keys, keys2, vals, order, (int)n, bb, 30,
                                              st));
    }
    ray_idx = order;
  }
  TraceArgs a{b.nodes, b.tris, O, D, tmin, tmax, start, n, ray_idx, count_dev, err, out};
  ProfScope ps(ray_idx ? P_TRACE_QUEUE : P_TRACE, st);
  if (g_trace_persistent) {
    static int* counters[64] = {nullptr};
    int dev = 0;
    cudaGetDevice(&dev);
    int*& counter = counters[dev & 63];
    if (!counter) HRPP_CK(cudaMalloc(&counter, sizeof(int)));
    HRPP_CK(cudaMemsetAsync(counter, 0, sizeof(int), st));
    if (closest) dispatch_persist<true>(b.stack, st, a, counter);
    else dispatch_persist<false>(b.stack, st, a, counter);
  } else {
    int grid = (int)((n + 127) / 128);
    if (closest) dispatch_trace<true>(b.stack, grid, st, a);
    else dispatch_trace<false>(b.stack, grid, st, a);
  }
  HRPP_LAUNCHED();
  return 0;
}

}  // namespace hrpp
