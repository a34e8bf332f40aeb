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

// lane_hash / ray_key / nonfinite: hrpp_device.cuh

// The word stored for ray i: its 48-bit key (ib = 0), or, for the wave's
// grouping sort, the three (1+2p)-bit lanes packed contiguously above the
// ray index, (packed << ib) | i (k_pack_keys_idx's word, written here so
// the sort needs no packing pass).
__device__ __forceinline__ uint64_t key_word(uint64_t k, int64_t i, int p, int ib) {
  if (ib == 0) return k;
  const int b = 1 + 2 * p;
  const uint64_t m = (1ull << b) - 1ull;
  const uint64_t pk = (k & m) | (((k >> 16) & m) << b) | (((k >> 32) & m) << (2 * b));
  return (pk << ib) | (uint64_t)i;
}

__global__ void __launch_bounds__(256) k_hash(const float* __restrict__ O,
                                              const float* __restrict__ D, int64_t n, int p,
                                              uint64_t* __restrict__ keys, int* err, int ib) {
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
      k01.x = key_word(ray_key(o[0], o[1], o[2], d[0], d[1], d[2], p), i0, p, ib);
      k01.y = key_word(ray_key(o[3], o[4], o[5], d[3], d[4], d[5], p), i0 + 1, p, ib);
      k23.x = key_word(ray_key(o[6], o[7], o[8], d[6], d[7], d[8], p), i0 + 2, p, ib);
      k23.y = key_word(ray_key(o[9], o[10], o[11], d[9], d[10], d[11], p), i0 + 3, p, ib);
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
        keys[i] = key_word(ray_key(o0, o1, o2, d0, d1, d2, p), i, p, ib);
      }
    }
  }
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(err, 1);
}

// Bulk-copy (TMA) variant for large aligned batches: a persistent grid, each
// block streaming 1024-ray tiles of O and D (2 x 12 KB) through a 4-stage
// shared-memory ring filled by cp.async.bulk and signalled by mbarriers (one
// elected thread issues; every thread hashes 4 rays of a landed tile), so
// ~96 KB per block stay in flight while the previous tiles are hashed.
constexpr int kHashTile = 1024;      // rays per tile (256 threads x 4)
constexpr int kHashStages = 4;
constexpr int kHashTileBytes = kHashTile * 12;  // one of O or D

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}

// Arm the stage's barrier with the tile's byte count and start both copies
// (bytes: a multiple of 48, i.e. whole groups of 4 rays; 0 for a tile of < 4).
__device__ __forceinline__ void bulk_tile(uint32_t bar, uint32_t dst_o, uint32_t dst_d,
                                          const float* src_o, const float* src_d,
                                          uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar),
               "r"(2 * bytes)
               : "memory");
  if (bytes == 0) return;
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(dst_o),
      "l"(src_o), "r"(bytes), "r"(bar)
      : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(dst_d),
      "l"(src_d), "r"(bytes), "r"(bar)
      : "memory");
}

__device__ __forceinline__ uint32_t tile_bytes(int64_t t, int64_t n) {
  const int64_t rays = n - t * kHashTile < kHashTile ? n - t * kHashTile : kHashTile;
  return (uint32_t)((rays / 4) * 48);
}

__global__ void __launch_bounds__(256) k_hash_bulk(const float* __restrict__ O,
                                                   const float* __restrict__ D, int64_t n,
                                                   int p, uint64_t* __restrict__ keys, int* err,
                                                   int ib) {
  const int64_t ntiles = (n + kHashTile - 1) / kHashTile;
  extern __shared__ __align__(128) unsigned char hsm[];
  float* so = reinterpret_cast<float*>(hsm);                                  // [stages][3072]
  float* sd = reinterpret_cast<float*>(hsm + kHashStages * kHashTileBytes);  // [stages][3072]
  __shared__ __align__(8) unsigned long long bars[kHashStages];
  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int sI = 0; sI < kHashStages; sI++)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bars[sI])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  // this block's tiles: blockIdx.x, + gridDim.x, ...
  const int64_t first = blockIdx.x, stride = gridDim.x;
  const int64_t mine = first < ntiles ? (ntiles - first + stride - 1) / stride : 0;
  if (tid == 0)
    for (int sI = 0; sI < kHashStages && sI < mine; sI++) {
      const int64_t t = first + sI * stride;
      bulk_tile(smem_u32(&bars[sI]), smem_u32(so + sI * (kHashTile * 3)),
                smem_u32(sd + sI * (kHashTile * 3)), O + t * (kHashTile * 3),
                D + t * (kHashTile * 3), tile_bytes(t, n));
    }
  bool bad = false;
  for (int64_t k = 0; k < mine; k++) {
    const int sI = (int)(k % kHashStages);
    const uint32_t parity = (uint32_t)((k / kHashStages) & 1);
    mbar_wait(smem_u32(&bars[sI]), parity);
    const int64_t t = first + k * stride;
    const int64_t i0 = t * kHashTile + 4 * tid;  // this thread's 4 rays
    if (i0 + 4 > n) {  // the batch's last < 4 rays: straight from global
      for (int64_t i = i0; i < n; i++) {
        const uint32_t o0 = __float_as_uint(O[3 * i]), o1 = __float_as_uint(O[3 * i + 1]),
                       o2 = __float_as_uint(O[3 * i + 2]);
        const uint32_t d0 = __float_as_uint(D[3 * i]), d1 = __float_as_uint(D[3 * i + 1]),
                       d2 = __float_as_uint(D[3 * i + 2]);
        bad |= nonfinite(o0) | nonfinite(o1) | nonfinite(o2) | nonfinite(d0) | nonfinite(d1) |
               nonfinite(d2);
        keys[i] = key_word(ray_key(o0, o1, o2, d0, d1, d2, p), i, p, ib);
      }
    } else {
    const float4* o4 = reinterpret_cast<const float4*>(so + sI * (kHashTile * 3) + 12 * tid);
    const float4* d4 = reinterpret_cast<const float4*>(sd + sI * (kHashTile * 3) + 12 * tid);
    const float4 oa = o4[0], ob = o4[1], oc = o4[2];
    const float4 da = d4[0], db = d4[1], dc = d4[2];
    const uint32_t o[12] = {__float_as_uint(oa.x), __float_as_uint(oa.y), __float_as_uint(oa.z),
                            __float_as_uint(oa.w), __float_as_uint(ob.x), __float_as_uint(ob.y),
                            __float_as_uint(ob.z), __float_as_uint(ob.w), __float_as_uint(oc.x),
                            __float_as_uint(oc.y), __float_as_uint(oc.z), __float_as_uint(oc.w)};
    const uint32_t d[12] = {__float_as_uint(da.x), __float_as_uint(da.y), __float_as_uint(da.z),
                            __float_as_uint(da.w), __float_as_uint(db.x), __float_as_uint(db.y),
                            __float_as_uint(db.z), __float_as_uint(db.w), __float_as_uint(dc.x),
                            __float_as_uint(dc.y), __float_as_uint(dc.z), __float_as_uint(dc.w)};
#pragma unroll
    for (int j = 0; j < 12; j++) bad |= nonfinite(o[j]) | nonfinite(d[j]);
    ulonglong2 k01, k23;
    k01.x = key_word(ray_key(o[0], o[1], o[2], d[0], d[1], d[2], p), i0, p, ib);
    k01.y = key_word(ray_key(o[3], o[4], o[5], d[3], d[4], d[5], p), i0 + 1, p, ib);
    k23.x = key_word(ray_key(o[6], o[7], o[8], d[6], d[7], d[8], p), i0 + 2, p, ib);
    k23.y = key_word(ray_key(o[9], o[10], o[11], d[9], d[10], d[11], p), i0 + 3, p, ib);
    ulonglong2* kp = reinterpret_cast<ulonglong2*>(keys + i0);
    __stcs(kp, k01);
    __stcs(kp + 1, k23);
    }
    __syncthreads();  // stage sI consumed by every thread: refill it
    if (tid == 0 && k + kHashStages < mine) {
      const int64_t tn = first + (k + kHashStages) * stride;
      bulk_tile(smem_u32(&bars[sI]), smem_u32(so + sI * (kHashTile * 3)),
                smem_u32(sd + sI * (kHashTile * 3)), O + tn * (kHashTile * 3),
                D + tn * (kHashTile * 3), tile_bytes(tn, n));
    }
  }
  if (__any_sync(0xffffffffu, bad) && (tid & 31) == 0) atomicOr(err, 1);
}

int launch_hash(const float* O, const float* D, int64_t n, int p, uint64_t* keys, int* err,
                cudaStream_t st, int ib) {
  if (n <= 0) return 0;
  ProfScope ps(P_HASH, st);
  const bool aligned = ((reinterpret_cast<uintptr_t>(O) | reinterpret_cast<uintptr_t>(D) |
                         reinterpret_cast<uintptr_t>(keys)) & 15) == 0;
  const int64_t ntiles = (n + kHashTile - 1) / kHashTile;
  if (aligned && ntiles >= 2 * (int64_t)num_sms()) {
    // the attribute applies to the current device only: set once per device
    static std::atomic<uint64_t> smem_set{0};
    const int smem = 2 * kHashStages * kHashTileBytes;
    int dev = 0;
    HRPP_CK(cudaGetDevice(&dev));
    const uint64_t bit = 1ull << (dev & 63);
    if (!(smem_set.load() & bit)) {
      HRPP_CK(cudaFuncSetAttribute(k_hash_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
      smem_set.fetch_or(bit);
    }
    k_hash_bulk<<<2 * num_sms(), 256, smem, st>>>(O, D, n, p, keys, err, ib);
  } else {  // small or unaligned batches
    k_hash<<<grid_for((n + 3) / 4, 256, num_sms() * 8), 256, 0, st>>>(O, D, n, p, keys, err, ib);
  }
  HRPP_LAUNCHED();
  return 0;
}

// Precision p -> p - 1 of a key (hrpp/rayhash.py:125-147).  A lane is the xor
// of two float hashes; dropping the lowest exponent and mantissa bit commutes
// with the xor, so each 16-bit lane {sign, p exponent bits, p mantissa bits}
// is re-packed as {sign, top p-1 of each}.
__device__ __forceinline__ uint64_t coarsen_lanes(uint64_t k, int p) {
  const uint32_t fm = (1u << p) - 1u;
  uint64_t out = 0;
#pragma unroll
  for (int l = 0; l < 3; l++) {
    const uint32_t v = (uint32_t)(k >> (16 * l)) & 0xFFFFu;
    const uint32_t man = v & fm, ex = (v >> p) & fm, sg = (v >> (2 * p)) & 1u;
    const uint32_t w = (sg << (2 * (p - 1))) | ((ex >> 1) << (p - 1)) | (man >> 1);
    out |= (uint64_t)w << (16 * l);
  }
  return out;
}

__global__ void k_coarsen(const uint64_t* __restrict__ keys, int64_t n, int p,
                          uint64_t* __restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = coarsen_lanes(keys[i], p);
}

int launch_coarsen(const uint64_t* keys, int64_t n, int p, uint64_t* out, cudaStream_t st) {
  if (n <= 0) return 0;
  k_coarsen<<<grid_for(n, 256, num_sms() * 8), 256, 0, st>>>(keys, n, p, out);
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

// Register cap from the resident-block target: 8 x 128 threads -> 64
// registers, no spills with the float32 slab test (measured against 6, 7, 9
// and 10 blocks on c2).  Warp-synchronous variants (leaf batching,
// cooperative leaves) measured 25-90 % slower; see DESIGN.md section 8.
#ifndef HRPP_TRACE_BS
#define HRPP_TRACE_BS 32  // one warp per block: a warp frees its slot as soon as its own rays finish
#endif
#ifndef HRPP_TRACE_MINB
#define HRPP_TRACE_MINB 8
#endif

template <bool CLOSEST, int STACK>
__global__ void __launch_bounds__(HRPP_TRACE_BS, HRPP_TRACE_MINB * 128 / HRPP_TRACE_BS) k_trace(TraceArgs a) {
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
    if (o.t) o.t[i] = (o.zero_miss_t && !h.found) ? 0.0 : h.t;
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
    if (o.box32) o.box32[i] = h.boxes;
    if (o.tri32) o.tri32[i] = h.tris;
    if (o.fa_f1 && h.found) {  // k_first_append's test, fused (k_consult.cu)
      const int32_t s = o.fa_seg_of_ray[i];
      const int32_t node = o.fa_anc[h.leaf];
      const int64_t off = o.fa_exoff[s];
      const int32_t len = o.fa_exlen[s];
      bool dup = false;
      for (int32_t k = 0; k < len && !dup; k++) dup = o.fa_arena[off + k] == node;
      if (!dup) atomicMin(o.fa_f1 + s, (int32_t)i);
    }
    if (o.known) o.known[i] = 1;
    sb = h.boxes;
    stt = h.tris;
  }
  if (a.out.sums) {  // one atomic pair per block (a.out.sums is uniform)
    __shared__ unsigned long long part[2][HRPP_TRACE_BS / 32];
    sb = warp_sum(sb);
    stt = warp_sum(stt);
    if ((threadIdx.x & 31) == 0) {
      part[0][threadIdx.x >> 5] = sb;
      part[1][threadIdx.x >> 5] = stt;
    }
    __syncthreads();
    if (threadIdx.x < 2) {
      unsigned long long v = 0;
#pragma unroll
      for (int w = 0; w < HRPP_TRACE_BS / 32; w++) v += part[threadIdx.x][w];
      if (v) atomicAdd(a.out.sums + threadIdx.x, v);
    }
  }
}

template <bool CLOSEST>
static void dispatch_trace(int stack, int grid, cudaStream_t st, const TraceArgs& a) {
  switch (stack) {
    case 32: k_trace<CLOSEST, 32><<<grid, HRPP_TRACE_BS, 0, st>>>(a); break;
    case 64: k_trace<CLOSEST, 64><<<grid, HRPP_TRACE_BS, 0, st>>>(a); break;
    case 128: k_trace<CLOSEST, 128><<<grid, HRPP_TRACE_BS, 0, st>>>(a); break;
    case 256: k_trace<CLOSEST, 256><<<grid, HRPP_TRACE_BS, 0, st>>>(a); break;
    default: k_trace<CLOSEST, 512><<<grid, HRPP_TRACE_BS, 0, st>>>(a); break;
  }
}

int launch_trace(const BvhDev& b, bool closest, const float* O, const float* D,
                 const double* tmin, const double* tmax, int32_t start, int64_t n,
                 const int32_t* ray_idx, const int* count_dev, const TraceOut& out,
                 const int* err, cudaStream_t st, Workspace* ws, bool fallback) {
  (void)ws;
  if (n <= 0) return 0;
  TraceArgs a{b.nodes, b.tris, O, D, tmin, tmax, start, n, ray_idx, count_dev, err, out};
  ProfScope ps(ray_idx || fallback ? P_TRACE_QUEUE : P_TRACE, st);
  const int grid = (int)((n + HRPP_TRACE_BS - 1) / HRPP_TRACE_BS);
  if (closest) dispatch_trace<true>(b.stack, grid, st, a);
  else dispatch_trace<false>(b.stack, grid, st, a);
  HRPP_LAUNCHED();
  return 0;
}

}  // namespace hrpp
