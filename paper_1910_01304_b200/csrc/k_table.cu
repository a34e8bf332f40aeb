// k_table.cu -- predictor table in HBM (hrpp/predictor.py:117-211).
//
// Index: open-addressed (linear probing) buckets {u64 key, i32 entry id},
// load factor <= 0.5, inserted with atomicCAS.  Entries: SoA {key, arena
// offset, length} in creation order.  Node lists live contiguously in an
// int32 arena; an entry that grows during a wave is relocated to the arena
// tail (old list + appended nodes), so every list stays contiguous for the
// consult kernel's broadcast reads.  The arena is compacted when garbage
// would overflow it.
#include <cub/cub.cuh>

#include "hrpp_internal.h"

namespace hrpp {

// ---------------------------------------------------------------------------
// grouping: stable (key, ray) sort + key segments
// ---------------------------------------------------------------------------

__global__ void k_iota(int32_t* v, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    v[i] = (int32_t)i;
}

// Hash keys use b = 1 + 2p bits of each 16-bit lane; packing the three lanes
// contiguously (3b bits, 39 at p = 6) lets the radix sort skip the empty bits.
__global__ void k_pack_keys(const unsigned long long* __restrict__ keys, int64_t n, int b,
                            unsigned long long* __restrict__ packed, int32_t* __restrict__ iota) {
  const unsigned long long m = (1ull << b) - 1ull;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const unsigned long long k = keys[i];
    packed[i] = (k & m) | (((k >> 16) & m) << b) | (((k >> 32) & m) << (2 * b));
    iota[i] = (int32_t)i;
  }
}

// Packed key and ray index in one word, (key << ib) | i: a keys-only sort of
// bits [ib, ib + 3b) then moves 8 instead of 12 bytes per ray and pass (the
// LSD radix sort is stable, so rays of one key stay in ray order).
__global__ void k_pack_keys_idx(const unsigned long long* __restrict__ keys, int64_t n, int b,
                                int ib, unsigned long long* __restrict__ packed) {
  const unsigned long long m = (1ull << b) - 1ull;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const unsigned long long k = keys[i];
    const unsigned long long pk = (k & m) | (((k >> 16) & m) << b) | (((k >> 32) & m) << (2 * b));
    packed[i] = (pk << ib) | (unsigned long long)i;
  }
}

__global__ void k_head_flags_idx(const unsigned long long* __restrict__ src, int64_t n, int b,
                                 int ib, int32_t* __restrict__ flags,
                                 unsigned long long* __restrict__ out, int32_t* __restrict__ sidx) {
  const unsigned long long m = (1ull << b) - 1ull;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const unsigned long long w = src[i];
    const unsigned long long k = w >> ib;
    flags[i] = (i == 0) || (k != (src[i - 1] >> ib));
    out[i] = (k & m) | (((k >> b) & m) << 16) | (((k >> (2 * b)) & m) << 32);
    sidx[i] = (int32_t)(w & ((1ull << ib) - 1ull));
  }
}

// Segment heads of the sorted keys `src`; with b > 0 they are packed and are
// written unpacked (48-bit hash keys) to `out`.
__global__ void k_head_flags(const unsigned long long* __restrict__ src, int64_t n, int b,
                             int32_t* __restrict__ flags, unsigned long long* __restrict__ out) {
  const unsigned long long m = b ? (1ull << b) - 1ull : 0ull;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const unsigned long long k = src[i];
    flags[i] = (i == 0) || (k != src[i - 1]);
    if (b) out[i] = (k & m) | (((k >> b) & m) << 16) | (((k >> (2 * b)) & m) << 32);
  }
}

// Segment construction fused into one scan over the sorted words: the scan
// input is the head flag of each sorted position (its key differs from the
// previous one), the inclusive sum is the segment id (+1), and the output
// iterator writes seg_id[p], sidx[p] and, at segment heads, seg_start and the
// unpacked 48-bit key skeys[p] (read only at heads).  Replaces a head-flag
// pass, a flagged select and a separate scan.
struct HeadFlag {
  const unsigned long long* w;
  int ib;
  __host__ __device__ __forceinline__ int operator()(int64_t p) const {
    return p == 0 || (w[p] >> ib) != (w[p - 1] >> ib);
  }
};

struct SegWriter {
  using value_type = int;
  using difference_type = std::ptrdiff_t;
  using pointer = void;
  using iterator_category = std::random_access_iterator_tag;
  const unsigned long long* w;
  int ib, b;
  int64_t base;
  int32_t* seg_id;
  int32_t* seg_start;
  unsigned long long* skeys;
  int32_t* sidx;
  struct Ref {
    const unsigned long long* w;
    int ib, b;
    int64_t p;
    int32_t* seg_id;
    int32_t* seg_start;
    unsigned long long* skeys;
    int32_t* sidx;
    __device__ __forceinline__ void operator=(int incl) const {
      const unsigned long long x = w[p];
      const unsigned long long k = x >> ib;
      seg_id[p] = incl;
      sidx[p] = (int32_t)(x & ((1ull << ib) - 1ull));
      if (p == 0 || k != (w[p - 1] >> ib)) {
        const unsigned long long m = (1ull << b) - 1ull;
        seg_start[incl - 1] = (int32_t)p;
        skeys[p] = (k & m) | (((k >> b) & m) << 16) | (((k >> (2 * b)) & m) << 32);
      }
    }
  };
  using reference = Ref;
  __host__ __device__ __forceinline__ Ref operator[](int64_t i) const {
    return Ref{w, ib, b, base + i, seg_id, seg_start, skeys, sidx};
  }
  __host__ __device__ __forceinline__ Ref operator*() const { return (*this)[0]; }
  __host__ __device__ __forceinline__ SegWriter operator+(int64_t k) const {
    SegWriter r = *this;
    r.base += k;
    return r;
  }
};

__global__ void k_seg_finish(const int32_t* __restrict__ seg_id, int64_t n, int* nsegs,
                             int32_t* seg_start, int* nsegs_mapped) {
  const int ns = seg_id[n - 1];
  *nsegs = ns;
  seg_start[ns] = (int32_t)n;
  if (nsegs_mapped) *nsegs_mapped = ns;  // host-visible (mapped pinned memory)
}

__global__ void k_seg_sentinel(int32_t* seg_start, const int* nsegs, int64_t n,
                               int* nsegs_mapped) {
  seg_start[*nsegs] = (int32_t)n;
  if (nsegs_mapped) *nsegs_mapped = *nsegs;  // host-visible (mapped pinned memory)
}

int group_by_key(Workspace& ws, const uint64_t* keys, int64_t n, int lane_bits, Segments* seg,
                 cudaStream_t st, int* nsegs_mapped, bool prepacked) {
  int32_t* iota;
  int32_t* flags;
  unsigned long long* packed = nullptr;
  unsigned long long* sorted_out;
  int rc;
  if ((rc = ws.get("g_skeys", n, &seg->skeys))) return rc;
  if ((rc = ws.get("g_iota", n, &iota))) return rc;
  if ((rc = ws.get("g_sidx", n, &seg->sidx))) return rc;
  if ((rc = ws.get("g_flags", n, &flags))) return rc;
  if ((rc = ws.get("g_segstart", n + 1, &seg->seg_start))) return rc;
  if ((rc = ws.get("g_nsegs", 1, &seg->nsegs))) return rc;
  if ((rc = ws.get("g_segid", n, &seg->seg_id))) return rc;
  int grid = grid_for(n, 256, num_sms() * 8);
  ProfScope ps(P_GROUP, st);
  const unsigned long long* kin = reinterpret_cast<const unsigned long long*>(keys);
  int ib = 1;  // ray index bits
  while (ib < 31 && (1ll << ib) < n) ib++;
  if (lane_bits > 0 && 3 * lane_bits + ib <= 64) {
    unsigned long long *packed2, *sorted2;
    if ((rc = ws.get("g_packed", n, &packed2)) || (rc = ws.get("g_psorted", n, &sorted2)))
      return rc;
    if (prepacked) {  // the hash kernel already wrote (packed << ib) | i
      packed2 = const_cast<unsigned long long*>(kin);
    } else {
      k_pack_keys_idx<<<grid, 256, 0, st>>>(kin, n, lane_bits, ib, packed2);
      HRPP_LAUNCHED();
    }
    size_t b_sort = 0, b_scan = 0;
    cub::DeviceRadixSort::SortKeys(nullptr, b_sort, packed2, sorted2, (int)n, ib,
                                   ib + 3 * lane_bits, st);
    cub::TransformInputIterator<int, HeadFlag, cub::CountingInputIterator<int64_t>> heads(
        cub::CountingInputIterator<int64_t>(0), HeadFlag{sorted2, ib});
    SegWriter out{sorted2, ib, lane_bits, 0, seg->seg_id, seg->seg_start, seg->skeys,
                  seg->sidx};
    cub::DeviceScan::InclusiveSum(nullptr, b_scan, heads, out, (int)n, st);
    size_t b = b_sort > b_scan ? b_sort : b_scan;
    void* tmp;
    if ((rc = ws.get_raw("g_cubtmp", b, &tmp))) return rc;
    HRPP_CK(cub::DeviceRadixSort::SortKeys(tmp, b_sort, packed2, sorted2, (int)n, ib,
                                           ib + 3 * lane_bits, st));
    HRPP_CK(cub::DeviceScan::InclusiveSum(tmp, b_scan, heads, out, (int)n, st));
    k_seg_finish<<<1, 1, 0, st>>>(seg->seg_id, n, seg->nsegs, seg->seg_start, nsegs_mapped);
    HRPP_LAUNCHED();
    return 0;
  }
  int end_bit = 64;  // generic keys (record API)
  sorted_out = seg->skeys;
  if (lane_bits > 0) {
    if ((rc = ws.get("g_packed", n, &packed)) || (rc = ws.get("g_psorted", n, &sorted_out)))
      return rc;
    k_pack_keys<<<grid, 256, 0, st>>>(kin, n, lane_bits, packed, iota);
    kin = packed;
    end_bit = 3 * lane_bits;
  } else {
    k_iota<<<grid, 256, 0, st>>>(iota, n);
  }
  HRPP_LAUNCHED();
  size_t b_sort = 0, b_sel = 0, b_scan = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, b_sort, kin, sorted_out, iota, seg->sidx, (int)n,
                                  0, end_bit, st);
  cub::CountingInputIterator<int32_t> cnt(0);
  cub::DeviceSelect::Flagged(nullptr, b_sel, cnt, flags, seg->seg_start, seg->nsegs, (int)n,
                             st);
  cub::DeviceScan::InclusiveSum(nullptr, b_scan, flags, seg->seg_id, (int)n, st);
  size_t b = b_sort > b_sel ? b_sort : b_sel;
  b = b > b_scan ? b : b_scan;
  void* tmp;
  if ((rc = ws.get_raw("g_cubtmp", b, &tmp))) return rc;
  HRPP_CK(cub::DeviceRadixSort::SortPairs(tmp, b_sort, kin, sorted_out, iota, seg->sidx, (int)n,
                                          0, end_bit, st));
  k_head_flags<<<grid, 256, 0, st>>>(sorted_out, n, lane_bits, flags, seg->skeys);
  HRPP_LAUNCHED();
  HRPP_CK(cub::DeviceSelect::Flagged(tmp, b_sel, cnt, flags, seg->seg_start, seg->nsegs, (int)n,
                                     st));
  // seg_id[p] = 1 + index of the key segment holding sorted position p
  HRPP_CK(cub::DeviceScan::InclusiveSum(tmp, b_scan, flags, seg->seg_id, (int)n, st));
  k_seg_sentinel<<<1, 1, 0, st>>>(seg->seg_start, seg->nsegs, n, nsegs_mapped);
  HRPP_LAUNCHED();
  return 0;
}

int compact_flags(Workspace& ws, const uint8_t* flags, int64_t n, int32_t* out, int* count_dev,
                  cudaStream_t st) {
  cub::CountingInputIterator<int32_t> cnt(0);
  size_t b = 0;
  cub::DeviceSelect::Flagged(nullptr, b, cnt, flags, out, count_dev, (int)n, st);
  void* tmp;
  int rc;
  if ((rc = ws.get_raw("cf_tmp", b, &tmp))) return rc;
  ProfScope ps(P_GROUP, st);
  HRPP_CK(cub::DeviceSelect::Flagged(tmp, b, cnt, flags, out, count_dev, (int)n, st));
  return 0;
}

int compact_by_flags(Workspace& ws, const int32_t* values, const uint8_t* flags, int64_t n,
                     int32_t* out, int* count_dev, cudaStream_t st) {
  size_t b = 0;
  cub::DeviceSelect::Flagged(nullptr, b, values, flags, out, count_dev, (int)n, st);
  void* tmp;
  int rc;
  if ((rc = ws.get_raw("cbf_tmp", b, &tmp))) return rc;
  ProfScope ps(P_GROUP, st);
  HRPP_CK(cub::DeviceSelect::Flagged(tmp, b, values, flags, out, count_dev, (int)n, st));
  return 0;
}

// ---------------------------------------------------------------------------
// index maintenance
// ---------------------------------------------------------------------------

__device__ __forceinline__ void index_insert(Bucket* idx, uint64_t mask, unsigned long long key,
                                             int32_t id) {
  uint64_t h = mix64(key) & mask;
  for (;;) {
    unsigned long long prev = atomicCAS(&idx[h].key, kEmptyKey, key);
    if (prev == kEmptyKey || prev == key) {
      idx[h].val = id;
      return;
    }
    h = (h + 1) & mask;
  }
}

__global__ void k_rehash(const unsigned long long* __restrict__ e_key, int64_t n_entries,
                         Bucket* idx, uint64_t mask) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n_entries;
       e += (int64_t)gridDim.x * blockDim.x)
    index_insert(idx, mask, e_key[e], (int32_t)e);
}

__global__ void k_len_to_i64(const int32_t* __restrict__ len, int64_t n, long long* out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = len[i];
}

__global__ void k_compact(const int32_t* __restrict__ src, int32_t* __restrict__ dst,
                          int64_t* e_off, const int32_t* __restrict__ e_len,
                          const long long* __restrict__ new_off, int64_t n_entries) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n_entries;
       e += (int64_t)gridDim.x * blockDim.x) {
    int64_t o = e_off[e], no = new_off[e];
    for (int32_t j = 0; j < e_len[e]; j++) dst[no + j] = src[o + j];
    e_off[e] = no;
  }
}

static int64_t next_pow2(int64_t x) {
  int64_t p = 1024;
  while (p < x) p <<= 1;
  return p;
}

template <typename T>
static int grow(T** p, int64_t old_count, int64_t new_count, cudaStream_t st) {
  T* np = nullptr;
  HRPP_CK(cudaMalloc(&np, sizeof(T) * new_count));
  if (*p && old_count) HRPP_CK(cudaMemcpyAsync(np, *p, sizeof(T) * old_count,
                                               cudaMemcpyDeviceToDevice, st));
  if (*p) {
    HRPP_CK(cudaStreamSynchronize(st));
    HRPP_CK(cudaFree(*p));
  }
  *p = np;
  return 0;
}

int TableDev::reserve(int64_t extra_e, int64_t extra, cudaStream_t st) {
  int rc;
  if (!meta) {
    HRPP_CK(cudaMalloc(&meta, sizeof(long long) * 4));
    HRPP_CK(cudaMemsetAsync(meta, 0, sizeof(long long) * 4, st));
  }
  int64_t need_e = n_entries + extra_e + 16;
  if (e_cap < need_e) {
    int64_t nc = need_e > 2 * e_cap ? need_e : 2 * e_cap;
    if ((rc = grow(&e_key, n_entries, nc, st))) return rc;
    if ((rc = grow(&e_off, n_entries, nc, st))) return rc;
    if ((rc = grow(&e_len, n_entries, nc, st))) return rc;
    e_cap = nc;
  }
  int64_t need_idx = next_pow2(2 * need_e);
  if (idx_cap < need_idx) {
    if (idx) {
      HRPP_CK(cudaStreamSynchronize(st));
      HRPP_CK(cudaFree(idx));
    }
    HRPP_CK(cudaMalloc(&idx, sizeof(Bucket) * need_idx));
    HRPP_CK(cudaMemsetAsync(idx, 0xFF, sizeof(Bucket) * need_idx, st));
    idx_cap = need_idx;
    if (n_entries) {
      k_rehash<<<grid_for(n_entries, 256, num_sms() * 8), 256, 0, st>>>(
          e_key, n_entries, idx, (uint64_t)idx_cap - 1);
      HRPP_LAUNCHED();
    }
  }
  int64_t need_arena = arena_used + stored + extra + 16;
  if (arena_cap < need_arena) {
    // compact live lists into a fresh arena sized with headroom
    int64_t nc = 2 * (stored + extra) + 1024;
    if (nc < 2 * arena_cap && arena_used <= 2 * stored) nc = 2 * arena_cap;
    int32_t* na = nullptr;
    HRPP_CK(cudaMalloc(&na, sizeof(int32_t) * nc));
    if (n_entries) {
      long long *len64, *off64;
      if ((rc = ws.get("c_len64", n_entries, &len64))) return rc;
      if ((rc = ws.get("c_off64", n_entries, &off64))) return rc;
      int grid = grid_for(n_entries, 256, num_sms() * 8);
      k_len_to_i64<<<grid, 256, 0, st>>>(e_len, n_entries, len64);
      HRPP_LAUNCHED();
      size_t b = 0;
      cub::DeviceScan::ExclusiveSum(nullptr, b, len64, off64, (int)n_entries, st);
      void* tmp;
      if ((rc = ws.get_raw("c_tmp", b, &tmp))) return rc;
      HRPP_CK(cub::DeviceScan::ExclusiveSum(tmp, b, len64, off64, (int)n_entries, st));
      k_compact<<<grid, 256, 0, st>>>(arena, na, e_off, e_len, off64, n_entries);
      HRPP_LAUNCHED();
    }
    if (arena) {
      HRPP_CK(cudaStreamSynchronize(st));
      HRPP_CK(cudaFree(arena));
    }
    arena = na;
    arena_cap = nc;
    arena_used = stored;
    if ((rc = set_i64(meta + 2, stored, st))) return rc;
  }
  return 0;
}

TableDev::~TableDev() {
  if (clear_ev) cudaEventDestroy(clear_ev);
  cudaFree(idx);
  cudaFree(e_key);
  cudaFree(e_off);
  cudaFree(e_len);
  cudaFree(arena);
  cudaFree(meta);
}

// ---------------------------------------------------------------------------
// commit the per-segment appends of one wave (or one record batch)
// ---------------------------------------------------------------------------

// Block-wide exclusive scan of two counters (128 threads = 4 warps).
__device__ __forceinline__ void block_scan2(long long a, long long b, long long& ea, long long& eb,
                                            long long& ta, long long& tb) {
  __shared__ long long wa[4], wb[4];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  long long ia = a, ib = b;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    long long xa = __shfl_up_sync(0xffffffffu, ia, o);
    long long xb = __shfl_up_sync(0xffffffffu, ib, o);
    if (lane >= o) {
      ia += xa;
      ib += xb;
    }
  }
  if (lane == 31) {
    wa[w] = ia;
    wb[w] = ib;
  }
  __syncthreads();
  long long pa = 0, pb = 0;
  ta = 0;
  tb = 0;
  for (int k = 0; k < 4; k++) {
    if (k < w) {
      pa += wa[k];
      pb += wb[k];
    }
    ta += wa[k];
    tb += wb[k];
  }
  ea = pa + ia - a;
  eb = pb + ib - b;
}

// Commit of the touched segments: per block (128 segments) the counts of new
// entries, relocated list nodes and appended nodes; an exclusive scan over
// the block totals; then every block places its entries and lists.  No
// contended atomics; entry ids and arena layout are deterministic.
struct Tot3 {
  long long n_new, reloc, app;
};
struct Tot3Sum {
  __host__ __device__ Tot3 operator()(const Tot3& a, const Tot3& b) const {
    return Tot3{a.n_new + b.n_new, a.reloc + b.reloc, a.app + b.app};
  }
};

__device__ __forceinline__ void seg_commit_counts(const int ns, int64_t s,
                                                  const int32_t* __restrict__ seg_eid,
                                                  const int32_t* __restrict__ seg_napp,
                                                  const int32_t* __restrict__ e_len,
                                                  int32_t& napp, int32_t& eid,
                                                  int32_t& old_len) {
  napp = 0;
  eid = -1;
  old_len = 0;
  if (s < ns) {
    napp = seg_napp[s];
    if (napp > 0) {
      eid = seg_eid[s];
      old_len = eid >= 0 ? e_len[eid] : 0;
    }
  }
}

__global__ void __launch_bounds__(128) k_commit_count(const int* nsegs,
                                                      const int32_t* __restrict__ seg_eid,
                                                      const int32_t* __restrict__ seg_napp,
                                                      const int32_t* __restrict__ e_len,
                                                      Tot3* block_tot, int* err,
                                                      const int32_t* __restrict__ seg_start,
                                                      const int32_t* __restrict__ seg_cursor) {
  if (*err) return;
  const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  // (consult) every segment replayed to its end, else an internal error
  if (seg_cursor && s < *nsegs && seg_cursor[s] < seg_start[s + 1]) atomicCAS(err, 0, 4);
  int32_t napp, eid, old_len;
  seg_commit_counts(*nsegs, s, seg_eid, seg_napp, e_len, napp, eid, old_len);
  long long ex_new, ex_reloc, t_new, t_reloc;
  block_scan2(napp > 0 && eid < 0, napp > 0 ? old_len + napp : 0, ex_new, ex_reloc, t_new,
              t_reloc);
  __shared__ long long wapp[4];
  long long a = warp_sum((long long)napp);
  if ((threadIdx.x & 31) == 0) wapp[threadIdx.x >> 5] = a;
  __syncthreads();
  if (threadIdx.x == 0)
    block_tot[blockIdx.x] = Tot3{t_new, t_reloc, wapp[0] + wapp[1] + wapp[2] + wapp[3]};
}

__global__ void k_commit_check(const Tot3* block_tot, const Tot3* block_off, int nblocks,
                               const long long* meta, long long max_entries, int* err,
                               Tot3* total) {
  const Tot3 t = Tot3Sum()(block_off[nblocks - 1], block_tot[nblocks - 1]);
  *total = t;
  if (*err == 0 && meta[0] + t.n_new > max_entries) *err = 2;  // CapacityExceeded
}

__global__ void __launch_bounds__(128) k_commit_apply(
    const int* nsegs, const int32_t* __restrict__ seg_start,
    const unsigned long long* __restrict__ skeys, const int32_t* __restrict__ seg_eid,
    const int32_t* __restrict__ seg_napp, const int32_t* __restrict__ app, const long long* meta,
    unsigned long long* e_key, int64_t* e_off, int32_t* e_len, int32_t* arena, Bucket* idx,
    uint64_t mask, const Tot3* __restrict__ block_off, const int* err) {
  if (*err) return;
  const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int32_t napp, eid, old_len;
  seg_commit_counts(*nsegs, s, seg_eid, seg_napp, e_len, napp, eid, old_len);
  long long ex_new, ex_reloc, t_new, t_reloc;
  block_scan2(napp > 0 && eid < 0, napp > 0 ? old_len + napp : 0, ex_new, ex_reloc, t_new,
              t_reloc);
  if (napp <= 0) return;
  const Tot3 base = block_off[blockIdx.x];
  const int64_t old_off = eid >= 0 ? e_off[eid] : 0;
  if (eid < 0) {
    eid = (int32_t)(meta[0] + base.n_new + ex_new);
    const unsigned long long key = skeys[seg_start[s]];
    e_key[eid] = key;
    index_insert(idx, mask, key, eid);
  }
  const int64_t no = meta[2] + base.reloc + ex_reloc;
  for (int32_t j = 0; j < old_len; j++) arena[no + j] = arena[old_off + j];
  const int32_t* a = app + seg_start[s];
  for (int32_t j = 0; j < napp; j++) arena[no + old_len + j] = a[j];
  e_off[eid] = no;
  e_len[eid] = old_len + napp;
}

__global__ void k_commit_finish(long long* meta, const Tot3* total, const int* err) {
  if (*err) return;
  meta[0] += total->n_new;
  meta[1] += total->app;
  meta[2] += total->reloc;
}

int table_commit(TableDev& t, const Segments& seg, int64_t n, int32_t* seg_eid,
                 int32_t* seg_napp, const int32_t* app, int* err, cudaStream_t st,
                 const int32_t* seg_cursor) {
  const int nblocks = (int)((n + 127) / 128);
  Tot3 *btot, *boff, *total;
  int rc;
  if ((rc = t.ws.get("m_btot", nblocks, &btot)) || (rc = t.ws.get("m_boff", nblocks, &boff)) ||
      (rc = t.ws.get("m_total", 1, &total)))
    return rc;
  size_t b = 0;
  cub::DeviceScan::ExclusiveScan(nullptr, b, btot, boff, Tot3Sum(), Tot3{0, 0, 0}, nblocks, st);
  void* tmp;
  if ((rc = t.ws.get_raw("m_tmp", b, &tmp))) return rc;
  ProfScope ps(P_COMMIT, st);
  k_commit_count<<<nblocks, 128, 0, st>>>(seg.nsegs, seg_eid, seg_napp, t.e_len, btot, err,
                                          seg.seg_start, seg_cursor);
  HRPP_LAUNCHED();
  HRPP_CK(cub::DeviceScan::ExclusiveScan(tmp, b, btot, boff, Tot3Sum(), Tot3{0, 0, 0}, nblocks,
                                         st));
  k_commit_check<<<1, 1, 0, st>>>(btot, boff, nblocks, t.meta, (long long)t.max_entries, err,
                                  total);
  HRPP_LAUNCHED();
  k_commit_apply<<<nblocks, 128, 0, st>>>(seg.nsegs, seg.seg_start, seg.skeys, seg_eid, seg_napp,
                                          app, t.meta, t.e_key, t.e_off, t.e_len, t.arena, t.idx,
                                          (uint64_t)t.idx_cap - 1, boff, err);
  HRPP_LAUNCHED();
  k_commit_finish<<<1, 1, 0, st>>>(t.meta, total, err);
  HRPP_LAUNCHED();
  return 0;
}

// ---------------------------------------------------------------------------
// deferred mode: gather the wave's append records, sorted by ray index
// ---------------------------------------------------------------------------

__global__ void k_pend_count(const int* nsegs, int64_t n, const int32_t* __restrict__ seg_napp,
                             long long* cnt, const int* err) {
  const int ns = *nsegs;
  const bool dead = *err != 0;
  for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < n;
       s += (int64_t)gridDim.x * blockDim.x)
    cnt[s] = (s < ns && !dead) ? seg_napp[s] : 0;
}

__global__ void k_pend_scatter(const int* nsegs, const int32_t* __restrict__ seg_start,
                               const unsigned long long* __restrict__ skeys,
                               const int32_t* __restrict__ seg_napp,
                               const int32_t* __restrict__ app,
                               const int32_t* __restrict__ app_ray,
                               const long long* __restrict__ off, unsigned long long* pk,
                               int32_t* pn, int32_t* pr, int32_t* iota, const int* err) {
  if (*err) return;
  const int ns = *nsegs;
  for (int s = blockIdx.x * blockDim.x + threadIdx.x; s < ns; s += gridDim.x * blockDim.x) {
    const int32_t napp = seg_napp[s], b = seg_start[s];
    const long long o = off[s];
    for (int32_t j = 0; j < napp; j++) {
      pk[o + j] = skeys[b];
      pn[o + j] = app[b + j];
      pr[o + j] = app_ray[b + j];
      iota[o + j] = (int32_t)(o + j);
    }
  }
}

__global__ void k_pend_total(const long long* cnt, const long long* off, int64_t n,
                             long long* meta) {
  meta[3] = off[n - 1] + cnt[n - 1];
}

__global__ void k_pend_gather(const int32_t* __restrict__ perm, const long long* meta,
                              const unsigned long long* __restrict__ pk,
                              const int32_t* __restrict__ pn, unsigned long long* ok,
                              int32_t* on) {
  const long long m = meta[3];
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < m;
       i += (long long)gridDim.x * blockDim.x) {
    ok[i] = pk[perm[i]];
    on[i] = pn[perm[i]];
  }
}

int table_collect_pending(TableDev& t, const Segments& seg, int64_t n, const int32_t* seg_napp,
                          const int32_t* app, const int32_t* app_ray, int* err,
                          cudaStream_t st) {
  long long *cnt, *off;
  unsigned long long *pk, *okeys;
  int32_t *pn, *pr, *iota, *rays_sorted, *perm, *onodes;
  int rc;
  if ((rc = t.ws.get("q_cnt", n, &cnt)) || (rc = t.ws.get("q_off", n, &off)) ||
      (rc = t.ws.get("q_pk", n, &pk)) || (rc = t.ws.get("q_pn", n, &pn)) ||
      (rc = t.ws.get("q_pr", n, &pr)) || (rc = t.ws.get("q_iota", n, &iota)) ||
      (rc = t.ws.get("p_rays", n, &rays_sorted)) || (rc = t.ws.get("q_perm", n, &perm)) ||
      (rc = t.ws.get("p_keys", n, &okeys)) || (rc = t.ws.get("p_nodes", n, &onodes)))
    return rc;
  int grid = grid_for(n, 256, num_sms() * 8);
  ProfScope ps(P_COMMIT, st);
  HRPP_CK(cudaMemsetAsync(pr, 0x7F, sizeof(int32_t) * n, st));  // pad rays sort last
  k_pend_count<<<grid, 256, 0, st>>>(seg.nsegs, n, seg_napp, cnt, err);
  HRPP_LAUNCHED();
  size_t b1 = 0, b2 = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, b1, cnt, off, (int)n, st);
  cub::DeviceRadixSort::SortPairs(nullptr, b2, pr, rays_sorted, iota, perm, (int)n, 0, 32, st);
  void* tmp;
  if ((rc = t.ws.get_raw("q_tmp", b1 > b2 ? b1 : b2, &tmp))) return rc;
  HRPP_CK(cub::DeviceScan::ExclusiveSum(tmp, b1, cnt, off, (int)n, st));
  k_pend_scatter<<<grid, 256, 0, st>>>(seg.nsegs, seg.seg_start, seg.skeys, seg_napp, app,
                                       app_ray, off, pk, pn, pr, iota, err);
  HRPP_LAUNCHED();
  k_pend_total<<<1, 1, 0, st>>>(cnt, off, n, t.meta);
  HRPP_LAUNCHED();
  // ray indices are < 2^31, padding 0x7F7F7F7F sorts after every real record
  HRPP_CK(cub::DeviceRadixSort::SortPairs(tmp, b2, pr, rays_sorted, iota, perm, (int)n, 0, 32,
                                          st));
  k_pend_gather<<<grid, 256, 0, st>>>(perm, t.meta, pk, pn, okeys, onodes);
  HRPP_LAUNCHED();
  return 0;
}

// ---------------------------------------------------------------------------
// record (predictor.py:147-160), batched with sequential semantics
// ---------------------------------------------------------------------------

__global__ void k_record_seg(const int* nsegs, const int32_t* __restrict__ seg_start,
                             const unsigned long long* __restrict__ skeys,
                             const int32_t* __restrict__ sidx, const int32_t* __restrict__ nodes,
                             const Bucket* __restrict__ idx, uint64_t mask,
                             const int64_t* __restrict__ e_off, const int32_t* __restrict__ e_len,
                             const int32_t* __restrict__ arena, int32_t* app, int32_t* seg_eid,
                             int32_t* seg_napp, uint8_t* inserted) {
  const int ns = *nsegs;
  for (int s = blockIdx.x * blockDim.x + threadIdx.x; s < ns; s += gridDim.x * blockDim.x) {
    int32_t beg = seg_start[s], end = seg_start[s + 1];
    int32_t eid = index_lookup(idx, mask, skeys[beg]);
    int64_t off = eid >= 0 ? e_off[eid] : 0;
    int32_t len = eid >= 0 ? e_len[eid] : 0;
    int32_t* ap = app + beg;
    int32_t napp = 0;
    for (int32_t j = beg; j < end; j++) {
      int32_t idx = sidx[j];
      int32_t node = nodes[idx];
      bool dup = false;
      for (int32_t k = 0; k < len && !dup; k++) dup = arena[off + k] == node;
      for (int32_t k = 0; k < napp && !dup; k++) dup = ap[k] == node;
      if (!dup) ap[napp++] = node;
      if (inserted) inserted[idx] = !dup;
    }
    seg_eid[s] = eid;
    seg_napp[s] = napp;
  }
}

int table_record(TableDev& t, const uint64_t* keys, const int32_t* nodes, int64_t n,
                 uint8_t* inserted, int* err, cudaStream_t st) {
  int rc;
  if ((rc = t.reserve(n, n, st))) return rc;
  Segments seg;
  if ((rc = group_by_key(t.ws, keys, n, 0, &seg, st))) return rc;
  int32_t *app, *seg_eid, *seg_napp;
  if ((rc = t.ws.get("r_app", n, &app))) return rc;
  if ((rc = t.ws.get("r_eid", n, &seg_eid))) return rc;
  if ((rc = t.ws.get("r_napp", n, &seg_napp))) return rc;
  k_record_seg<<<grid_for(n, 128, num_sms() * 16), 128, 0, st>>>(
      seg.nsegs, seg.seg_start, seg.skeys, seg.sidx, nodes, t.idx,
      (uint64_t)t.idx_cap - 1, t.e_off, t.e_len, t.arena, app, seg_eid, seg_napp, inserted);
  HRPP_LAUNCHED();
  return table_commit(t, seg, n, seg_eid, seg_napp, app, err, st);
}

// ---------------------------------------------------------------------------
// export (dump_lines order), lookup, max length
// ---------------------------------------------------------------------------

__global__ void k_export_len(const int32_t* __restrict__ ids, const int32_t* __restrict__ e_len,
                             int64_t n, long long* lens) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    lens[i] = e_len[ids[i]];
}

__global__ void k_export_nodes(const int32_t* __restrict__ ids, const int64_t* __restrict__ e_off,
                               const int32_t* __restrict__ e_len, const int32_t* __restrict__ arena,
                               const long long* __restrict__ offs, int64_t n, int32_t* out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    int32_t e = ids[i];
    int64_t o = e_off[e];
    for (int32_t j = 0; j < e_len[e]; j++) out[offs[i] + j] = arena[o + j];
  }
}

int table_export(TableDev& t, uint64_t* keys_h, int64_t* offs_h, int32_t* nodes_h) {
  const int64_t n = t.n_entries;
  offs_h[0] = 0;
  if (n == 0) return 0;
  cudaStream_t st = 0;
  int rc;
  unsigned long long* sk;
  int32_t *iota, *ids, *nodes;
  long long *lens, *offs;
  if ((rc = t.ws.get("x_sk", n, &sk))) return rc;
  if ((rc = t.ws.get("x_iota", n, &iota))) return rc;
  if ((rc = t.ws.get("x_ids", n, &ids))) return rc;
  if ((rc = t.ws.get("x_len", n + 1, &lens))) return rc;
  if ((rc = t.ws.get("x_off", n + 1, &offs))) return rc;
  if ((rc = t.ws.get("x_nodes", t.stored + 1, &nodes))) return rc;
  int grid = grid_for(n, 256, num_sms() * 8);
  k_iota<<<grid, 256, 0, st>>>(iota, n);
  HRPP_LAUNCHED();
  size_t b1 = 0, b2 = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, b1, t.e_key, sk, iota, ids, (int)n, 0, 48, st);
  cub::DeviceScan::ExclusiveSum(nullptr, b2, lens, offs, (int)n + 1, st);
  void* tmp;
  if ((rc = t.ws.get_raw("x_tmp", b1 > b2 ? b1 : b2, &tmp))) return rc;
  HRPP_CK(cub::DeviceRadixSort::SortPairs(tmp, b1, t.e_key, sk, iota, ids, (int)n, 0, 48, st));
  HRPP_CK(cudaMemsetAsync(lens + n, 0, sizeof(long long), st));
  k_export_len<<<grid, 256, 0, st>>>(ids, t.e_len, n, lens);
  HRPP_LAUNCHED();
  HRPP_CK(cub::DeviceScan::ExclusiveSum(tmp, b2, lens, offs, (int)n + 1, st));
  k_export_nodes<<<grid, 256, 0, st>>>(ids, t.e_off, t.e_len, t.arena, offs, n, nodes);
  HRPP_LAUNCHED();
  HRPP_CK(cudaMemcpyAsync(keys_h, sk, sizeof(uint64_t) * n, cudaMemcpyDeviceToHost, st));
  HRPP_CK(cudaMemcpyAsync(offs_h, offs, sizeof(int64_t) * (n + 1), cudaMemcpyDeviceToHost, st));
  if (t.stored)
    HRPP_CK(cudaMemcpyAsync(nodes_h, nodes, sizeof(int32_t) * t.stored, cudaMemcpyDeviceToHost,
                            st));
  HRPP_CK(cudaStreamSynchronize(st));
  return 0;
}

__global__ void k_lookup1(const Bucket* __restrict__ idx, uint64_t mask, uint64_t key,
                          const int64_t* __restrict__ e_off, const int32_t* __restrict__ e_len,
                          long long* out) {
  int32_t e = idx ? index_lookup(idx, mask, key) : -1;
  out[0] = e >= 0 ? e_off[e] : 0;
  out[1] = e >= 0 ? e_len[e] : 0;
}

int table_lookup1(TableDev& t, uint64_t key, int32_t* nodes_h, int64_t cap, int64_t* len) {
  *len = 0;
  if (t.n_entries == 0) return 0;
  long long* out;
  int rc;
  if ((rc = t.ws.get("l_out", 2, &out))) return rc;
  k_lookup1<<<1, 1>>>(t.idx, (uint64_t)t.idx_cap - 1, key, t.e_off, t.e_len, out);
  HRPP_LAUNCHED();
  long long h[2];
  HRPP_CK(cudaMemcpy(h, out, sizeof(h), cudaMemcpyDeviceToHost));
  *len = h[1];
  int64_t m = h[1] < cap ? h[1] : cap;
  if (m > 0 && nodes_h)
    HRPP_CK(cudaMemcpy(nodes_h, t.arena + h[0], sizeof(int32_t) * m, cudaMemcpyDeviceToHost));
  return 0;
}

int table_max_len(TableDev& t, int64_t* out) {
  *out = 0;
  if (t.n_entries == 0) return 0;
  int32_t* r;
  int rc;
  if ((rc = t.ws.get("mx_out", 1, &r))) return rc;
  size_t b = 0;
  cub::DeviceReduce::Max(nullptr, b, t.e_len, r, (int)t.n_entries);
  void* tmp;
  if ((rc = t.ws.get_raw("mx_tmp", b, &tmp))) return rc;
  HRPP_CK(cub::DeviceReduce::Max(tmp, b, t.e_len, r, (int)t.n_entries));
  int32_t h = 0;
  HRPP_CK(cudaMemcpy(&h, r, sizeof(h), cudaMemcpyDeviceToHost));
  *out = h;
  return 0;
}

// ---------------------------------------------------------------------------
// predict (hrpp/predictor.py:167-192) against a frozen table
// ---------------------------------------------------------------------------

struct PredictArgs {
  const DNode* nodes;
  const DTri* tris;
  const int32_t* depth;
  const Bucket* idx;
  uint64_t mask;
  const int64_t* e_off;
  const int32_t* e_len;
  const int32_t* arena;
  const uint64_t* keys;
  const float* O;
  const float* D;
  const double* tmin;
  const double* tmax;
  int64_t n;
  int8_t* cls;
  double* t;
  int32_t* slot;
  int32_t* leaf;
  double* u;
  double* v;
  int64_t* box;
  int64_t* tri;
  int64_t* vis;
  int64_t* est;
};

template <bool CLOSEST, int STACK>
__global__ void __launch_bounds__(128) k_predict(PredictArgs a) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= a.n) return;
  int32_t e = a.idx ? index_lookup(a.idx, a.mask, a.keys[i]) : -1;
  Hit acc = empty_entry_result(CLOSEST);
  int8_t c = 2;
  if (e >= 0) {
    Ray r = make_ray(a.O, a.D, a.tmin, a.tmax, i);
    const int32_t* nl = a.arena + a.e_off[e];
    int32_t L = a.e_len[e];
    for (int32_t j = 0; j < L; j++) {
      if (!CLOSEST && acc.found) break;  // eval_entry_any stops at the first hit
      fold_entry<CLOSEST>(acc, trace_from<CLOSEST, STACK>(a.nodes, a.tris, r, nl[j]));
    }
    c = acc.found ? 0 : 1;
  } else {
    acc.t = __longlong_as_double(0x7ff0000000000000LL);
  }
  a.cls[i] = c;
  if (a.t) a.t[i] = acc.t;
  if (a.slot) a.slot[i] = acc.slot;
  if (a.leaf) a.leaf[i] = acc.leaf;
  if (a.u || a.v) {
    double u = 0.0, v = 0.0;
    if (e >= 0) hit_uv(a.tris, make_ray(a.O, a.D, a.tmin, a.tmax, i), acc, u, v);
    if (a.u) a.u[i] = u;
    if (a.v) a.v[i] = v;
  }
  if (a.box) a.box[i] = acc.boxes;
  if (a.tri) a.tri[i] = acc.tris;
  if (a.vis) a.vis[i] = acc.boxes;
  if (a.est) {
    int64_t x = acc.found ? (int64_t)a.depth[acc.leaf] + 1 - acc.boxes : 0;
    a.est[i] = x > 0 ? x : 0;
  }
}

int predict_batch(const BvhDev& b, TableDev& t, const uint64_t* keys, const float* O,
                  const float* D, const double* tmin, const double* tmax, int64_t n,
                  int8_t* cls, double* tt, int32_t* slot, int32_t* leaf, double* u, double* v,
                  int64_t* box, int64_t* tri, int64_t* vis, int64_t* est, cudaStream_t st) {
  if (n <= 0) return 0;
  PredictArgs a{b.nodes, b.tris, b.depth, t.n_entries ? t.idx : nullptr,
                (uint64_t)t.idx_cap - 1, t.e_off, t.e_len, t.arena, keys, O, D, tmin, tmax, n,
                cls, tt, slot, leaf, u, v, box, tri, vis, est};
  int grid = (int)((n + 127) / 128);
#define PRED_CASE(S)                                                        \
  case S:                                                                   \
    if (t.closest) k_predict<true, S><<<grid, 128, 0, st>>>(a);             \
    else k_predict<false, S><<<grid, 128, 0, st>>>(a);                      \
    break;
  switch (b.stack) {
    PRED_CASE(32)
    PRED_CASE(64)
    PRED_CASE(128)
    PRED_CASE(256)
    default:
      if (t.closest) k_predict<true, 512><<<grid, 128, 0, st>>>(a);
      else k_predict<false, 512><<<grid, 128, 0, st>>>(a);
  }
#undef PRED_CASE
  HRPP_LAUNCHED();
  return 0;
}

}  // namespace hrpp
