// k_shard.cu -- key ownership for the exact multi-GPU mode.
//
// Key sharding: the owner of key k among G ranks is (mix64(k) >> 32) % G.
// Every rank partitions its contiguous block of a wave by owner, stably, so
// after an all-to-all each owner holds all rays of its keys in global ray
// order (source blocks arrive in rank order).  The consult of a key only
// reads and writes that key's entry (hrpp/tracer.py:233-267, 295-331), so an
// owner's replay of its rays against its table partition is exactly the
// single-GPU replay restricted to those keys: results and statistics sum to
// the single-GPU ones at any G.
#include <cub/cub.cuh>

#include "../../include/hrpp_b200.h"
#include "hrpp_internal.h"

namespace hrpp {

__device__ __forceinline__ uint32_t key_owner(uint64_t key, uint32_t world) {
  return (uint32_t)((mix64(key) >> 32) % world);
}

__global__ void k_owner(const uint64_t* __restrict__ keys, int64_t n, uint32_t world,
                        uint8_t* __restrict__ owner, int32_t* __restrict__ iota,
                        unsigned long long* __restrict__ counts) {
  __shared__ unsigned int hist[256];
  for (int k = threadIdx.x; k < 256; k += blockDim.x) hist[k] = 0;
  __syncthreads();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t o = key_owner(keys[i], world);
    owner[i] = (uint8_t)o;
    iota[i] = (int32_t)i;
    atomicAdd(&hist[o], 1u);
  }
  __syncthreads();
  for (int k = threadIdx.x; k < (int)world; k += blockDim.x)
    if (hist[k]) atomicAdd(counts + k, (unsigned long long)hist[k]);
}

// Exchange rows (one all-to-all each way instead of four): a ray is 40 bytes
// {O.xyz f32, D.xyz f32, tmin f64, tmax f64}; a hit is 24 bytes {t f64,
// slot i32, leaf i32, found u8, pad}.
struct __align__(8) RayRow {
  float o[3], d[3];
  double t0, t1;
};
struct __align__(8) HitRow {
  double t;
  int32_t slot, leaf;
  uint8_t found;
  uint8_t pad[7];
};

__global__ void k_pack_rays(const int32_t* __restrict__ perm, int64_t n,
                            const float* __restrict__ O, const float* __restrict__ D,
                            const double* __restrict__ t0, const double* __restrict__ t1,
                            RayRow* __restrict__ rows) {
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = perm[k];
    RayRow r;
    r.o[0] = O[3 * i]; r.o[1] = O[3 * i + 1]; r.o[2] = O[3 * i + 2];
    r.d[0] = D[3 * i]; r.d[1] = D[3 * i + 1]; r.d[2] = D[3 * i + 2];
    r.t0 = t0[i];
    r.t1 = t1[i];
    rows[k] = r;
  }
}

__global__ void k_unpack_rays(const RayRow* __restrict__ rows, int64_t n, float* __restrict__ O,
                              float* __restrict__ D, double* __restrict__ t0,
                              double* __restrict__ t1) {
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * blockDim.x) {
    const RayRow r = rows[k];
    O[3 * k] = r.o[0]; O[3 * k + 1] = r.o[1]; O[3 * k + 2] = r.o[2];
    D[3 * k] = r.d[0]; D[3 * k + 1] = r.d[1]; D[3 * k + 2] = r.d[2];
    t0[k] = r.t0;
    t1[k] = r.t1;
  }
}

__global__ void k_pack_hits(int64_t n, const uint8_t* __restrict__ found,
                            const double* __restrict__ t, const int32_t* __restrict__ slot,
                            const int32_t* __restrict__ leaf, HitRow* __restrict__ rows) {
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * blockDim.x) {
    HitRow h{};
    h.t = t[k];
    h.slot = slot[k];
    h.leaf = leaf[k];
    h.found = found[k];
    rows[k] = h;
  }
}

__global__ void k_unpack_hits(const HitRow* __restrict__ rows, const int32_t* __restrict__ perm,
                              int64_t n, uint8_t* __restrict__ found, double* __restrict__ t,
                              int32_t* __restrict__ slot, int32_t* __restrict__ leaf) {
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * blockDim.x) {
    const HitRow h = rows[k];
    const int64_t i = perm[k];
    found[i] = h.found;
    t[i] = h.t;
    slot[i] = h.slot;
    leaf[i] = h.leaf;
  }
}

__global__ void k_counts_out(const unsigned long long* cnt, int world, long long* out) {
  for (int k = threadIdx.x; k < world; k += blockDim.x) out[k] = (long long)cnt[k];
}

}  // namespace hrpp

using namespace hrpp;

extern "C" int hrpp_partition_by_owner(const uint64_t* keys, int64_t n, int world,
                                       int32_t* perm, int64_t* counts, void* stream) {
  if (world < 1 || world > 256 || n < 0 || n >= (1LL << 31) || !counts || (n > 0 && !perm) ||
      (n > 0 && !keys)) {
    set_error("partition_by_owner: bad arguments (world in [1, 256], n < 2^31)");
    return HRPP_INVALID_ARG;
  }
  cudaStream_t st = (cudaStream_t)stream;
  Workspace& ws = device_ws();  // per host thread and device
  uint8_t *own, *own2;
  int32_t* iota;
  unsigned long long* cnt;
  int rc;
  const int64_t m = n > 0 ? n : 1;
  if ((rc = ws.get("pt_own", m, &own)) || (rc = ws.get("pt_own2", m, &own2)) ||
      (rc = ws.get("pt_iota", m, &iota)) || (rc = ws.get("pt_cnt", 256, &cnt)))
    return rc;
  HRPP_CK(cudaMemsetAsync(cnt, 0, sizeof(unsigned long long) * 256, st));
  if (n > 0) {
    k_owner<<<grid_for(n, 256, num_sms() * 8), 256, 0, st>>>(keys, n, (uint32_t)world, own, iota,
                                                               cnt);
    HRPP_LAUNCHED();
    int bits = 0;
    while ((1 << bits) < world) bits++;
    if (bits == 0) {
      HRPP_CK(cudaMemcpyAsync(perm, iota, sizeof(int32_t) * n, cudaMemcpyDeviceToDevice, st));
    } else {
      size_t bytes = 0;  // LSD radix sort is stable: ray order within each owner
      cub::DeviceRadixSort::SortPairs(nullptr, bytes, own, own2, iota, perm, (int)n, 0, bits, st);
      void* tmp;
      if ((rc = ws.get_raw("pt_tmp", bytes, &tmp))) return rc;
      HRPP_CK(cub::DeviceRadixSort::SortPairs(tmp, bytes, own, own2, iota, perm, (int)n, 0, bits,
                                              st));
    }
  }
  cudaPointerAttributes attr{};
  if (cudaPointerGetAttributes(&attr, counts) == cudaSuccess &&
      (attr.type == cudaMemoryTypeDevice || attr.type == cudaMemoryTypeManaged)) {
    // device counts: no host round trip (the caller exchanges them on the device)
    k_counts_out<<<1, 256, 0, st>>>(cnt, world, (long long*)counts);
    HRPP_LAUNCHED();
    return HRPP_OK;
  }
  cudaGetLastError();  // a host pointer is not an error
  long long* pin = pinned_scratch();
  if (!pin) return HRPP_CUDA;
  for (int k0 = 0; k0 < world; k0 += 32) {  // 32 counters per readback
    const int m2 = world - k0 < 32 ? world - k0 : 32;
    if ((rc = to_host(pin + 32, cnt + k0, sizeof(unsigned long long) * m2, st))) return rc;
    HRPP_CK(cudaStreamSynchronize(st));
    for (int k = 0; k < m2; k++) counts[k0 + k] = ((volatile long long*)pin)[32 + k];
  }
  return HRPP_OK;
}

extern "C" int hrpp_pack_rays(const int32_t* perm, int64_t n, const float* O, const float* D,
                              const double* tmin, const double* tmax, void* rows, void* stream) {
  if (n < 0 || (n > 0 && (!perm || !O || !D || !tmin || !tmax || !rows))) {
    set_error("pack_rays: bad arguments");
    return HRPP_INVALID_ARG;
  }
  if (n == 0) return HRPP_OK;
  k_pack_rays<<<grid_for(n, 256, num_sms() * 16), 256, 0, (cudaStream_t)stream>>>(
      perm, n, O, D, tmin, tmax, (RayRow*)rows);
  HRPP_LAUNCHED();
  return HRPP_OK;
}

extern "C" int hrpp_unpack_rays(const void* rows, int64_t n, float* O, float* D, double* tmin,
                                double* tmax, void* stream) {
  if (n < 0 || (n > 0 && (!rows || !O || !D || !tmin || !tmax))) {
    set_error("unpack_rays: bad arguments");
    return HRPP_INVALID_ARG;
  }
  if (n == 0) return HRPP_OK;
  k_unpack_rays<<<grid_for(n, 256, num_sms() * 16), 256, 0, (cudaStream_t)stream>>>(
      (const RayRow*)rows, n, O, D, tmin, tmax);
  HRPP_LAUNCHED();
  return HRPP_OK;
}

extern "C" int hrpp_pack_hits(int64_t n, const uint8_t* found, const double* t,
                              const int32_t* slot, const int32_t* leaf, void* rows,
                              void* stream) {
  if (n < 0 || (n > 0 && (!found || !t || !slot || !leaf || !rows))) {
    set_error("pack_hits: bad arguments");
    return HRPP_INVALID_ARG;
  }
  if (n == 0) return HRPP_OK;
  k_pack_hits<<<grid_for(n, 256, num_sms() * 16), 256, 0, (cudaStream_t)stream>>>(
      n, found, t, slot, leaf, (HitRow*)rows);
  HRPP_LAUNCHED();
  return HRPP_OK;
}

extern "C" int hrpp_unpack_hits(const void* rows, const int32_t* perm, int64_t n,
                                uint8_t* found, double* t, int32_t* slot, int32_t* leaf,
                                void* stream) {
  if (n < 0 || (n > 0 && (!rows || !perm || !found || !t || !slot || !leaf))) {
    set_error("unpack_hits: bad arguments");
    return HRPP_INVALID_ARG;
  }
  if (n == 0) return HRPP_OK;
  k_unpack_hits<<<grid_for(n, 256, num_sms() * 16), 256, 0, (cudaStream_t)stream>>>(
      (const HitRow*)rows, perm, n, found, t, slot, leaf);
  HRPP_LAUNCHED();
  return HRPP_OK;
}
