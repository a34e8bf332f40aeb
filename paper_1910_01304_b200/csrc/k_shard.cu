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
  static thread_local Workspace ws;
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
