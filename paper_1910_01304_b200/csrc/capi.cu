// capi.cu -- the extern "C" boundary (include/hrpp_b200.h).
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <tuple>
#include <vector>

#include "../../include/hrpp_b200.h"
#include "hrpp_internal.h"

namespace hrpp {

std::atomic<int64_t> g_launches{0};
static thread_local std::string g_err;

void set_error(const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
}

int num_sms() {
  static int cached[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 0;
  if (!cached[dev]) {
    int v = 0;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0)
      v = 148;
    cached[dev] = v;
  }
  return cached[dev];
}

Workspace::~Workspace() {
  for (auto& kv : bufs) cudaFree(kv.second.p);
}

int Workspace::get_raw(const char* name, size_t bytes, void** out) {
  Buf& b = bufs[name];
  if (b.bytes < bytes) {
    if (b.p) HRPP_CK(cudaFree(b.p));
    b.p = nullptr;
    size_t nb = bytes + bytes / 4 + 256;
    HRPP_CK(cudaMalloc(&b.p, nb));
    b.bytes = nb;
  }
  *out = b.p;
  return 0;
}

BvhDev::~BvhDev() {
  cudaFree(nodes);
  cudaFree(tris);
  cudaFree(depth);
  for (auto& kv : anc) cudaFree(kv.second);
}

__global__ void k_ancestor(const int32_t* __restrict__ parent, int64_t n, int level,
                           int32_t* lut) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    int32_t x = (int32_t)i;
    for (int k = 0; k < level; k++) {  // hrpp/bvh.py:147-149, clamped at the root
      int32_t up = parent[x];
      if (up < 0) break;
      x = up;
    }
    lut[i] = x;
  }
}

int BvhDev::ancestor_lut(int level, const int32_t** out) {
  auto it = anc.find(level);
  if (it != anc.end()) {
    *out = it->second;
    return 0;
  }
  int32_t *par = nullptr, *lut = nullptr;
  HRPP_CK(cudaMalloc(&lut, sizeof(int32_t) * n_nodes));
  HRPP_CK(cudaMalloc(&par, sizeof(int32_t) * n_nodes));
  HRPP_CK(cudaMemcpy(par, parent_host.data(), sizeof(int32_t) * n_nodes, cudaMemcpyHostToDevice));
  k_ancestor<<<grid_for(n_nodes, 256, num_sms() * 8), 256>>>(par, n_nodes, level, lut);
  HRPP_LAUNCHED();
  HRPP_CK(cudaDeviceSynchronize());
  HRPP_CK(cudaFree(par));
  anc[level] = lut;
  *out = lut;
  return 0;
}

// ---- per-stage CUDA-event profiler --------------------------------------------
// Calls may run concurrently from several host threads (one stream each, e.g.
// waves on different tables); the profiler's shared state is under a mutex.
bool g_prof_on = false;
static unsigned g_prof_mask = ~0u;  // stages recorded while enabled
static std::mutex g_prof_mu;
struct ProfState {
  std::vector<cudaEvent_t> pool;
  std::vector<std::tuple<int, cudaEvent_t, cudaEvent_t>> pending;
  double ms[P_NCAT] = {0};
  long long count[P_NCAT] = {0};
  cudaEvent_t get() {
    if (!pool.empty()) {
      cudaEvent_t e = pool.back();
      pool.pop_back();
      return e;
    }
    cudaEvent_t e = nullptr;
    cudaEventCreate(&e);
    return e;
  }
};
static ProfState g_prof;

ProfScope::ProfScope(int c, cudaStream_t s) : cat(c), st(s) {
  if (!g_prof_on || !((g_prof_mask >> c) & 1u)) return;
  {
    std::lock_guard<std::mutex> lk(g_prof_mu);
    a = g_prof.get();
    b = g_prof.get();
  }
  cudaEventRecord(a, st);
}

ProfScope::~ProfScope() {
  if (!a) return;
  cudaEventRecord(b, st);
  std::lock_guard<std::mutex> lk(g_prof_mu);
  g_prof.pending.emplace_back(cat, a, b);
}

void prof_flush() {
  std::lock_guard<std::mutex> lk(g_prof_mu);
  for (auto& p : g_prof.pending) {
    float ms = 0.f;
    cudaEventSynchronize(std::get<2>(p));
    if (cudaEventElapsedTime(&ms, std::get<1>(p), std::get<2>(p)) == cudaSuccess) {
      g_prof.ms[std::get<0>(p)] += ms;
      g_prof.count[std::get<0>(p)] += 1;
    }
    g_prof.pool.push_back(std::get<1>(p));
    g_prof.pool.push_back(std::get<2>(p));
  }
  g_prof.pending.clear();
}

// Scratch for calls without a table (and host staging): one per host thread
// and device, so concurrent calls from different threads never share it.
Workspace& device_ws() {
  static thread_local Workspace ws[64];
  int dev = 0;
  cudaGetDevice(&dev);
  ws[dev & 63].device = dev;
  return ws[dev & 63];
}
static Workspace& global_ws() { return device_ws(); }

static bool is_device_ptr(const void* p);

// Host/device pointer staging for one call: every array is checked on its
// own; host (pageable or pinned) arrays go through the device workspace.
struct Stager {
  Workspace& ws;
  cudaStream_t st;
  std::vector<std::tuple<void*, const void*, size_t>> back;
  int k = 0;
  Stager(Workspace& w, cudaStream_t s) : ws(w), st(s) {}
  std::string name() { return "stage" + std::to_string(k++); }
  template <typename T>
  int in(const T* p, size_t count, const T** out) {
    if (!p || count == 0 || is_device_ptr(p)) {
      *out = p;
      return 0;
    }
    T* d;
    int rc = ws.get(name().c_str(), count, &d);
    if (rc) return rc;
    HRPP_CK(cudaMemcpyAsync(d, p, sizeof(T) * count, cudaMemcpyHostToDevice, st));
    *out = d;
    return 0;
  }
  template <typename T>
  int out(T* p, size_t count, T** dev) {
    if (!p || count == 0 || is_device_ptr(p)) {
      *dev = p;
      return 0;
    }
    T* d;
    int rc = ws.get(name().c_str(), count, &d);
    if (rc) return rc;
    back.emplace_back((void*)p, (const void*)d, sizeof(T) * count);
    *dev = d;
    return 0;
  }
  // scratch when the caller passed NULL but the pipeline needs the array
  template <typename T>
  int need(T** p, size_t count) {
    if (*p) return 0;
    return ws.get(name().c_str(), count, p);
  }
  int finish() {
    for (auto& b : back)
      HRPP_CK(cudaMemcpyAsync(std::get<0>(b), std::get<1>(b), std::get<2>(b),
                              cudaMemcpyDeviceToHost, st));
    HRPP_CK(cudaStreamSynchronize(st));
    return 0;
  }
};

static bool is_device_ptr(const void* p) {
  if (!p) return false;
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
}

static int choose_stack(int height) {
  if (height + 2 <= 64) return 64;
  if (height + 2 <= 256) return 256;
  if (height + 2 <= 512) return 512;
  return -1;
}

struct Pinned {
  long long* p = nullptr;
  int get() {
    if (!p) HRPP_CK(cudaHostAlloc(&p, sizeof(long long) * 64, cudaHostAllocMapped | cudaHostAllocPortable));
    return 0;
  }
};
static thread_local Pinned g_pinned;  // per host thread (see global_ws)

long long* pinned_scratch() { return g_pinned.get() ? nullptr : g_pinned.p; }

__global__ void k_to_host(char* dst, const char* src, int bytes) {
  for (int i = threadIdx.x; i < bytes; i += blockDim.x) dst[i] = src[i];
}
__global__ void k_set_i32(int32_t* dst, int32_t v) { *dst = v; }
// end-of-wave readback into the pinned buffer: meta -> [28, 32), err -> [3],
// stats -> [4, 20)
__global__ void k_wave_readback(const long long* meta, const int* err,
                                const unsigned long long* stats, long long* pin) {
  const int k = threadIdx.x;
  if (k < 4) pin[28 + k] = meta[k];
  if (k == 4) *reinterpret_cast<int*>(pin + 3) = *err;
  if (stats && k < 16) pin[4 + k] = (long long)stats[k];
}
__global__ void k_set_i64(long long* dst, long long v) { *dst = v; }

int to_host(void* pinned_dst, const void* dev_src, size_t bytes, cudaStream_t st) {
  if (bytes == 0) return 0;
  k_to_host<<<1, 128, 0, st>>>((char*)pinned_dst, (const char*)dev_src, (int)bytes);
  HRPP_LAUNCHED();
  return 0;
}
int set_i32(int32_t* dst, int32_t v, cudaStream_t st) {
  k_set_i32<<<1, 1, 0, st>>>(dst, v);
  HRPP_LAUNCHED();
  return 0;
}
int set_i64(long long* dst, long long v, cudaStream_t st) {
  k_set_i64<<<1, 1, 0, st>>>(dst, v);
  HRPP_LAUNCHED();
  return 0;
}

}  // namespace hrpp

using namespace hrpp;

struct hrpp_bvh_s : BvhDev {};
struct hrpp_table_s : TableDev {};

#define CHECK_ARG(cond, msg)          \
  do {                                \
    if (!(cond)) {                    \
      set_error("%s", msg);           \
      return HRPP_INVALID_ARG;        \
    }                                 \
  } while (0)

extern "C" {

const char* hrpp_last_error(void) { return g_err.c_str(); }
int hrpp_version(void) { return 1; }
int64_t hrpp_launch_count(void) { return g_launches.load(); }
int hrpp_device_count(int* count) {
  *count = 0;
  HRPP_CK(cudaGetDeviceCount(count));
  return HRPP_OK;
}
int hrpp_set_consult_short(int len) {
  CHECK_ARG(len >= 0, "short segment length must be >= 0");
  g_consult_short = len;
  return HRPP_OK;
}
int hrpp_profile_enable(int on) {
  g_prof_on = on != 0;
  g_prof_mask = ~0u;
  return HRPP_OK;
}
int hrpp_profile_stages(unsigned mask) {
  g_prof_on = mask != 0;
  g_prof_mask = mask;
  return HRPP_OK;
}
int hrpp_profile_read(double* ms, int64_t* counts, int n, int reset) {
  cudaDeviceSynchronize();
  prof_flush();
  std::lock_guard<std::mutex> lk(g_prof_mu);
  for (int k = 0; k < n && k < P_NCAT; k++) {
    if (ms) ms[k] = g_prof.ms[k];
    if (counts) counts[k] = g_prof.count[k];
  }
  if (reset)
    for (int k = 0; k < P_NCAT; k++) {
      g_prof.ms[k] = 0;
      g_prof.count[k] = 0;
    }
  return P_NCAT;
}
int hrpp_set_fast_rounds(int rounds, int stop_div) {
  CHECK_ARG(rounds >= 0 && rounds < 100000, "fast rounds must be in [0, 100000)");
  CHECK_ARG(stop_div >= 0, "stop_div must be >= 0");
  g_fast_rounds = rounds;
  g_fast_stop_div = stop_div;
  return HRPP_OK;
}
int hrpp_set_live_rounds(int rounds) {
  CHECK_ARG(rounds >= 0 && rounds < 1000, "live rounds must be in [0, 1000)");
  g_live_rounds = rounds;
  return HRPP_OK;
}

// ---- hash -----------------------------------------------------------------

int hrpp_hash_rays(const float* O, const float* D, int64_t n, int p, uint64_t* keys,
                   void* stream) {
  CHECK_ARG(p >= 1 && p <= 7, "precision_bits must be in [1, 7]");
  CHECK_ARG(n >= 0, "n must be >= 0");
  if (n == 0) return HRPP_OK;
  cudaStream_t st = (cudaStream_t)stream;
  Stager sg(global_ws(), st);
  const float *dO, *dD;
  uint64_t* dk;
  int* err;
  int rc;
  if ((rc = sg.in(O, 3 * n, &dO)) || (rc = sg.in(D, 3 * n, &dD)) || (rc = sg.out(keys, n, &dk)))
    return rc;
  if ((rc = global_ws().get("hash_err", 1, &err))) return rc;
  HRPP_CK(cudaMemsetAsync(err, 0, sizeof(int), st));
  if ((rc = launch_hash(dO, dD, n, p, dk, err, st))) return rc;
  if ((rc = g_pinned.get())) return rc;
  if ((rc = to_host(g_pinned.p, err, sizeof(int), st))) return rc;
  if ((rc = sg.finish())) return rc;
  if (*(int*)g_pinned.p) {
    set_error("non-finite ray component in hash batch");
    return HRPP_NONFINITE;
  }
  return HRPP_OK;
}

int hrpp_hash_floats(const float* f, int64_t n, int p, uint32_t* out, void* stream) {
  CHECK_ARG(p >= 1 && p <= 7, "precision_bits must be in [1, 7]");
  if (n <= 0) return HRPP_OK;
  cudaStream_t st = (cudaStream_t)stream;
  Stager sg(global_ws(), st);
  const float* df;
  uint32_t* dout;
  int* err;
  int rc;
  if ((rc = sg.in(f, n, &df)) || (rc = sg.out(out, n, &dout))) return rc;
  if ((rc = global_ws().get("hashf_err", 1, &err))) return rc;
  HRPP_CK(cudaMemsetAsync(err, 0, sizeof(int), st));
  if ((rc = launch_hash_floats(df, n, p, dout, err, st))) return rc;
  if ((rc = g_pinned.get())) return rc;
  if ((rc = to_host(g_pinned.p, err, sizeof(int), st))) return rc;
  if ((rc = sg.finish())) return rc;
  if (*(int*)g_pinned.p) {
    set_error("cannot hash non-finite float");
    return HRPP_NONFINITE;
  }
  return HRPP_OK;
}

int hrpp_coarsen_keys(const uint64_t* keys, int64_t n, int p, uint64_t* out, void* stream) {
  CHECK_ARG(p >= 2 && p <= 7, "cannot coarsen below the minimum precision");
  CHECK_ARG(n >= 0 && (n == 0 || (keys && out)), "bad arguments");
  if (n == 0) return HRPP_OK;
  cudaStream_t st = (cudaStream_t)stream;
  Stager sg(global_ws(), st);
  const uint64_t* dk;
  uint64_t* dout;
  int rc;
  if ((rc = sg.in(keys, n, &dk)) || (rc = sg.out(out, n, &dout))) return rc;
  if ((rc = launch_coarsen(dk, n, p, dout, st))) return rc;
  return sg.finish();
}

// ---- BVH ------------------------------------------------------------------

int hrpp_bvh_create(const float* bmin, const float* bmax, const int32_t* left,
                    const int32_t* right, const int8_t* axis, const int32_t* first,
                    const int32_t* count, const int32_t* parent, const int32_t* depth,
                    const float* tv0, const float* tv1, const float* tv2,
                    const int32_t* tri_ids, int64_t n_nodes, int64_t n_tris, int device,
                    hrpp_bvh_t* out) {
  (void)tri_ids;
  CHECK_ARG(n_nodes >= 1 && n_nodes < (1LL << 27), "node count must be in [1, 2^27)");
  CHECK_ARG(n_tris >= 0 && n_tris < (1LL << 31), "triangle count out of range");
  HRPP_CK(cudaSetDevice(device));
  std::vector<DNode> hn(n_nodes);
  for (int64_t i = 0; i < n_nodes; i++) {
    if (left[i] < 0) {
      CHECK_ARG(first[i] >= 0 && count[i] >= 0 && (int64_t)first[i] + count[i] <= n_tris,
                "leaf triangle range out of bounds");
      pack_node(hn[i], bmin + 3 * i, bmax + 3 * i, ~first[i], count[i]);
    } else {
      CHECK_ARG(left[i] < n_nodes && right[i] >= 0 && right[i] < n_nodes,
                "child index out of range");
      int ax = axis[i] == 1 ? 1 : (axis[i] == 2 ? 2 : 0);
      pack_node(hn[i], bmin + 3 * i, bmax + 3 * i, left[i],
                (int32_t)((uint32_t)right[i] | (1u << (27 + ax))));
    }
  }
  // tree height from the root (stack bound); guards against cycles
  int height = 0;
  {
    std::vector<std::pair<int32_t, int32_t>> stk{{0, 0}};
    int64_t steps = 0;
    while (!stk.empty()) {
      auto [nd, dep] = stk.back();
      stk.pop_back();
      CHECK_ARG(++steps <= 2 * n_nodes + 2, "BVH is not a tree");
      if (dep > height) height = dep;
      if (left[nd] >= 0) {
        stk.push_back({left[nd], dep + 1});
        stk.push_back({right[nd], dep + 1});
      }
    }
  }
  int stack = choose_stack(height);
  CHECK_ARG(stack > 0, "BVH deeper than the 512-entry traversal stack");
  // slot -> leaf (the traversal reads a hit's leaf from its triangle record)
  std::vector<int32_t> leaf_of(n_tris > 0 ? n_tris : 1, -1);
  for (int64_t nd = 0; nd < n_nodes; nd++) {
    if (left[nd] >= 0) continue;
    for (int64_t k = first[nd]; k < (int64_t)first[nd] + count[nd]; k++) {
      CHECK_ARG(leaf_of[k] < 0, "leaf slot ranges overlap");
      leaf_of[k] = (int32_t)nd;
    }
  }
  std::vector<DTri> ht(n_tris > 0 ? n_tris : 1);
  for (int64_t k = 0; k < n_tris; k++)
    pack_tri(ht[k], tv0 + 3 * k, tv1 + 3 * k, tv2 + 3 * k, leaf_of[k]);
  auto* h = new hrpp_bvh_s();
  h->device = device;
  h->n_nodes = n_nodes;
  h->n_tris = n_tris;
  h->height = height;
  h->stack = stack;
  h->parent_host.assign(parent, parent + n_nodes);
  for (int k = 0; k < 3; k++) {
    h->root_lo[k] = bmin[k];
    h->root_hi[k] = bmax[k];
  }
  bool ok = cudaMalloc(&h->nodes, sizeof(DNode) * n_nodes) == cudaSuccess &&
            cudaMalloc(&h->tris, sizeof(DTri) * ht.size()) == cudaSuccess &&
            cudaMalloc(&h->depth, sizeof(int32_t) * n_nodes) == cudaSuccess &&
            cudaMemcpy(h->nodes, hn.data(), sizeof(DNode) * n_nodes, cudaMemcpyHostToDevice) ==
                cudaSuccess &&
            cudaMemcpy(h->tris, ht.data(), sizeof(DTri) * ht.size(), cudaMemcpyHostToDevice) ==
                cudaSuccess &&
            cudaMemcpy(h->depth, depth, sizeof(int32_t) * n_nodes, cudaMemcpyHostToDevice) ==
                cudaSuccess;
  if (!ok) {
    set_error("BVH upload failed: %s", cudaGetErrorString(cudaGetLastError()));
    delete h;
    return HRPP_CUDA;
  }
  *out = h;
  return HRPP_OK;
}

int hrpp_bvh_destroy(hrpp_bvh_t bvh) {
  delete bvh;
  return HRPP_OK;
}

int hrpp_bvh_ancestor_lut(hrpp_bvh_t bvh, int go_up_level, int32_t* lut_host) {
  CHECK_ARG(bvh, "null BVH");
  CHECK_ARG(go_up_level >= 0, "go_up_level must be >= 0");
  HRPP_CK(cudaSetDevice(bvh->device));
  const int32_t* lut;
  int rc = bvh->ancestor_lut(go_up_level, &lut);
  if (rc) return rc;
  HRPP_CK(cudaMemcpy(lut_host, lut, sizeof(int32_t) * bvh->n_nodes, cudaMemcpyDeviceToHost));
  return HRPP_OK;
}

// ---- traversal batch --------------------------------------------------------

int hrpp_trace_batch(hrpp_bvh_t bvh, int kind, const float* O, const float* D,
                     const double* tmin, const double* tmax, int32_t start, int64_t n,
                     hrpp_wave_out* out, void* stream) {
  CHECK_ARG(bvh && out, "null argument");
  CHECK_ARG(kind == HRPP_HIT_ANY || kind == HRPP_CLOSEST_HIT, "bad ray kind");
  CHECK_ARG(start >= 0 && start < bvh->n_nodes, "start node out of range");
  CHECK_ARG(n >= 0 && n < (1LL << 31), "ray count out of range");
  if (n == 0) return HRPP_OK;
  HRPP_CK(cudaSetDevice(bvh->device));
  cudaStream_t st = (cudaStream_t)stream;
  const bool closest = kind == HRPP_CLOSEST_HIT;
  Stager sg(global_ws(), st);
  const float *dO, *dD;
  const double *d0, *d1;
  TraceOut to;
  int rc;
  if ((rc = sg.in(O, 3 * n, &dO)) || (rc = sg.in(D, 3 * n, &dD)) ||
      (rc = sg.in(tmin, n, &d0)) || (rc = sg.in(tmax, n, &d1)) ||
      (rc = sg.out(out->found, n, &to.found)) || (rc = sg.out(out->t, n, &to.t)) ||
      (rc = sg.out(out->slot, n, &to.slot)) || (rc = sg.out(out->leaf, n, &to.leaf)) ||
      (rc = sg.out(out->box, n, &to.box)) || (rc = sg.out(out->tri, n, &to.tri)) ||
      (rc = sg.out(out->visited, n, &to.vis)))
    return rc;
  if (closest) {
    if ((rc = sg.out(out->u, n, &to.u)) || (rc = sg.out(out->v, n, &to.v))) return rc;
  }
  if ((rc = launch_trace(*bvh, closest, dO, dD, d0, d1, start, n, nullptr, nullptr, to, nullptr,
                         st, &global_ws())))
    return rc;
  return sg.finish();
}

// ---- table ------------------------------------------------------------------

int hrpp_table_create(int precision, int go_up_level, int kind, int64_t max_entries, int device,
                      hrpp_table_t* out) {
  CHECK_ARG(precision >= 1 && precision <= 7, "precision_bits must be in [1, 7]");
  CHECK_ARG(go_up_level >= 0, "go_up_level must be >= 0");
  CHECK_ARG(kind == HRPP_HIT_ANY || kind == HRPP_CLOSEST_HIT, "bad ray kind");
  CHECK_ARG(max_entries >= 0, "max_entries must be >= 0");
  HRPP_CK(cudaSetDevice(device));
  auto* t = new hrpp_table_s();
  t->device = device;
  t->precision = precision;
  t->go_up = go_up_level;
  t->closest = kind == HRPP_CLOSEST_HIT;
  t->max_entries = max_entries;
  t->ws.device = device;
  int rc = t->reserve(0, 0, 0);
  if (rc) {
    delete t;
    return rc;
  }
  HRPP_CK(cudaDeviceSynchronize());
  *out = t;
  return HRPP_OK;
}

int hrpp_table_destroy(hrpp_table_t table) {
  delete table;
  return HRPP_OK;
}

int hrpp_table_clear_async(hrpp_table_t t, void* stream) {
  CHECK_ARG(t, "null table");
  HRPP_CK(cudaSetDevice(t->device));
  cudaStream_t st = (cudaStream_t)stream;
  HRPP_CK(t->wait_clear(st));
  if (t->meta) HRPP_CK(cudaMemsetAsync(t->meta, 0, sizeof(long long) * 4, st));
  if (t->idx) HRPP_CK(cudaMemsetAsync(t->idx, 0xFF, sizeof(Bucket) * t->idx_cap, st));
  t->n_entries = t->stored = t->arena_used = t->pending = 0;
  // Later calls may run on other streams (host arrays use the legacy stream,
  // export/lookup stream 0): each waits for this event before touching the
  // table, so none reads the stale index or races the memsets.
  if (!t->clear_ev) HRPP_CK(cudaEventCreateWithFlags(&t->clear_ev, cudaEventDisableTiming));
  HRPP_CK(cudaEventRecord(t->clear_ev, st));
  t->clear_recorded = true;
  return HRPP_OK;
}

int hrpp_table_clear(hrpp_table_t t) {
  int rc = hrpp_table_clear_async(t, nullptr);
  if (rc) return rc;
  HRPP_CK(cudaStreamSynchronize(nullptr));
  return HRPP_OK;
}

int hrpp_table_info(hrpp_table_t t, int64_t* entries, int64_t* stored, int64_t* max_len) {
  CHECK_ARG(t, "null table");
  HRPP_CK(cudaSetDevice(t->device));
  *entries = t->n_entries;
  *stored = t->stored;
  HRPP_CK(t->wait_clear(0));
  if (max_len) return table_max_len(*t, max_len);
  return HRPP_OK;
}

static int read_meta_and_finish(TableDev& t, int* err, cudaStream_t st, Stager& sg,
                                unsigned long long* stats_dev) {
  int rc;
  if ((rc = g_pinned.get())) return rc;
  k_wave_readback<<<1, 32, 0, st>>>(t.meta, err, stats_dev, g_pinned.p);  // one launch
  HRPP_LAUNCHED();
  if ((rc = sg.finish())) return rc;
  int e = *(int*)(g_pinned.p + 3);
  if (e == 0) {
    t.n_entries = g_pinned.p[28];
    t.stored = g_pinned.p[29];
    t.arena_used = g_pinned.p[30];
    t.pending = t.deferred ? g_pinned.p[31] : 0;
  }
  return 0;
}

int hrpp_table_record(hrpp_table_t t, const uint64_t* keys, const int32_t* nodes, int64_t n,
                      uint8_t* inserted, void* stream) {
  CHECK_ARG(t, "null table");
  CHECK_ARG(n >= 0 && n < (1LL << 31), "record count out of range");
  if (n == 0) return HRPP_OK;
  HRPP_CK(cudaSetDevice(t->device));
  cudaStream_t st = (cudaStream_t)stream;
  HRPP_CK(t->wait_clear(st));
  Stager sg(global_ws(), st);
  const uint64_t* dk;
  const int32_t* dn;
  uint8_t* di;
  int* err;
  int rc;
  if ((rc = sg.in(keys, n, &dk)) || (rc = sg.in(nodes, n, &dn)) ||
      (rc = sg.out(inserted, n, &di)))
    return rc;
  if ((rc = t->ws.get("t_err", 1, &err))) return rc;
  HRPP_CK(cudaMemsetAsync(err, 0, sizeof(int), st));
  if ((rc = table_record(*t, dk, dn, n, di, err, st))) return rc;
  if ((rc = read_meta_and_finish(*t, err, st, sg, nullptr))) return rc;
  int e = *(int*)(g_pinned.p + 3);
  if (e == 2) {
    set_error("predictor table reached its cap of %lld entries", (long long)t->max_entries);
    return HRPP_CAPACITY;
  }
  if (e) {
    set_error("internal error %d in record", e);
    return HRPP_CUDA;
  }
  return HRPP_OK;
}

int hrpp_table_set_deferred(hrpp_table_t t, int on) {
  CHECK_ARG(t, "null table");
  t->deferred = on != 0;
  t->pending = 0;
  return HRPP_OK;
}

int hrpp_table_pending(hrpp_table_t t, uint64_t* keys, int32_t* nodes, int32_t* rays,
                       int64_t cap, int64_t* count) {
  CHECK_ARG(t && count, "null argument");
  HRPP_CK(cudaSetDevice(t->device));
  *count = t->pending;
  HRPP_CK(t->wait_clear(0));
  int64_t m = t->pending < cap ? t->pending : cap;
  if (m <= 0) return HRPP_OK;
  void *pk, *pn, *pr;
  int rc;
  if ((rc = t->ws.get_raw("p_keys", 0, &pk)) || (rc = t->ws.get_raw("p_nodes", 0, &pn)) ||
      (rc = t->ws.get_raw("p_rays", 0, &pr)))
    return rc;
  if (keys) HRPP_CK(cudaMemcpy(keys, pk, sizeof(uint64_t) * m, cudaMemcpyDefault));
  if (nodes) HRPP_CK(cudaMemcpy(nodes, pn, sizeof(int32_t) * m, cudaMemcpyDefault));
  if (rays) HRPP_CK(cudaMemcpy(rays, pr, sizeof(int32_t) * m, cudaMemcpyDefault));
  return HRPP_OK;
}

int hrpp_table_lookup(hrpp_table_t t, uint64_t key, int32_t* nodes_host, int64_t cap,
                      int64_t* len_out) {
  CHECK_ARG(t && len_out, "null argument");
  HRPP_CK(cudaSetDevice(t->device));
  HRPP_CK(t->wait_clear(0));
  return table_lookup1(*t, key, nodes_host, cap, len_out);
}

int hrpp_table_export(hrpp_table_t t, uint64_t* keys, int64_t* offsets, int32_t* nodes) {
  CHECK_ARG(t && keys && offsets, "null argument");
  HRPP_CK(cudaSetDevice(t->device));
  HRPP_CK(t->wait_clear(0));
  return table_export(*t, keys, offsets, nodes);
}

// ---- predict ------------------------------------------------------------------

int hrpp_predict_batch(hrpp_bvh_t bvh, hrpp_table_t t, const uint64_t* keys, const float* O,
                       const float* D, const double* tmin, const double* tmax, int64_t n,
                       int8_t* cls, double* tt, int32_t* slot, int32_t* leaf, double* u,
                       double* v, int64_t* box, int64_t* tri, int64_t* visited, int64_t* est,
                       void* stream) {
  CHECK_ARG(bvh && t && cls, "null argument");
  CHECK_ARG(n >= 0 && n < (1LL << 31), "ray count out of range");
  if (n == 0) return HRPP_OK;
  HRPP_CK(cudaSetDevice(bvh->device));
  cudaStream_t st = (cudaStream_t)stream;
  HRPP_CK(t->wait_clear(st));
  Stager sg(global_ws(), st);
  const uint64_t* dk;
  const float *dO, *dD;
  const double *d0, *d1;
  int8_t* dc;
  double *dt, *du, *dv;
  int32_t *ds, *dl;
  int64_t *db, *dtr, *dvis, *de;
  int rc;
  if ((rc = sg.in(keys, n, &dk)) || (rc = sg.in(O, 3 * n, &dO)) || (rc = sg.in(D, 3 * n, &dD)) ||
      (rc = sg.in(tmin, n, &d0)) || (rc = sg.in(tmax, n, &d1)) || (rc = sg.out(cls, n, &dc)) ||
      (rc = sg.out(tt, n, &dt)) || (rc = sg.out(slot, n, &ds)) || (rc = sg.out(leaf, n, &dl)) ||
      (rc = sg.out(u, n, &du)) || (rc = sg.out(v, n, &dv)) || (rc = sg.out(box, n, &db)) ||
      (rc = sg.out(tri, n, &dtr)) || (rc = sg.out(visited, n, &dvis)) ||
      (rc = sg.out(est, n, &de)))
    return rc;
  if ((rc = predict_batch(*bvh, *t, dk, dO, dD, d0, d1, n, dc, dt, ds, dl, du, dv, db, dtr, dvis,
                          de, st)))
    return rc;
  return sg.finish();
}

// ---- the wave -----------------------------------------------------------------

int hrpp_trace_wave(hrpp_bvh_t bvh, hrpp_table_t t, int mode, int closest, const float* O,
                    const float* D, const double* tmin, const double* tmax, int64_t n,
                    hrpp_wave_out* out, hrpp_outcome_log* log, int64_t* stats, void* stream) {
  CHECK_ARG(bvh && stats, "null argument");
  CHECK_ARG(mode >= HRPP_MODE_BASELINE && mode <= HRPP_MODE_FAST, "bad mode");
  CHECK_ARG(mode != HRPP_MODE_FAST || !t || !t->deferred,
            "fast mode does not support deferred commits");
  const bool live_like = mode == HRPP_MODE_LIVE || mode == HRPP_MODE_FAST;
  CHECK_ARG(mode == HRPP_MODE_BASELINE || t, "limit and live modes need a table");
  CHECK_ARG(!t || mode == HRPP_MODE_BASELINE || t->closest == (closest != 0),
            "table kind does not match the wave's ray kind");
  CHECK_ARG(n >= 0 && n < (1LL << 31), "ray count out of range");
  stats[0] += n;  // hrpp/tracer.py:350 counts the rays before hashing
  if (n == 0) return HRPP_OK;
  HRPP_CK(cudaSetDevice(bvh->device));
  cudaStream_t st = (cudaStream_t)stream;
  if (t) HRPP_CK(t->wait_clear(st));
  hrpp_wave_out none{};
  if (!out) out = &none;
  Workspace& ws = t ? t->ws : global_ws();
  Stager sg(ws, st);
  const float *dO, *dD;
  const double *d0, *d1;
  int rc;
  if ((rc = sg.in(O, 3 * n, &dO)) || (rc = sg.in(D, 3 * n, &dD)) || (rc = sg.in(tmin, n, &d0)) ||
      (rc = sg.in(tmax, n, &d1)))
    return rc;
  TraceOut to;
  uint64_t* keys = nullptr;
  if ((rc = sg.out(out->found, n, &to.found)) || (rc = sg.out(out->t, n, &to.t)) ||
      (rc = sg.out(out->slot, n, &to.slot)) || (rc = sg.out(out->leaf, n, &to.leaf)) ||
      (rc = sg.out(out->keys, n, &keys)))
    return rc;
  if (!live_like) {
    if ((rc = sg.out(out->box, n, &to.box)) || (rc = sg.out(out->tri, n, &to.tri)) ||
        (rc = sg.out(out->visited, n, &to.vis)))
      return rc;
    if (closest && ((rc = sg.out(out->u, n, &to.u)) || (rc = sg.out(out->v, n, &to.v))))
      return rc;
  }
  hrpp_outcome_log lg{};
  if (log && mode == HRPP_MODE_LIMIT) {
    if ((rc = sg.out(log->cls, n, &lg.cls)) || (rc = sg.out(log->eval_box, n, &lg.eval_box)) ||
        (rc = sg.out(log->pred_t, n, &lg.pred_t)) ||
        (rc = sg.out(log->pred_slot, n, &lg.pred_slot)))
      return rc;
  }
  // arrays the pipeline needs even if the caller did not ask for them
  if (mode != HRPP_MODE_BASELINE) {
    if ((rc = sg.need(&keys, n)) || (rc = sg.need(&to.found, n)) || (rc = sg.need(&to.t, n)) ||
        (rc = sg.need(&to.leaf, n)))
      return rc;
    if (mode == HRPP_MODE_LIMIT && (rc = sg.need(&to.box, n))) return rc;
    if (live_like && (rc = sg.need(&to.slot, n))) return rc;
  }
  int* err;
  unsigned long long* sdev;
  // stats [0, 16) and the error flag (slot 16) in one buffer: one memset
  if ((rc = ws.get("w_stats", 17, &sdev))) return rc;
  err = reinterpret_cast<int*>(sdev + 16);
  HRPP_CK(cudaMemsetAsync(sdev, 0, sizeof(unsigned long long) * 17, st));
  // keys nobody asked for go straight into the grouping sort's packed form
  bool prepacked = false;
  if (mode == HRPP_MODE_FAST) {  // hashing is fused into the fast consult
    FastIO io{dO, dD, d0, d1, n, to.found, to.t, to.slot, to.leaf, keys};
    if ((rc = run_fast(*bvh, *t, io, sdev, err, st))) return rc;
    if ((rc = read_meta_and_finish(*t, err, st, sg, sdev))) return rc;
  } else if (mode != HRPP_MODE_BASELINE) {
    int ib = 1;  // ray index bits, as group_by_key computes them
    while (ib < 31 && (1ll << ib) < n) ib++;
    prepacked = out->keys == nullptr && 3 * (1 + 2 * t->precision) + ib <= 64;
    if ((rc = launch_hash(dO, dD, n, t->precision, keys, err, st, prepacked ? ib : 0)))
      return rc;
  }
  if (!live_like) {
    to.sums = sdev + 4;  // baseline_box_tests, baseline_tri_tests (tracer.py:361-362)
    if ((rc = launch_trace(*bvh, closest != 0, dO, dD, d0, d1, 0, n, nullptr, nullptr, to, err,
                           st, &ws)))
      return rc;
  }
  if (mode != HRPP_MODE_BASELINE && mode != HRPP_MODE_FAST) {
    Consult c;
    c.live = mode == HRPP_MODE_LIVE;
    c.O = dO;
    c.D = dD;
    c.tmin = d0;
    c.tmax = d1;
    c.n = n;
    c.base_found = to.found;
    c.base_t = to.t;
    c.base_leaf = to.leaf;
    c.base_box = to.box;
    c.o_found = to.found;
    c.o_t = to.t;
    c.o_slot = to.slot;
    c.o_leaf = to.leaf;
    c.log_cls = lg.cls;
    c.log_eval_box = lg.eval_box;
    c.log_pred_t = lg.pred_t;
    c.log_pred_slot = lg.pred_slot;
    if ((rc = run_consult(*bvh, *t, c, keys, sdev, err, st, prepacked))) return rc;
    if ((rc = read_meta_and_finish(*t, err, st, sg, sdev))) return rc;
  } else if (mode == HRPP_MODE_BASELINE) {
    if ((rc = g_pinned.get())) return rc;
    if ((rc = to_host(g_pinned.p + 3, err, sizeof(int), st))) return rc;
    if ((rc = to_host(g_pinned.p + 4, sdev, sizeof(long long) * 16, st))) return rc;
    if ((rc = sg.finish())) return rc;
  }
  const int e = *(int*)(g_pinned.p + 3);
  const long long* s = g_pinned.p + 4;
  if (e == 1) {
    set_error("non-finite ray component in hash batch");
    return HRPP_NONFINITE;
  }
  if (mode == HRPP_MODE_LIMIT || mode == HRPP_MODE_BASELINE) {
    stats[4] += s[4];  // the baseline sums precede the consult (tracer.py:361-362)
    stats[5] += s[5];
  }
  if (mode == HRPP_MODE_LIVE && t && e == 0) {  // slot 14: wave-start TPs (k_eval0)
    t->start_tp_frac = (double)s[14] / (double)n;
    if (t->wave_started_empty) t->empty_tp_frac = (double)s[1] / (double)n;
  }
  if (e == 2) {
    set_error("predictor table reached its cap of %lld entries", (long long)t->max_entries);
    return HRPP_CAPACITY;
  }
  if (e) {
    set_error("internal error %d in trace_wave", e);
    return HRPP_CUDA;
  }
  for (int k = 1; k < HRPP_STATS_LEN; k++)
    if (live_like || !(k == 4 || k == 5)) stats[k] += s[k];
  return HRPP_OK;
}

}  // extern "C"
