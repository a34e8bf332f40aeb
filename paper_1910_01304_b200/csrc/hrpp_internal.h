// hrpp_internal.h -- host-side structures shared by the library's .cu files.
#pragma once
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <map>
#include <string>
#include <vector>

#include "hrpp_device.cuh"

namespace hrpp {

extern std::atomic<int64_t> g_launches;
void set_error(const char* fmt, ...);

#define HRPP_CK(call)                                                                   \
  do {                                                                                  \
    cudaError_t e_ = (call);                                                            \
    if (e_ != cudaSuccess) {                                                            \
      ::hrpp::set_error("%s:%d: %s -> %s", __FILE__, __LINE__, #call,                   \
                        cudaGetErrorString(e_));                                        \
      return 4;                                                                         \
    }                                                                                   \
  } while (0)

#define HRPP_LAUNCHED()                                                                 \
  do {                                                                                  \
    ::hrpp::g_launches.fetch_add(1, std::memory_order_relaxed);                         \
    cudaError_t e_ = cudaGetLastError();                                                \
    if (e_ != cudaSuccess) {                                                            \
      ::hrpp::set_error("%s:%d: kernel launch -> %s", __FILE__, __LINE__,               \
                        cudaGetErrorString(e_));                                        \
      return 4;                                                                         \
    }                                                                                   \
  } while (0)

// Grow-only scratch buffers (contents are not preserved across growth).
struct Workspace {
  struct Buf {
    void* p = nullptr;
    size_t bytes = 0;
  };
  std::map<std::string, Buf> bufs;
  int device = 0;
  ~Workspace();
  int get_raw(const char* name, size_t bytes, void** out);
  template <typename T>
  int get(const char* name, size_t count, T** out) {
    void* p = nullptr;
    int rc = get_raw(name, count * sizeof(T) + 16, &p);
    *out = static_cast<T*>(p);
    return rc;
  }
};

// Scratch of calls without a table: one per host thread and CUDA device
// (the current one), so neither threads nor devices share buffers.
Workspace& device_ws();

// Result arrays of a traversal (any pointer may be null = not stored).
struct TraceOut {
  uint8_t* found = nullptr;
  double* t = nullptr;
  int32_t* slot = nullptr;
  int32_t* leaf = nullptr;
  double* u = nullptr;
  double* v = nullptr;
  int64_t* box = nullptr;
  int64_t* tri = nullptr;
  int64_t* vis = nullptr;
  uint8_t* known = nullptr;               // set to 1 for every traced ray
  unsigned long long* sums = nullptr;     // [0] += boxes, [1] += tris
  int32_t* box32 = nullptr;               // per-ray counts, 32-bit (live mode)
  int32_t* tri32 = nullptr;
  bool zero_miss_t = false;               // t = 0 on a miss (live-mode outputs)
  // live consult hook: a traced ray that hits a node not yet in its key's
  // wave-start entry bids (atomicMin) to be its segment's first append
  const int32_t* fa_seg_of_ray = nullptr;
  const int64_t* fa_exoff = nullptr;
  const int32_t* fa_exlen = nullptr;
  const int32_t* fa_arena = nullptr;
  const int32_t* fa_anc = nullptr;
  int32_t* fa_f1 = nullptr;
};

struct BvhDev {
  int device = 0;
  DNode* nodes = nullptr;
  DTri* tris = nullptr;
  int32_t* depth = nullptr;
  int32_t* tri_ids = nullptr;
  int64_t n_nodes = 0, n_tris = 0;
  int height = 0;      // longest root-to-leaf edge count (stack bound)
  float root_lo[3] = {0, 0, 0}, root_hi[3] = {1, 1, 1};  // scene bounds (coherence keys)
  int stack = 64;      // template stack size chosen from height
  std::vector<int32_t> parent_host;
  std::map<int, int32_t*> anc;  // go-up level -> device LUT
  ~BvhDev();
  int ancestor_lut(int level, const int32_t** out);
};

struct TableDev {
  int device = 0;
  int precision = 6, go_up = 0;
  bool closest = true;
  int64_t max_entries = 1 << 26;
  // hash index: key -> entry id
  Bucket* idx = nullptr;
  int64_t idx_cap = 0;
  // entries (creation order), node lists in the arena
  unsigned long long* e_key = nullptr;
  int64_t* e_off = nullptr;
  int32_t* e_len = nullptr;
  int64_t e_cap = 0;
  int32_t* arena = nullptr;
  int64_t arena_cap = 0;
  // device meta: [0] entries, [1] stored, [2] arena_used, [3] pending records
  long long* meta = nullptr;
  // host mirrors (exact after every call returns)
  int64_t n_entries = 0, stored = 0, arena_used = 0;
  // deferred mode (multi-GPU): a wave does not commit; its append records
  // (key, node, ray index) wait in ws "p_keys"/"p_nodes"/"p_rays", sorted by ray
  bool deferred = false;
  int64_t pending = 0;
  double start_tp_frac = 1.0;  // wave-start TP fraction of the last live wave
  double empty_tp_frac = -1.0;  // TP fraction of the last live wave that started on an empty table
  bool wave_started_empty = false;
  int64_t fast_wcap = 0;  // fast mode: initialised wave-slot capacity
  // stream-ordered clear: every later call on the table waits for it
  cudaEvent_t clear_ev = nullptr;
  bool clear_recorded = false;
  cudaError_t wait_clear(cudaStream_t st) {
    return clear_recorded ? cudaStreamWaitEvent(st, clear_ev, 0) : cudaSuccess;
  }
  Workspace ws;
  ~TableDev();
  // capacity for up to extra_entries new entries and extra_nodes new nodes
  int reserve(int64_t extra_entries, int64_t extra_nodes, cudaStream_t st);
};

// ---- launchers (return HRPP status) ----
// ib > 0: store (packed key << ib) | ray index, the grouping sort's word
int launch_hash(const float* O, const float* D, int64_t n, int p, uint64_t* keys, int* err,
                cudaStream_t st, int ib = 0);
int launch_coarsen(const uint64_t* keys, int64_t n, int p, uint64_t* out, cudaStream_t st);
int launch_hash_floats(const float* f, int64_t n, int p, uint32_t* out, int* err,
                       cudaStream_t st);
// Traces n rays (or the device-counted queue ray_idx[0..*count_dev)), one
// ray per thread.
int launch_trace(const BvhDev& b, bool closest, const float* O, const float* D,
                 const double* tmin, const double* tmax, int32_t start, int64_t n,
                 const int32_t* ray_idx, const int* count_dev, const TraceOut& out,
                 const int* err, cudaStream_t st, Workspace* ws = nullptr,
                 bool fallback = false);  // fallback: profiled as the live fallback traversal

// Group a batch of keys: stable sort (key, ray) and find key segments.
struct Segments {
  unsigned long long* skeys = nullptr;  // 48-bit keys; valid at segment heads
  int32_t* sidx = nullptr;
  int32_t* seg_start = nullptr;  // nsegs + 1 entries (device count)
  int* nsegs = nullptr;          // device scalar
  int32_t* seg_id = nullptr;     // per sorted position: segment index + 1
};
// lane_bits = 1 + 2p for hash keys (sorted on their 3(1+2p) used bits), 0 for
// arbitrary 64-bit keys.
int group_by_key(Workspace& ws, const uint64_t* keys, int64_t n, int lane_bits, Segments* seg,
                 cudaStream_t st, int* nsegs_mapped = nullptr, bool prepacked = false);
// indices i < n with flags[i] != 0, ascending, count to *count_dev
int compact_flags(Workspace& ws, const uint8_t* flags, int64_t n, int32_t* out, int* count_dev,
                  cudaStream_t st);
extern int g_consult_short;
// values[i] for i < n with flags[i] != 0, in order, count to *count_dev
int compact_by_flags(Workspace& ws, const int32_t* values, const uint8_t* flags, int64_t n,
                     int32_t* out, int* count_dev, cudaStream_t st);

struct Consult {
  bool live = false;
  const float* O = nullptr;
  const float* D = nullptr;
  const double* tmin = nullptr;
  const double* tmax = nullptr;
  int64_t n = 0;
  // per-ray baseline (limit) results
  const uint8_t* base_found = nullptr;
  const double* base_t = nullptr;
  const int32_t* base_leaf = nullptr;
  const int64_t* base_box = nullptr;
  // live outputs
  uint8_t* o_found = nullptr;
  double* o_t = nullptr;
  int32_t* o_slot = nullptr;
  int32_t* o_leaf = nullptr;
  // limit log
  int8_t* log_cls = nullptr;
  int64_t* log_eval_box = nullptr;
  double* log_pred_t = nullptr;
  int64_t* log_pred_slot = nullptr;
};

// Runs the ray-ordered per-key consult of one wave and commits the table.
// stats_dev: unsigned long long[16] device (RayKindStats order).
int run_consult(const BvhDev& b, TableDev& t, const Consult& c, const uint64_t* keys,
                unsigned long long* stats_dev, int* err, cudaStream_t st, bool prepacked = false);
int table_record(TableDev& t, const uint64_t* keys, const int32_t* nodes, int64_t n,
                 uint8_t* inserted, int* err, cudaStream_t st);
int table_commit(TableDev& t, const Segments& seg, int64_t n, int32_t* seg_eid,
                 int32_t* seg_napp, const int32_t* app, int* err, cudaStream_t st,
                 const int32_t* seg_cursor = nullptr);
int table_collect_pending(TableDev& t, const Segments& seg, int64_t n, const int32_t* seg_napp,
                          const int32_t* app, const int32_t* app_ray, int* err,
                          cudaStream_t st);
int table_export(TableDev& t, uint64_t* keys_h, int64_t* offs_h, int32_t* nodes_h);
int table_max_len(TableDev& t, int64_t* out);
int table_lookup1(TableDev& t, uint64_t key, int32_t* nodes_h, int64_t cap, int64_t* len);
int predict_batch(const BvhDev& b, TableDev& t, const uint64_t* keys, const float* O,
                  const float* D, const double* tmin, const double* tmax, int64_t n,
                  int8_t* cls, double* tt, int32_t* slot, int32_t* leaf, double* u, double* v,
                  int64_t* box, int64_t* tri, int64_t* vis, int64_t* est, cudaStream_t st);

// Small device->host reads without a copy engine: a one-block kernel stores
// into this host thread's pinned buffer (UVA-mapped), then the caller syncs
// the stream.  Large user copies keep the DMA engines to themselves, so a
// 4-byte readback never queues behind a 100-MB upload or download.
long long* pinned_scratch();  // 64 entries; [32, 64) free for kernels' use
int to_host(void* pinned_dst, const void* dev_src, size_t bytes, cudaStream_t st);
// Small host->device values as kernel arguments (no copy engine either).
int set_i32(int32_t* dst, int32_t v, cudaStream_t st);
int set_i64(long long* dst, long long v, cudaStream_t st);

extern int g_live_rounds;

// Fast mode (k_fast.cu): the wave's rays and outputs (device pointers).
struct FastIO {
  const float* O;
  const float* D;
  const double* tmin;
  const double* tmax;
  int64_t n;
  uint8_t* found;
  double* t;
  int32_t* slot;
  int32_t* leaf;
  uint64_t* keys;
};
extern int g_fast_rounds, g_fast_stop_div;
int run_fast(const BvhDev& b, TableDev& t, const FastIO& io, unsigned long long* stats_dev,
             int* err, cudaStream_t st);

inline int grid_for(int64_t n, int block, int max_blocks) {
  int64_t g = (n + block - 1) / block;
  if (g < 1) g = 1;
  if (g > max_blocks) g = max_blocks;
  return (int)g;
}

int num_sms();

// ---- optional per-stage CUDA-event profiler (hrpp_profile_*) ----
enum ProfCat { P_HASH = 0, P_TRACE, P_TRACE_QUEUE, P_GROUP, P_CONSULT, P_COMMIT, P_OTHER, P_NCAT };
extern bool g_prof_on;
struct ProfScope {
  int cat;
  cudaStream_t st;
  cudaEvent_t a = nullptr, b = nullptr;
  ProfScope(int c, cudaStream_t s);
  ~ProfScope();
};
void prof_flush();

}  // namespace hrpp
