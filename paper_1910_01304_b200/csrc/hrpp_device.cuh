// hrpp_device.cuh -- device data layout and the bit-exact traversal core.
//
// Layout in HBM:
//   DNode  32 B  {float lo.xyz; a; float hi.xyz; b}: one 256-bit load per
//          visit (the reference's float32 boxes, exact in float64).
//          interior: a = left (>= 0), b = right | 1 << (27 + axis)
//          leaf:     a = ~first (< 0, so the reference's `left < 0` test
//                    becomes `a < 0`), b = count
//   DTri   96 B  {double v0.xyz, e1.xyz, e2.xyz; leaf}: the reference's
//          float64 vertex and edges (e = v - v0 rounded once, as it does per
//          test), two 256-bit loads and one 64-bit load.
//   (HRPP_BOX32=0 / HRPP_NODE_F64=0: the earlier float64-node and
//   float32-triangle layouts, kept for experiments.)
//
// Arithmetic restates hrpp/kernels.py:23-206 operation by operation: the
// slab test runs in float32 with a certified error margin and falls back to
// the reference's float64 test inside it (box_hit32); the triangle test is
// float64.  The whole library is compiled with --fmad=false so no
// multiply-add is contracted (numba emits none either), and double division
// is IEEE round-to-nearest, so results are bit-identical to the reference.
#pragma once
#include <cstdint>
#include <cstring>
#include <cuda_runtime.h>

namespace hrpp {

// HRPP_NODE_F64 (default 1): node boxes and triangle vertices are stored
// pre-widened to float64 (exact), so the traversal loop does no f32->f64
// conversions; 0 keeps the compact float32 records.
#ifndef HRPP_NODE_F64
#define HRPP_NODE_F64 1
#endif
#ifndef HRPP_OPAQUE_SIGNS
#define HRPP_OPAQUE_SIGNS 1
#endif
// HRPP_BOX32 (default 1): the slab test runs in float32 with a certified
// error margin and falls back to the reference's float64 test only when the
// float32 result is within the margin (see box_hit32).  Nodes are stored as
// 32-B float32 records (the reference's own bmin/bmax values, exact in
// float64); triangles stay pre-widened float64 (HRPP_NODE_F64).
#ifndef HRPP_BOX32
#define HRPP_BOX32 1
#endif
#ifndef HRPP_SLAB_MINMAX
#define HRPP_SLAB_MINMAX 1
#endif
#ifndef HRPP_LDG256
#define HRPP_LDG256 1
#endif



#if HRPP_NODE_F64 && !HRPP_BOX32
struct __align__(16) DNode {  // 64 B: four 16-B loads
  double lo[3], hi[3];
  int32_t a, b;
  int64_t pad;
};
#else
struct __align__(16) DNode {  // 32 B: two 16-B loads
  float bmin[3];
  int32_t a;
  float bmax[3];
  int32_t b;
};
#endif
#if HRPP_NODE_F64
struct __align__(32) DTri {  // 96 B: three 32-B loads
  double v[9];  // v0, then the edges e1 = v1 - v0, e2 = v2 - v0 in float64
                // (hrpp/kernels.py:60-65; the same rounding the reference does
                // per test, done once when the BVH is created)
  int32_t leaf;  // the leaf node whose slot range holds this slot (-1: none)
  int32_t pad[5];
};
#else
struct __align__(16) DTri {  // 48 B: three 16-B loads
  float4 p0, p1, p2;
};
#endif

// Host-side packing of the reference's arrays into the device records.
__host__ __device__ inline void pack_node(DNode& d, const float* lo, const float* hi, int32_t a,
                                          int32_t b) {
#if HRPP_NODE_F64 && !HRPP_BOX32
  for (int k = 0; k < 3; k++) {
    d.lo[k] = lo[k];
    d.hi[k] = hi[k];
  }
  d.a = a;
  d.b = b;
  d.pad = 0;
#else
  for (int k = 0; k < 3; k++) {
    d.bmin[k] = lo[k];
    d.bmax[k] = hi[k];
  }
  d.a = a;
  d.b = b;
#endif
}

__host__ __device__ inline void pack_tri(DTri& t, const float* a, const float* b, const float* c,
                                         int32_t leaf) {
#if HRPP_NODE_F64
  for (int k = 0; k < 3; k++) {
    t.v[k] = a[k];
    t.v[3 + k] = (double)b[k] - (double)a[k];
    t.v[6 + k] = (double)c[k] - (double)a[k];
  }
  t.leaf = leaf;
  for (int k = 0; k < 5; k++) t.pad[k] = 0;
#else
  t.p0 = make_float4(a[0], a[1], a[2], b[0]);
  t.p1 = make_float4(b[1], b[2], c[0], c[1]);
  float leaf_bits;
  memcpy(&leaf_bits, &leaf, sizeof(float));
  t.p2 = make_float4(c[2], leaf_bits, 0.f, 0.f);
#endif
}

// The leaf node holding slot k (leaf slot ranges are disjoint, checked when
// the BVH is created), so the traversal loop need not carry it.
__device__ __forceinline__ int32_t slot_leaf(const DTri* __restrict__ tris, int32_t k) {
#if HRPP_NODE_F64
  return __ldg(&tris[k].leaf);
#else
  return __float_as_int(__ldg(&tris[k].p2.y));
#endif
}

// Ray hash of one float (hrpp/rayhash.py:67-78, :118-122): sign, top p
// exponent bits, top p mantissa bits.
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

constexpr double kDetEps = 1e-9;          // hrpp/kernels.py:20
constexpr double kWrongClosestEps = 1e-9; // hrpp/tracer.py:52

// Traversal result.  The barycentrics (u, v) of the hit are not carried
// through the loop (4 registers): hit_uv recomputes them from the winning
// slot with the same arithmetic when an output needs them.
struct Hit {
  bool found;
  double t;
  int32_t slot, leaf;
  int32_t boxes, tris;  // per-ray counts are small; widened when stored
};

__device__ __forceinline__ double recip(double d) {
  // hrpp/kernels.py:97-99
  return d != 0.0 ? 1.0 / d : copysign(__longlong_as_double(0x7ff0000000000000LL), d);
}

struct NodeBox {
  double lx, ly, lz, hx, hy, hz;
  int32_t a, b;
};

__device__ __forceinline__ NodeBox load_node(const DNode* __restrict__ nodes, int32_t nd) {
  NodeBox n;
#if HRPP_NODE_F64 && !HRPP_BOX32
  const double2* p = reinterpret_cast<const double2*>(nodes + nd);
  const double2 q0 = __ldg(p), q1 = __ldg(p + 1), q2 = __ldg(p + 2);
  const int4 q3 = __ldg(reinterpret_cast<const int4*>(nodes + nd) + 3);
  n.lx = q0.x; n.ly = q0.y; n.lz = q1.x; n.hx = q1.y; n.hy = q2.x; n.hz = q2.y;
  n.a = q3.x;
  n.b = q3.y;
#else
  const float4* p = reinterpret_cast<const float4*>(nodes + nd);
  const float4 lo = __ldg(p), hi = __ldg(p + 1);
  n.lx = lo.x; n.ly = lo.y; n.lz = lo.z; n.hx = hi.x; n.hy = hi.y; n.hz = hi.z;
  n.a = __float_as_int(lo.w);
  n.b = __float_as_int(hi.w);
#endif
  return n;
}

// hrpp/kernels.py:23-51 (inclusive slab test; NaN compares are ignored)
__device__ __forceinline__ bool box_hit(const NodeBox& n, double ox, double oy, double oz,
                                        double ivx, double ivy, double ivz, double t0,
                                        double t1) {
  double tn = t0, tf = t1, a, b, s;
  a = (n.lx - ox) * ivx;
  b = (n.hx - ox) * ivx;
  if (ivx < 0.0) { s = a; a = b; b = s; }
  if (a > tn) tn = a;
  if (b < tf) tf = b;
  a = (n.ly - oy) * ivy;
  b = (n.hy - oy) * ivy;
  if (ivy < 0.0) { s = a; a = b; b = s; }
  if (a > tn) tn = a;
  if (b < tf) tf = b;
  a = (n.lz - oz) * ivz;
  b = (n.hz - oz) * ivz;
  if (ivz < 0.0) { s = a; a = b; b = s; }
  if (a > tn) tn = a;
  if (b < tf) tf = b;
  return tn <= tf;
}

// box_hit with the swap decisions (inv < 0 per axis) precomputed per ray as
// bits of `ivneg`: integer tests instead of three float64 compares per box.
__device__ __forceinline__ bool box_hit_s(const NodeBox& n, double ox, double oy, double oz,
                                          double ivx, double ivy, double ivz, uint32_t ivneg,
                                          double t0, double t1) {
  double tn = t0, tf = t1, a, b, s;
  a = (n.lx - ox) * ivx;
  b = (n.hx - ox) * ivx;
  if (ivneg & 1u) { s = a; a = b; b = s; }
  if (a > tn) tn = a;
  if (b < tf) tf = b;
  a = (n.ly - oy) * ivy;
  b = (n.hy - oy) * ivy;
  if (ivneg & 2u) { s = a; a = b; b = s; }
  if (a > tn) tn = a;
  if (b < tf) tf = b;
  a = (n.lz - oz) * ivz;
  b = (n.hz - oz) * ivz;
  if (ivneg & 4u) { s = a; a = b; b = s; }
  if (a > tn) tn = a;
  if (b < tf) tf = b;
  return tn <= tf;
}

// Triangle v0 and edges e1, e2 in float64 (the reference's values).
__device__ __forceinline__ void load_tri(const DTri* __restrict__ tris, int32_t k, double v[9]) {
#if HRPP_NODE_F64
  const double* p = reinterpret_cast<const double*>(tris + k);
  double w;  // the leaf / pad word
  asm("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];"
      : "=d"(v[0]), "=d"(v[1]), "=d"(v[2]), "=d"(v[3]) : "l"(p));
  asm("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];"
      : "=d"(v[4]), "=d"(v[5]), "=d"(v[6]), "=d"(v[7]) : "l"(p + 4));
  v[8] = __ldg(p + 8);
  (void)w;
#else
  const float4* p = reinterpret_cast<const float4*>(tris + k);
  const float4 q0 = __ldg(p), q1 = __ldg(p + 1), q2 = __ldg(p + 2);
  v[0] = q0.x; v[1] = q0.y; v[2] = q0.z; v[3] = q0.w; v[4] = q1.x; v[5] = q1.y;
  v[6] = q1.z; v[7] = q1.w; v[8] = q2.x;
  for (int k = 3; k < 9; k++) v[k] -= v[k % 3];
#endif
}

// hrpp/kernels.py:54-86 (Moller-Trumbore, |det| <= 1e-9 rejected)
__device__ __forceinline__ bool tri_test(const DTri* __restrict__ tris, int32_t k, double ox,
                                         double oy, double oz, double dx, double dy, double dz,
                                         double& t, double& u, double& v) {
  double q[9];
  load_tri(tris, k, q);
  double ax = q[0], ay = q[1], az = q[2];
  double e1x = q[3], e1y = q[4], e1z = q[5];
  double e2x = q[6], e2y = q[7], e2z = q[8];
  double px = dy * e2z - dz * e2y;
  double py = dz * e2x - dx * e2z;
  double pz = dx * e2y - dy * e2x;
  double det = e1x * px + e1y * py + e1z * pz;
  if (fabs(det) <= kDetEps) return false;
  double inv_det = 1.0 / det;
  double tx = ox - ax, ty = oy - ay, tz = oz - az;
  double uu = (tx * px + ty * py + tz * pz) * inv_det;
  if (uu < 0.0 || uu > 1.0) return false;
  double qx = ty * e1z - tz * e1y;
  double qy = tz * e1x - tx * e1z;
  double qz = tx * e1y - ty * e1x;
  double vv = (dx * qx + dy * qy + dz * qz) * inv_det;
  if (vv < 0.0 || uu + vv > 1.0) return false;
  t = (e2x * qx + e2y * qy + e2z * qz) * inv_det;
  u = uu;
  v = vv;
  return true;
}

#if HRPP_BOX32
// The ray as the wave stores it (float32 O and D, exact in float64) plus its
// float32 slab-test constants; the float64 values the reference computes
// with are exact widenings of these (o, d) or recomputed on demand (1/d).
struct Ray {
  float ox, oy, oz, dx, dy, dz;
  float ivx, ivy, ivz;  // correctly rounded float32 1/d (signed inf for 0)
  float t0f;            // float32 tmin; +inf for rays outside the certified
                        // range (tn = +inf: every box test then runs in float64)
  double tmin, tmax;
};

// The certified range of box_hit32: every direction component is 0 or has a
// magnitude in [2^-60, 2^60] (1/d is finite, normal and not near overflow in
// float32), the origin is finite with magnitude < 2^60, tmin/tmax not NaN.
__device__ __forceinline__ bool dir_ok32(float d) {
  const float a = fabsf(d);
  return d == 0.0f || (a >= 0x1p-60f && a <= 0x1p60f);
}

__device__ __forceinline__ Ray make_ray(const float* __restrict__ O, const float* __restrict__ D,
                                        const double* __restrict__ tmin,
                                        const double* __restrict__ tmax, int64_t i) {
  Ray r;
  r.ox = O[3 * i]; r.oy = O[3 * i + 1]; r.oz = O[3 * i + 2];
  r.dx = D[3 * i]; r.dy = D[3 * i + 1]; r.dz = D[3 * i + 2];
  r.ivx = __frcp_rn(r.dx); r.ivy = __frcp_rn(r.dy); r.ivz = __frcp_rn(r.dz);
  r.tmin = tmin[i];
  r.tmax = tmax[i];
  const bool ok = dir_ok32(r.dx) && dir_ok32(r.dy) && dir_ok32(r.dz) &&
                  fabsf(r.ox) < 0x1p60f && fabsf(r.oy) < 0x1p60f && fabsf(r.oz) < 0x1p60f &&
                  r.tmin == r.tmin && r.tmax == r.tmax;
  r.t0f = ok ? (float)r.tmin : __int_as_float(0x7f800000);
  return r;
}

struct NodeBox32 {
  float lx, ly, lz, hx, hy, hz;
  int32_t a, b;
};

// One 256-bit load per node (sm_100 LDG.E.ENL2.256; records are 32-B aligned).
__device__ __forceinline__ NodeBox32 load_node32(const DNode* __restrict__ nodes, int32_t nd) {
  NodeBox32 n;
#if HRPP_LDG256
  float aw, bw;
  asm("ld.global.nc.v8.f32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
      : "=f"(n.lx), "=f"(n.ly), "=f"(n.lz), "=f"(aw), "=f"(n.hx), "=f"(n.hy), "=f"(n.hz),
        "=f"(bw)
      : "l"(nodes + nd));
  n.a = __float_as_int(aw);
  n.b = __float_as_int(bw);
#else
  const float4* p = reinterpret_cast<const float4*>(nodes + nd);
  const float4 lo = __ldg(p), hi = __ldg(p + 1);
  n.lx = lo.x; n.ly = lo.y; n.lz = lo.z; n.hx = hi.x; n.hy = hi.y; n.hz = hi.z;
  n.a = __float_as_int(lo.w);
  n.b = __float_as_int(hi.w);
#endif
  return n;
}

// The reference's float64 slab test (hrpp/kernels.py:23-51) on the same
// node and ray, every float64 value rebuilt exactly (widenings of the
// float32 inputs, 1/d recomputed as the reference does).  Out of line: it
// runs only for the rare box tests box_hit32 cannot certify.
static __device__ __noinline__ bool box_hit_exact(float lx, float ly, float lz, float hx, float hy,
                                           float hz, float ox, float oy, float oz, float dx,
                                           float dy, float dz, double t0, double t1) {
  NodeBox n;
  n.lx = lx; n.ly = ly; n.lz = lz; n.hx = hx; n.hy = hy; n.hz = hz;
  return box_hit(n, ox, oy, oz, recip(dx), recip(dy), recip(dz), t0, t1);
}

// Slab test in float32 with a certified decision.
//
// For a ray in the certified range each float32 slab value a = (lo - o) * iv
// is within 3u|a| (u = 2^-24: one rounding in the subtraction of exact
// float32 inputs, one in the correctly rounded reciprocal, one in the
// product) of the real value, and the reference's float64 value within
// 3*2^-53|a|; infinities and NaNs (zero direction components) arise
// identically in both.  max/min of such values keep the bound relative to
// the result, so with tn, tf the float32 entry/exit and s = |tn| + |tf|:
//   |(tf - tn) - (tf64 - tn64)| <= ~4u s + 2^-149 (underflow)  <  m,
//   m = 2^-18 s + 2^-126.
// So d = tf - tn > m certifies tn64 <= tf64 (hit) and d < -m certifies a
// miss; anything else -- including every inf/NaN in d or m, and every test
// of a ray outside the certified range (t0f = +inf makes tn = +inf, so d is
// -inf or NaN and m is inf or NaN) -- is decided by the
// float64 test.  The result is therefore always the reference's.
__device__ __forceinline__ bool box_hit32(const NodeBox32& n, const Ray& r, uint32_t ivneg,
                                          float t1f, double t1) {
#if HRPP_SLAB_MINMAX
  // Slab entry/exit by min/max instead of swapping on the sign of 1/d: the
  // same values whenever no slab value is NaN (rounding is monotone, so the
  // smaller of the two is the one the swap picks); with a NaN (d = 0 and the
  // origin on that slab plane) the two differ only by putting an infinity
  // into tn or tf, which sends the test to the float64 path below.
  (void)ivneg;
  const float lx = (n.lx - r.ox) * r.ivx, hx = (n.hx - r.ox) * r.ivx;
  const float ly = (n.ly - r.oy) * r.ivy, hy = (n.hy - r.oy) * r.ivy;
  const float lz = (n.lz - r.oz) * r.ivz, hz = (n.hz - r.oz) * r.ivz;
  const float tn = fmaxf(fmaxf(r.t0f, fminf(lx, hx)), fmaxf(fminf(ly, hy), fminf(lz, hz)));
  const float tf = fminf(fminf(t1f, fmaxf(lx, hx)), fminf(fmaxf(ly, hy), fmaxf(lz, hz)));
#else
  const float nx = (ivneg & 1u) ? n.hx : n.lx, fx = (ivneg & 1u) ? n.lx : n.hx;
  const float ny = (ivneg & 2u) ? n.hy : n.ly, fy = (ivneg & 2u) ? n.ly : n.hy;
  const float nz = (ivneg & 4u) ? n.hz : n.lz, fz = (ivneg & 4u) ? n.lz : n.hz;
  const float ax = (nx - r.ox) * r.ivx, bx = (fx - r.ox) * r.ivx;
  const float ay = (ny - r.oy) * r.ivy, by = (fy - r.oy) * r.ivy;
  const float az = (nz - r.oz) * r.ivz, bz = (fz - r.oz) * r.ivz;
  const float tn = fmaxf(fmaxf(r.t0f, ax), fmaxf(ay, az));
  const float tf = fminf(fminf(t1f, bx), fminf(by, bz));
#endif
  const float d = tf - tn;
  const float m = __fmaf_ru(fabsf(tn) + fabsf(tf), 0x1p-18f, 0x1p-126f);
  if (d > m) return true;
  if (d < -m) return false;
  return box_hit_exact(n.lx, n.ly, n.lz, n.hx, n.hy, n.hz, r.ox, r.oy, r.oz, r.dx, r.dy, r.dz,
                       r.tmin, t1);
}
#else
struct Ray {
  double ox, oy, oz, dx, dy, dz, ivx, ivy, ivz, tmin, tmax;
};

__device__ __forceinline__ Ray make_ray(const float* __restrict__ O, const float* __restrict__ D,
                                        const double* __restrict__ tmin,
                                        const double* __restrict__ tmax, int64_t i) {
  Ray r;
  r.ox = O[3 * i]; r.oy = O[3 * i + 1]; r.oz = O[3 * i + 2];
  r.dx = D[3 * i]; r.dy = D[3 * i + 1]; r.dz = D[3 * i + 2];

  r.ivx = recip(r.dx); r.ivy = recip(r.dy); r.ivz = recip(r.dz);
  r.tmin = tmin[i];
  r.tmax = tmax[i];
  return r;
}
#endif

// Per-thread traversal stack in local memory.  (A shared-memory column per
// thread measured 8-15 % slower: it takes L1 capacity from the node reads.)
template <int STACK>
struct LocalStack {
  int32_t s[STACK];
  __device__ __forceinline__ int32_t& operator[](int i) { return s[i]; }
};

// trace_closest / trace_any from `start` (hrpp/kernels.py:89-206).
// Traversal order: pop, count visit + box test, leaf = slots [first,
// first+count) in order, interior pushes far then near (near = left iff
// d[axis] >= 0, so -0.0 goes left).
template <bool CLOSEST, typename Stack>
__device__ __forceinline__ Hit trace_stk(const DNode* __restrict__ nodes,
                                         const DTri* __restrict__ tris, const Ray& r,
                                         int32_t start, Stack& stack) {
  // The reference pushes far then near and pops near next; visiting the near
  // child directly (only far goes to the stack) is the same visit order with
  // one local-memory store and load less per interior node.
  // Only slot and t live in the loop: found = slot >= 0 and the leaf is
  // read from the slot's triangle record at the end.
  int top = 0;
  int32_t nd = start;
  // d[axis] < 0 per axis (bit axis): the near child is the right one
#if HRPP_BOX32
  // bits 0-2: 1/d < 0 per axis (slab swap); bits 3-5: d < 0 (near child right)
  uint32_t ivneg = (r.ivx < 0.0f ? 1u : 0u) | (r.ivy < 0.0f ? 2u : 0u) |
                   (r.ivz < 0.0f ? 4u : 0u) | (r.dx >= 0.0f ? 0u : 8u) |
                   (r.dy >= 0.0f ? 0u : 16u) | (r.dz >= 0.0f ? 0u : 32u);
#else
  const uint32_t dneg = (r.dx >= 0.0 ? 0u : 1u) | (r.dy >= 0.0 ? 0u : 2u) |
                        (r.dz >= 0.0 ? 0u : 4u);
  uint32_t ivneg = (r.ivx < 0.0 ? 1u : 0u) | (r.ivy < 0.0 ? 2u : 0u) |
                   (r.ivz < 0.0 ? 4u : 0u);
#endif
#if HRPP_OPAQUE_SIGNS
  asm volatile("mov.u32 %0, %0;" : "+r"(ivneg));  // keep the bits, not 3 float64 compares
#endif
  // d[axis] < 0 at bit 27 + axis, matching the interior nodes' axis bit
#if HRPP_BOX32
  const uint32_t dmask = (ivneg & 0x38u) << 24;
#else
  const uint32_t dmask = dneg << 27;
#endif
  // h.t starts at tmax for both kinds: the closest-hit box interval is
  // [tmin, best t] and a hit needs t <= tmax before the first hit and
  // t < best t after it; an any-hit ray's interval stays [tmin, tmax] until
  // its first hit ends the traversal.  So tmax itself is not live here.
  Hit h;
  h.t = r.tmax;
  h.slot = -1;
  h.boxes = 0;
  h.tris = 0;
#if HRPP_BOX32
  float t1f = (float)h.t;  // float32 copy of the interval end for box_hit32
#endif
  for (;;) {
    h.boxes++;
#if HRPP_BOX32
    const NodeBox32 nb = load_node32(nodes, nd);
    if (box_hit32(nb, r, ivneg, t1f, h.t)) {
#else
    const NodeBox nb = load_node(nodes, nd);
    if (box_hit_s(nb, r.ox, r.oy, r.oz, r.ivx, r.ivy, r.ivz, ivneg, r.tmin, h.t)) {
#endif
      const int32_t a = nb.a;
      const int32_t b = nb.b;
      if (a >= 0) {
        // b = right | 1 << (27 + axis): one AND against the ray's sign mask
        const int32_t right = b & 0x07FFFFFF;
        const bool go_right = ((uint32_t)b & dmask) != 0u;
        stack[top++] = go_right ? a : right;  // far
        nd = go_right ? right : a;             // near, visited next
        continue;
      }
      const int32_t f = ~a, e = f + b;
#pragma unroll 1
      for (int32_t k = f; k < e; k++) {
        double t, u, v;
        h.tris++;
#if HRPP_BOX32
        // widen the ray inside the leaf loop (opaque, so the compiler does not
        // keep float64 copies of o and d live across the whole traversal)
        float fo[3] = {r.ox, r.oy, r.oz}, fd[3] = {r.dx, r.dy, r.dz};
#pragma unroll
        for (int c = 0; c < 3; c++) {
          asm volatile("mov.b32 %0, %0;" : "+f"(fo[c]));
          asm volatile("mov.b32 %0, %0;" : "+f"(fd[c]));
        }
        if (tri_test(tris, k, fo[0], fo[1], fo[2], fd[0], fd[1], fd[2], t, u, v) &&
            t >= r.tmin &&
#else
        if (tri_test(tris, k, r.ox, r.oy, r.oz, r.dx, r.dy, r.dz, t, u, v) && t >= r.tmin &&
#endif
            (h.slot < 0 ? t <= h.t : t < h.t)) {
          h.t = t;
#if HRPP_BOX32
          t1f = (float)t;
#endif
          h.slot = k;
          if (!CLOSEST) {
            top = 0;
            break;
          }
        }
      }
      if (!CLOSEST && h.slot >= 0) break;
    }
    if (top == 0) break;
    nd = stack[--top];
  }
  h.found = h.slot >= 0;
  if (!CLOSEST && !h.found) h.t = 0.0;  // trace_any's miss (hrpp/kernels.py:206)
  h.leaf = h.found ? slot_leaf(tris, h.slot) : -1;
  return h;
}

template <bool CLOSEST, int STACK>
__device__ __forceinline__ Hit trace_from(const DNode* __restrict__ nodes,
                                          const DTri* __restrict__ tris, const Ray& r,
                                          int32_t start) {
  LocalStack<STACK> st;
  return trace_stk<CLOSEST>(nodes, tris, r, start, st);
}

// One step of eval_entry_{closest,any} (hrpp/kernels.py:251-297): fold the
// subtree result of the next stored node into the running entry result.
template <bool CLOSEST>
__device__ __forceinline__ void fold_entry(Hit& acc, const Hit& r) {
  acc.boxes += r.boxes;
  acc.tris += r.tris;
  if (r.found && (!acc.found || (CLOSEST && r.t < acc.t))) {
    acc.found = true; acc.t = r.t; acc.slot = r.slot; acc.leaf = r.leaf;
  }
}

// (u, v) of h's triangle: the reference's values, recomputed (0, 0 on a miss).
__device__ __forceinline__ void hit_uv(const DTri* __restrict__ tris, const Ray& r, const Hit& h,
                                       double& u, double& v) {
  u = 0.0;
  v = 0.0;
  if (h.found) {
    double t;
    tri_test(tris, h.slot, r.ox, r.oy, r.oz, r.dx, r.dy, r.dz, t, u, v);
  }
}

__device__ __forceinline__ Hit empty_entry_result(bool closest) {
  Hit h;
  h.found = false;
  h.t = closest ? __longlong_as_double(0x7ff0000000000000LL) : 0.0;
  h.slot = -1; h.leaf = -1; h.boxes = 0; h.tris = 0;
  return h;
}

// Predictor table hash index (open addressing, linear probing).
constexpr unsigned long long kEmptyKey = ~0ull;

__device__ __forceinline__ uint64_t mix64(uint64_t x) {
  x ^= x >> 33; x *= 0xff51afd7ed558ccdULL; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ULL;
  x ^= x >> 33;
  return x;
}

// One 16-B bucket per probe: {key, entry id}.
struct __align__(16) Bucket {
  unsigned long long key;
  int32_t val;
  int32_t pad;
};

__device__ __forceinline__ int32_t index_lookup(const Bucket* __restrict__ idx, uint64_t mask,
                                                uint64_t key) {
  uint64_t h = mix64(key) & mask;
  for (;;) {
    const ulonglong2 b = *reinterpret_cast<const ulonglong2*>(idx + h);
    if (b.x == key) return (int32_t)(b.y & 0xffffffffull);
    if (b.x == kEmptyKey) return -1;
    h = (h + 1) & mask;
  }
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

}  // namespace hrpp
