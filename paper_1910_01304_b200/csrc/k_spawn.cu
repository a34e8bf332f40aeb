// k_spawn.cu -- ray waves generated and spawned on the device, so waves
// never leave HBM between bounces.
//
//  k_gen_primary  restates generate_primary_rays (hrpp/tracer.py:173-211)
//                 with the counter RNG unit_floats (hrpp/rng.py:15-31):
//                 pixel-major / sample-minor, stratified jitter, float64
//                 arithmetic in numpy's order, no FMA -> bit-identical rays.
//  k_spawn        hit points offset 1e-4 along the geometric normal flipped
//                 to face the ray (hrpp/tracer.py:442-453), then
//                 * shadow rays to a point light (hrpp/tracer.py:456-464) or
//                   to uniform samples of a y-facing square area light;
//                 * mirror bounces (hrpp/tracer.py:488-492) or
//                   cosine-weighted diffuse bounces.
//                 Point-light shadows and mirror bounces are bit-identical
//                 to the reference renderer's numpy arithmetic; area-light
//                 and diffuse spawns (absent from the reference) are
//                 bit-identical to this repo's host generators
//                 (scenes.area_light_samples, scenes.cosine_bounce).
#include <cub/cub.cuh>

#include "../../include/hrpp_b200.h"
#include "hrpp_internal.h"

namespace hrpp {

__device__ __forceinline__ uint64_t rng_mix(uint64_t x) {
  x ^= x >> 30;
  x *= 0xBF58476D1CE4E5B9ull;
  x ^= x >> 27;
  x *= 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

// hrpp/rng.py:23-31
__device__ __forceinline__ double unit_float(uint64_t seed, uint64_t pixel, uint64_t sample,
                                             uint64_t dim) {
  const uint64_t G = 0x9E3779B97F4A7C15ull, M1 = 0xBF58476D1CE4E5B9ull,
                 M2 = 0x94D049BB133111EBull;
  uint64_t h = rng_mix(seed + G);
  h = rng_mix(h ^ (pixel * G + 1ull));
  h = rng_mix(h ^ (sample * M1 + dim * M2 + 1ull));
  return (double)(h >> 11) * 1.1102230246251565e-16;  // 2**-53
}

struct PrimaryArgs {
  float pos[3];
  double fwd[3], right[3], up[3];
  double tan_half, tan_aspect;  // tan_half, tan_half * aspect
  int64_t w, h, spp, sx, sy;
  uint64_t seed;
  int jitter;
  int64_t n;
  float* O;
  float* D;
};

__global__ void k_gen_primary(PrimaryArgs a) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < a.n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t pixel = (uint64_t)i / (uint64_t)a.spp;
    const uint64_t sample = (uint64_t)i % (uint64_t)a.spp;
    const double px = (double)(pixel % (uint64_t)a.w);
    const double py = (double)(pixel / (uint64_t)a.w);
    double offx = 0.5, offy = 0.5;
    if (a.jitter) {
      const double six = (double)(sample % (uint64_t)a.sx);
      const double siy = (double)(sample / (uint64_t)a.sx);
      offx = (six + unit_float(a.seed, pixel, sample, 0)) / (double)a.sx;
      offy = (siy + unit_float(a.seed, pixel, sample, 1)) / (double)a.sy;
    }
    const double ndc_x = ((px + offx) / (double)a.w) * 2.0 - 1.0;
    const double ndc_y = 1.0 - ((py + offy) / (double)a.h) * 2.0;
    double d[3];
    for (int k = 0; k < 3; k++)
      d[k] = (a.fwd[k] + (ndc_x * a.tan_aspect) * a.right[k]) + (ndc_y * a.tan_half) * a.up[k];
    const double nrm = sqrt((d[0] * d[0] + d[1] * d[1]) + d[2] * d[2]);
    for (int k = 0; k < 3; k++) {
      a.D[3 * i + k] = (float)(d[k] / nrm);
      a.O[3 * i + k] = a.pos[k];
    }
  }
}

struct SpawnArgs {
  const float* O;
  const float* D;
  const uint8_t* found;
  const double* t;
  const int32_t* slot;
  const DTri* tris;
  const int32_t* pos;  // compacted hit index -> ray index
  const int* count;
  int shadow_kind;     // 0 none, 1 point light, 2 area light
  double light[3];
  double half;         // area light half extent
  int bounce_kind;     // 0 none, 1 mirror, 2 diffuse
  uint64_t seed;
  float *so, *sd;
  double *s0, *s1;
  float *bo, *bd;
  double *b0, *b1;
};

// (cos, sin) of 2 pi u, u in [0, 1): scenes.cos_sin_turn's plain float64
// operations in the same order (no FMA: the library is built with
// --fmad=false), so diffuse bounces match the host generator bit for bit.
__device__ __forceinline__ void cos_sin_turn(double u, double* cs, double* sn) {
  const double x = 4.0 * u;
  const double q = floor(x);
  const double t = (x - q) * 1.5707963267948966;
  const double t2 = t * t;
  const double S[8] = {-1.0 / 6, 1.0 / 120, -1.0 / 5040, 1.0 / 362880, -1.0 / 39916800,
                       1.0 / 6227020800, -1.0 / 1307674368000, 1.0 / 355687428096000};
  const double C[8] = {-1.0 / 2, 1.0 / 24, -1.0 / 720, 1.0 / 40320, -1.0 / 3628800,
                       1.0 / 479001600, -1.0 / 87178291200, 1.0 / 20922789888000};
  double s = S[7], c = C[7];
#pragma unroll
  for (int k = 6; k >= 0; k--) {
    s = S[k] + t2 * s;
    c = C[k] + t2 * c;
  }
  s = t * (1.0 + t2 * s);
  c = 1.0 + t2 * c;
  switch ((int)q & 3) {
    case 0: *cs = c; *sn = s; break;
    case 1: *cs = -s; *sn = c; break;
    case 2: *cs = -c; *sn = -s; break;
    default: *cs = s; *sn = -c; break;
  }
}

__global__ void k_spawn(SpawnArgs a) {
  const int m = *a.count;
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < m;
       j += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = a.pos[j];
    double o[3], d[3];
    for (int k = 0; k < 3; k++) {
      o[k] = a.O[3 * i + k];
      d[k] = a.D[3 * i + k];
    }
    const double t = a.t[i];
    double P[3];
    for (int k = 0; k < 3; k++) P[k] = o[k] + t * d[k];
    // geometric normal of the slot (Bvh.slot_normals, hrpp/bvh.py:130-138)
    double q[9];
    load_tri(a.tris, a.slot[i], q);
    // q = v0, e1 = v1 - v0, e2 = v2 - v0 (float64, as load_tri returns them)
    const double e1[3] = {q[3], q[4], q[5]};
    const double e2[3] = {q[6], q[7], q[8]};
    double N[3];
    N[0] = e1[1] * e2[2] - e1[2] * e2[1];
    N[1] = e1[2] * e2[0] - e1[0] * e2[2];
    N[2] = e1[0] * e2[1] - e1[1] * e2[0];
    const double nn = sqrt((N[0] * N[0] + N[1] * N[1]) + N[2] * N[2]);
    for (int k = 0; k < 3; k++) N[k] /= nn;
    const double facing = (N[0] * d[0] + N[1] * d[1]) + N[2] * d[2];
    if (facing > 0.0)
      for (int k = 0; k < 3; k++) N[k] = -N[k];
    double op[3];
    for (int k = 0; k < 3; k++) op[k] = P[k] + 1e-4 * N[k];
    if (a.shadow_kind) {
      double lp[3] = {a.light[0], a.light[1], a.light[2]};
      if (a.shadow_kind == 2) {
        const double u = unit_float(a.seed, (uint64_t)j, 0, 10);
        const double v = unit_float(a.seed, (uint64_t)j, 0, 11);
        lp[0] = a.light[0] + (2.0 * u - 1.0) * a.half;
        lp[2] = a.light[2] + (2.0 * v - 1.0) * a.half;
      }
      double lv[3];
      for (int k = 0; k < 3; k++) lv[k] = lp[k] - op[k];
      double dist = sqrt((lv[0] * lv[0] + lv[1] * lv[1]) + lv[2] * lv[2]);
      dist = dist > 1e-9 ? dist : 1e-9;
      for (int k = 0; k < 3; k++) {
        a.so[3 * j + k] = (float)op[k];
        a.sd[3 * j + k] = (float)(lv[k] / dist);
      }
      const double tm = dist - 1e-4;
      a.s0[j] = 0.0;
      a.s1[j] = tm > 1e-6 ? tm : 1e-6;
    }
    if (a.bounce_kind == 1) {  // mirror
      const double rdot = (d[0] * N[0] + d[1] * N[1]) + d[2] * N[2];
      double rd[3];
      for (int k = 0; k < 3; k++) rd[k] = d[k] - (2.0 * rdot) * N[k];
      const double rn = sqrt((rd[0] * rd[0] + rd[1] * rd[1]) + rd[2] * rd[2]);
      for (int k = 0; k < 3; k++) {
        a.bo[3 * j + k] = (float)op[k];
        a.bd[3 * j + k] = (float)(rd[k] / rn);
      }
      a.b0[j] = 0.0;
      a.b1[j] = __longlong_as_double(0x7ff0000000000000LL);
    } else if (a.bounce_kind == 2) {  // cosine-weighted about N
      const double u1 = unit_float(a.seed, (uint64_t)j, 0, 20);
      const double u2 = unit_float(a.seed, (uint64_t)j, 0, 21);
      const double rr = sqrt(u1);
      double sphi, cphi;
      cos_sin_turn(u2, &cphi, &sphi);
      const double lx = rr * cphi, ly = rr * sphi, lz = sqrt(fmax(0.0, 1.0 - u1));
      double ax[3] = {1.0, 0.0, 0.0};
      if (fabs(N[0]) > 0.9) {
        ax[0] = 0.0;
        ax[1] = 1.0;
      }
      double tx[3] = {N[1] * ax[2] - N[2] * ax[1], N[2] * ax[0] - N[0] * ax[2],
                      N[0] * ax[1] - N[1] * ax[0]};
      const double tn = sqrt((tx[0] * tx[0] + tx[1] * tx[1]) + tx[2] * tx[2]);
      for (int k = 0; k < 3; k++) tx[k] /= tn;
      const double ty[3] = {N[1] * tx[2] - N[2] * tx[1], N[2] * tx[0] - N[0] * tx[2],
                            N[0] * tx[1] - N[1] * tx[0]};
      double bd[3];
      for (int k = 0; k < 3; k++) bd[k] = lx * tx[k] + ly * ty[k] + lz * N[k];
      const double bn = sqrt((bd[0] * bd[0] + bd[1] * bd[1]) + bd[2] * bd[2]);
      for (int k = 0; k < 3; k++) {
        a.bo[3 * j + k] = (float)op[k];
        a.bd[3 * j + k] = (float)(bd[k] / bn);
      }
      a.b0[j] = 0.0;
      a.b1[j] = __longlong_as_double(0x7ff0000000000000LL);
    }
  }
}

}  // namespace hrpp

using namespace hrpp;

extern "C" int hrpp_gen_primary(const float* cam_pos, const double* basis9, double tan_half,
                                double aspect, int64_t width, int64_t height, int64_t spp,
                                int64_t sx, int64_t sy, uint64_t seed, int jitter, float* O,
                                float* D, void* stream) {
  if (width < 1 || height < 1 || spp < 1 || sx < 1 || sy < 1) {
    set_error("bad camera resolution or spp");
    return HRPP_INVALID_ARG;
  }
  PrimaryArgs a;
  for (int k = 0; k < 3; k++) {
    a.pos[k] = cam_pos[k];
    a.fwd[k] = basis9[k];
    a.right[k] = basis9[3 + k];
    a.up[k] = basis9[6 + k];
  }
  a.tan_half = tan_half;
  a.tan_aspect = tan_half * aspect;
  a.w = width;
  a.h = height;
  a.spp = spp;
  a.sx = sx;
  a.sy = sy;
  a.seed = seed;
  a.jitter = jitter;
  a.n = width * height * spp;
  a.O = O;
  a.D = D;
  cudaStream_t st = (cudaStream_t)stream;
  k_gen_primary<<<grid_for(a.n, 256, num_sms() * 16), 256, 0, st>>>(a);
  HRPP_LAUNCHED();
  HRPP_CK(cudaStreamSynchronize(st));
  return HRPP_OK;
}

extern "C" int hrpp_spawn(hrpp_bvh_t bvh, const float* O, const float* D, const uint8_t* found,
                          const double* t, const int32_t* slot, int64_t n, int shadow_kind,
                          const double* light3, double half, int bounce_kind, uint64_t seed,
                          float* so, float* sd, double* s0, double* s1, float* bo, float* bd,
                          double* b0, double* b1, int64_t* count_out, void* stream) {
  const BvhDev* b = reinterpret_cast<const BvhDev*>(bvh);
  if (!b || !count_out || n < 0 || n >= (1LL << 31)) {
    set_error("bad spawn arguments");
    return HRPP_INVALID_ARG;
  }
  *count_out = 0;
  if (n == 0) return HRPP_OK;
  cudaStream_t st = (cudaStream_t)stream;
  Workspace& ws = device_ws();  // per host thread and device
  int32_t* pos;
  int* cnt;
  int rc;
  if ((rc = ws.get("sp_pos", n, &pos)) || (rc = ws.get("sp_cnt", 1, &cnt))) return rc;
  size_t bytes = 0;
  cub::CountingInputIterator<int32_t> it(0);
  cub::DeviceSelect::Flagged(nullptr, bytes, it, found, pos, cnt, (int)n, st);
  void* tmp;
  if ((rc = ws.get_raw("sp_tmp", bytes, &tmp))) return rc;
  HRPP_CK(cub::DeviceSelect::Flagged(tmp, bytes, it, found, pos, cnt, (int)n, st));
  SpawnArgs a;
  a.O = O;
  a.D = D;
  a.found = found;
  a.t = t;
  a.slot = slot;
  a.tris = b->tris;
  a.pos = pos;
  a.count = cnt;
  a.shadow_kind = shadow_kind;
  for (int k = 0; k < 3; k++) a.light[k] = light3 ? light3[k] : 0.0;
  a.half = half;
  a.bounce_kind = bounce_kind;
  a.seed = seed;
  a.so = so;
  a.sd = sd;
  a.s0 = s0;
  a.s1 = s1;
  a.bo = bo;
  a.bd = bd;
  a.b0 = b0;
  a.b1 = b1;
  k_spawn<<<grid_for(n, 128, num_sms() * 16), 128, 0, st>>>(a);
  HRPP_LAUNCHED();
  long long* pin = pinned_scratch();
  if (!pin) return HRPP_CUDA;
  if ((rc = to_host(pin + 32, cnt, sizeof(int), st))) return rc;
  HRPP_CK(cudaStreamSynchronize(st));
  *count_out = *(volatile int*)(pin + 32);
  return HRPP_OK;
}
