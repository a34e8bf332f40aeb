// bvh_build.cpp -- native BVH builder (host C++).
//
// Restates the reference builder hrpp/bvh.py:184-357 operation by operation
// so that its arrays are bit-identical to the reference's on the same
// triangles (checked against tests/golden/bvh_*.npz): degenerate filter
// (area > 2e-12, bvh.py:195), binned SAH with 16 bins over all three axes
// (bvh.py:290-345), the improvement test 1 + cost/parent_area < n
// (bvh.py:344-345), the stable median fallback on the widest centroid axis
// (bvh.py:351-357), coincident centroids -> oversized leaf, DFS preorder
// with the left child created first (bvh.py:255-257).  The Python builder
// runs at ~0.36 ms/triangle; this one builds the 60k-1M triangle configs in
// seconds.  median_split selects a plain median-split tree (BASELINE c1).
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <limits>
#include <vector>

namespace {

constexpr int kBins = 16;
constexpr int kMaxDepth = 512 / 2 - 2;  // bvh.py:34 (_MAX_SUPPORTED_DEPTH)

inline double half_area(const double lo[3], const double hi[3]) {
  double d0 = std::max(hi[0] - lo[0], 0.0);
  double d1 = std::max(hi[1] - lo[1], 0.0);
  double d2 = std::max(hi[2] - lo[2], 0.0);
  return d0 * d1 + d1 * d2 + d2 * d0;
}

struct Builder {
  int64_t m;
  const float *tmin, *tmax;  // per-triangle f32 boxes (m,3)
  const double* cent;        // (m,3)
  int max_leaf;
  bool median;

  // returns false for "no split" (leaf)
  bool find_split(const std::vector<int64_t>& idx, int* axis_out, std::vector<int64_t>& L,
                  std::vector<int64_t>& R) {
    const int64_t n = (int64_t)idx.size();
    double cmin[3], cmax[3], ext[3];
    for (int a = 0; a < 3; a++) {
      cmin[a] = std::numeric_limits<double>::infinity();
      cmax[a] = -std::numeric_limits<double>::infinity();
    }
    for (int64_t i : idx)
      for (int a = 0; a < 3; a++) {
        double c = cent[3 * i + a];
        if (c < cmin[a]) cmin[a] = c;
        if (c > cmax[a]) cmax[a] = c;
      }
    for (int a = 0; a < 3; a++) ext[a] = cmax[a] - cmin[a];
    bool all_flat = ext[0] <= 0.0 && ext[1] <= 0.0 && ext[2] <= 0.0;

    double best_cost = std::numeric_limits<double>::infinity();
    int best_ax = -1, best_k = -1;
    if (!median) {
      for (int ax = 0; ax < 3; ax++) {
        if (ext[ax] <= 0.0) continue;
        double scale = kBins / ext[ax];
        int64_t counts[kBins] = {0};
        double blo[kBins][3], bhi[kBins][3];
        for (int b = 0; b < kBins; b++)
          for (int a = 0; a < 3; a++) {
            blo[b][a] = std::numeric_limits<double>::infinity();
            bhi[b][a] = -std::numeric_limits<double>::infinity();
          }
        for (int64_t j = 0; j < n; j++) {
          int64_t i = idx[j];
          int64_t b = (int64_t)((cent[3 * i + ax] - cmin[ax]) * scale);
          if (b > kBins - 1) b = kBins - 1;
          counts[b]++;
          for (int a = 0; a < 3; a++) {
            double lo = tmin[3 * i + a], hi = tmax[3 * i + a];
            if (lo < blo[b][a]) blo[b][a] = lo;
            if (hi > bhi[b][a]) bhi[b][a] = hi;
          }
        }
        double lol[kBins][3], hil[kBins][3], lor[kBins][3], hir[kBins][3];
        for (int a = 0; a < 3; a++) {
          lol[0][a] = blo[0][a];
          hil[0][a] = bhi[0][a];
          for (int b = 1; b < kBins; b++) {
            lol[b][a] = std::min(lol[b - 1][a], blo[b][a]);
            hil[b][a] = std::max(hil[b - 1][a], bhi[b][a]);
          }
          lor[kBins - 1][a] = blo[kBins - 1][a];
          hir[kBins - 1][a] = bhi[kBins - 1][a];
          for (int b = kBins - 2; b >= 0; b--) {
            lor[b][a] = std::min(lor[b + 1][a], blo[b][a]);
            hir[b][a] = std::max(hir[b + 1][a], bhi[b][a]);
          }
        }
        int64_t cl = 0;
        for (int k = 0; k < kBins - 1; k++) {
          cl += counts[k];
          int64_t nl = cl, nr = n - cl;
          if (nl == 0 || nr == 0) continue;
          double cost = half_area(lol[k], hil[k]) * (double)nl +
                        half_area(lor[k + 1], hir[k + 1]) * (double)nr;
          if (cost < best_cost) {
            best_cost = cost;
            best_ax = ax;
            best_k = k;
          }
        }
      }
    }
    if (all_flat) return false;
    bool improving = false;
    if (best_ax >= 0) {
      double plo[3], phi[3];
      for (int a = 0; a < 3; a++) {
        plo[a] = std::numeric_limits<double>::infinity();
        phi[a] = -std::numeric_limits<double>::infinity();
      }
      for (int64_t i : idx)
        for (int a = 0; a < 3; a++) {
          plo[a] = std::min(plo[a], (double)tmin[3 * i + a]);
          phi[a] = std::max(phi[a], (double)tmax[3 * i + a]);
        }
      double parent_area = half_area(plo, phi);
      improving = parent_area > 0.0 && 1.0 + best_cost / parent_area < (double)n;
    }
    L.clear();
    R.clear();
    if (improving) {
      // the winning axis's bins, recomputed with the same arithmetic
      const double scale = kBins / ext[best_ax];
      for (int64_t j = 0; j < n; j++) {
        const int64_t i = idx[j];
        int64_t b = (int64_t)((cent[3 * i + best_ax] - cmin[best_ax]) * scale);
        if (b > kBins - 1) b = kBins - 1;
        (b <= best_k ? L : R).push_back(i);
      }
      *axis_out = best_ax;
      return true;
    }
    if (n <= max_leaf) return false;
    int ax = 0;
    for (int a = 1; a < 3; a++)
      if (ext[a] > ext[ax]) ax = a;
    std::vector<int64_t> order(n);
    for (int64_t j = 0; j < n; j++) order[j] = j;
    std::stable_sort(order.begin(), order.end(), [&](int64_t x, int64_t y) {
      return cent[3 * idx[x] + ax] < cent[3 * idx[y] + ax];
    });
    int64_t half = n / 2;
    for (int64_t j = 0; j < n; j++) (j < half ? L : R).push_back(idx[order[j]]);
    *axis_out = ax;
    return true;
  }
};

struct Item {
  std::vector<int64_t> idx;
  int32_t parent;
  bool is_left;
  int32_t depth;
};

}  // namespace

extern "C" int hrpp_build_bvh(const float* v0, const float* v1, const float* v2,
                              const int32_t* ids, int64_t n_tris, int max_leaf_size,
                              int median_split, float* bmin, float* bmax, int32_t* left,
                              int32_t* right, int8_t* axis, int32_t* first, int32_t* count,
                              int32_t* parent, int32_t* depth, float* tv0, float* tv1,
                              float* tv2, int32_t* tri_ids, int64_t* n_nodes_out,
                              int64_t* n_tris_out, int32_t* max_depth_out) {
  if (max_leaf_size < 1 || n_tris < 0) return 3;
  // degenerate filter (bvh.py:195, _area2_f64 :279-282)
  std::vector<int64_t> keep;
  keep.reserve(n_tris);
  for (int64_t i = 0; i < n_tris; i++) {
    double e1x = (double)v1[3 * i] - (double)v0[3 * i];
    double e1y = (double)v1[3 * i + 1] - (double)v0[3 * i + 1];
    double e1z = (double)v1[3 * i + 2] - (double)v0[3 * i + 2];
    double e2x = (double)v2[3 * i] - (double)v0[3 * i];
    double e2y = (double)v2[3 * i + 1] - (double)v0[3 * i + 1];
    double e2z = (double)v2[3 * i + 2] - (double)v0[3 * i + 2];
    double cx = e1y * e2z - e1z * e2y;
    double cy = e1z * e2x - e1x * e2z;
    double cz = e1x * e2y - e1y * e2x;
    double a2 = std::sqrt(cx * cx + cy * cy + cz * cz);
    if (a2 > 2.0 * 1e-12) keep.push_back(i);
  }
  const int64_t m = (int64_t)keep.size();
  *n_tris_out = m;
  if (m == 0) return 3;  // EmptyScene
  std::vector<float> tb_min(3 * m), tb_max(3 * m), kv0(3 * m), kv1(3 * m), kv2(3 * m);
  std::vector<int32_t> kid(m);
  std::vector<double> cent(3 * m);
  for (int64_t j = 0; j < m; j++) {
    int64_t i = keep[j];
    for (int a = 0; a < 3; a++) {
      float x = v0[3 * i + a], y = v1[3 * i + a], z = v2[3 * i + a];
      kv0[3 * j + a] = x;
      kv1[3 * j + a] = y;
      kv2[3 * j + a] = z;
      tb_min[3 * j + a] = std::min(std::min(x, y), z);
      tb_max[3 * j + a] = std::max(std::max(x, y), z);
      cent[3 * j + a] = ((double)tb_min[3 * j + a] + (double)tb_max[3 * j + a]) * 0.5;
    }
    kid[j] = ids ? ids[i] : (int32_t)i;
  }
  Builder B{m, tb_min.data(), tb_max.data(), cent.data(), max_leaf_size, median_split != 0};
  std::vector<Item> stack;
  Item root;
  root.idx.resize(m);
  for (int64_t j = 0; j < m; j++) root.idx[j] = j;
  root.parent = -1;
  root.is_left = false;
  root.depth = 0;
  stack.push_back(std::move(root));
  int64_t nn = 0, order_len = 0;
  int32_t maxd = 0;
  std::vector<int64_t> L, R;
  while (!stack.empty()) {
    Item it = std::move(stack.back());
    stack.pop_back();
    int64_t me = nn++;
    float lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
    for (int64_t i : it.idx)
      for (int a = 0; a < 3; a++) {
        lo[a] = std::min(lo[a], tb_min[3 * i + a]);
        hi[a] = std::max(hi[a], tb_max[3 * i + a]);
      }
    for (int a = 0; a < 3; a++) {
      bmin[3 * me + a] = lo[a];
      bmax[3 * me + a] = hi[a];
    }
    left[me] = -1;
    right[me] = -1;
    axis[me] = 0;
    first[me] = -1;
    count[me] = 0;
    parent[me] = it.parent;
    depth[me] = it.depth;
    if (it.parent >= 0) (it.is_left ? left : right)[it.parent] = (int32_t)me;
    const int64_t n = (int64_t)it.idx.size();
    int ax = 0;
    bool split = n > 1 && B.find_split(it.idx, &ax, L, R);
    if (!split) {
      first[me] = (int32_t)order_len;
      count[me] = (int32_t)n;
      for (int64_t j = 0; j < n; j++) {
        int64_t i = it.idx[j];
        for (int a = 0; a < 3; a++) {
          tv0[3 * (order_len + j) + a] = kv0[3 * i + a];
          tv1[3 * (order_len + j) + a] = kv1[3 * i + a];
          tv2[3 * (order_len + j) + a] = kv2[3 * i + a];
        }
        tri_ids[order_len + j] = kid[i];
      }
      order_len += n;
      maxd = std::max(maxd, it.depth);
      continue;
    }
    axis[me] = (int8_t)ax;
    if (it.depth + 1 > kMaxDepth) return 3;  // bvh.py:252-254
    Item r{R, (int32_t)me, false, it.depth + 1};
    Item l{L, (int32_t)me, true, it.depth + 1};
    stack.push_back(std::move(r));
    stack.push_back(std::move(l));
  }
  *n_nodes_out = nn;
  *max_depth_out = maxd;
  return 0;
}
