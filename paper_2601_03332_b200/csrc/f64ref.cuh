// f64ref.cuh — the reference's scalar f64 expressions on the device, for eval_accuracy
// (eval.cu) and the element primitives (elements.cu). Both files build with -fmad=false, so every
// expression below rounds exactly as the reference's (proj/core built without contraction).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

namespace lkg {
namespace f64ref {

constexpr int kMaxP = 7;   // spline degree bound
constexpr int kMaxT = 96;  // extended knots bound
constexpr int kMaxK = 64;  // artifact segments bound

__device__ __forceinline__ double silu(double x) { return x / (1.0 + exp(-x)); }  // spline.cpp:85

// basis_into (spline.cpp:69-83) restricted to the degree+1 functions that can be non-zero at x:
// b[o] = B_{mu-p+o}(x), *r0 = mu - p (mu = -1: x outside the extended knots, every value 0). The
// reference's full recursion adds exact zeros outside this window, so the values are identical.
__device__ __forceinline__ void basis_window(const double* T, int nT, int p, double x, double (&b)[kMaxP + 1],
                                             int* r0) {
  const int n0 = nT - 1;
  int mu = -1;
  for (int s = 0; s < n0; s++)
    if (T[s] <= x && x < T[s + 1]) mu = s;
  for (int o = 0; o <= kMaxP; o++) b[o] = 0.0;
  if (mu >= 0) {
    b[p] = 1.0;
    for (int q = 1; q <= p; q++) {
      for (int o = p - q; o <= p; o++) {
        const int rr = mu - p + o;
        if (rr < 0 || rr >= n0 - q) {
          b[o] = 0.0;
          continue;
        }
        double acc = 0.0;
        const double d1 = T[rr + q] - T[rr];
        if (d1 > 0.0) acc += (x - T[rr]) / d1 * b[o];
        const double d2 = T[rr + q + 1] - T[rr + 1];
        if (d2 > 0.0 && o + 1 <= p) acc += (T[rr + q + 1] - x) / d2 * b[o + 1];
        b[o] = acc;
      }
    }
  }
  *r0 = mu - p;
}

// runtime.cpp:45-75 over the artifact's f32 knots widened to f64 (kn[0..K])
struct Coord64 {
  bool in;
  double xp, w;
  int k, l0, l1;
};
__device__ __forceinline__ Coord64 coords(const double* kn, int K, int L, bool half_open, double hi_clip, double x) {
  Coord64 c;
  const double lo = kn[0], hi = kn[K];
  c.in = half_open ? (lo <= x && x < hi) : (lo <= x && x <= hi);  // in_range
  c.xp = x < lo ? lo : (x > hi_clip ? hi_clip : x);                 // safe_clip (std::clamp)
  int k = 0;
  while (k + 1 <= K && kn[k + 1] <= c.xp) k++;                     // upper_bound - 1
  c.k = k > K - 1 ? K - 1 : k;
  const double u = (c.xp - kn[c.k]) / (kn[c.k + 1] - kn[c.k]);     // interp_coords
  const double z = u * (double)(L - 1);
  int l0 = (int)floor(z);
  c.l0 = l0 < 0 ? 0 : (l0 > L - 1 ? L - 1 : l0);
  c.l1 = c.l0 + 1 < L - 1 ? c.l0 + 1 : L - 1;
  c.w = z - (double)c.l0;
  return c;
}

// fetch_cell (runtime.cpp:81-88)
__device__ __forceinline__ double fetch(const uint8_t* q, const float* scale, const float* ymin, const double* ftab,
                                        bool i8, int L, int64_t cell, int l) {
  const int64_t off = cell * L + l;
  if (ftab) return ftab[off];
  const double qv = i8 ? (double)(int8_t)q[off] : (double)q[off];
  return (double)ymin[cell] + (double)scale[cell] * qv;
}

}  // namespace f64ref
}  // namespace lkg
