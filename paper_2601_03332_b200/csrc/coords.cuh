// coords.cuh — steps 1-4 of the reference's 5-step LUT evaluation for one coordinate
// (forward_quant phase 1, proj/core/src/runtime.cpp:170-190), shared by every forward kernel
// and by lkg_layer_coords (so the exposed segment indices / masks are the ones the kernels use).
//
//   in   = t_0 <= x <= hi_clip          (hi_clip = nextafterf(t_K, -inf) when half_open, else
//                                         t_K — for fp32 x this is exactly the reference's
//                                         lo <= x && (half_open ? x < hi : x <= hi) over f32 knots)
//   x'   = clamp(x, t_0, hi_clip)
//   k    = #{r in 1..K-1 : x' >= t_r}   (uniform knots: estimate + one exact correction step)
//   z    = (x' - t_k) * (L-1)/(t_k+1 - t_k) in fp32; within z_thr of a sample node, u and z are
//          re-evaluated in f64 exactly as runtime.cpp:178-181 so l0 matches the reference
//   l0   = clamp(floor(z), 0, L-1), w1 = z - l0 (w1 = 0 at l0 = L-1), rounded to a multiple of
//          2^-23 (keeps the magic-float constants of the table walk exact; |change| <= 2^-24)
#pragma once
#include <cuda_runtime.h>

namespace lkg {

constexpr int kMaxKT = 64;

struct CoordConst {
  float lo, hi_clip, inv_h, z_thr;
  int32_t K, L, top_l0;  // (top_l0, top_w1): exact coordinates of x' == hi_clip
  float top_w1;
};

struct Coord {
  int k, l0;
  float w1, xp;
  bool in;
};

#ifdef __CUDACC__
__device__ __forceinline__ Coord lut_coords(const CoordConst& c, const float4* ktab, float x) {
  Coord o;
  o.in = c.lo <= x && x <= c.hi_clip;  // false for NaN
  const float xp = fminf(fmaxf(x, c.lo), c.hi_clip);
  o.xp = xp;
  int k = min(__float2int_rd((xp - c.lo) * c.inv_h), c.K - 1);
  float4 kt = ktab[k];
  k = k - (xp < kt.x ? 1 : 0) + ((xp >= kt.y && k < c.K - 1) ? 1 : 0);
  kt = ktab[k];
  const float dx = xp - kt.x, z = dx * kt.z, fl = floorf(z);
  float w1 = z - fl;
  int l0 = (int)fl;
  const bool top = xp == c.hi_clip;
  l0 = top ? c.top_l0 : l0;
  w1 = top ? c.top_w1 : w1;
  if (!top && dx != 0.0f && (w1 < c.z_thr || w1 > 1.0f - c.z_thr)) {
    // near a sample node: u and z exactly as runtime.cpp:178-181 (f64)
    const double u = ((double)xp - (double)kt.x) / ((double)kt.y - (double)kt.x);
    const double zz = u * (double)(c.L - 1);
    int ll = (int)floor(zz);
    ll = ll < 0 ? 0 : (ll > c.L - 1 ? c.L - 1 : ll);
    l0 = ll;
    w1 = (float)(zz - (double)ll);
  }
  w1 = l0 >= c.L - 1 ? 0.0f : w1;
  l0 = min(max(l0, 0), c.L - 1);
  o.k = k;
  o.l0 = l0;
  o.w1 = (w1 + 1.0f) - 1.0f;
  return o;
}
#endif

}  // namespace lkg
