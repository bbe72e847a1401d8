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
  float fast_half;       // lut_coords_fast: 0.5 - (node distance below which the exact path runs)
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
  k = k - (xp < kt.x ? 1 : 0) + ((xp >= kt.z && k < c.K - 1) ? 1 : 0);
  kt = ktab[k];
  const float dx = xp - kt.x, z = dx * kt.y, fl = floorf(z);
  float w1 = z - fl;
  int l0 = (int)fl;
  const bool top = xp == c.hi_clip;
  l0 = top ? c.top_l0 : l0;
  w1 = top ? c.top_w1 : w1;
  if (!top && dx != 0.0f && (w1 < c.z_thr || w1 > 1.0f - c.z_thr)) {
    // near a sample node: u and z exactly as runtime.cpp:178-181 (f64)
    const double u = ((double)xp - (double)kt.x) / ((double)kt.z - (double)kt.x);
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

// silu(x) = x / (1 + 2^(-x log2 e)) with the flush-to-zero MUFU forms (no denormal guards):
// relative error ~3e-7; x -> -inf gives -0 (rcp(inf) = 0), x -> +inf gives x.
__device__ __forceinline__ float silu_fast(float x) {
  float e, r;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(x * -1.4426950408889634f));
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(1.0f + e));
  return x * r;
}

// silu(x) = x / (1 + exp(-x)) evaluated in f64 (spline.cpp:105-108) and rounded once to f32.
__device__ __forceinline__ float silu_exact(float x) {
  const double xd = x;
  return (float)(xd / (1.0 + exp(-xd)));
}

// Fast path of lut_coords for the table walk: the segment from the uniform-grid estimate, with no
// knot compares, and z from that segment's constants. An estimate can only be off by one within a
// few fp32 roundings of a knot, where z lands next to a sample node; every coordinate closer than
// 0.5 - c.fast_half to a node takes the exact path above (a grid that failed the host's uniformity
// bound has fast_half = -1: always exact). Elsewhere floor(z) has no tie to resolve, so k, l0 and
// the mask equal the reference's. z is formed as 1 + z so that w1 is a multiple of 2^-23.
// Branch-free half of lut_coords_fast: the fast coordinates and whether the exact path must
// replace them (lets a caller run several rows' coordinate chains side by side and take the
// exact path once for all of them).
// floor() of a value in [0, 2^23) on the FMA/ALU pipes: the round-down add leaves 2^23 + floor(v)
// in the float and floor(v) in its low mantissa bits (no F2I / FRND, which issue at 1/8 rate).
__device__ __forceinline__ float floor_magic(float v) { return __fadd_rd(v, 8388608.0f); }
__device__ __forceinline__ int floor_magic_int(float m) { return __float_as_int(m) - 0x4B000000; }

// kf: the compact per-segment table {T_k, (L-1)/h_k} (8-byte entries: a warp's 64-bit loads of up to
// 16 distinct segments hit distinct banks; the 16-byte ktab rows conflicted for K > 8)
__device__ __forceinline__ Coord lut_coords_fast_nb(const CoordConst& c, const float2* kf, float x, bool& slow) {
  const float xp = fminf(fmaxf(x, c.lo), c.hi_clip);
  const int k = min(floor_magic_int(floor_magic((xp - c.lo) * c.inv_h)), c.K - 1);
  const float2 kt = kf[k];  // {T_k, (L-1)/h_k}
  const float dx = xp - kt.x, z1 = fmaf(dx, kt.y, 1.0f), zm = floor_magic(z1), zf = zm - 8388608.0f;
  const float w1 = z1 - zf;
  const bool top = xp == c.hi_clip;
  slow = !top && dx != 0.0f && fabsf(w1 - 0.5f) > c.fast_half;
  Coord o;
  o.in = xp == x;  // == (t_0 <= x <= hi_clip): clamping changes every other x; NaN compares false
  o.xp = xp;
  o.k = k;
  o.l0 = top ? c.top_l0 : floor_magic_int(zm) - 1;
  o.w1 = top ? c.top_w1 : w1;
  return o;
}

__device__ __forceinline__ Coord lut_coords_fast(const CoordConst& c, const float4* ktab, const float2* kf, float x) {
  const float xp = fminf(fmaxf(x, c.lo), c.hi_clip);
  const int k = min(floor_magic_int(floor_magic((xp - c.lo) * c.inv_h)), c.K - 1);
  const float2 kt = kf[k];  // {T_k, (L-1)/h_k}
  const float dx = xp - kt.x, z1 = fmaf(dx, kt.y, 1.0f), zm = floor_magic(z1), zf = zm - 8388608.0f;
  const float w1 = z1 - zf;
  const bool top = xp == c.hi_clip;  // exact host-side coordinates; dx == 0: z = 0 exactly
  if (!top && dx != 0.0f && fabsf(w1 - 0.5f) > c.fast_half) return lut_coords(c, ktab, x);
  Coord o;
  o.in = c.lo <= x && x <= c.hi_clip;
  o.xp = xp;
  o.k = k;
  o.l0 = top ? c.top_l0 : floor_magic_int(zm) - 1;
  o.w1 = top ? c.top_w1 : w1;
  return o;
}
#endif

}  // namespace lkg
