// compile.cu — K1: LUT compile on the device, bit-exact with the reference
// compile_layer (proj/core/src/compiler.cpp:132-209).
//
// One warp per (edge, segment) cell; lanes stride over the L samples. The host
// supplies, per sample point p = k*L + l, the exact f64 basis window {b_t} starting
// at r0[p] (every basis value outside the window is exactly 0, checked on the host)
// and, for value_repr = phi, silu(x_p) — both computed with the reference's own f64
// expressions and libm (model_gen.cpp). The device then forms
//   s = sum_r c_r * b_r          (compiler.cpp:65-66; zero terms are exact no-ops)
//   v = out*(base*silu + spline*s)   (phi, compiler.cpp:67-69)
// with unfused __dmul_rn/__dadd_rn in the reference order, reduces the segment's
// amax (symmetric) or min/max (asymmetric) exactly, rounds the parameters through
// f32 (or f16) like round_param (compiler.cpp:97-101), and computes the codes with
// round-half-away division (codes_for, compiler.cpp:86-95). This file is compiled
// with -fmad=false as well.
#include <cuda_runtime.h>

#include <cstdint>

#include "lkg_internal.h"

namespace {

// float16.cpp:7-42 restated for the device (round to nearest even).
__device__ uint16_t f32_to_f16_bits(float f) {
  const uint32_t x = __float_as_uint(f);
  const uint32_t sign = (x >> 16) & 0x8000u;
  const uint32_t ex = (x >> 23) & 0xffu;
  uint32_t man = x & 0x7fffffu;
  if (ex == 0xffu) return (uint16_t)(sign | 0x7c00u | (man ? 0x200u | (man >> 13) : 0u));
  const int e = (int)ex - 127 + 15;
  if (e >= 0x1f) return (uint16_t)(sign | 0x7c00u);
  if (e <= 0) {
    if (e < -10) return (uint16_t)sign;
    man |= 0x800000u;
    const int sh = 14 - e;
    uint32_t hm = man >> sh;
    const uint32_t rem = man & ((1u << sh) - 1u), half = 1u << (sh - 1);
    if (rem > half || (rem == half && (hm & 1u))) hm++;
    return (uint16_t)(sign | hm);
  }
  uint32_t h = sign | ((uint32_t)e << 10) | (man >> 13);
  const uint32_t rem = man & 0x1fffu;
  if (rem > 0x1000u || (rem == 0x1000u && (h & 1u))) h++;
  return (uint16_t)h;
}

// float16.cpp:44-71.
__device__ float f16_bits_to_f32(uint16_t h) {
  const uint32_t sign = ((uint32_t)h & 0x8000u) << 16;
  const uint32_t ex = (h >> 10) & 0x1fu;
  uint32_t man = h & 0x3ffu, out;
  if (ex == 0x1fu) {
    out = sign | 0x7f800000u | (man << 13);
  } else if (ex == 0) {
    if (man == 0) {
      out = sign;
    } else {
      int e = -1;
      do {
        man <<= 1;
        e++;
      } while ((man & 0x400u) == 0);
      out = sign | ((uint32_t)(127 - 15 - e) << 23) | ((man & 0x3ffu) << 13);
    }
  } else {
    out = sign | ((ex - 15 + 127) << 23) | (man << 13);
  }
  return __uint_as_float(out);
}

__device__ __forceinline__ double round_param(double v, int f16) {
  const float f = __double2float_rn(v);
  return f16 ? (double)f16_bits_to_f32(f32_to_f16_bits(f)) : (double)f;
}

struct CompileArgs {
  const double* coeffs;  // [E, R]
  const double* gains;   // [3][E]: base, spline, out
  const double* basis;   // [K*L, W]
  const int32_t* r0;     // [K*L]
  const double* silu;    // [K*L] (phi only)
  uint8_t* q;            // [E, K, L]
  float* scale;          // [E, K]
  float* ymin;           // [E, K]
  double* float_table;   // [E, K, L] or null
  int* nonfinite;
  int64_t E;
  int32_t K, L, R, W, phi, asym, f16;
};

constexpr int kCache = 4;  // samples cached per lane (L <= 128 without recomputation)

__device__ __forceinline__ double sample_value(const CompileArgs& a, const double* c, double base,
                                               double spline, double out, int p) {
  const double* b = a.basis + (int64_t)p * a.W;
  const double* cr = c + a.r0[p];
  double s = 0.0;  // starts at +0.0 like the reference (keeps the sign of an all-zero sum)
  for (int t = 0; t < a.W; t++) s = __dadd_rn(s, __dmul_rn(cr[t], b[t]));
  if (!a.phi) return s;
  return __dmul_rn(out, __dadd_rn(__dmul_rn(base, a.silu[p]), __dmul_rn(spline, s)));
}

__global__ void __launch_bounds__(256) compile_kernel(CompileArgs a) {
  const int lane = threadIdx.x & 31;
  const int64_t cell = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (cell >= a.E * a.K) return;
  const int64_t e = cell / a.K;
  const int k = (int)(cell - e * a.K);
  const double* c = a.coeffs + e * a.R;
  const double base = a.gains[e], spline = a.gains[a.E + e], out = a.gains[2 * a.E + e];
  const int p0 = k * a.L;

  // Pass 1: segment statistics (quantize_segment_*, compiler.cpp:105-128). min/max
  // follow std::min/std::max over the samples in ascending l: on ties (only +0/-0 can
  // tie with different bits) the earliest sample wins, so indices ride along.
  double amax = 0.0, lo = 0.0, hi = 0.0;
  int lo_i = 0x7fffffff, hi_i = 0x7fffffff;
  bool finite = true;
  double vc[kCache];  // the lane's samples (L <= 32 * kCache), reused by the code pass
#pragma unroll
  for (int t = 0; t < kCache; t++) vc[t] = 0.0;
  for (int l = lane; l < a.L; l += 32) {
    const double v = sample_value(a, c, base, spline, out, p0 + l);
#pragma unroll
    for (int t = 0; t < kCache; t++)
      if (l == lane + 32 * t) vc[t] = v;
    finite = finite && isfinite(v);
    amax = amax < fabs(v) ? fabs(v) : amax;            // std::max(amax, fabs(v))
    if (lo_i == 0x7fffffff || v < lo) { lo = v; lo_i = l; }
    if (hi_i == 0x7fffffff || hi < v) { hi = v; hi_i = l; }
    if (a.float_table) a.float_table[cell * a.L + l] = v;
  }
  for (int o = 16; o; o >>= 1) {
    const double am = __shfl_xor_sync(0xffffffffu, amax, o);
    amax = amax < am ? am : amax;
    const double ol = __shfl_xor_sync(0xffffffffu, lo, o), oh = __shfl_xor_sync(0xffffffffu, hi, o);
    const int oli = __shfl_xor_sync(0xffffffffu, lo_i, o), ohi = __shfl_xor_sync(0xffffffffu, hi_i, o);
    if (oli != 0x7fffffff && (lo_i == 0x7fffffff || ol < lo || (ol == lo && oli < lo_i))) { lo = ol; lo_i = oli; }
    if (ohi != 0x7fffffff && (hi_i == 0x7fffffff || hi < oh || (oh == hi && ohi < hi_i))) { hi = oh; hi_i = ohi; }
  }
  if (!__all_sync(0xffffffffu, finite)) {
    if (lane == 0) atomicExch(a.nonfinite, 1);
    return;
  }

  // Storage-width parameters, then codes against them (compiler.cpp:176-204).
  double sc, ym;
  int qlo, qhi;
  if (!a.asym) {
    ym = 0.0;
    sc = round_param(__ddiv_rn(amax, 127.0), a.f16);
    qlo = -127;
    qhi = 127;
  } else {
    ym = round_param(lo, a.f16);
    const double s = round_param(__ddiv_rn(__dsub_rn(hi, ym), 255.0), a.f16);
    sc = s < 0.0 ? 0.0 : s;  // std::max(s, 0.0)
    qlo = 0;
    qhi = 255;
  }
  if (lane == 0) {
    a.scale[cell] = (float)sc;
    a.ymin[cell] = (float)ym;
  }
  uint8_t* dst = a.q + cell * a.L;
  // codes_for (compiler.cpp:86-95): round_half_away((v - y_min) / scale). The quotient is
  // estimated with one reciprocal; round() can only differ from round(correctly rounded quotient)
  // when the quotient is within a few ulp of a half-integer, so those (rare) cases take the exact
  // IEEE division. The result is identical to dividing every time.
  const double inv = sc > 0.0 ? __drcp_rn(sc) : 0.0;
  for (int l = lane, t = 0; l < a.L; l += 32, t++) {
    int q = 0;
    if (sc > 0.0) {
      double v = 0.0;
#pragma unroll
      for (int tt = 0; tt < kCache; tt++)
        if (tt == t) v = vc[tt];
      if (t >= kCache) v = sample_value(a, c, base, spline, out, p0 + l);
      const double num = __dsub_rn(v, ym);
      double r = __dmul_rn(num, inv);
      if (fabs(r - floor(r) - 0.5) < 1e-6) r = __ddiv_rn(num, sc);
      r = round(r);
      r = r < (double)qlo ? (double)qlo : (r > (double)qhi ? (double)qhi : r);
      q = (int)r;
    }
    dst[l] = (uint8_t)(a.asym ? q : (int)(int8_t)q);
  }
}

// Per-edge gains narrowed to the artifact's f32 (compiler.cpp:151-160).
__global__ void gains_to_f32(const double* g, float* out, int64_t n) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t < n) out[t] = __double2float_rn(g[t]);
}

}  // namespace

namespace lkg {

void launch_compile(lkg_ctx* ctx, const lkg_spec* S, const lkg_quant_config* qc, lkg_layer* out,
                    const double* d_basis, const int32_t* d_r0, const double* d_silu, int32_t W,
                    bool keep_float) {
  const int64_t E = (int64_t)S->in_dim * (S->col1 - S->col0);
  const int K = S->K, L = qc->L;
  DBuf flag;
  flag.alloc(sizeof(int));
  LKG_CUDA(cudaMemsetAsync(flag.p, 0, sizeof(int), ctx->stream));
  CompileArgs a;
  a.coeffs = S->coeffs.as<double>();
  a.gains = S->gains.as<double>();
  a.basis = d_basis;
  a.r0 = d_r0;
  a.silu = d_silu;
  a.q = out->q.as<uint8_t>();
  a.scale = out->scale.as<float>();
  a.ymin = out->ymin.as<float>();
  a.float_table = keep_float ? out->float_table.as<double>() : nullptr;
  a.nonfinite = flag.as<int>();
  a.E = E;
  a.K = K;
  a.L = L;
  a.R = K + S->degree;
  a.W = W;
  a.phi = qc->value_repr == LKG_REPR_PHI;
  a.asym = qc->scheme == LKG_SCHEME_ASYMMETRIC;
  a.f16 = qc->param_dtype == LKG_PARAM_F16;
  const int64_t cells = E * K, warps_per_block = 8;
  const int64_t blocks = (cells + warps_per_block - 1) / warps_per_block;
  compile_kernel<<<(unsigned)blocks, 256, 0, ctx->stream>>>(a);
  LKG_CUDA(cudaGetLastError());
  ctx->launches++;
  if (out->value_repr == LKG_REPR_SPLINE_COMPONENT) {
    const int64_t n = 3 * E;
    gains_to_f32<<<(unsigned)((n + 255) / 256), 256, 0, ctx->stream>>>(S->gains.as<double>(),
                                                                         out->gains.as<float>(), n);
    LKG_CUDA(cudaGetLastError());
    ctx->launches++;
  }
  int h = 0;
  LKG_CUDA(cudaMemcpyAsync(&h, flag.p, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  LKG_CUDA(cudaStreamSynchronize(ctx->stream));
  if (h) throw Error{LKG_ERR_NON_FINITE, "non-finite table value"};
}

}  // namespace lkg
