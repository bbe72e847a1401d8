// elements.cu — the reference's scalar primitives, batched on the device in f64 (SURVEY §8a rows
// F7-F13, S2, CM3-CM5, CM9), built with -fmad=false so every value equals the reference's:
//   coords      safe_clip / segment_index / interp_coords / in_range   runtime.cpp:45-75
//   lut_eval    lut_eval_value / lut_eval_phi                          runtime.cpp:96-120
//   basis       basis_values                                           spline.cpp:89-94
//   edge_phi    eval_edge_phi (eval_spline + base_fn)                  spline.cpp:96-115
//   quantize    quantize_segment_symmetric / _asymmetric + codes_for   compiler.cpp:86-128
// One thread per element; the C-ABI (api.cpp) stages host arrays.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <vector>

#include "f64ref.cuh"
#include "lkg_internal.h"

namespace {

using lkg::f64ref::kMaxK;
using lkg::f64ref::kMaxP;
using lkg::f64ref::kMaxT;

struct LayerRef {  // artifact side (runtime.cpp)
  const uint8_t* q;
  const float* scale;
  const float* ymin;
  const float* g;  // [3][E]: base, spline, out
  const double* ftab;
  int32_t K, L, E, half_open, zs, phi, i8;
  double hi_clip;
  double kn[kMaxK + 1];
};

struct SpecRef {  // spline side (spline.cpp)
  const double* coeffs;  // [E][R]
  const double* g;       // [3][E]
  int32_t R, p, nT, E;
  double T[kMaxT];
};

__global__ void coords_kernel(const __grid_constant__ LayerRef a, const double* x, int64_t n, uint8_t* in,
                              double* xc, int32_t* k, int32_t* l0, int32_t* l1, double* w) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  const lkg::f64ref::Coord64 c = lkg::f64ref::coords(a.kn, a.K, a.L, a.half_open, a.hi_clip, x[t]);
  in[t] = c.in;
  xc[t] = c.xp;
  k[t] = c.k;
  l0[t] = c.l0;
  l1[t] = c.l1;
  w[t] = c.w;
}

// lut_eval_value / lut_eval_phi for (edge, x) pairs; flags[0] |= 1 on a non-finite x,
// flags[1] |= 1 on an edge index out of range (runtime.cpp:97-98)
__global__ void lut_eval_kernel(const __grid_constant__ LayerRef a, const int32_t* e, const double* x, int64_t n,
                                double* value, uint8_t* was_oob, double* phi, int* flags) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  const double xv = x[t];
  const int32_t ev = e[t];
  if (!isfinite(xv)) {
    atomicOr(flags + 0, 1);
    return;
  }
  if (ev < 0 || ev >= a.E) {
    atomicOr(flags + 1, 1);
    return;
  }
  const lkg::f64ref::Coord64 c = lkg::f64ref::coords(a.kn, a.K, a.L, a.half_open, a.hi_clip, xv);
  const int64_t cell = (int64_t)ev * a.K + c.k;
  const double v0 = lkg::f64ref::fetch(a.q, a.scale, a.ymin, a.ftab, a.i8, a.L, cell, c.l0);
  const double v1 = lkg::f64ref::fetch(a.q, a.scale, a.ymin, a.ftab, a.i8, a.L, cell, c.l1);
  double v = (1.0 - c.w) * v0 + c.w * v1;
  if (a.zs && !c.in) v = 0.0;
  value[t] = v;
  was_oob[t] = !c.in;
  if (a.phi) {
    phi[t] = v;
  } else {
    const double bx = lkg::f64ref::silu(a.zs ? xv : c.xp);
    phi[t] = (double)a.g[2 * a.E + ev] * ((double)a.g[ev] * bx + (double)a.g[a.E + ev] * v);
  }
}

__global__ void basis_kernel(const __grid_constant__ SpecRef s, const double* x, int64_t n, double* out) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  double b[kMaxP + 1];
  int r0;
  lkg::f64ref::basis_window(s.T, s.nT, s.p, x[t], b, &r0);
  double* o = out + t * s.R;
  for (int r = 0; r < s.R; r++) o[r] = 0.0;
  for (int q = 0; q <= s.p; q++)
    if (r0 + q >= 0 && r0 + q < s.R) o[r0 + q] = b[q];
}

// eval_edge_phi: out*(base*silu(x) + spline*eval_spline(x)), eval_spline summing r ascending
__global__ void edge_phi_kernel(const __grid_constant__ SpecRef s, const int32_t* e, const double* x, int64_t n,
                                double* phi, int* flags) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  const int32_t ev = e[t];
  if (ev < 0 || ev >= s.E) {
    atomicOr(flags + 1, 1);
    return;
  }
  const double xv = x[t];
  double b[kMaxP + 1];
  int r0;
  lkg::f64ref::basis_window(s.T, s.nT, s.p, xv, b, &r0);
  double sp = 0.0;
  for (int q = 0; q <= s.p; q++) {
    const int rr = r0 + q;
    if (rr >= 0 && rr < s.R) sp += s.coeffs[(int64_t)ev * s.R + rr] * b[q];
  }
  phi[t] = s.g[2 * s.E + ev] * (s.g[ev] * lkg::f64ref::silu(xv) + s.g[s.E + ev] * sp);
}

// quantize_segment_symmetric / _asymmetric (compiler.cpp:105-128): one thread per segment
__global__ void quantize_kernel(const double* v, int64_t nseg, int L, int asym, int32_t* q, double* scale,
                                double* ymin, int* flags) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nseg) return;
  const double* s = v + t * L;
  for (int l = 0; l < L; l++)
    if (!isfinite(s[l])) {
      atomicOr(flags + 0, 1);
      return;
    }
  double sc, y0;
  int qlo, qhi;
  if (!asym) {
    double amax = 0.0;
    for (int l = 0; l < L; l++) amax = fmax(amax, fabs(s[l]));  // std::max(amax, |v|): amax first
    sc = amax / 127.0;
    y0 = 0.0;
    qlo = -127;
    qhi = 127;
  } else {
    double lo = s[0], hi = s[0];
    for (int l = 0; l < L; l++) {
      lo = s[l] < lo ? s[l] : lo;  // std::min / std::max: keep the first of equal values
      hi = hi < s[l] ? s[l] : hi;
    }
    y0 = lo;
    sc = (hi - lo) / 255.0;
    qlo = 0;
    qhi = 255;
  }
  scale[t] = sc;
  ymin[t] = y0;
  for (int l = 0; l < L; l++) {  // codes_for (compiler.cpp:86-95)
    int c = 0;
    if (sc > 0.0) {
      const double r = round((s[l] - y0) / sc);  // round half away from zero
      c = (int)(r < qlo ? qlo : (r > qhi ? qhi : r));
    }
    q[t * L + l] = c;
  }
}

LayerRef layer_ref(const lkg_layer* L) {
  LayerRef a{};
  if (L->K > kMaxK) throw lkg::Error{LKG_ERR_CONFIG, "element primitives: more than 64 segments"};
  if (!L->q.p && !L->float_table.p)
    throw lkg::Error{LKG_ERR_CONFIG, "element primitives need the reference-layout table (layer stored tiles-only)"};
  a.q = L->q.as<uint8_t>();
  a.scale = L->scale.as<float>();
  a.ymin = L->ymin.as<float>();
  a.g = L->gains.as<float>();
  a.ftab = L->float_table.p ? L->float_table.as<double>() : nullptr;
  a.K = L->K;
  a.L = L->L;
  a.E = L->in_dim * (L->col1 - L->col0);
  a.half_open = L->boundary_mode == LKG_BOUNDARY_HALF_OPEN;
  a.zs = L->oob_policy == LKG_OOB_ZERO_SPLINE;
  a.phi = L->value_repr == LKG_REPR_PHI;
  a.i8 = L->scheme == LKG_SCHEME_SYMMETRIC;
  a.hi_clip = a.half_open ? (double)std::nextafterf(L->knots[L->K], -INFINITY) : (double)L->knots[L->K];
  for (int k = 0; k <= L->K; k++) a.kn[k] = (double)L->knots[k];
  return a;
}

SpecRef spec_ref(const lkg_spec* S) {
  SpecRef s{};
  std::vector<double> ext;
  lkg::knot_grid(S->breakpoints, S->degree, ext);
  if ((int)ext.size() > kMaxT || S->degree > kMaxP) throw lkg::Error{LKG_ERR_CONFIG, "element primitives: grid too large"};
  s.coeffs = S->coeffs.as<double>();
  s.g = S->gains.as<double>();
  s.R = S->K + S->degree;
  s.p = S->degree;
  s.nT = (int)ext.size();
  s.E = S->in_dim * (S->col1 - S->col0);
  for (size_t k = 0; k < ext.size(); k++) s.T[k] = ext[k];
  return s;
}

unsigned blocks(int64_t n) { return (unsigned)((n + 255) / 256); }

}  // namespace

namespace lkg {

void launch_coords64(lkg_ctx* ctx, const lkg_layer* L, const double* x, int64_t n, uint8_t* in, double* xc,
                     int32_t* k, int32_t* l0, int32_t* l1, double* w) {
  coords_kernel<<<blocks(n), 256, 0, ctx->stream>>>(layer_ref(L), x, n, in, xc, k, l0, l1, w);
  LKG_CUDA(cudaGetLastError());
  ctx->launches++;
}

void launch_lut_eval(lkg_ctx* ctx, const lkg_layer* L, const int32_t* e, const double* x, int64_t n, double* value,
                     uint8_t* was_oob, double* phi, int* flags) {
  lut_eval_kernel<<<blocks(n), 256, 0, ctx->stream>>>(layer_ref(L), e, x, n, value, was_oob, phi, flags);
  LKG_CUDA(cudaGetLastError());
  ctx->launches++;
}

void launch_basis(lkg_ctx* ctx, const std::vector<double>& bp, int degree, const double* x, int64_t n,
                  double* out) {
  SpecRef s{};
  std::vector<double> ext;
  knot_grid(bp, degree, ext);
  if ((int)ext.size() > kMaxT || degree > kMaxP) throw Error{LKG_ERR_CONFIG, "element primitives: grid too large"};
  s.R = (int)bp.size() - 1 + degree;
  s.p = degree;
  s.nT = (int)ext.size();
  for (size_t k = 0; k < ext.size(); k++) s.T[k] = ext[k];
  basis_kernel<<<blocks(n), 256, 0, ctx->stream>>>(s, x, n, out);
  LKG_CUDA(cudaGetLastError());
  ctx->launches++;
}

void launch_edge_phi(lkg_ctx* ctx, const lkg_spec* S, const int32_t* e, const double* x, int64_t n, double* phi,
                     int* flags) {
  edge_phi_kernel<<<blocks(n), 256, 0, ctx->stream>>>(spec_ref(S), e, x, n, phi, flags);
  LKG_CUDA(cudaGetLastError());
  ctx->launches++;
}

void launch_quantize(lkg_ctx* ctx, const double* v, int64_t nseg, int L, int asym, int32_t* q, double* scale,
                     double* ymin, int* flags) {
  quantize_kernel<<<blocks(nseg), 256, 0, ctx->stream>>>(v, nseg, L, asym, q, scale, ymin, flags);
  LKG_CUDA(cudaGetLastError());
  ctx->launches++;
}

}  // namespace lkg
