// eval.cu — GPU eval_accuracy (reference metrics.cpp:30-103).
//
// Every (sample, input, edge) evaluation contributes |lut_eval_phi - eval_edge_phi|:
//   * the spline side is basis_values (spline.cpp:69-94) over the spec's extended knots and
//     out*(base*silu(x) + spline*sum_r c_r B_r(x)) (metrics.cpp:62-68), all in f64;
//   * the table side is lut_eval_phi (runtime.cpp:96-120): in_range / safe_clip / segment_index
//     / interp_coords over the artifact's f32 knots widened to f64, two dequantized cells, the
//     zero_spline mask, and the base branch at x' (clip_x) or x (zero_spline).
// Both are evaluated with the reference's own expressions in the reference's order; this file is
// built with -fmad=false, so no product is contracted into an FMA and the per-evaluation errors
// equal the reference's up to exp() (CUDA vs glibc, <= 1 ulp). The non-zero basis window is
// evaluated locally (degree+1 functions): the reference's full recursion adds exact zeros
// outside it, so the window values are bit-identical.
// Buckets (metrics.cpp:55-79): OOB when the artifact's In(x) is false, in range when
// t_0 <= x < t_K, boundary otherwise (closed mode, x == t_K). Sums are f64 atomics (their order
// is not the reference's sequential order: mae agrees to ~1e-15 relative); maxima and counts are
// exact.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <vector>

#include "f64ref.cuh"
#include "lkg_internal.h"

namespace {

constexpr int kThreads = 256;
using lkg::f64ref::kMaxK;
using lkg::f64ref::kMaxP;
using lkg::f64ref::kMaxT;

struct EvalArgs {
  const void* X;         // f32, or f64 (x_f64: the reference's Matrix values unrounded)
  int32_t x_f64;
  int64_t rows;
  int32_t d, m, R, p, nT, K, L;
  int32_t half_open, zs, phi, i8, JT, RB;
  const double* coeffs;  // spec [E, R]
  const double* sg;      // spec gains [3][E]: base, spline, out
  const uint8_t* q;      // artifact [E, K, L]
  const float* scale;    // [E, K]
  const float* ymin;     // [E, K]
  const float* ag;       // artifact gains [3][E] (spline_component)
  const double* ftab;    // float_table [E, K, L] or null
  double lo, hi, hi_clip;
  double T[kMaxT];       // spec extended knots
  double kn[kMaxK + 1];  // artifact knots (f32 widened)
  double* dsum;                // [2]: in-range, OOB error sums
  unsigned long long* u;       // [0,1] max bits (in, oob), [2..5] n_in, n_oob, n_boundary, n_oob_samples, [6] nonfinite
};

__device__ __forceinline__ double fetch(const EvalArgs& a, int64_t cell, int l) {  // runtime.cpp:81-88
  return lkg::f64ref::fetch(a.q, a.scale, a.ymin, a.ftab, a.i8, a.L, cell, l);
}

__global__ void __launch_bounds__(kThreads) eval_kernel(const __grid_constant__ EvalArgs a) {
  __shared__ double s_b[kThreads][kMaxP + 1];
  __shared__ double s_base[kThreads], s_w[kThreads], s_bxl[kThreads];
  __shared__ int s_r0[kThreads], s_k[kThreads], s_l0[kThreads], s_l1[kThreads], s_fl[kThreads];
  __shared__ int s_rowoob[kThreads];
  const int t = threadIdx.x;
  const int r = t / a.JT, jt = t - r * a.JT;
  const int64_t row = (int64_t)blockIdx.x * a.RB + r;
  const int j = blockIdx.y * a.JT + jt;
  const int p = a.p;
  const int64_t E = (int64_t)a.d * a.m;
  double sum_in = 0.0, max_in = 0.0, sum_oob = 0.0, max_oob = 0.0;
  unsigned long long n_in = 0, n_oob = 0, n_bd = 0;
  bool nonfinite = false;
  s_rowoob[t] = 0;
  for (int c0 = 0; c0 < a.d; c0 += a.JT) {
    __syncthreads();
    const int i = c0 + jt;
    if (row < a.rows && i < a.d) {
      const double x = a.x_f64 ? static_cast<const double*>(a.X)[row * a.d + i]
                               : (double)static_cast<const float*>(a.X)[row * a.d + i];
      int fl = 0;
      if (!isfinite(x)) nonfinite = true;
      const bool in = a.half_open ? (a.lo <= x && x < a.hi) : (a.lo <= x && x <= a.hi);  // runtime.cpp:71-75
      const bool interior = a.lo <= x && x < a.hi;
      fl = (in ? 1 : 0) | (interior ? 2 : 0);
      if (!in) s_rowoob[r] = 1;
      // spline basis window (spline.cpp:69-83): b[o] = B_{r0+o}(x)
      double b[kMaxP + 1];
      int r0;
      lkg::f64ref::basis_window(a.T, a.nT, p, x, b, &r0);
      for (int o = 0; o <= kMaxP; o++) s_b[t][o] = b[o];
      s_r0[t] = r0;
      s_base[t] = lkg::f64ref::silu(x);  // base_fn(silu, x) on the raw input (metrics.cpp:60)
      // table coordinates (runtime.cpp:45-69)
      const lkg::f64ref::Coord64 c = lkg::f64ref::coords(a.kn, a.K, a.L, a.half_open, a.hi_clip, x);
      const double xp = c.xp;
      s_k[t] = c.k;
      s_l0[t] = c.l0;
      s_l1[t] = c.l1;
      s_w[t] = c.w;
      s_bxl[t] = a.phi ? 0.0 : lkg::f64ref::silu(a.zs ? x : xp);  // runtime.cpp:113-115
      s_fl[t] = fl;
    }
    __syncthreads();
    if (row < a.rows && j < a.m) {
      const int n = min(a.JT, a.d - c0);
      const int cb0 = r * a.JT;
      for (int ii = 0; ii < n; ii++) {
        const int s = cb0 + ii;
        const int64_t e = (int64_t)(c0 + ii) * a.m + j;
        // spline reference (metrics.cpp:62-68)
        double sp = 0.0;
        const int r0 = s_r0[s];
        for (int o = 0; o <= p; o++) {
          const int rr = r0 + o;
          if (rr >= 0 && rr < a.R) sp += a.coeffs[e * a.R + rr] * s_b[s][o];
        }
        const double ref = a.sg[2 * E + e] * (a.sg[e] * s_base[s] + a.sg[E + e] * sp);
        // lut_eval_phi (runtime.cpp:96-120)
        const int fl = s_fl[s];
        const int64_t cell = e * a.K + s_k[s];
        const double w = s_w[s];
        double v = (1.0 - w) * fetch(a, cell, s_l0[s]) + w * fetch(a, cell, s_l1[s]);
        if (a.zs && !(fl & 1)) v = 0.0;
        const double lut =
            a.phi ? v
                  : (double)a.ag[2 * E + e] * ((double)a.ag[e] * s_bxl[s] + (double)a.ag[E + e] * v);
        const double err = fabs(lut - ref);
        if (!(fl & 1)) {
          sum_oob += err;
          max_oob = fmax(max_oob, err);
          n_oob++;
        } else if (fl & 2) {
          sum_in += err;
          max_in = fmax(max_in, err);
          n_in++;
        } else {
          n_bd++;
        }
      }
    }
  }
  // block partials -> global
  for (int o = 16; o; o >>= 1) {
    sum_in += __shfl_xor_sync(0xffffffffu, sum_in, o);
    sum_oob += __shfl_xor_sync(0xffffffffu, sum_oob, o);
    max_in = fmax(max_in, __shfl_xor_sync(0xffffffffu, max_in, o));
    max_oob = fmax(max_oob, __shfl_xor_sync(0xffffffffu, max_oob, o));
    n_in += __shfl_xor_sync(0xffffffffu, n_in, o);
    n_oob += __shfl_xor_sync(0xffffffffu, n_oob, o);
    n_bd += __shfl_xor_sync(0xffffffffu, n_bd, o);
  }
  const bool nf = __any_sync(0xffffffffu, nonfinite);
  if ((t & 31) == 0) {
    if (sum_in != 0.0) atomicAdd(a.dsum + 0, sum_in);
    if (sum_oob != 0.0) atomicAdd(a.dsum + 1, sum_oob);
    // non-negative doubles order like their bit patterns
    atomicMax(a.u + 0, (unsigned long long)__double_as_longlong(max_in));
    atomicMax(a.u + 1, (unsigned long long)__double_as_longlong(max_oob));
    if (n_in) atomicAdd(a.u + 2, n_in);
    if (n_oob) atomicAdd(a.u + 3, n_oob);
    if (n_bd) atomicAdd(a.u + 4, n_bd);
    if (nf) atomicExch(a.u + 6, 1ull);
  }
  // samples with at least one masked input: once per row (column block 0, first lane of the row)
  if (blockIdx.y == 0 && jt == 0 && row < a.rows && s_rowoob[r]) atomicAdd(a.u + 5, 1ull);
}

}  // namespace

namespace lkg {

void launch_eval(lkg_ctx* ctx, const lkg_spec* S, const lkg_layer* L, const void* X, bool x_f64, int64_t rows,
                 double* dsum, unsigned long long* u) {
  EvalArgs a{};
  std::vector<double> ext;
  knot_grid(S->breakpoints, S->degree, ext);
  if ((int)ext.size() > kMaxT || S->degree > kMaxP || L->K > kMaxK)
    throw Error{LKG_ERR_CONFIG, "eval_accuracy: grid above kernel limits"};
  if (!L->q.p && !L->float_table.p)
    throw Error{LKG_ERR_CONFIG, "eval_accuracy needs the reference-layout table (layer stored tiles-only)"};
  a.X = X;
  a.x_f64 = x_f64;
  a.rows = rows;
  a.d = S->in_dim;
  a.m = S->col1 - S->col0;
  a.R = S->K + S->degree;
  a.p = S->degree;
  a.nT = (int)ext.size();
  a.K = L->K;
  a.L = L->L;
  a.half_open = L->boundary_mode == LKG_BOUNDARY_HALF_OPEN;
  a.zs = L->oob_policy == LKG_OOB_ZERO_SPLINE;
  a.phi = L->value_repr == LKG_REPR_PHI;
  a.i8 = L->scheme == LKG_SCHEME_SYMMETRIC;
  a.coeffs = S->coeffs.as<double>();
  a.sg = S->gains.as<double>();
  a.q = L->q.as<uint8_t>();
  a.scale = L->scale.as<float>();
  a.ymin = L->ymin.as<float>();
  a.ag = L->gains.as<float>();
  a.ftab = L->float_table.p ? L->float_table.as<double>() : nullptr;
  a.lo = (double)L->knots[0];
  a.hi = (double)L->knots[L->K];
  a.hi_clip = a.half_open ? (double)std::nextafterf(L->knots[L->K], -INFINITY) : a.hi;  // runtime.cpp:45-51
  for (size_t s = 0; s < ext.size(); s++) a.T[s] = ext[s];
  for (int k = 0; k <= L->K; k++) a.kn[k] = (double)L->knots[k];
  a.dsum = dsum;
  a.u = u;
  int jt = 1;
  while (jt < a.m && jt < kThreads) jt <<= 1;
  a.JT = jt;
  a.RB = kThreads / jt;
  dim3 g((unsigned)((rows + a.RB - 1) / a.RB), (unsigned)((a.m + jt - 1) / jt));
  eval_kernel<<<g, kThreads, 0, ctx->stream>>>(a);
  LKG_CUDA(cudaGetLastError());
  ctx->launches++;
}

}  // namespace lkg
