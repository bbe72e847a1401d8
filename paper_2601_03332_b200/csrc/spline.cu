// spline.cu — K3: same-backend B-spline forward, the paper's "honest baseline"
// (layer_forward_batch → forward_optimized, proj/core/src/spline.cpp:145-187).
//
// spline_simple is the any-grid, any-degree kernel and the PRECISE one: everything in f64, in the
// reference's own expressions. Per (row, i): Cox-de Boor basis of x over the f64 extended knots
// (spline.cpp:69-83), evaluated locally — only the degree+1 functions that can be non-zero at x —
// plus silu(x) of the UNCLIPPED input (spline.cpp:166; the float model has no OOB handling: outside
// the extended knots every basis value is 0). Per (row, i, j): sp = sum_r c_r B_r(x);
// y_j += os*(bs*silu(x) + ss*sp) (spline.cpp:174) with the f64 coefficients and gains.
// The fast kernels (spline_tc.cu, spline_tiled.cu) carry fp32 terms and fp32 tile partial sums: a
// spec whose terms are large (spline_bound_kernel: the estimate of that rounding above kFastErrMax —
// a 600-seed fuzz campaign found d = 300 specs with terms of ~10 at 1.5-2.2e-5) comes here instead.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "lkg_internal.h"

namespace {

constexpr int kThreads = 256;
constexpr int kMaxP = 7;
constexpr int kMaxT = 96;

struct SplArgs {
  const float* X;
  int64_t rows;
  float* Y;
  const double* coeffs;  // [E, R] f64
  const double* gains;   // [3][E] f64: base, spline, out
  int32_t d, mc, R, p, nT, JT, RB;
  double T[kMaxT];
};

__device__ __forceinline__ double silu_d(double x) { return x / (1.0 + exp(-x)); }  // spline.cpp:105-108

__global__ void __launch_bounds__(kThreads) spline_simple(const __grid_constant__ SplArgs a) {
  __shared__ double s_b[kThreads][kMaxP + 1];
  __shared__ int s_r0[kThreads];
  __shared__ double s_bx[kThreads];
  const int t = threadIdx.x;
  const int r = t / a.JT, jt = t - r * a.JT;
  const int64_t row = (int64_t)blockIdx.x * a.RB + r;
  const int j = blockIdx.y * a.JT + jt;
  const int p = a.p, n0 = a.nT - 1;
  const int64_t E = (int64_t)a.d * a.mc;
  double acc = 0.0;
  for (int c0 = 0; c0 < a.d; c0 += a.JT) {
    __syncthreads();
    const int i = c0 + jt;
    if (row < a.rows && i < a.d) {
      const double x = (double)a.X[row * a.d + i];
      // span mu with T[mu] <= x < T[mu+1]; none -> every basis value is 0
      int mu = -1;
      for (int q = 0; q < n0; q++)
        if (a.T[q] <= x && x < a.T[q + 1]) mu = q;
      double b[kMaxP + 1];
      for (int q = 0; q <= kMaxP; q++) b[q] = 0.0;
      // b[o] holds buf[mu - p + o] of the reference recursion (spline.cpp:72-82)
      if (mu >= 0) {
        b[p] = 1.0;
        for (int q = 1; q <= p; q++) {
          for (int o = p - q; o <= p; o++) {
            const int rr = mu - p + o;
            if (rr < 0 || rr >= n0 - q) {
              b[o] = 0.0;
              continue;
            }
            double accq = 0.0;
            const double d1 = a.T[rr + q] - a.T[rr];
            if (d1 > 0.0) accq += (x - a.T[rr]) / d1 * b[o];
            const double d2 = a.T[rr + q + 1] - a.T[rr + 1];
            if (d2 > 0.0 && o + 1 <= p) accq += (a.T[rr + q + 1] - x) / d2 * b[o + 1];
            b[o] = accq;
          }
        }
      }
      for (int q = 0; q <= p; q++) s_b[t][q] = b[q];
      s_r0[t] = mu - p;  // may be negative or >= R at the ends: masked in phase 2
      s_bx[t] = silu_d(x);
    }
    __syncthreads();
    if (row < a.rows && j < a.mc) {
      const int n = min(a.JT, a.d - c0);
      const int cb0 = r * a.JT;
      for (int ii = 0; ii < n; ii++) {
        const int64_t e = (int64_t)(c0 + ii) * a.mc + j;
        const int r0 = s_r0[cb0 + ii];
        double sp = 0.0;
        if (r0 > -p - 1) {
          const double* c = a.coeffs + e * a.R;
          for (int q = 0; q <= p; q++) {
            const int rr = r0 + q;
            if (rr >= 0 && rr < a.R) sp += c[rr] * s_b[cb0 + ii][q];
          }
        }
        acc += a.gains[2 * E + e] * (a.gains[e] * s_bx[cb0 + ii] + a.gains[E + e] * sp);
      }
    }
  }
  if (row < a.rows && j < a.mc) a.Y[row * a.mc + j] = (float)acc;
}

// Spline-forward operands: fp32 coefficients and fused gains out*base, out*spline
// (forward_optimized computes os*(bs*b + ss*sp), spline.cpp:174; fused in f64 here).
__global__ void spec_prepare_kernel(const double* coeffs, const double* gains, float* c32, float* g32,
                                    int64_t n_coeffs, int64_t E) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t < n_coeffs) c32[t] = __double2float_rn(coeffs[t]);
  if (t < E) {
    const double bs = gains[t], ss = gains[E + t], os = gains[2 * E + t];
    g32[t] = __double2float_rn(os * bs);
    g32[E + t] = __double2float_rn(os * ss);
  }
}

// Scale of the fast kernels' rounding, per output column j: sum over inputs i of the squared largest
// term edge (i, j) can contribute, (|os ss| max_r |c_r| + |os bs| silu_max)^2 (a B-spline is a convex
// combination of its coefficients); one thread per edge, f64 atomics.
__global__ void spline_bound_kernel(const double* coeffs, const double* gains, int64_t E, int32_t mc, int32_t R,
                                    double silu_max, double* acc) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= E) return;
  double cmax = 0.0;
  for (int r = 0; r < R; r++) cmax = fmax(cmax, fabs(coeffs[e * R + r]));
  const double os = fabs(gains[2 * E + e]);
  const double term = os * (fabs(gains[E + e]) * cmax + fabs(gains[e]) * silu_max);
  atomicAdd(acc + (e % mc), term * term);
}

}  // namespace

namespace lkg {

// fp32 terms and fp32 partial sums over a tile of 8 inputs (the fast kernels): each of the d adds
// rounds at the ulp of a tile partial, |partial| ~ t sqrt(8) for terms of rms t -> ~2^-24 t sqrt(8 d / 3).
static constexpr double kFastErrMax = 3e-6;

static double spline_fast_err(lkg_ctx* ctx, lkg_spec* S) {
  if (S->fast_err >= 0.0) return S->fast_err;
  const int mc = S->col1 - S->col0;
  const int64_t E = (int64_t)S->in_dim * mc;
  DBuf acc;
  acc.alloc(sizeof(double) * mc);
  LKG_CUDA(cudaMemsetAsync(acc.p, 0, acc.bytes, ctx->stream));
  auto silu = [](double x) { return x / (1.0 + std::exp(-x)); };
  // (the input is not clipped; the bound takes the breakpoint range as its typical extent)
  const double lo = S->breakpoints.front(), hi = S->breakpoints.back(), ext = 0.0;
  const double silu_max = std::max({std::fabs(silu(lo - ext)), std::fabs(silu(hi + ext)), 0.2785});
  spline_bound_kernel<<<(unsigned)((E + 255) / 256), 256, 0, ctx->stream>>>(
      S->coeffs.as<double>(), S->gains.as<double>(), E, mc, S->K + S->degree, silu_max, acc.as<double>());
  LKG_CUDA(cudaGetLastError());
  ctx->launches++;
  std::vector<double> h(mc);
  LKG_CUDA(cudaMemcpyAsync(h.data(), acc.p, acc.bytes, cudaMemcpyDeviceToHost, ctx->stream));
  LKG_CUDA(cudaStreamSynchronize(ctx->stream));
  double t2 = 0.0;
  for (double v : h) t2 = std::max(t2, v);
  // rms term t = sqrt(t2 / (3 d)); d roundings at the ulp of a partial sum of 8 terms (f64 flush per
  // tile, d > 256) or of up to d terms (fp32 accumulation)
  S->fast_err = 0x1p-24 * std::sqrt(t2 / 3.0) * std::sqrt(S->in_dim > 256 ? 8.0 : (double)S->in_dim);
  static const bool verbose = getenv("LKG_VERBOSE") != nullptr;
  if (verbose)
    fprintf(stderr, "lkg spline %dx%d K%d deg%d: fast_err %.3g\n", S->in_dim, mc, S->K, S->degree, S->fast_err);
  return S->fast_err;
}

void launch_spec_prepare(lkg_ctx* ctx, lkg_spec* S) {
  const int64_t E = (int64_t)S->in_dim * (S->col1 - S->col0);
  const int64_t nc = E * (S->K + S->degree);
  S->coeffs32.alloc(sizeof(float) * nc);
  S->gains32.alloc(sizeof(float) * 2 * E);
  const int64_t n = nc > E ? nc : E;
  spec_prepare_kernel<<<(unsigned)((n + 255) / 256), 256, 0, ctx->stream>>>(
      S->coeffs.as<double>(), S->gains.as<double>(), S->coeffs32.as<float>(), S->gains32.as<float>(), nc, E);
  LKG_CUDA(cudaGetLastError());
  ctx->launches++;
}

void launch_spline(lkg_ctx* ctx, const lkg_spec* S, const float* X, int64_t rows, float* Y,
                   const float* /*d_ext*/) {
  if (rows <= 0) return;
  static const bool env_simple = getenv("LKG_SPLINE_SIMPLE") != nullptr;  // test hook
  // (the bound needs the f64 operands of the spec; a spec uploaded without them stays on the fast kernels)
  const bool force_simple =
      env_simple || (S->coeffs.p && S->gains.p && spline_fast_err(ctx, const_cast<lkg_spec*>(S)) > kFastErrMax);
  // tensor-core GEMM form first (spline_tc.cu) unless the context asks for the SIMT kernels
  // (lkg_ctx_set_spline_kernel) or LKG_SPLINE_SIMT=1 (experiment hook)
  static const char* simt = getenv("LKG_SPLINE_SIMT");
  const bool no_tc = (simt && simt[0] == '1') || ctx->spline_kernel == LKG_SPLINE_SIMT;
  if (!force_simple && !no_tc && launch_spline_tc(ctx, S, X, rows, Y)) return;
  if (!force_simple && launch_spline_tiled(ctx, S, X, rows, Y)) return;
  std::vector<double> ext;
  knot_grid(S->breakpoints, S->degree, ext);
  if ((int)ext.size() > kMaxT || S->degree > kMaxP)
    throw Error{LKG_ERR_CONFIG, "spline grid above kernel limits"};
  SplArgs a{};
  a.X = X;
  a.rows = rows;
  a.Y = Y;
  if (!S->coeffs.p || !S->gains.p) throw Error{LKG_ERR_CONFIG, "spline forward needs the spec's coefficients"};
  a.coeffs = S->coeffs.as<double>();
  a.gains = S->gains.as<double>();
  a.d = S->in_dim;
  a.mc = S->col1 - S->col0;
  a.R = S->K + S->degree;
  a.p = S->degree;
  a.nT = (int)ext.size();
  for (size_t q = 0; q < ext.size(); q++) a.T[q] = ext[q];
  int jt = 1;
  while (jt < a.mc && jt < kThreads) jt <<= 1;
  a.JT = jt;
  a.RB = kThreads / jt;
  dim3 g((unsigned)((rows + a.RB - 1) / a.RB), (unsigned)((a.mc + jt - 1) / jt));
  spline_simple<<<g, kThreads, 0, ctx->stream>>>(a);
  LKG_CUDA(cudaGetLastError());
  ctx->launches++;
}

}  // namespace lkg
