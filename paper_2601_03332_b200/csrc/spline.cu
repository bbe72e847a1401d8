// spline.cu — K3: same-backend B-spline forward, the paper's "honest baseline"
// (layer_forward_batch → forward_optimized, proj/core/src/spline.cpp:145-187).
//
// Per (row, i): Cox-de Boor basis of x over the extended knots (spline.cpp:69-83),
// evaluated locally — only the degree+1 functions that can be non-zero at x — in
// fp32, plus silu(x) of the UNCLIPPED input (spline.cpp:166; the float model has no
// OOB handling: outside the extended knots every basis value is 0). Per (row, i, j):
// sp = sum_r c_r B_r(x); y_j += out*(base*silu(x) + spline*sp), fp32 terms with f64
// accumulation (<= 3e-6 against the f64 reference).
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>

#include "lkg_internal.h"

namespace {

constexpr int kThreads = 256;
constexpr int kMaxP = 7;
constexpr int kMaxT = 96;

struct SplArgs {
  const float* X;
  int64_t rows;
  float* Y;
  const float* coeffs;  // [E, R] fp32
  const float* cbcs;    // [2][E]: out*base, out*spline
  int32_t d, mc, R, p, nT, JT, RB;
  float T[kMaxT];
};

__device__ __forceinline__ float silu_f(float x) { return x / (1.0f + expf(-x)); }

__global__ void __launch_bounds__(kThreads) spline_simple(SplArgs a) {
  __shared__ float s_b[kThreads][kMaxP + 1];
  __shared__ int s_r0[kThreads];
  __shared__ float s_bx[kThreads];
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
      const float x = a.X[row * a.d + i];
      // span mu with T[mu] <= x < T[mu+1]; none -> every basis value is 0
      int mu = -1;
      for (int q = 0; q < n0; q++)
        if (a.T[q] <= x && x < a.T[q + 1]) mu = q;
      float b[kMaxP + 1];
      for (int q = 0; q <= kMaxP; q++) b[q] = 0.0f;
      // b[o] holds buf[mu - p + o] of the reference recursion (spline.cpp:72-82)
      if (mu >= 0) {
        b[p] = 1.0f;
        for (int q = 1; q <= p; q++) {
          for (int o = p - q; o <= p; o++) {
            const int rr = mu - p + o;
            if (rr < 0 || rr >= n0 - q) {
              b[o] = 0.0f;
              continue;
            }
            float accq = 0.0f;
            const float d1 = a.T[rr + q] - a.T[rr];
            if (d1 > 0.0f) accq += (x - a.T[rr]) / d1 * b[o];
            const float d2 = a.T[rr + q + 1] - a.T[rr + 1];
            if (d2 > 0.0f && o + 1 <= p) accq += (a.T[rr + q + 1] - x) / d2 * b[o + 1];
            b[o] = accq;
          }
        }
      }
      for (int q = 0; q <= p; q++) s_b[t][q] = b[q];
      s_r0[t] = mu - p;  // may be negative or >= R at the ends: masked in phase 2
      s_bx[t] = silu_f(x);
    }
    __syncthreads();
    if (row < a.rows && j < a.mc) {
      const int n = min(a.JT, a.d - c0);
      const int cb0 = r * a.JT;
      for (int ii = 0; ii < n; ii++) {
        const int64_t e = (int64_t)(c0 + ii) * a.mc + j;
        const int r0 = s_r0[cb0 + ii];
        float sp = 0.0f;
        if (r0 > -p - 1) {
          const float* c = a.coeffs + e * a.R;
          for (int q = 0; q <= p; q++) {
            const int rr = r0 + q;
            if (rr >= 0 && rr < a.R) sp += c[rr] * s_b[cb0 + ii][q];
          }
        }
        acc += (double)(a.cbcs[e] * s_bx[cb0 + ii] + a.cbcs[E + e] * sp);
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

}  // namespace

namespace lkg {

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
  static const bool force_simple = getenv("LKG_SPLINE_SIMPLE") != nullptr;  // test hook
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
  if (!S->coeffs32.p) launch_spec_prepare(ctx, const_cast<lkg_spec*>(S));
  a.coeffs = S->coeffs32.as<float>();
  a.cbcs = S->gains32.as<float>();
  a.d = S->in_dim;
  a.mc = S->col1 - S->col0;
  a.R = S->K + S->degree;
  a.p = S->degree;
  a.nT = (int)ext.size();
  for (size_t q = 0; q < ext.size(); q++) a.T[q] = (float)ext[q];
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
