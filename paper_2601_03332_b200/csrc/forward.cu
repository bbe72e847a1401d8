// forward.cu — K2: LUT-KAN layer forward (lut_layer_forward_batch → forward_quant,
// proj/core/src/runtime.cpp:135-285).
//
// Per (row s, input i) the 5-step coordinate pipeline runs once (runtime.cpp:170-190):
// finite check, in-range mask, clip (hi_clip = nextafterf(t_K, -inf) at f32 width for
// half_open), linear segment scan, u/z/l0/l1/w, mask folded into the weights, SiLU of
// the clipped (clip_x) or raw (zero_spline) input. Segment index and mask are
// computed with fp32 compares against the stored fp32 knots, which is exactly the
// reference's f64 comparison of the same values. Per (s, i, j) the table walk gathers
// two codes, dequantizes, interpolates and accumulates y_j = sum_i phi_ij in f64.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>

#include "lkg_internal.h"

namespace {

constexpr int kThreads = 256;
constexpr int kMaxK = 64;

struct FwdArgs {
  const float* X;
  int64_t rows;
  int32_t x_blk;        // 0: row-major [rows, d]; >0: rank-major column blocks
  float* Y;             // [rows, mc]
  const uint8_t* q;     // [E, K, L]
  const float* scale;   // [E, K]
  const float* ymin;    // [E, K]
  const float* cb;      // [E] out*base (spline_component)
  const float* cs;      // [E] out*spline
  const double* ft;     // float table (debug artifacts) or null
  unsigned long long* counters;  // {oob_samples, oob_inputs, nonfinite, -}
  int32_t d, mc, K, L, half_open, JT, RB;
  float lo, hi, hi_clip;
  float knots[kMaxK + 1];
};

__device__ __forceinline__ float load_x(const FwdArgs& a, int64_t r, int i) {
  if (a.x_blk <= 0) return a.X[r * a.d + i];
  const int b = i / a.x_blk;
  return a.X[(int64_t)b * a.rows * a.x_blk + r * a.x_blk + (i - b * a.x_blk)];
}

__device__ __forceinline__ float silu_f(float x) { return x / (1.0f + expf(-x)); }

// Steps 1-4 of the 5-step pipeline for one coordinate (runtime.cpp:170-190). k and the
// mask come from fp32 compares of fp32 values (exactly the reference's f64 compares);
// u, z, l0, w are formed in f64 exactly as runtime.cpp:178-181.
struct Coord {
  int k, l0, l1;
  float w0m, w1m, bx;
  bool in, finite;
};

template <bool ZS>
__device__ __forceinline__ Coord coord_of(const FwdArgs& a, float x) {
  Coord c;
  c.finite = isfinite(x);
  c.in = a.lo <= x && (a.half_open ? x < a.hi : x <= a.hi);
  const float xp = x < a.lo ? a.lo : (x > a.hi_clip ? a.hi_clip : x);
  int k = 0;
  for (int q = 1; q < a.K; q++) k += xp >= a.knots[q];
  const double u = ((double)xp - (double)a.knots[k]) / ((double)a.knots[k + 1] - (double)a.knots[k]);
  const double z = u * (double)(a.L - 1);
  int l0 = (int)floor(z);
  l0 = l0 < 0 ? 0 : (l0 > a.L - 1 ? a.L - 1 : l0);
  const double w1 = z - (double)l0;
  const float mask = (ZS && !c.in) ? 0.0f : 1.0f;
  c.k = k;
  c.l0 = l0;
  c.l1 = l0 + 1 < a.L ? l0 + 1 : a.L - 1;
  c.w0m = mask * (float)(1.0 - w1);
  c.w1m = mask * (float)w1;
  c.bx = silu_f(ZS ? x : xp);  // clip_x clips the base branch too (runtime.cpp:189)
  return c;
}

template <bool ZS>
__global__ void coords_kernel(FwdArgs a, const float* x, int64_t n, int32_t* in_range, int32_t* k, int32_t* l0) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  const Coord c = coord_of<ZS>(a, x[t]);
  if (in_range) in_range[t] = c.in;
  if (k) k[t] = c.k;
  if (l0) l0[t] = c.l0;
}

struct CoordArgs {
  lkg::CoordConst cc;
  float4 ktab[lkg::kMaxKT];
};

__global__ void coords_tiled_kernel(const __grid_constant__ CoordArgs c, const float* x, int64_t n,
                                    int32_t* in_range, int32_t* k, int32_t* l0) {
  __shared__ float4 ktab[lkg::kMaxKT];
  __shared__ float2 kf[lkg::kMaxKT];
  for (int q = threadIdx.x; q < c.cc.K; q += blockDim.x) {
    ktab[q] = c.ktab[q];
    kf[q] = make_float2(c.ktab[q].x, c.ktab[q].y);
  }
  __syncthreads();
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  const lkg::Coord co = lkg::lut_coords_fast(c.cc, ktab, kf, x[t]);  // the table walk's own path
  if (in_range) in_range[t] = co.in;
  if (k) k[t] = co.k;
  if (l0) l0[t] = co.l0;
}

template <bool SR, bool ZS, bool I8, bool FT>
__global__ void __launch_bounds__(kThreads) fwd_simple(FwdArgs a) {
  // coordinate scratch for RB rows x JT inputs
  __shared__ int s_k[kThreads], s_l0[kThreads], s_l1[kThreads];
  __shared__ float s_w0[kThreads], s_w1[kThreads], s_bx[kThreads];
  __shared__ int s_rowoob[kThreads];
  __shared__ unsigned long long s_oob_inputs;
  const int t = threadIdx.x;
  const int r = t / a.JT, jt = t - r * a.JT;
  const int64_t row = (int64_t)blockIdx.x * a.RB + r;
  const int j = blockIdx.y * a.JT + jt;
  const bool count = blockIdx.y == 0;
  if (t < a.RB) s_rowoob[t] = 0;
  if (t == 0) s_oob_inputs = 0;
  double acc = 0.0;
  for (int c0 = 0; c0 < a.d; c0 += a.JT) {
    __syncthreads();
    {  // phase 1: coordinates of (row, i = c0 + jt)
      const int i = c0 + jt;
      if (row < a.rows && i < a.d) {
        const float x = load_x(a, row, i);
        const Coord c = coord_of<ZS>(a, x);
        if (!c.finite) atomicExch(a.counters + 2, 1ull);
        const bool in = c.in;
        s_k[t] = c.k;
        s_l0[t] = c.l0;
        s_l1[t] = c.l1;
        s_w0[t] = c.w0m;
        s_w1[t] = c.w1m;
        s_bx[t] = SR ? c.bx : 0.0f;
        if (!in && count) {
          atomicOr(&s_rowoob[r], 1);
          atomicAdd(&s_oob_inputs, 1ull);
        }
      }
    }
    __syncthreads();
    if (row < a.rows && j < a.mc) {  // phase 2: table walk over the chunk
      const int n = min(a.JT, a.d - c0);
      const int cbase = r * a.JT;
      for (int ii = 0; ii < n; ii++) {
        const int i = c0 + ii;
        const int64_t e = (int64_t)i * a.mc + j;
        const int64_t cell = e * a.K + s_k[cbase + ii];
        const int64_t off = cell * a.L;
        float v;
        if (FT) {
          v = (float)((double)s_w0[cbase + ii] * a.ft[off + s_l0[cbase + ii]] +
                      (double)s_w1[cbase + ii] * a.ft[off + s_l1[cbase + ii]]);
        } else {
          const float q0 = I8 ? (float)(int8_t)a.q[off + s_l0[cbase + ii]] : (float)a.q[off + s_l0[cbase + ii]];
          const float q1 = I8 ? (float)(int8_t)a.q[off + s_l1[cbase + ii]] : (float)a.q[off + s_l1[cbase + ii]];
          const float sc = a.scale[cell], ym = a.ymin[cell];
          v = s_w0[cbase + ii] * (ym + sc * q0) + s_w1[cbase + ii] * (ym + sc * q1);
        }
        const float term = SR ? a.cb[e] * s_bx[cbase + ii] + a.cs[e] * v : v;
        acc += (double)term;
      }
    }
  }
  if (row < a.rows && j < a.mc) a.Y[row * a.mc + j] = (float)acc;
  __syncthreads();
  if (count && t < a.RB && (int64_t)blockIdx.x * a.RB + t < a.rows && s_rowoob[t])
    atomicAdd(a.counters + 0, 1ull);
  if (count && t == 0 && s_oob_inputs) atomicAdd(a.counters + 1, s_oob_inputs);
}

__global__ void fuse_gains_kernel(const float* gains, float* cbcs, int64_t E) {
  // runtime.cpp:263-273: cb = out*base, cs = out*spline (in f64, then narrowed)
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= E) return;
  const double bs = gains[e], ss = gains[E + e], os = gains[2 * E + e];
  cbcs[e] = (float)(os * bs);
  cbcs[E + e] = (float)(os * ss);
}

template <bool SR, bool ZS, bool I8, bool FT>
void launch_t(cudaStream_t st, dim3 g, const FwdArgs& a) {
  fwd_simple<SR, ZS, I8, FT><<<g, kThreads, 0, st>>>(a);
}

}  // namespace

namespace lkg {

void launch_fuse_gains(lkg_ctx* ctx, lkg_layer* L) {
  if (L->value_repr != LKG_REPR_SPLINE_COMPONENT) return;
  const int64_t E = (int64_t)L->in_dim * (L->col1 - L->col0);
  L->cbcs.alloc(sizeof(float) * 2 * E);
  fuse_gains_kernel<<<(unsigned)((E + 255) / 256), 256, 0, ctx->stream>>>(L->gains.as<float>(),
                                                                         L->cbcs.as<float>(), E);
  LKG_CUDA(cudaGetLastError());
  ctx->launches++;
}


static FwdArgs layer_args(const lkg_layer* L) {
  if (L->K > kMaxK) throw Error{LKG_ERR_CONFIG, "segment count above kernel limit"};
  FwdArgs a{};
  a.K = L->K;
  a.L = L->L;
  a.half_open = L->boundary_mode == LKG_BOUNDARY_HALF_OPEN;
  for (int k = 0; k <= L->K; k++) a.knots[k] = L->knots[k];
  a.lo = L->knots[0];
  a.hi = L->knots[L->K];
  a.hi_clip = a.half_open ? std::nextafterf(a.hi, -INFINITY) : a.hi;
  return a;
}

void launch_coords(lkg_ctx* ctx, const lkg_layer* L, const float* x, int64_t n, int32_t* in_range, int32_t* k,
                   int32_t* l0) {
  if (n <= 0) return;
  if (L->geom.tile_bytes > 0) {  // the tiled / small kernels' coordinate path (coords.cuh)
    CoordArgs c{};
    fill_coord_const(L, c.cc, c.ktab);
    coords_tiled_kernel<<<(unsigned)((n + 255) / 256), 256, 0, ctx->stream>>>(c, x, n, in_range, k, l0);
    LKG_CUDA(cudaGetLastError());
    ctx->launches++;
    return;
  }
  FwdArgs a = layer_args(L);
  const unsigned g = (unsigned)((n + 255) / 256);
  if (L->oob_policy == LKG_OOB_ZERO_SPLINE) coords_kernel<true><<<g, 256, 0, ctx->stream>>>(a, x, n, in_range, k, l0);
  else coords_kernel<false><<<g, 256, 0, ctx->stream>>>(a, x, n, in_range, k, l0);
  LKG_CUDA(cudaGetLastError());
  ctx->launches++;
}

void launch_forward(lkg_ctx* ctx, const lkg_layer* L, const float* X, int64_t rows, int32_t x_blk,
                    float* Y, int slot, bool count_oob) {
  if (rows <= 0) return;
  if (tiled_eligible(L)) {
    launch_forward_tiled(ctx, L, X, rows, x_blk, Y, slot);
    return;
  }
  FwdArgs a = layer_args(L);
  a.X = X;
  a.rows = rows;
  a.x_blk = x_blk;
  a.Y = Y;
  a.q = L->q.as<uint8_t>();
  a.scale = L->scale.as<float>();
  a.ymin = L->ymin.as<float>();
  const int64_t E = (int64_t)L->in_dim * (L->col1 - L->col0);
  a.cb = L->cbcs.p ? L->cbcs.as<float>() : nullptr;
  a.cs = L->cbcs.p ? L->cbcs.as<float>() + E : nullptr;
  a.ft = L->float_table.p ? L->float_table.as<double>() : nullptr;
  a.counters = ctx->counters.as<unsigned long long>() + 4 * slot;
  a.d = L->in_dim;
  a.mc = L->col1 - L->col0;
  int jt = 1;
  while (jt < a.mc && jt < kThreads) jt <<= 1;
  a.JT = jt;
  a.RB = kThreads / jt;
  dim3 g((unsigned)((rows + a.RB - 1) / a.RB), (unsigned)((a.mc + jt - 1) / jt));
  (void)count_oob;
  const bool sr = L->value_repr == LKG_REPR_SPLINE_COMPONENT, zs = L->oob_policy == LKG_OOB_ZERO_SPLINE;
  const bool i8 = L->scheme == LKG_SCHEME_SYMMETRIC, ft = a.ft != nullptr;
  const int sel = (sr << 3) | (zs << 2) | (i8 << 1) | (int)ft;
  switch (sel) {
#define CASE(S) \
  case S: launch_t<(S >> 3) & 1, (S >> 2) & 1, (S >> 1) & 1, S & 1>(ctx->stream, g, a); break;
    CASE(0) CASE(1) CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7)
    CASE(8) CASE(9) CASE(10) CASE(11) CASE(12) CASE(13) CASE(14) CASE(15)
#undef CASE
  }
  LKG_CUDA(cudaGetLastError());
  ctx->launches++;
}

}  // namespace lkg
