// spline_tiled.cu — K3 on sm_100a: the same-backend B-spline forward ("honest baseline",
// layer_forward_batch -> forward_optimized, proj/core/src/spline.cpp:145-187), built like the LUT
// kernel (forward_tiled.cu) so the two are compared on equal footing.
//
//  * Uniform knots, degree 3 (all BASELINE grids): the extended knot vector (spline.cpp:8-27) is
//    uniform, so the 4 non-zero Cox-de Boor basis values at x are the uniform cubic B-spline
//    polynomials of u = frac((x - T_0)/h) (the recursion of spline.cpp:69-83 in closed form;
//    agreement ~1e-7, C2-continuous at knots). Outside the extended knots every basis value is 0
//    (the float model has no OOB handling, spline.cpp:165).
//  * Device layout (built once per spec): tiles of 8 inputs x 16 outputs,
//      C' [R][8 i_lo][20] f32   C' = f32(out*spline*c_r)       (80-byte rows: conflict-free)
//      CB [8][20]        f32   out*base
//    streamed through shared memory by TMA bulk copies (double-buffered, mbarriers); lanes own
//    rows and walk the 8 inputs of a tile in rotated order (conflict-free LDS.128 phases).
//  * Per (row, input, 16 outputs): y += sum_{t<4} b_t * C'[r0+t] + CB * silu(x) with FFMA2 pairs;
//    fp32 terms, f64 flush per tile when d > 256 (<= 3e-6).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>

#include "lkg_internal.h"
#include "tma.cuh"

namespace {

constexpr int G = 8, JB = 16, PROW = 80, kFp32MaxD = 256;
constexpr int RR = 2, NS = 2;  // 2 rows per lane; 16 warps (8 in f64 mode: 32 f64 accumulators)

struct SplArgs {
  const uint8_t* tiles;
  int64_t tile_bytes;
  int32_t n_ih, n_jb, cb_off, R, n0;
  const float* X;
  int64_t rows;
  int32_t d;
  float* Y;
  int32_t m;
  float t0, inv_h;  // first extended knot, 1/h
  int64_t n_items;
};

template <bool F64, int W>
__global__ void __launch_bounds__(W * 32, 1) spline_tiled(const __grid_constant__ SplArgs a) {
  extern __shared__ __align__(128) uint8_t smem[];
  constexpr int ROWS_W = 32 * RR, XS = ROWS_W + 4, NX = 4 * RR;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t tb = a.tile_bytes;
  uint8_t* stage = smem;
  float* xs = reinterpret_cast<float*>(smem + NS * tb) + warp * G * XS;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + NS * tb + W * G * XS * 4);
  if (tid == 0) {
    for (int s = 0; s < NS; s++) lkg::mbar_init(&full[s], 1);
    lkg::mbar_fence_init();
  }
  __syncthreads();
  // Balanced rows for one-j-block layers, as the LUT table walk (forward_tiled.cu): CTA b owns an
  // equal, 64-aligned row range walked in W*ROWS_W-row tiles.
  constexpr int64_t TILE_ROWS = W * ROWS_W;
  const bool bal = a.n_jb == 1;
  int64_t r_lo = 0, r_hi = a.rows;
  if (bal) {
    auto split = [&](int64_t b) -> int64_t {
      return b >= (int64_t)gridDim.x ? a.rows : (a.rows * b / (int64_t)gridDim.x) / 64 * 64;
    };
    r_lo = split(blockIdx.x);
    r_hi = split((int64_t)blockIdx.x + 1);
  }
  const int64_t n_local = bal ? (r_hi - r_lo + TILE_ROWS - 1) / TILE_ROWS
                              : (a.n_items > blockIdx.x ? (a.n_items - 1 - blockIdx.x) / gridDim.x + 1 : 0);
  const int64_t n_stages = n_local * a.n_ih;
  auto issue = [&](int64_t g) {
    const int64_t item = blockIdx.x + (g / a.n_ih) * gridDim.x;
    const int jb = (int)(item % a.n_jb), ih = (int)(g % a.n_ih);
    lkg::stage_copy(stage + (g % NS) * tb, a.tiles + ((int64_t)jb * a.n_ih + ih) * tb, tb, &full[g % NS]);
  };
  if (tid == 0)
    for (int64_t g = 0; g < NS && g < n_stages; g++) issue(g);
  const int xr_row = lane >> 2, xr_col = 2 * (lane & 3);
  int64_t g = 0;
  for (int64_t li = 0; li < n_local; li++) {
    const int64_t item = blockIdx.x + li * gridDim.x;
    const int64_t rt = item / a.n_jb;
    const int jb = bal ? 0 : (int)(item % a.n_jb);
    const int64_t row0 = bal ? r_lo + li * TILE_ROWS + warp * ROWS_W : rt * TILE_ROWS + warp * ROWS_W;
    const int64_t rows_left = r_hi - row0;
    float2 acc[RR][8];
    double acc64[F64 ? RR : 1][F64 ? 16 : 1];
#pragma unroll
    for (int r = 0; r < RR; r++) {
#pragma unroll
      for (int q = 0; q < 8; q++) acc[r][q] = make_float2(0.f, 0.f);
      if (F64)
#pragma unroll
        for (int q = 0; q < 16; q++) acc64[r][q] = 0.0;
    }
    float2 xr[NX];
#define SPL_LOAD_X(IH)                                                     \
  {                                                                        \
    const int i_ = (IH) * G + xr_col;                                      \
    const float* p_ = a.X + (row0 + xr_row) * a.d + i_;                    \
    _Pragma("unroll") for (int t = 0; t < NX; t++) {                       \
      float2 v_ = make_float2(0.f, 0.f);                                   \
      if (xr_row + 8 * t < rows_left) {                                    \
        const float* q_ = p_ + (int64_t)(8 * t) * a.d;                     \
        if (i_ < a.d) v_.x = __ldg(q_);                                    \
        if (i_ + 1 < a.d) v_.y = __ldg(q_ + 1);                            \
      }                                                                    \
      xr[t] = v_;                                                          \
    }                                                                      \
  }
    SPL_LOAD_X(0);
    for (int ih = 0; ih < a.n_ih; ih++, g++) {
      __syncwarp();
#pragma unroll
      for (int t = 0; t < NX; t++) {
        xs[xr_col * XS + xr_row + 8 * t] = xr[t].x;
        xs[(xr_col + 1) * XS + xr_row + 8 * t] = xr[t].y;
      }
      __syncwarp();
      if (ih + 1 < a.n_ih) SPL_LOAD_X(ih + 1);
      lkg::mbar_wait(&full[g % NS], (uint32_t)((g / NS) & 1));
      const uint8_t* T = stage + (g % NS) * tb;
#pragma unroll 1
      for (int s = 0; s < G; s++) {
        const int il = (s + lane) & 7;
        const uint8_t* Tc = T + il * PROW;
        float2 cb[8];
        {
          const float4* cbp = reinterpret_cast<const float4*>(T + a.cb_off + il * PROW);
#pragma unroll
          for (int q = 0; q < 4; q++) {
            const float4 v = cbp[q];
            cb[2 * q] = make_float2(v.x, v.y);
            cb[2 * q + 1] = make_float2(v.z, v.w);
          }
        }
#pragma unroll
        for (int r = 0; r < RR; r++) {
          const float x = xs[il * XS + lane + 32 * r];
          // uniform cubic B-spline basis at x (spline.cpp:69-83 in closed form)
          const float tt = (x - a.t0) * a.inv_h;
          const float fl = floorf(tt);
          const int mu = (int)fl;
          const bool inside = tt >= 0.0f && mu < a.n0;  // false for NaN
          const float u = tt - fl, om = 1.0f - u, u2 = u * u, u3 = u2 * u;
          const float s6 = 1.0f / 6.0f;
          float bt[4] = {om * om * om * s6, fmaf(3.0f, u3, fmaf(-6.0f, u2, 4.0f)) * s6,
                         fmaf(-3.0f, u3, fmaf(3.0f, u2, fmaf(3.0f, u, 1.0f))) * s6, u3 * s6};
          const int r0 = mu - 3;
          const float bx = __fdividef(x, 1.0f + __expf(-x));  // silu of the unclipped input
          float2 BX = make_float2(bx, bx);
#pragma unroll
          for (int q = 0; q < 8; q++) acc[r][q] = __ffma2_rn(cb[q], BX, acc[r][q]);
#pragma unroll
          for (int t = 0; t < 4; t++) {
            const int rr = r0 + t;
            const bool ok = inside && rr >= 0 && rr < a.R;
            const float b = ok ? bt[t] : 0.0f;
            const float4* cp = reinterpret_cast<const float4*>(Tc + (ok ? rr : 0) * (G * PROW));
            const float2 B = make_float2(b, b);
#pragma unroll
            for (int q = 0; q < 4; q++) {
              const float4 c = cp[q];
              acc[r][2 * q] = __ffma2_rn(make_float2(c.x, c.y), B, acc[r][2 * q]);
              acc[r][2 * q + 1] = __ffma2_rn(make_float2(c.z, c.w), B, acc[r][2 * q + 1]);
            }
          }
        }
      }
      if (F64) {
#pragma unroll
        for (int r = 0; r < RR; r++)
#pragma unroll
          for (int q = 0; q < 8; q++) {
            acc64[r][2 * q] += (double)acc[r][q].x;
            acc64[r][2 * q + 1] += (double)acc[r][q].y;
            acc[r][q] = make_float2(0.f, 0.f);
          }
      }
      __syncthreads();
      if (tid == 0 && g + NS < n_stages) issue(g + NS);
    }
#undef SPL_LOAD_X
    const int j0 = jb * JB;
#pragma unroll
    for (int r = 0; r < RR; r++) {
      const int64_t row = row0 + lane + 32 * r;
      if (lane + 32 * r < rows_left) {
        float* yr = a.Y + row * a.m + j0;
#pragma unroll
        for (int q = 0; q < 8; q++) {
          const float v0 = F64 ? (float)acc64[r][2 * q] : acc[r][q].x;
          const float v1 = F64 ? (float)acc64[r][2 * q + 1] : acc[r][q].y;
          if (j0 + 2 * q < a.m) yr[2 * q] = v0;
          if (j0 + 2 * q + 1 < a.m) yr[2 * q + 1] = v1;
        }
      }
    }
  }
}

// coeffs f64 [E, R], gains f64 [3][E] (base, spline, out) -> spline tiles.
__global__ void build_spline_tiles_kernel(const double* coeffs, const double* gains, uint8_t* tiles, int64_t tile_bytes,
                                          int32_t n_ih, int32_t d, int32_t m, int32_t R, int32_t cb_off) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t E = (int64_t)d * m;
  if (e >= E) return;
  const int i = (int)(e / m), j = (int)(e - (int64_t)i * m);
  uint8_t* t = tiles + ((int64_t)(j / JB) * n_ih + i / G) * tile_bytes;
  const double bs = gains[e], ss = gains[E + e], os = gains[2 * E + e];
  for (int r = 0; r < R; r++)
    reinterpret_cast<float*>(t + (r * G + i % G) * PROW)[j % JB] = (float)(os * ss * coeffs[e * R + r]);
  reinterpret_cast<float*>(t + cb_off + (i % G) * PROW)[j % JB] = (float)(os * bs);
}

}  // namespace

namespace lkg {

// Builds the spline tiles of a spec if its grid qualifies (uniform knots, degree 3); returns false
// otherwise (the generic spline kernel is used).
bool build_spline_tiles(lkg_ctx* ctx, lkg_spec* S) {
  if (S->spline_tiles.p) return true;
  if (S->degree != 3 || S->K < 1) return false;
  double hmin = 1e300, hmax = 0;
  for (int k = 0; k < S->K; k++) {
    hmin = std::min(hmin, S->breakpoints[k + 1] - S->breakpoints[k]);
    hmax = std::max(hmax, S->breakpoints[k + 1] - S->breakpoints[k]);
  }
  if (hmax > hmin * (1.0 + 1e-9)) return false;
  const int d = S->in_dim, m = S->col1 - S->col0, R = S->K + 3;
  const int64_t tb = ((int64_t)(R + 1) * G * PROW + 127) / 128 * 128;
  const size_t smem = 2 * tb + (size_t)16 * G * (32 * RR + 4) * 4 + 64;
  if (smem > 227 * 1024) return false;
  S->sp_tile_bytes = tb;
  S->sp_n_ih = (d + G - 1) / G;
  S->sp_n_jb = (m + JB - 1) / JB;
  S->spline_tiles.alloc((size_t)S->sp_n_ih * S->sp_n_jb * tb);
  LKG_CUDA(cudaMemsetAsync(S->spline_tiles.p, 0, S->spline_tiles.bytes, ctx->stream));
  const int64_t E = (int64_t)d * m;
  build_spline_tiles_kernel<<<(unsigned)((E + 255) / 256), 256, 0, ctx->stream>>>(
      S->coeffs.as<double>(), S->gains.as<double>(), S->spline_tiles.as<uint8_t>(), tb, S->sp_n_ih, d, m, R,
      R * G * PROW);
  LKG_CUDA(cudaGetLastError());
  ctx->launches++;
  return true;
}

template <bool F64, int W>
void launch_w(lkg_ctx* ctx, SplArgs& a, int64_t rows, int sms) {
  const int64_t row_tile = (int64_t)W * 32 * RR;
  a.n_items = ((rows + row_tile - 1) / row_tile) * a.n_jb;
  const int grid = (int)std::min<int64_t>(a.n_items, sms);
  const size_t smem = 2 * a.tile_bytes + (size_t)W * G * (32 * RR + 4) * 4 + 64;
  static bool attr = false;
  if (!attr) {
    LKG_CUDA(cudaFuncSetAttribute(spline_tiled<F64, W>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
    attr = true;
  }
  spline_tiled<F64, W><<<grid, W * 32, smem, ctx->stream>>>(a);
}

bool launch_spline_tiled(lkg_ctx* ctx, const lkg_spec* S_, const float* X, int64_t rows, float* Y) {
  lkg_spec* S = const_cast<lkg_spec*>(S_);
  if (!build_spline_tiles(ctx, S)) return false;
  SplArgs a{};
  a.tiles = S->spline_tiles.as<uint8_t>();
  a.tile_bytes = S->sp_tile_bytes;
  a.n_ih = S->sp_n_ih;
  a.n_jb = S->sp_n_jb;
  a.R = S->K + 3;
  a.n0 = S->K + 6;  // intervals of the extended knot vector (K + 2p)
  a.cb_off = a.R * G * PROW;
  a.X = X;
  a.rows = rows;
  a.d = S->in_dim;
  a.Y = Y;
  a.m = S->col1 - S->col0;
  const double h = (S->breakpoints[S->K] - S->breakpoints[0]) / S->K;
  a.t0 = (float)(S->breakpoints[0] - 3.0 * (S->breakpoints[1] - S->breakpoints[0]));
  a.inv_h = (float)(1.0 / h);
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->device);
  if (S->in_dim > kFp32MaxD)
    launch_w<true, 8>(ctx, a, rows, sms);
  else
    launch_w<false, 16>(ctx, a, rows, sms);
  LKG_CUDA(cudaGetLastError());
  ctx->launches++;
  return true;
}

}  // namespace lkg
