// forward_tiled.cu — K2 on sm_100a: shared-memory-staged LUT forward.
//
// Replaces forward_quant<SR,ZS,I8> (proj/core/src/runtime.cpp:135-223) for artifacts whose
// per-stage LUT tile fits shared memory. Design:
//
//  * Device layout ("tiles", built once at upload by build_tiles): the layer's edges are cut
//    into tiles of 8 inputs (i_lo) x 16 outputs (j_lo). A tile is one contiguous block:
//      codes  [(K*L)+1 lines][8 i_lo][16 j_lo]  bytes — one 128-byte line per (k, l)
//      P      [(K+1)*8 rows][20] f32   P = out*spline*scale per (k, i_lo, j) (+1 zero block)
//      Q      [(K+1)*8 rows][20] f32   Q = out*spline*y_min (asymmetric only)
//      CB     [8 rows][20] f32          out*base per (i_lo, j) (spline_component only)
//    Symmetric codes are stored biased (q ^ 0x80 = q + 128) so every code is an unsigned byte.
//  * A CTA owns a 1024-row tile x one 16-column j-block and streams the tiles of its j-block
//    through shared memory with cp.async.bulk (TMA bulk copies) completing on mbarriers,
//    double-buffered. CTAs are persistent over (row tile, j-block) items.
//  * Lane = row (R rows per lane). Within a tile the lanes walk the 8 inputs in a ROTATED order
//    (step s: i_lo = (s + lane) & 7), so the 8 lanes of every LDS.128 phase hit 8 different
//    16-byte bank groups of each 128-byte line: code, P and CB reads are conflict-free no matter
//    which (segment, sample) each row selects, and each (row, j) accumulator lives in exactly
//    one lane (no cross-lane reduction).
//  * Per (row, input): coordinates once (exact fp32 mask/segment, f64 re-evaluation of u, z
//    near sample nodes so l0 matches runtime.cpp:178-181), SiLU of the clipped/raw input.
//    Per (row, input, 16 outputs): a code byte becomes the float 2^23 + u with one PRMT; the
//    magic offset cancels exactly inside the FMA: a = fma(w0, 2^23+u0, -(w0*2^23 + 128)),
//    b = fma(w1, 2^23+u1, -w1*2^23) (w1 is a multiple of 2^-23, so both constants are exact);
//    acc += P*a + P*b (+ CB*silu) (+ Q) with packed FFMA2 over pairs of outputs.
//  * Zero_spline masking is folded into the P/Q offset: an out-of-bounds input reads the zero
//    block, so its table term vanishes while the base branch stays live (runtime.cpp:183-189).
//  * Accumulation: fp32 per lane; for long reductions (d > kFp32MaxD) the fp32 partial is
//    flushed into an f64 accumulator every 64 inputs.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>

#include "lkg_internal.h"

namespace {

constexpr int G = 8;                // inputs per line
constexpr int JB = 16;              // outputs per line / j-block
constexpr int LINE = G * JB;        // 128 bytes
constexpr int PROW = 80;            // bytes per P/Q/CB row (16 floats + 16 B pad, conflict-free)
constexpr int kMaxKT = 64;
constexpr int kFlushBlocks = 8;     // f64 flush every 8 tiles = 64 inputs
constexpr int kFp32MaxD = 256;      // fp32 accumulation bound

struct TiledArgs {
  const uint8_t* tiles;
  int64_t tile_bytes;
  int32_t n_ih, n_jb;
  int32_t p_off, q_off, cb_off;
  const float* X;
  int64_t rows;
  int32_t d, x_blk;
  float* Y;
  int32_t m;
  unsigned long long* counters;
  int32_t K, L;
  float lo, hi, hi_clip, est_scale;
  int32_t half_open;
  int64_t n_items;
  float4 ktab[kMaxKT];  // {T_k, T_k+1, (L-1)/(T_k+1 - T_k), 0}
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok = 0;
  do {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
  } while (!ok);
}

// TMA bulk copy global -> shared, completion counted on the mbarrier.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ float load_x(const TiledArgs& a, int64_t r, int i) {
  if (a.x_blk <= 0) return __ldg(a.X + r * a.d + i);
  const int b = i / a.x_blk;
  return __ldg(a.X + (int64_t)b * a.rows * a.x_blk + r * a.x_blk + (i - b * a.x_blk));
}

__device__ __forceinline__ float magic(uint32_t w, uint32_t sel) {
  return __uint_as_float(__byte_perm(w, 0x4B000000u, sel));  // 2^23 + byte
}

template <int R, int W, bool ASYM, bool SR, bool ZS, bool F64>
__global__ void __launch_bounds__(W * 32, 1) fwd_tiled(const __grid_constant__ TiledArgs a) {
  extern __shared__ __align__(128) uint8_t smem[];
  constexpr int NS = 2;
  constexpr int ROWS_W = 32 * R;        // rows per warp
  constexpr int XS = ROWS_W + 4;        // padded row stride of the transposed x tile
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t tb = a.tile_bytes;
  uint8_t* stage = smem;                                             // NS * tile_bytes
  float* xs = reinterpret_cast<float*>(smem + NS * tb) + warp * G * XS;  // per-warp x tile
  float4* ktab = reinterpret_cast<float4*>(smem + NS * tb + W * G * XS * 4);
  uint64_t* full = reinterpret_cast<uint64_t*>(ktab + kMaxKT);

  for (int k = tid; k < a.K; k += W * 32) ktab[k] = a.ktab[k];
  if (tid == 0) {
    for (int s = 0; s < NS; s++) mbar_init(&full[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  const int64_t n_local = a.n_items > blockIdx.x ? (a.n_items - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const int64_t n_stages = n_local * a.n_ih;
  auto tile_src = [&](int64_t g) {
    const int64_t item = blockIdx.x + (g / a.n_ih) * gridDim.x;
    const int jb = (int)(item % a.n_jb), ih = (int)(g % a.n_ih);
    return a.tiles + ((int64_t)jb * a.n_ih + ih) * tb;
  };
  auto issue = [&](int64_t g) {
    uint8_t* dst = stage + (g % NS) * tb;
    const uint8_t* src = tile_src(g);
    mbar_expect_tx(&full[g % NS], (uint32_t)tb);
    for (int64_t off = 0; off < tb; off += 32768) {
      const uint32_t n = (uint32_t)(tb - off < 32768 ? tb - off : 32768);
      bulk_g2s(dst + off, src + off, n, &full[g % NS]);
    }
  };
  if (tid == 0)
    for (int64_t g = 0; g < NS && g < n_stages; g++) issue(g);

  const float M = 8388608.0f;  // 2^23
  const float OFF = ASYM ? 0.0f : 128.0f;
  unsigned long long oob_inputs = 0, oob_rows = 0;
  bool nonfinite = false;
  int64_t g = 0;

  for (int64_t li = 0; li < n_local; li++) {
    const int64_t item = blockIdx.x + li * gridDim.x;
    const int64_t rt = item / a.n_jb;
    const int jb = (int)(item % a.n_jb);
    const bool count = jb == 0;
    const int64_t row0 = rt * (int64_t)(W * ROWS_W) + warp * ROWS_W;
    float2 acc[R][8];
    double acc64[F64 ? R : 1][F64 ? 16 : 1];
    bool row_oob[R];
#pragma unroll
    for (int r = 0; r < R; r++) {
      row_oob[r] = false;
#pragma unroll
      for (int q = 0; q < 8; q++) acc[r][q] = make_float2(0.f, 0.f);
      if (F64)
#pragma unroll
        for (int q = 0; q < 16; q++) acc64[r][q] = 0.0;
    }
    // prefetch x for tile 0 into registers
    float xr[R * G];
#define LOAD_XBLOCK(IH)                                             \
  _Pragma("unroll") for (int t = 0; t < R * G; t++) {               \
    const int e = t * 32 + lane, rr = e >> 3, c = e & 7;            \
    const int64_t row = row0 + rr;                                  \
    const int i = (IH) * G + c;                                     \
    xr[t] = (row < a.rows && i < a.d) ? load_x(a, row, i) : 0.0f;   \
  }
    LOAD_XBLOCK(0);

    for (int ih = 0; ih < a.n_ih; ih++, g++) {
      // stage this warp's x tile transposed: xs[c][row] (conflict-free)
      __syncwarp();
#pragma unroll
      for (int t = 0; t < R * G; t++) {
        const int e = t * 32 + lane;
        xs[(e & 7) * XS + (e >> 3)] = xr[t];
      }
      __syncwarp();
      if (ih + 1 < a.n_ih) {
        LOAD_XBLOCK(ih + 1);
      }
      mbar_wait(&full[g % NS], (uint32_t)((g / NS) & 1));
      const uint8_t* T = stage + (g % NS) * tb;

#pragma unroll 1
      for (int s = 0; s < G; s++) {
        const int il = (s + lane) & 7;
        const int i = ih * G + il;
        float2 cb[8];
        if (SR) {
          const float4* cbp = reinterpret_cast<const float4*>(T + a.cb_off + il * PROW);
#pragma unroll
          for (int q = 0; q < 4; q++) {
            const float4 v = cbp[q];
            cb[2 * q] = make_float2(v.x, v.y);
            cb[2 * q + 1] = make_float2(v.z, v.w);
          }
        }
#pragma unroll
        for (int r = 0; r < R; r++) {
          const float x = xs[il * XS + lane + 32 * r];
          // ---- steps 1-4: mask, clip, segment, interpolation coordinates
          const bool valid_i = i < a.d;
          const bool in = a.lo <= x && (a.half_open ? x < a.hi : x <= a.hi);
          if (valid_i) {
            nonfinite |= !isfinite(x);
            if (count && row0 + lane + 32 * r < a.rows && !in) {
              oob_inputs++;
              row_oob[r] = true;
            }
          }
          const float xp = fminf(fmaxf(x, a.lo), a.hi_clip);
          int k = (int)((xp - a.lo) * a.est_scale);
          k = k < 0 ? 0 : (k > a.K - 1 ? a.K - 1 : k);
          float4 kt = ktab[k];
          while (k > 0 && xp < kt.x) kt = ktab[--k];
          while (k < a.K - 1 && xp >= kt.y) kt = ktab[++k];
          const float z = (xp - kt.x) * kt.z;
          float fl = floorf(z);
          float w1 = z - fl;
          int l0 = (int)fl;
          if (w1 < 0x1p-12f || w1 > 1.0f - 0x1p-12f || l0 >= a.L - 1 || l0 < 0) {
            // near a sample node: runtime.cpp:178-181 in f64
            const double u = ((double)xp - (double)kt.x) / ((double)kt.y - (double)kt.x);
            const double zz = u * (double)(a.L - 1);
            int ll = (int)floor(zz);
            ll = ll < 0 ? 0 : (ll > a.L - 1 ? a.L - 1 : ll);
            l0 = ll;
            w1 = (float)(zz - (double)ll);
          }
          if (l0 >= a.L - 1) w1 = 0.0f;
          w1 = (w1 + 1.0f) - 1.0f;  // multiple of 2^-23: keeps the magic constants exact
          const float w0 = 1.0f - w1;
          const float cA = -fmaf(w0, M, OFF), cB = -w1 * M;
          const bool masked = ZS && !in;
          const uint8_t* qp = T + (k * a.L + l0) * LINE + il * JB;
          const uint4 c0 = *reinterpret_cast<const uint4*>(qp);
          const uint4 c1 = *reinterpret_cast<const uint4*>(qp + LINE);
          const int prow = (masked ? a.K : k) * G + il;
          const float4* pp = reinterpret_cast<const float4*>(T + a.p_off + prow * PROW);
          float bx = 0.0f;
          if (SR) {
            const float xb = ZS ? x : xp;  // clip_x clips the base branch too (runtime.cpp:189)
            bx = __fdividef(xb, 1.0f + __expf(-xb));
          }
          const float2 W0 = make_float2(w0, w0), W1 = make_float2(w1, w1);
          const float2 CA = make_float2(cA, cA), CB = make_float2(cB, cB), BX = make_float2(bx, bx);
          const uint32_t w0w[4] = {c0.x, c0.y, c0.z, c0.w}, w1w[4] = {c1.x, c1.y, c1.z, c1.w};
#pragma unroll
          for (int q = 0; q < 4; q++) {
            const float4 P = pp[q];
            const float2 Pl = make_float2(P.x, P.y), Ph = make_float2(P.z, P.w);
            const float2 fa0 = make_float2(magic(w0w[q], 0x7440), magic(w0w[q], 0x7441));
            const float2 fa1 = make_float2(magic(w0w[q], 0x7442), magic(w0w[q], 0x7443));
            const float2 fb0 = make_float2(magic(w1w[q], 0x7440), magic(w1w[q], 0x7441));
            const float2 fb1 = make_float2(magic(w1w[q], 0x7442), magic(w1w[q], 0x7443));
            const float2 a0 = __ffma2_rn(W0, fa0, CA), a1 = __ffma2_rn(W0, fa1, CA);
            const float2 b0 = __ffma2_rn(W1, fb0, CB), b1 = __ffma2_rn(W1, fb1, CB);
            float2 s0 = acc[r][2 * q], s1 = acc[r][2 * q + 1];
            s0 = __ffma2_rn(Pl, a0, s0);
            s1 = __ffma2_rn(Ph, a1, s1);
            s0 = __ffma2_rn(Pl, b0, s0);
            s1 = __ffma2_rn(Ph, b1, s1);
            if (SR) {
              s0 = __ffma2_rn(cb[2 * q], BX, s0);
              s1 = __ffma2_rn(cb[2 * q + 1], BX, s1);
            }
            if (ASYM) {
              const float4 Q = reinterpret_cast<const float4*>(T + a.q_off + prow * PROW)[q];
              s0 = __fadd2_rn(s0, make_float2(Q.x, Q.y));
              s1 = __fadd2_rn(s1, make_float2(Q.z, Q.w));
            }
            acc[r][2 * q] = s0;
            acc[r][2 * q + 1] = s1;
          }
        }
      }
      if (F64 && ((ih + 1) % kFlushBlocks == 0 || ih + 1 == a.n_ih)) {
#pragma unroll
        for (int r = 0; r < R; r++)
#pragma unroll
          for (int q = 0; q < 8; q++) {
            acc64[r][2 * q] += (double)acc[r][q].x;
            acc64[r][2 * q + 1] += (double)acc[r][q].y;
            acc[r][q] = make_float2(0.f, 0.f);
          }
      }
      __syncthreads();  // every warp is done with this stage buffer
      if (tid == 0 && g + NS < n_stages) issue(g + NS);
    }
    // epilogue: rows of this lane, 16 outputs of the j-block
    const int j0 = jb * JB;
#pragma unroll
    for (int r = 0; r < R; r++) {
      const int64_t row = row0 + lane + 32 * r;
      if (row < a.rows) {
        float out[16];
#pragma unroll
        for (int q = 0; q < 8; q++) {
          out[2 * q] = F64 ? (float)acc64[r][2 * q] : acc[r][q].x;
          out[2 * q + 1] = F64 ? (float)acc64[r][2 * q + 1] : acc[r][q].y;
        }
        float* yr = a.Y + row * a.m + j0;
        if (j0 + 16 <= a.m && (a.m & 3) == 0) {
#pragma unroll
          for (int q = 0; q < 4; q++)
            reinterpret_cast<float4*>(yr)[q] = make_float4(out[4 * q], out[4 * q + 1], out[4 * q + 2], out[4 * q + 3]);
        } else {
          for (int q = 0; q < 16 && j0 + q < a.m; q++) yr[q] = out[q];
        }
        if (row_oob[r]) oob_rows++;
      }
    }
  }
  // OOB counters (runtime.cpp:216-222) and the non-finite flag (runtime.cpp:172)
  for (int o = 16; o; o >>= 1) {
    oob_inputs += __shfl_xor_sync(0xffffffffu, oob_inputs, o);
    oob_rows += __shfl_xor_sync(0xffffffffu, oob_rows, o);
  }
  if (lane == 0) {
    if (oob_rows) atomicAdd(a.counters + 0, oob_rows);
    if (oob_inputs) atomicAdd(a.counters + 1, oob_inputs);
  }
  if (__any_sync(0xffffffffu, nonfinite) && lane == 0) atomicExch(a.counters + 2, 1ull);
}

// Reference layout -> tiles (one thread per (edge, segment) cell).
__global__ void build_tiles_kernel(const uint8_t* q, const float* scale, const float* ymin, const float* gains,
                                   uint8_t* tiles, int64_t tile_bytes, int32_t n_ih, int32_t d, int32_t m,
                                   int32_t K, int32_t L, int32_t p_off, int32_t q_off, int32_t cb_off, int sym,
                                   int sr, int asym) {
  const int64_t cell = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t E = (int64_t)d * m;
  if (cell >= E * K) return;
  const int64_t e = cell / K;
  const int k = (int)(cell - e * K);
  const int i = (int)(e / m), j = (int)(e - (int64_t)i * m);
  const int ih = i / G, il = i % G, jb = j / JB, jl = j % JB;
  uint8_t* t = tiles + ((int64_t)jb * n_ih + ih) * tile_bytes;
  const uint8_t* src = q + cell * L;
  for (int l = 0; l < L; l++) t[(k * L + l) * LINE + il * JB + jl] = sym ? (uint8_t)(src[l] ^ 0x80u) : src[l];
  // fused gains in f64 (runtime.cpp:263-273), then one rounding to f32
  const double cs = sr ? (double)gains[2 * E + e] * (double)gains[E + e] : 1.0;
  float* P = reinterpret_cast<float*>(t + p_off + (k * G + il) * PROW) + jl;
  *P = (float)(cs * (double)scale[cell]);
  if (asym) *reinterpret_cast<float*>(t + q_off + (k * G + il) * PROW + jl * 4) = (float)(cs * (double)ymin[cell]);
  if (sr && k == 0)
    *reinterpret_cast<float*>(t + cb_off + il * PROW + jl * 4) = (float)((double)gains[2 * E + e] * (double)gains[e]);
}

template <int R, int W, bool ASYM, bool SR, bool ZS, bool F64>
void launch_tiled(cudaStream_t st, const TiledArgs& a, size_t smem, int grid) {
  auto kern = fwd_tiled<R, W, ASYM, SR, ZS, F64>;
  static bool attr = false;
  if (!attr) {
    LKG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
    attr = true;
  }
  kern<<<grid, W * 32, smem, st>>>(a);
}

}  // namespace

namespace lkg {

static constexpr int kW = 16, kR = 2;          // fp32 mode: 16 warps x 64 rows = 1024-row tiles
static constexpr int kW64 = 8, kR64 = 2;       // f64-flush mode: 8 warps x 64 rows = 512-row tiles

bool tiled_eligible(const lkg_layer* L) {
  if (L->float_table.p || L->K > kMaxKT) return false;
  return L->geom.tile_bytes > 0;
}

void build_tiles(lkg_ctx* ctx, lkg_layer* L) {
  TileGeom& gm = L->geom;
  gm = TileGeom{};
  if (L->float_table.p || L->K > kMaxKT) return;
  const int d = L->in_dim, m = L->col1 - L->col0, K = L->K, Ls = L->L;
  const bool asym = L->scheme == LKG_SCHEME_ASYMMETRIC, sr = L->value_repr == LKG_REPR_SPLINE_COMPONENT;
  int64_t off = (int64_t)(K * Ls + 1) * LINE;
  gm.p_off = (int32_t)off;
  off += (int64_t)(K + 1) * G * PROW;
  if (asym) {
    gm.q_off = (int32_t)off;
    off += (int64_t)(K + 1) * G * PROW;
  }
  if (sr) {
    gm.cb_off = (int32_t)off;
    off += G * PROW;
  }
  off = (off + 127) / 128 * 128;
  const size_t xs_bytes = (size_t)kW * G * (32 * kR + 4) * 4;
  if (2 * off + xs_bytes + kMaxKT * 16 + 64 > 227 * 1024) return;  // tile too large: generic kernel
  gm.tile_bytes = off;
  gm.JB = JB;
  gm.IC = G;
  gm.n_ih = (d + G - 1) / G;
  gm.n_jb = (m + JB - 1) / JB;
  L->tiles.alloc((size_t)gm.n_ih * gm.n_jb * off);
  LKG_CUDA(cudaMemsetAsync(L->tiles.p, 0, L->tiles.bytes, ctx->stream));
  const int64_t cells = (int64_t)d * m * K;
  build_tiles_kernel<<<(unsigned)((cells + 255) / 256), 256, 0, ctx->stream>>>(
      L->q.as<uint8_t>(), L->scale.as<float>(), L->ymin.as<float>(), L->gains.as<float>(), L->tiles.as<uint8_t>(),
      off, gm.n_ih, d, m, K, Ls, gm.p_off, gm.q_off, gm.cb_off, !asym, sr, asym);
  LKG_CUDA(cudaGetLastError());
  ctx->launches++;
}

void launch_forward_tiled(lkg_ctx* ctx, const lkg_layer* L, const float* X, int64_t rows, int32_t x_blk, float* Y,
                          int slot) {
  const TileGeom& gm = L->geom;
  TiledArgs a{};
  a.tiles = L->tiles.as<uint8_t>();
  a.tile_bytes = gm.tile_bytes;
  a.n_ih = gm.n_ih;
  a.n_jb = gm.n_jb;
  a.p_off = gm.p_off;
  a.q_off = gm.q_off;
  a.cb_off = gm.cb_off;
  a.X = X;
  a.rows = rows;
  a.d = L->in_dim;
  a.x_blk = x_blk;
  a.Y = Y;
  a.m = L->col1 - L->col0;
  a.counters = ctx->counters.as<unsigned long long>() + 4 * slot;
  a.K = L->K;
  a.L = L->L;
  a.half_open = L->boundary_mode == LKG_BOUNDARY_HALF_OPEN;
  a.lo = L->knots[0];
  a.hi = L->knots[L->K];
  a.hi_clip = a.half_open ? std::nextafterf(a.hi, -INFINITY) : a.hi;
  a.est_scale = (float)L->K / (a.hi - a.lo);
  for (int k = 0; k < L->K; k++) {
    const float t0 = L->knots[k], t1 = L->knots[k + 1];
    a.ktab[k] = make_float4(t0, t1, (float)(L->L - 1) / (t1 - t0), 0.f);
  }
  const bool f64 = L->in_dim > kFp32MaxD;
  const int W = f64 ? kW64 : kW, R = f64 ? kR64 : kR;
  const int64_t row_tile = (int64_t)W * 32 * R;
  a.n_items = ((rows + row_tile - 1) / row_tile) * gm.n_jb;
  int dev = ctx->device, sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int grid = (int)std::min<int64_t>(a.n_items, sms);
  const size_t smem = 2 * gm.tile_bytes + (size_t)W * G * (32 * R + 4) * 4 + kMaxKT * 16 + 64;
  const bool asym = L->scheme == LKG_SCHEME_ASYMMETRIC, sr = L->value_repr == LKG_REPR_SPLINE_COMPONENT;
  const bool zs = L->oob_policy == LKG_OOB_ZERO_SPLINE;
  const int sel = (f64 << 3) | (asym << 2) | (sr << 1) | (int)zs;
  switch (sel) {
#define CASE(S)                                                                                           \
  case S:                                                                                                 \
    if ((S >> 3) & 1)                                                                                     \
      launch_tiled<kR64, kW64, (S >> 2) & 1, (S >> 1) & 1, S & 1, true>(ctx->stream, a, smem, grid);     \
    else                                                                                                  \
      launch_tiled<kR, kW, (S >> 2) & 1, (S >> 1) & 1, S & 1, false>(ctx->stream, a, smem, grid);        \
    break;
    CASE(0) CASE(1) CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7)
    CASE(8) CASE(9) CASE(10) CASE(11) CASE(12) CASE(13) CASE(14) CASE(15)
#undef CASE
  }
  LKG_CUDA(cudaGetLastError());
  ctx->launches++;
}

}  // namespace lkg
