// forward_chain.cu — the whole artifact chain in ONE launch for models whose every layer is a
// "small" layer (out_dim <= 8, dequantized value table resident in shared memory: build_tiles'
// small == 2 layout). SURVEY §8f rank 3: the reference chain (proj/core/src/runtime.cpp:298-314)
// copies a Matrix between layers (runtime.cpp:306-310); here the hidden activations of a row never
// leave its thread — every layer's table is staged into shared memory once per CTA and a lane walks
// its row through all layers (configs[0], the PyKAN-style [2,5,1] model: one launch instead of two).
//
// Each layer is evaluated exactly as fwd_small evaluates it (forward_tiled.cu: same coordinates,
// same lane-rotated input order i = lane + t mod d, same fma sequence), so the fused chain's
// outputs and OobStats are bit-identical to the layer-by-layer chain (tests/test_gpu_parity.py).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>

#include "checks.cuh"
#include "coords.cuh"
#include "lkg_internal.h"
#include "tma.cuh"

namespace {

constexpr int kChainMaxLayers = 4;
constexpr int kChainMaxK = 16;  // knot segments per layer (the per-layer tables travel as kernel parameters)

struct ChainLayer {
  const uint8_t* lut;  // value table + CB (build_small_vt_kernel)
  int32_t lut_bytes, cb_off, MP, vp, d, m, sr, zs;
  lkg::CoordConst cc;
  float4 ktab[kChainMaxK];
};

struct ChainArgs {
  ChainLayer l[kChainMaxLayers];
  int32_t n;
  const float* X;
  int64_t rows;
  float* Y;
  unsigned long long* counters;  // [slot][4]
};

// One layer for one row. FIRST: inputs from global memory (row pointer xg), else from this thread's
// column of the hidden-activation scratch (hs[i * bd]). Returns the outputs in y[0..m).
template <bool FIRST>
__device__ __forceinline__ void chain_layer(const ChainLayer& P, const float* V, const float* CBt, const float4* ktab,
                                            const float2* kf, const float* xg, const float* hs, int bd, bool vrow,
                                            int lane, float (&y)[8], uint32_t& oob_inputs, bool& any_oob,
                                            float& nfacc) {
  const int d = P.d, L = P.cc.L, MP = P.MP, ES = P.vp ? 2 * MP : MP;
  const float lo = P.cc.lo;
  const bool sr = P.sr != 0, zs = P.zs != 0;
#pragma unroll
  for (int j = 0; j < 8; j++) y[j] = 0.0f;
  auto X = [&](int i) -> float { return FIRST ? __ldg(xg + i) : hs[i * bd]; };
  auto nxt = [&](int v) { return v + 1 == d ? 0 : v + 1; };
  auto accum = [&](int i, float x, const lkg::Coord& co) {  // fwd_small's VT accum, runtime MP
    oob_inputs += (uint32_t)!co.in;
    any_oob |= !co.in;
    const bool tab = !(zs && !co.in);
    float bx = 0.0f;
    if (sr) bx = lkg::silu_fast(zs ? x : co.xp);  // clip_x clips the base branch too (runtime.cpp:189)
    const float w1 = co.w1, w0 = 1.0f - w1;
    const float* V0 = V + ((int64_t)(co.k * L + co.l0) * d + i) * ES;
    const float* V1 = P.vp ? V0 + MP : V0 + d * ES;
    const float* CB = CBt + i * MP;
    LKG_DCHECK(co.k >= 0 && co.k < P.cc.K && co.l0 >= 0 && co.l0 < L && i >= 0 && i < d, "value-table index");
    LKG_DCHECK((V1 - V + MP) * 4 <= P.cb_off, "value-table entry past the table");
    LKG_DCHECK((i + 1) * MP * 4 + P.cb_off <= P.lut_bytes, "CB row past the layer image");
#pragma unroll
    for (int j = 0; j < 8; j++) {
      if (j < MP) {
        const float v = tab ? fmaf(w1, V1[j], w0 * V0[j]) : 0.0f;
        y[j] += sr ? fmaf(CB[j], bx, v) : v;
      }
    }
  };
  int i = lane % d;
  float xa_n = lo, xb_n = lo;
  if (vrow) {
    xa_n = X(i);
    if (d > 1) xb_n = X(nxt(i));
  }
  for (int t = 0; t < d; t += 2) {
    const int ia = i, ib = nxt(i);
    const float xa = xa_n, xb = xb_n;
    i = nxt(ib);
    if (vrow && t + 2 < d) {
      xa_n = X(i);
      if (t + 3 < d) xb_n = X(nxt(i));
    }
    const bool two = t + 1 < d;
    bool s0, s1;
    lkg::Coord c0 = lkg::lut_coords_fast_nb(P.cc, kf, xa, s0);
    lkg::Coord c1 = lkg::lut_coords_fast_nb(P.cc, kf, two ? xb : lo, s1);
    if (s0 || s1) {
      if (s0) c0 = lkg::lut_coords(P.cc, ktab, xa);
      if (s1) c1 = lkg::lut_coords(P.cc, ktab, xb);
    }
    nfacc = fmaf(xa, 0.0f, nfacc);  // NaN once any input is NaN or inf (runtime.cpp:172)
    accum(ia, xa, c0);
    if (two) {
      nfacc = fmaf(xb, 0.0f, nfacc);
      accum(ib, xb, c1);
    }
  }
}

__global__ void __launch_bounds__(1024) fwd_chain_small(const __grid_constant__ ChainArgs a) {
  extern __shared__ __align__(128) uint8_t smem[];
  const int tid = threadIdx.x, lane = tid & 31, bd = blockDim.x;
  // shared memory: per layer {value table + CB, ktab[kChainMaxK], kf[kChainMaxK]}, then the hidden
  // activations hs[8][bd] (a thread's own column: no synchronisation between layers)
  const float* V[kChainMaxLayers];
  const float* CB[kChainMaxLayers];
  const float4* ktab[kChainMaxLayers];
  const float2* kf[kChainMaxLayers];
  // the tables arrive by TMA bulk copies issued by one thread (a per-thread copy loop left a
  // 128-thread CTA ~26 dependent L2 round trips: most of a small batch's latency)
  __shared__ __align__(8) uint64_t tbar;
  if (tid == 0) {
    lkg::mbar_init(&tbar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    uint32_t total = 0, o2 = 0;
    for (int l = 0; l < a.n; l++) total += (uint32_t)a.l[l].lut_bytes;
    lkg::mbar_expect_tx(&tbar, total);
    for (int l = 0; l < a.n; l++) {
      const ChainLayer& P = a.l[l];
      for (int32_t o = 0; o < P.lut_bytes; o += 32768)
        lkg::bulk_g2s(smem + o2 + o, P.lut + o, (uint32_t)(P.lut_bytes - o < 32768 ? P.lut_bytes - o : 32768), &tbar);
      o2 += (uint32_t)((P.lut_bytes + 15) & ~15) + kChainMaxK * (16 + 8);
    }
  }
  uint32_t off = 0;
#pragma unroll
  for (int l = 0; l < kChainMaxLayers; l++) {
    if (l < a.n) {
      const ChainLayer& P = a.l[l];
      uint8_t* lut = smem + off;
      off += (uint32_t)((P.lut_bytes + 15) & ~15);
      float4* kt = reinterpret_cast<float4*>(smem + off);
      float2* kc = reinterpret_cast<float2*>(kt + kChainMaxK);
      for (int k = tid; k < P.cc.K; k += bd) {
        kt[k] = P.ktab[k];
        kc[k] = make_float2(P.ktab[k].x, P.ktab[k].y);
      }
      off += kChainMaxK * (16 + 8);
      V[l] = reinterpret_cast<const float*>(lut);
      CB[l] = reinterpret_cast<const float*>(lut + P.cb_off);
      ktab[l] = kt;
      kf[l] = kc;
    }
  }
  float* hs = reinterpret_cast<float*>(smem + off) + tid;
  __syncthreads();  // the barrier is initialised and the knot tables are written ...
  lkg::mbar_wait(&tbar, 0);  // ... and the value tables have landed

  uint32_t oob_inputs[kChainMaxLayers] = {}, oob_rows[kChainMaxLayers] = {};
  float nfacc[kChainMaxLayers] = {};
  // equal 64-aligned row ranges per block (a row keeps its lane, hence its input rotation and bits)
  const int64_t b_lo = (a.rows * blockIdx.x / gridDim.x) / 64 * 64;
  const int64_t b_hi = blockIdx.x + 1 == gridDim.x ? a.rows : (a.rows * (blockIdx.x + 1) / gridDim.x) / 64 * 64;
  for (int64_t rb = b_lo; rb < b_hi; rb += bd) {
    const int64_t row = rb + tid;
    if (rb + (tid & ~31) >= b_hi) break;  // this warp has no row left (warp-uniform)
    const bool vrow = row < b_hi;
    float y[8];
#pragma unroll
    for (int l = 0; l < kChainMaxLayers; l++) {
      if (l < a.n) {
        const ChainLayer& P = a.l[l];
        bool any_oob = false;
        if (l == 0)
          chain_layer<true>(P, V[l], CB[l], ktab[l], kf[l], a.X + row * P.d, hs, bd, vrow, lane, y, oob_inputs[l],
                            any_oob, nfacc[l]);
        else
          chain_layer<false>(P, V[l], CB[l], ktab[l], kf[l], nullptr, hs, bd, vrow, lane, y, oob_inputs[l], any_oob,
                             nfacc[l]);
        if (vrow) oob_rows[l] += (uint32_t)any_oob;
        if (l + 1 < a.n) {  // hidden activations: this thread's column of hs
#pragma unroll
          for (int j = 0; j < 8; j++)
            if (j < P.m) hs[j * bd] = y[j];
        } else if (vrow) {
          float* yr = a.Y + row * P.m;
#pragma unroll
          for (int j = 0; j < 8; j++)
            if (j < P.m) yr[j] = y[j];
        }
      }
    }
  }
  // OOB counters per layer slot (runtime.cpp:216-222) and the non-finite flags (runtime.cpp:172)
#pragma unroll
  for (int l = 0; l < kChainMaxLayers; l++) {
    if (l < a.n) {
      unsigned long long oi = oob_inputs[l], orow = oob_rows[l];
      for (int o = 16; o; o >>= 1) {
        oi += __shfl_xor_sync(0xffffffffu, oi, o);
        orow += __shfl_xor_sync(0xffffffffu, orow, o);
      }
      unsigned long long* c = a.counters + 4 * l;
      if (lane == 0) {
        if (orow) atomicAdd(c + 0, orow);
        if (oi) atomicAdd(c + 1, oi);
      }
      const bool nonfinite = !(nfacc[l] == 0.0f);
      if (__any_sync(0xffffffffu, nonfinite) && lane == 0) atomicExch(c + 2, 1ull);
    }
  }
}

size_t chain_table_bytes(const lkg_layer* const* chain, int n) {
  size_t b = 0;
  for (int l = 0; l < n; l++) b += (((size_t)chain[l]->geom.tile_bytes + 15) & ~(size_t)15) + kChainMaxK * (16 + 8);
  return b;
}

}  // namespace

namespace lkg {

// A chain of >= 2 layers that are all value-table small layers whose tables fit shared memory
// together runs as one launch. LKG_CHAIN_FUSE=0 keeps the layer-by-layer launches (A/B and the
// bit-identity test).
bool can_fuse_chain(const lkg_layer* const* chain, int n) {
  static const char* env = getenv("LKG_CHAIN_FUSE");
  if (env && env[0] == '0') return false;
  if (n < 2 || n > kChainMaxLayers) return false;
  for (int l = 0; l < n; l++) {
    const lkg_layer* L = chain[l];
    if (L->geom.small != 2 || L->K > kChainMaxK || L->col1 - L->col0 != L->out_dim || L->out_dim > 8) return false;
    if (L->geom.tile_bytes % 16 != 0) return false;  // the tables are staged by TMA bulk copies
  }
  return chain_table_bytes(chain, n) + 8 * 128 * sizeof(float) <= 200 * 1024;
}

void launch_forward_chain(lkg_ctx* ctx, const lkg_layer* const* chain, int n, const float* X, int64_t rows, float* Y) {
  ChainArgs a{};
  a.n = n;
  a.X = X;
  a.rows = rows;
  a.Y = Y;
  a.counters = ctx->counters.as<unsigned long long>();
  for (int l = 0; l < n; l++) {
    const lkg_layer* L = chain[l];
    ChainLayer& P = a.l[l];
    P.lut = L->tiles.as<uint8_t>();
    P.lut_bytes = (int32_t)L->geom.tile_bytes;
    P.cb_off = L->geom.cb_off;
    P.MP = L->geom.MP;
    P.vp = L->geom.p_off;  // small == 2: p_off carries the pair-entry flag
    P.d = L->in_dim;
    P.m = L->out_dim;
    P.sr = L->value_repr == LKG_REPR_SPLINE_COMPONENT;
    P.zs = L->oob_policy == LKG_OOB_ZERO_SPLINE;
    float4 kt[kMaxKT];
    fill_coord_const(L, P.cc, kt);
    for (int k = 0; k < L->K; k++) P.ktab[k] = kt[k];
  }
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->device);
  // block size: the largest that still spreads the batch over every SM and leaves room for the
  // hidden-activation scratch next to the tables
  const size_t tables = chain_table_bytes(chain, n);
  int bd = 1024;
  while (bd > 128 && (rows < (int64_t)sms * bd || tables + (size_t)8 * bd * sizeof(float) > 220 * 1024)) bd >>= 1;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((rows + bd - 1) / bd, sms));
  const size_t smem = tables + (size_t)8 * bd * sizeof(float);
  static bool attr = false;
  if (!attr) {
    LKG_CUDA(cudaFuncSetAttribute(fwd_chain_small, cudaFuncAttributeMaxDynamicSharedMemorySize, 224 * 1024));  // (+ the static barrier)
    attr = true;
  }
  fwd_chain_small<<<grid, bd, smem, ctx->stream>>>(a);
  LKG_CUDA(cudaGetLastError());
  ctx->launches++;
}

}  // namespace lkg
