// fwd_tiled.cuh — K2 on sm_100a: the shared-memory-staged LUT forward kernel (table walk) and its launchers.
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
//    double-buffered; the last warp to finish with a buffer refills it (no CTA barrier per tile,
//    so warps drift apart: C4 layers -6% time). CTAs are persistent over (row tile, j-block) items.
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
//    flushed after every tile (8 inputs) into f64 accumulators held in Tensor Memory (tmem.cuh;
//    SURVEY Appendix B.4).
//  * Coordinates: lut_coords_fast (coords.cuh) for both rows side by side, the exact path once
//    per step for any coordinate next to a sample node; x blocks arrive by cp.async one tile
//    ahead; items are grouped (item_coords) so x blocks and tiles are reused in L2.
#pragma once
#include <cuda.h>  // CUtensorMap (the x-block tensor map of the XT mode)
#include <cuda_runtime.h>

#include <cmath>
#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "checks.cuh"
#include "coords.cuh"
#include "lkg_internal.h"
#include "tma.cuh"
#include "tmem.cuh"

#ifndef LKG_NS
#define LKG_NS 2  // fwd_tiled stage buffers (see the kernel)
#endif

#ifndef LKG_W
#define LKG_W 16
#endif
#ifndef LKG_R
#define LKG_R 2
#endif

namespace lkg {
namespace tiled {

constexpr int kW = LKG_W, kR = LKG_R;    // fp32 mode: 16 warps x 64 rows = 1024-row tiles
constexpr int kW64 = kW, kR64 = kR;      // f64 mode: same shape, f64 accumulators in TMEM

struct TiledArgs {
  const uint8_t* tiles;
  int64_t tile_bytes, tiles_bytes;  // one tile; the whole layer (bounds checks)
  int32_t n_ih, n_jb;
  int32_t p_off, q_off, cb_off;
  const float* X;
  int64_t rows;
  int32_t d, x_blk, x_vec2;  // x_vec2: even row stride and 8-aligned column blocks -> float2 loads
  float* Y;
  int32_t m;
  unsigned long long* counters;
  lkg::CoordConst cc;        // coordinate constants (coords.cuh)
  int64_t n_items, n_rt;
  uint32_t rt_group;    // row tiles per item group (item_coords)
  // Input split (split-K) of f64-accumulating layers: an item covers n_ihs = n_ih / ksplit
  // consecutive input tiles of its (row tile, j-block); ksplit > 1 when the layer has too few items to
  // fill the SMs evenly (a configs[4] column shard on 8 GPUs: 512 items on 148 SMs = 3.46 waves).
  // A split writes its f64 sums to Ypart[ks][rows][m]; ksplit_reduce_kernel adds the planes in f64, in
  // split order, and rounds once — the unsplit result up to f64 reassociation (1e-16 relative).
  int32_t ksplit, n_ihs;
  double* Ypart;
  uint32_t* rowflags;   // ksplit > 1: one bit per row, set by the first split that saw it out of range
  int32_t lgL;          // REC: log2(L)
  float4 ktab[kMaxKT];  // {T_k, (L-1)/(T_k+1 - T_k), T_k+1, 0}
  // fused next layer (FUSE): a small-out_dim layer evaluated in the epilogue from the 16 hidden
  // activations each lane holds (the whole-layer "small" layout, resident in shared memory)
  const uint8_t* lut2;
  int32_t lut2_bytes, p_off2, q_off2, cb_off2, MP2, m2, vp2;  // vp2: pair value table (small layout)
  float* Y2;
  unsigned long long* counters2;
  lkg::CoordConst cc2;
  float4 ktab2[kMaxKT];
  // XT mode: the layer input was transposed to [d][rows] (launch_forward_tiled) and each warp's x
  // block [8 inputs][64 rows] is one 2D TMA box of this map
  alignas(64) CUtensorMap xmap;
  // ... and the layer's base-branch activations silu(x') of the same input, [d][rows] (computed
  // once per input element by the transpose pass, in f64: correctly rounded to f32)
  alignas(64) CUtensorMap smap;
};

// The kernel variants are instantiated in three translation units that compile side by side
// (forward_tiled_xt.cu, forward_tiled_gc.cu, forward_tiled_rows.cu); forward_tiled.cu holds the
// layouts, the small-layer kernel and the dispatch. sel = asym << 2 | spline_component << 1 | zero_spline.
void launch_xt(int sel, bool f64, bool gc, int idp, cudaStream_t st, const TiledArgs& a, size_t smem, int grid, bool rec);
void launch_gc(int sel, bool f64, int idp, cudaStream_t st, const TiledArgs& a, size_t smem, int grid);
void launch_fused(int sel, int idp, cudaStream_t st, const TiledArgs& a, size_t smem, int grid);
void launch_r1(int sel, int idp, cudaStream_t st, const TiledArgs& a, size_t smem, int grid);
void launch_rows(int sel, bool f64, bool xb2, bool bal, int idp, cudaStream_t st, const TiledArgs& a, size_t smem,
                 int grid);

}  // namespace tiled
}  // namespace lkg

namespace {

using lkg::kMaxKT;
constexpr int G = 8;                // inputs per line
constexpr int JB = 16;              // outputs per line / j-block
constexpr int LINE = G * JB;        // 128 bytes
constexpr int PROW = 80;            // bytes per P/Q/CB row (16 floats + 16 B pad, conflict-free)
constexpr int PLINE = 2 * LINE;     // IDP pair line: 8 inputs x 16 outputs x (code, next code)
constexpr int kFlushBlocks = 1;     // f64 flush after every tile (8 inputs): partial sums stay short
// IDP integer lerp: W0 + W1 = 2^15 (so W0*u0 + W1*u1 <= 2^15 * 255 < 2^23 stays a magic float's
// mantissa), packed as the dp2a weight word W0 | W1 << 16 = 2^15 + 65535*W1, formed from the float
// 2^23 + W1 by one IMAD with this bias (unsigned wrap-around intended)
constexpr uint32_t kWordBias = 32768u - 0x4B000000u * 65535u;
constexpr int kFp32MaxD = 256;      // fp32 accumulation bound

using lkg::tiled::TiledArgs;

using lkg::bulk_g2s;
using lkg::mbar_expect_tx;
using lkg::mbar_init;
using lkg::mbar_wait;

// GC mode: a 16-byte code read through the read-only path. The L1 hit rate (~28% on configs[4])
// matters: L1::no_allocate measured 1.6x slower, L1::evict_last no different.
__device__ __forceinline__ uint4 gc_load(const uint8_t* p) { return __ldg(reinterpret_cast<const uint4*>(p)); }

// GC pair entries (IDPM == 3, codes in global memory): per (input, segment, sample) one 32-byte
// entry holding the 16 outputs' codes of sample l NEXT TO those of sample l+1, already in dp2a word
// order [u_l(j), u_l+1(j), u_l(j+1), u_l+1(j+1)] — a (row, input) is ONE 256-bit load of one sector
// (the standard lines cost two 16-byte loads from two 128-byte lines plus 8 PRMT). Entries are
// input-major inside a tile: [8 i_lo][K][L][32 B]; sample L-1's successor slot is 0 (its weight is 0).
constexpr int GCE = 32;
__host__ __device__ __forceinline__ int64_t gce_off(int il, int k, int l, int K, int L) {
  return ((int64_t)(il * K + k) * L + l) * GCE;
}
__device__ __forceinline__ void gc_load256(const uint8_t* p, uint32_t (&w)[8]) {
  asm volatile("ld.global.nc.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]), "=r"(w[4]), "=r"(w[5]), "=r"(w[6]), "=r"(w[7])
               : "l"(p));
}

__device__ __forceinline__ float magic(uint32_t w, uint32_t sel) {
  return __uint_as_float(__byte_perm(w, 0x4B000000u, sel));  // 2^23 + byte
}

// IDP.2A: a.h0 * b.byte(0|2) + a.h1 * b.byte(1|3) + c (16-bit x 8-bit, unsigned)
__device__ __forceinline__ uint32_t dp2a_lo(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d;
  asm("dp2a.lo.u32.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}
__device__ __forceinline__ uint32_t dp2a_hi(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d;
  asm("dp2a.hi.u32.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}

// Byte offset of (input il, output j, sample l or l+1) inside an IDP pair line: output pairs
// (j, j+1) share a word [u_l(j), u_l+1(j), u_l(j+1), u_l+1(j+1)]; outputs 8h..8h+7 form a 16-byte
// half stored at chunk h ^ (il >> 2) of the input's 32 bytes, so the 8 lanes of an LDS.128 phase
// (8 distinct rotated inputs) hit 8 distinct 16-byte bank groups.
__host__ __device__ __forceinline__ int pair_off(int il, int j, int next) {
  return il * 32 + (((j >> 3) ^ (il >> 2)) << 4) + ((j & 7) >> 1) * 4 + (j & 1) * 2 + next;
}

// Item u -> (row tile, j-block). GC: row tiles fastest (every CTA in flight shares the current
// tile in L2). Otherwise groups of a.rt_group row tiles sweep all j-blocks with the row tile
// fastest: the group's x blocks stay in L2 across j-blocks and each tile is read once per group
// (C4: DRAM traffic per layer 17 GB -> ~5 GB).
__device__ __forceinline__ void item_coords(const TiledArgs& a, bool gc, uint32_t u, uint32_t& rt, int& jb,
                                            int& ks) {
  const uint32_t n_rt = (uint32_t)a.n_rt, rg = a.rt_group, S = (uint32_t)a.ksplit;
  const uint32_t n_js = (uint32_t)a.n_jb * S;  // (j-block, input split) pairs, split fastest
  uint32_t js;
  if (gc) {
    rt = u % n_rt;
    js = u / n_rt;
  } else {
    const uint32_t per = rg * n_js, g = u / per, base = g * rg;
    const uint32_t gsz = n_rt - base < rg ? n_rt - base : rg, ul = u - g * per;
    rt = base + ul % gsz;
    js = ul / gsz;
  }
  if (S == 1) {
    jb = (int)js;
    ks = 0;
  } else {
    jb = (int)(js / S);
    ks = (int)(js - (uint32_t)jb * S);
  }
}

template <int R, int W, bool ASYM, bool SR, bool ZS, bool F64, bool FUSE, int MINB = 1, bool GC = false,
          bool BAL = false, int XB = 1, bool XT = false, int IDPM = 0, bool REC = false, int NSX = 0>
__global__ void __launch_bounds__(W * 32, MINB) fwd_tiled(const __grid_constant__ TiledArgs a) {
  extern __shared__ __align__(128) uint8_t smem[];
  // Two stage buffers, a compile-time count: NS as a runtime value turned every per-tile
  // g mod NS into a 64-bit division (configs[1] layer 0: 0.567 -> 0.534 ms once removed). Three
  // (LKG_NS=3, the most that fits next to the x tiles) measured 8.5% slower on configs[1].
  // (NSX: the small-batch variant runs 4 stages — its chain of tile loads is latency-bound)
  constexpr int NS = NSX ? NSX : LKG_NS;
  constexpr int ROWS_W = 32 * R;        // rows per warp
  // row stride of the transposed x tile: padded for the 4-byte cp.async writes, or exactly the TMA
  // box (XT; the rotated reads xs[il][lane + 32r] are conflict-free either way)
  constexpr int XS = XT ? ROWS_W : ROWS_W + 4;
  constexpr int NXL = ROWS_W / 4;        // x elements each lane stages per tile (cp.async)
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t tb = a.tile_bytes;
  // GC (codes in global): tiles whose code block exceeds shared memory (K*L large, e.g. configs[4])
  // stage only P/Q/CB; the two code lines per (row, input) are read through the read-only path
  // from L2, and items are ordered row-tile fastest so concurrent CTAs share each tile in L2.
  const int64_t so = GC ? a.p_off : 0, sb = tb - so;
  uint8_t* stage = smem;                                                  // NS * sb
  // XB x-tile buffers per warp. One (the next block staged after the steps, from L1 mostly) leaves
  // 35 KB more L1 than two (staged a tile ahead): measured C4 -7%, C3 -5%, C5 -4%, C2a -2%; only the
  // int8 one-j-block layer (configs[1]) is faster with two (+2%).
  // XT: each x buffer is followed by its silu box (the base branch reads it instead of silu(x'))
  constexpr int XW = XT ? 2 : 1;
  float* xsw = reinterpret_cast<float*>(smem + NS * sb) + warp * XB * G * XS * XW;
  float4* ktab = reinterpret_cast<float4*>(smem + NS * sb + XB * W * G * XS * XW * 4);
  uint64_t* full = reinterpret_cast<uint64_t*>(ktab + kMaxKT);
  uint32_t* fin = reinterpret_cast<uint32_t*>(full + 4);  // warps done with each stage buffer
  uint64_t* xbar = full + 8;  // XT: per-warp x-block barriers (W <= 16)
  float2* kf = reinterpret_cast<float2*>(full + 24);  // compact {T_k, (L-1)/h_k} (coords.cuh)
  float2* kf2 = kf + kMaxKT;
  float4* ktab2 = reinterpret_cast<float4*>(kf2 + kMaxKT);
  uint8_t* lut2 = reinterpret_cast<uint8_t*>(ktab2 + kMaxKT);

  for (int k = tid; k < a.cc.K; k += W * 32) {
    ktab[k] = a.ktab[k];
    kf[k] = make_float2(a.ktab[k].x, a.ktab[k].y);
  }
  if (FUSE) {
    for (int k = tid; k < a.cc2.K; k += W * 32) {
      ktab2[k] = a.ktab2[k];
      kf2[k] = make_float2(a.ktab2[k].x, a.ktab2[k].y);
    }
    for (int o = tid * 16; o < a.lut2_bytes; o += W * 32 * 16)
      *reinterpret_cast<uint4*>(lut2 + o) = __ldg(reinterpret_cast<const uint4*>(a.lut2 + o));
  }
  if (tid == 0) {
    for (int s = 0; s < NS; s++) {
      mbar_init(&full[s], 1);
      fin[s] = 0;
    }
    if (XT)
      for (int w = 0; w < W; w++) mbar_init(&xbar[w], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // F64: the f64 accumulators live in Tensor Memory (tmem.cuh), not registers: each thread owns
  // R x 16 doubles = R x 32 columns of its TMEM lane; warps w and w+4k share a lane quarter.
  constexpr uint32_t kTmCols = F64 ? ((W / 4) * R * 32 <= 32 ? 32 : (W / 4) * R * 32 <= 64 ? 64
                                      : (W / 4) * R * 32 <= 128 ? 128 : (W / 4) * R * 32 <= 256 ? 256 : 512) : 32;
  uint32_t* tm_base_s = reinterpret_cast<uint32_t*>(full + 3);  // spare slot of the barrier block
  if (F64 && warp == 0) lkg::tmem_alloc(tm_base_s, kTmCols);
  if (F64) lkg::tmem_fence_before_sync();
  __syncthreads();
  if (F64) lkg::tmem_fence_after_sync();
  const uint32_t tm_base = F64 ? *tm_base_s : 0u;
  const uint32_t tm_warp = tm_base + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)((warp >> 2) * R * 32);
  LKG_DCHECK(!F64 || (uint32_t)((warp >> 2) * R * 32 + R * 32) <= kTmCols, "TMEM columns past the allocation");

  // Balanced rows (one j-block, e.g. configs[1] layer 0): CTA b owns rows [r_lo, r_hi) of an equal
  // split (starts at multiples of 64 rows, so every row keeps its lane and rotation and its result
  // bits), walked in 1024-row tiles; the warps past r_hi in the last tile only keep the stage
  // protocol. Whole 1024-row items over 148 CTAs would leave 6.6 items per CTA waiting on 7.
  constexpr int64_t TILE_ROWS = W * ROWS_W;
  // (a compile-time mode: the row-range bookkeeping measured 6.5% on configs[3] layers even when off)
  constexpr bool bal = BAL;  // launched only for one-j-block, codes-in-smem layers
  int64_t r_lo = 0, r_hi = a.rows;
  if (bal) {
    auto split = [&](int64_t b) -> int64_t {
      return b >= (int64_t)gridDim.x ? a.rows : (a.rows * b / (int64_t)gridDim.x) / ROWS_W * ROWS_W;
    };
    r_lo = split(blockIdx.x);
    r_hi = split((int64_t)blockIdx.x + 1);
  }
  const int64_t n_local = bal ? (r_hi - r_lo + TILE_ROWS - 1) / TILE_ROWS
                              : (a.n_items > blockIdx.x ? (a.n_items - 1 - blockIdx.x) / gridDim.x + 1 : 0);
  const int64_t n_stages = n_local * a.n_ihs;
  auto issue = [&](int64_t g, int st) {  // stage g into buffer st = g mod NS
    const uint32_t gs = (uint32_t)g, item = blockIdx.x + (gs / (uint32_t)a.n_ihs) * gridDim.x;
    uint32_t rt_ = 0;
    int jb = 0, ks_ = 0;  // balanced rows: the only j-block (local item numbers are not global item ids)
    if (!bal) item_coords(a, GC, item, rt_, jb, ks_);
    const int ih = ks_ * a.n_ihs + (int)(gs % (uint32_t)a.n_ihs);
    const uint8_t* src = a.tiles + ((int64_t)jb * a.n_ih + ih) * tb + so;
    uint8_t* dst = stage + st * sb;
    mbar_expect_tx(&full[st], (uint32_t)sb);
    for (int64_t off = 0; off < sb; off += 32768) {
      const uint32_t n = (uint32_t)(sb - off < 32768 ? sb - off : 32768);
      bulk_g2s(dst + off, src + off, n, &full[st]);
    }
  };
  if (tid == 0)
    for (int g0 = 0; g0 < NS && g0 < n_stages; g0++) issue(g0, g0);

  const float M = 8388608.0f;  // 2^23
  const float OFF = ASYM ? 0.0f : 128.0f;
  const float lo = a.cc.lo;
  const int K = a.cc.K, L = a.cc.L;  // knots are uniformly spaced (tiled_eligible)
  uint32_t oob_inputs = 0, oob_rows = 0, oob2_inputs = 0, oob2_rows = 0;
  bool nonfinite = false, nonfinite2 = false;
  float nfacc = 0.0f, nfacc2 = 0.0f;
  int64_t g = 0;
  const int64_t x_rs = a.x_blk > 0 ? a.x_blk : a.d;  // row stride of the input layout
  // x tiles (64 rows x 8 inputs per warp) go global -> shared with 4-byte cp.async, transposed to
  // xs[c][row] (conflict-free for the rotated reads), double-buffered one tile ahead. This lane
  // stages column (lane & 7) of rows (lane >> 3) + 4t. Cells outside [rows) x [d) are written as
  // t_0: finite and in range, so they never count as OOB; their P and CB entries are 0.
  // Row tile of local item li (32-bit division: item counts are far below 2^31).
  auto row0_of = [&](int64_t li_) -> int64_t {
    if (bal) return r_lo + li_ * TILE_ROWS + warp * ROWS_W;
    const uint32_t item_ = (uint32_t)(blockIdx.x + li_ * gridDim.x);
    uint32_t rt_;
    int jb_, ks_;
    item_coords(a, GC, item_, rt_, jb_, ks_);
    return (int64_t)rt_ * (W * ROWS_W) + warp * ROWS_W;
  };
  auto ih0_of = [&](int64_t li_) -> int {  // first input tile of local item li (its input split)
    if (bal || a.ksplit == 1) return 0;
    uint32_t rt_;
    int jb_, ks_;
    item_coords(a, GC, (uint32_t)(blockIdx.x + li_ * gridDim.x), rt_, jb_, ks_);
    return ks_ * a.n_ihs;
  };
  uint32_t xphase = 0;
  auto stage_x = [&](int64_t r0_, int ih_, int buf) {
    if constexpr (XT) {  // 2D TMA boxes [8 inputs][64 rows] of the transposed input and its silu
      if (lane == 0) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // the warp's reads, then TMA writes
        mbar_expect_tx(&xbar[warp], (uint32_t)(2 * G * ROWS_W * 4));
        float* dst = xsw + buf * G * XS * XW;
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
            ::"r"(lkg::smem_u32(dst)), "l"(&a.xmap), "r"((int)r0_), "r"(ih_ * G), "r"(lkg::smem_u32(&xbar[warp]))
            : "memory");
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
            ::"r"(lkg::smem_u32(dst + G * XS)), "l"(&a.smap), "r"((int)r0_), "r"(ih_ * G),
            "r"(lkg::smem_u32(&xbar[warp]))
            : "memory");
      }
      return;
    }
    const int c_ = lane & 7, i_ = ih_ * G + c_;
    float* dst = xsw + buf * G * XS + c_ * XS + (lane >> 3);
    int64_t col_ = i_;
    if (a.x_blk > 0) {
      const int b_ = i_ / a.x_blk;
      col_ = (int64_t)b_ * a.rows * a.x_blk + (i_ - b_ * a.x_blk);
    }
    const float* src = a.X + col_ + (r0_ + (lane >> 3)) * x_rs;
    const uint32_t sd = lkg::smem_u32(dst);
    if (ih_ * G + G <= a.d && r0_ + ROWS_W <= r_hi) {  // whole tile inside X (and this CTA's rows)
      // one running byte address (a 64-bit add per copy instead of an index-to-address chain)
      const uint64_t step = (uint64_t)(4 * x_rs) * sizeof(float);
      uint64_t pa = reinterpret_cast<uint64_t>(src);
#pragma unroll
      for (int t = 0; t < NXL; t++, pa += step)
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(sd + 16 * t), "l"(pa) : "memory");
    } else {
      const int64_t left = r_hi - r0_ - (lane >> 3);
      const bool cin = i_ < a.d;
#pragma unroll
      for (int t = 0; t < NXL; t++) {
        if (cin && 4 * t < left)
          asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(sd + 16 * t),
                       "l"(src + (int64_t)(4 * t) * x_rs)
                       : "memory");
        else
          dst[4 * t] = lo;
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  if (n_local > 0) stage_x(row0_of(0), ih0_of(0), 0);
  int xbuf = 0;

  for (int64_t li = 0; li < n_local; li++) {
    const uint32_t item = (uint32_t)(blockIdx.x + li * gridDim.x);
    uint32_t rt32 = 0;
    int jb = 0, ks = 0;
    if (!bal) item_coords(a, GC, item, rt32, jb, ks);
    const int64_t rt = rt32;
    const int64_t row0_next = li + 1 < n_local ? row0_of(li + 1) : 0;
    const int ih0 = ks * a.n_ihs, ih0_next = li + 1 < n_local ? ih0_of(li + 1) : 0;
    const int cnt = jb == 0;  // OOB statistics are counted once per row (j-block 0)
    const int64_t row0 = bal ? row0_of(li) : rt * TILE_ROWS + warp * ROWS_W;
    const int64_t rows_left = r_hi - row0;  // rows of this warp: [0, min(ROWS_W, rows_left))
    const bool wactive = rows_left > 0;     // else: a balanced CTA's last tile past its rows
    float2 acc[R][8];
    uint32_t row_oob = 0;   // bit r: row lane + 32 r saw an OOB coordinate
    uint32_t oob_item = 0;  // OOB coordinates of this lane's rows in this item
#pragma unroll
    for (int r = 0; r < R; r++) {
#pragma unroll
      for (int q = 0; q < 8; q++) acc[r][q] = make_float2(0.f, 0.f);
      if (F64) {
        const uint32_t zero[32] = {};
        lkg::tmem_st32(tm_warp + 32 * r, zero);
      }
    }

    for (int ih = ih0; ih < ih0 + a.n_ihs; ih++, g++) {
      // this tile's x block has landed (this lane's copies, then the warp's); prefetch the next
      if constexpr (XT) {
        mbar_wait(&xbar[warp], xphase);
        xphase ^= 1u;
      } else {
        asm volatile("cp.async.wait_group 0;" ::: "memory");
      }
      __syncwarp();
      const float* xs = xsw + (XB == 2 ? xbuf * G * XS * XW : 0);
      if constexpr (XB == 2) {
        if (ih + 1 < ih0 + a.n_ihs)
          stage_x(row0, ih + 1, xbuf ^ 1);
        else if (li + 1 < n_local)
          stage_x(row0_next, ih0_next, xbuf ^ 1);
        xbuf ^= 1;
      }
      const int st = (int)((uint32_t)g % NS);  // constant divisor: multiply-shift
      mbar_wait(&full[st], ((uint32_t)g / NS) & 1u);
      const uint8_t* T = stage + st * sb - so;  // T + p_off is the staged P block
      const uint8_t* Tcodes = GC ? a.tiles + ((int64_t)jb * a.n_ih + ih) * tb : T;

      // one step per iteration: unrolling by 2 spills 64 B and measured -5% (C2), -7% (C2a)
      const int n_steps = wactive ? G : 0;
#pragma unroll 1
      for (int s = 0; s < n_steps; s++) {
        const int il = (s + lane) & 7;
        const uint8_t* Tq = Tcodes + (IDPM == 3 ? gce_off(il, 0, 0, K, L) : IDPM == 1 ? pair_off(il, 0, 0) : il * JB);
        const uint8_t* Tp = T + a.p_off + il * PROW;
        // ---- steps 1-4 (runtime.cpp:170-190): mask, clip, segment, coordinates (coords.cuh),
        // the R rows' fast chains side by side, then the exact path once for any that need it
        // (REC: the coordinate pass did all of it once per input element; the box holds records)
        float xv[R];
        lkg::Coord cv[R];
        bool any_slow = false, slow_r[R];
        if constexpr (REC) {
          (void)any_slow;
          (void)slow_r;
#pragma unroll
          for (int r = 0; r < R; r++) xv[r] = xs[il * XS + lane + 32 * r];
        } else if constexpr (R > 1) {  // measured: -2% time at R=2, +2% at R=1 (where it has nothing to pair)
#pragma unroll
          for (int r = 0; r < R; r++) {
            xv[r] = xs[il * XS + lane + 32 * r];
            cv[r] = lkg::lut_coords_fast_nb(a.cc, kf, xv[r], slow_r[r]);
            any_slow |= slow_r[r];
          }
          if (any_slow) {
#pragma unroll
            for (int r = 0; r < R; r++)
              if (slow_r[r]) cv[r] = lkg::lut_coords(a.cc, ktab, xv[r]);
          }
        } else {
          xv[0] = xs[il * XS + lane];
          cv[0] = lkg::lut_coords_fast(a.cc, ktab, kf, xv[0]);
          (void)any_slow;
          (void)slow_r;
        }
#pragma unroll
        for (int r = 0; r < R; r++) {
          const float x = xv[r];
          bool in;
          int k, l0, cline;  // cline: the code line k*L + l0
          float xp, w1;
          uint32_t Wrec = 0;
          if constexpr (REC) {
            // record (coord_pass_kernel): W1 bits 0-14, code line k*L + l0 bits 15-27, OOB bit 31
            // (the line is used as it is: re-forming it from k and l0 cost an IMAD and a LOP per row)
            const uint32_t rec = __float_as_uint(x);
            in = (rec >> 31) == 0u;
            cline = (int)((rec >> 15) & 0x1FFFu);
            k = cline >> a.lgL;
            l0 = cline & (L - 1);  // (bounds checks only)
            Wrec = (rec & 0x7FFFu) * 65535u + 32768u;
            xp = 0.0f;
            w1 = 0.0f;
          } else {
            const lkg::Coord co = cv[r];
            in = co.in;
            k = co.k;
            l0 = co.l0;
            xp = co.xp;
            w1 = co.w1;  // w1: multiple of 2^-23 -> exact magic constants
            cline = k * L + l0;
            nfacc = fmaf(x, 0.0f, nfacc);  // NaN once any input is NaN or inf
          }
          if (!in) {  // (predicated adds: cheaper than materialising the flag)
            oob_item++;
            row_oob |= 1u << r;
          }
          const int prow = ((ZS && !in) ? K : k) * (G * PROW);  // zero block masks the table term
          const float4* pp = reinterpret_cast<const float4*>(Tp + prow);
          LKG_DCHECK(k >= 0 && k < K && l0 >= 0 && l0 < L, "segment / sample index out of range");
          LKG_DCHECK(prow >= 0 && prow <= K * G * PROW, "P row out of the staged block");
          LKG_DCHECK(GC || (int64_t)(k * L + l0 + 1) * (IDPM == 1 ? PLINE : LINE) + LINE <= a.p_off,
                     "code line past the staged code block");
          LKG_DCHECK(!GC || IDPM == 3 ||
                         ((int64_t)jb * a.n_ih + ih) * tb + (int64_t)(k * L + l0 + 2) * LINE <= a.tiles_bytes,
                     "code line past the layer's tiles (GC)");
          LKG_DCHECK(IDPM != 3 || gce_off(il, k, l0, K, L) + GCE <= a.p_off, "pair entry past the tile's code block (GC)");
          LKG_DCHECK(st >= 0 && st < NS, "stage index");
          (void)xp;
          if constexpr (IDPM != 0) {
            // Integer lerp: W1 = round(w1 * 2^15), W0 = 2^15 - W1; one dp2a per output
            // gives 2^23 + W0*u0 + W1*u1 exactly as a magic float, one FADD2 per output pair removes
            // the magic (and the symmetric codes' +128 bias), P arrives pre-scaled by 2^-15.
            const uint32_t Wd =
                REC ? Wrec : __float_as_uint(fmaf(w1, 32768.0f, 8388608.0f)) * 65535u + kWordBias;
            uint32_t wd[8];
            if constexpr (IDPM == 3) {  // GC pair entries: one 256-bit read-only load, words as stored
              gc_load256(Tq + cline * GCE, wd);
            } else if constexpr (IDPM == 1) {  // pair lines: the words are in shared memory as they are
              const uint8_t* qp = Tq + cline * PLINE;
              // Tq points at half 0 (chunk il >> 2 of the input's 32 bytes); half 1 is the other chunk
              const uint4 h0 = *reinterpret_cast<const uint4*>(qp);
              const uint4 h1 = *reinterpret_cast<const uint4*>(qp + 16 - ((il >> 2) << 5));
              wd[0] = h0.x, wd[1] = h0.y, wd[2] = h0.z, wd[3] = h0.w, wd[4] = h1.x, wd[5] = h1.y, wd[6] = h1.z, wd[7] = h1.w;
            } else {  // standard lines: pair each code with the next line's (one PRMT per 2 outputs)
              const uint8_t* qp = Tq + cline * LINE;
              const uint4 c0 = GC ? gc_load(qp) : *reinterpret_cast<const uint4*>(qp);
              const uint4 c1 = GC ? gc_load(qp + LINE) : *reinterpret_cast<const uint4*>(qp + LINE);
              const uint32_t u0[4] = {c0.x, c0.y, c0.z, c0.w}, u1[4] = {c1.x, c1.y, c1.z, c1.w};
#pragma unroll
              for (int q = 0; q < 4; q++) {
                wd[2 * q] = __byte_perm(u0[q], u1[q], 0x5140);
                wd[2 * q + 1] = __byte_perm(u0[q], u1[q], 0x7362);
              }
            }
            constexpr float MOFF = ASYM ? -8388608.0f : -12582912.0f;  // -(2^23 [+ 128 * 2^15])
            const float2 MO = make_float2(MOFF, MOFF);
#pragma unroll
            for (int q = 0; q < 4; q++) {
              const float4 P = pp[q];
              const float2 Pl = make_float2(P.x, P.y), Ph = make_float2(P.z, P.w);
              const float2 a01 = __fadd2_rn(make_float2(__uint_as_float(dp2a_lo(Wd, wd[2 * q], 0x4B000000u)),
                                                        __uint_as_float(dp2a_hi(Wd, wd[2 * q], 0x4B000000u))), MO);
              const float2 a23 = __fadd2_rn(make_float2(__uint_as_float(dp2a_lo(Wd, wd[2 * q + 1], 0x4B000000u)),
                                                        __uint_as_float(dp2a_hi(Wd, wd[2 * q + 1], 0x4B000000u))), MO);
              float2 s0 = acc[r][2 * q], s1 = acc[r][2 * q + 1];
              s0 = __ffma2_rn(Pl, a01, s0);
              s1 = __ffma2_rn(Ph, a23, s1);
              if (ASYM) {
                const float4 Q = reinterpret_cast<const float4*>(T + a.q_off + il * PROW + prow)[q];
                s0 = __fadd2_rn(s0, make_float2(Q.x, Q.y));
                s1 = __fadd2_rn(s1, make_float2(Q.z, Q.w));
              }
              acc[r][2 * q] = s0;
              acc[r][2 * q + 1] = s1;
            }
            continue;
          }
          const float w0 = 1.0f - w1;
          const float cA = -fmaf(w0, M, OFF), cB = -w1 * M;
          const uint8_t* qp = Tq + cline * LINE;
          const uint4 c0 = GC ? gc_load(qp) : *reinterpret_cast<const uint4*>(qp);
          const uint4 c1 = GC ? gc_load(qp + LINE) : *reinterpret_cast<const uint4*>(qp + LINE);
          const float2 W0 = make_float2(w0, w0), W1 = make_float2(w1, w1);
          const float2 CA = make_float2(cA, cA), CB = make_float2(cB, cB);
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
            if (ASYM) {
              const float4 Q = reinterpret_cast<const float4*>(T + a.q_off + il * PROW + prow)[q];
              s0 = __fadd2_rn(s0, make_float2(Q.x, Q.y));
              s1 = __fadd2_rn(s1, make_float2(Q.z, Q.w));
            }
            acc[r][2 * q] = s0;
            acc[r][2 * q + 1] = s1;
          }
        }
        if (SR) {
          // base branch sum_i cb_ij silu(x'_i) (runtime.cpp:189,206-212) in a lane-UNIFORM input
          // order (input s at step s): every lane reads the same CB row, so each LDS.128 is one
          // broadcast wavefront instead of four rotated ones; the x value comes from the tile again
          const float4* cbp = reinterpret_cast<const float4*>(T + a.cb_off + s * PROW);
          LKG_DCHECK(a.cb_off + (s + 1) * PROW <= tb, "CB row past the tile");
          float2 cbu[8];
#pragma unroll
          for (int q = 0; q < 4; q++) {
            const float4 v = cbp[q];
            cbu[2 * q] = make_float2(v.x, v.y);
            cbu[2 * q + 1] = make_float2(v.z, v.w);
          }
#pragma unroll
          for (int r = 0; r < R; r++) {
            float bx;
            if constexpr (XT) {
              bx = xs[G * XS + s * XS + lane + 32 * r];  // the transpose pass's silu(x') box
            } else {
              const float xr = xs[s * XS + lane + 32 * r];
              // clip_x clips the base branch too (runtime.cpp:189); zero_spline keeps the raw input
              const float xb = ZS ? xr : fminf(fmaxf(xr, a.cc.lo), a.cc.hi_clip);
              // long reductions (d > 256, f64 accumulators) take silu correctly rounded: the MUFU
              // approximation's ~2^-22 relative error, summed over thousands of inputs, reaches the
              // 1e-5 bar on configs[4]
              bx = F64 ? lkg::silu_exact(xb) : lkg::silu_fast(xb);
            }
            const float2 BX = make_float2(bx, bx);
#pragma unroll
            for (int q = 0; q < 8; q++) acc[r][q] = __ffma2_rn(cbu[q], BX, acc[r][q]);
          }
        }
      }
      if (F64 && ((ih + 1) % kFlushBlocks == 0 || ih + 1 == ih0 + a.n_ihs)) {
        // fp32 tile partials into the f64 accumulators in TMEM (lo/hi word pairs)
#pragma unroll
        for (int r = 0; r < R; r++) {
          uint32_t w[32];
          lkg::tmem_ld32(tm_warp + 32 * r, w);
#pragma unroll
          for (int q = 0; q < 8; q++) {
            const double d0 = __hiloint2double((int)w[4 * q + 1], (int)w[4 * q]) + (double)acc[r][q].x;
            const double d1 = __hiloint2double((int)w[4 * q + 3], (int)w[4 * q + 2]) + (double)acc[r][q].y;
            w[4 * q] = (uint32_t)__double2loint(d0);
            w[4 * q + 1] = (uint32_t)__double2hiint(d0);
            w[4 * q + 2] = (uint32_t)__double2loint(d1);
            w[4 * q + 3] = (uint32_t)__double2hiint(d1);
            acc[r][q] = make_float2(0.f, 0.f);
          }
          lkg::tmem_st32(tm_warp + 32 * r, w);
        }
      }
      if constexpr (XB == 1) {
        __syncwarp();  // one x buffer: the next block is staged once every lane is done with this one
        if (ih + 1 < ih0 + a.n_ihs)
          stage_x(row0, ih + 1, 0);
        else if (li + 1 < n_local)
          stage_x(row0_next, ih0_next, 0);
      }
      // Stage release without a CTA barrier: the last warp done with this buffer refills it, so
      // warps drift up to NS-1 stages apart instead of re-aligning at every tile.
      __syncwarp();
      if (lane == 0) {
        __threadfence_block();
        if (atomicAdd(&fin[st], 1u) == (uint32_t)(W - 1)) {
          fin[st] = 0;
          __threadfence_block();
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          if (g + NS < n_stages) issue(g + NS, st);
        }
      }
    }
    if (cnt) oob_inputs += oob_item;
    // epilogue: rows of this lane, 16 outputs of the j-block
    const int j0 = jb * JB;
#pragma unroll
    for (int r = 0; r < R; r++) {
      const int64_t row = row0 + lane + 32 * r;
      float out[16];
      if (F64) {  // warp-collective TMEM read: every lane, before the row bound
        uint32_t w[32];
        lkg::tmem_ld32(tm_warp + 32 * r, w);
        if (a.ksplit > 1) {  // input split: this split's f64 sums go to its plane (ksplit_reduce_kernel)
          if (lane + 32 * r < rows_left) {
            double* pr = a.Ypart + ((int64_t)ks * a.rows + row) * a.m + j0;
#pragma unroll
            for (int q = 0; q < 16; q++)
              if (j0 + q < a.m) pr[q] = __hiloint2double((int)w[2 * q + 1], (int)w[2 * q]);
          }
        }
#pragma unroll
        for (int q = 0; q < 16; q++) out[q] = (float)__hiloint2double((int)w[2 * q + 1], (int)w[2 * q]);
      } else {
#pragma unroll
        for (int q = 0; q < 8; q++) {
          out[2 * q] = acc[r][q].x;
          out[2 * q + 1] = acc[r][q].y;
        }
      }
      if (lane + 32 * r < rows_left) {
        if (FUSE) {
          // next layer (runtime.cpp:298-314 chain) on this row's hidden activations out[0..m):
          // its whole value table is in shared memory (small layout, 2 outputs, MP2 == 2);
          // inputs in pairs with both fast coordinate chains side by side
          const int K2 = a.cc2.K, L2 = a.cc2.L;
          const float2* V2 = reinterpret_cast<const float2*>(lut2);
          const float2* CB2 = reinterpret_cast<const float2*>(lut2 + a.cb_off2);
          float2 y2 = make_float2(0.f, 0.f);
          bool r_oob2 = false;
#pragma unroll
          for (int i2 = 0; i2 < 16; i2 += 2) {
            if (i2 < a.m) {
              const float h0 = out[i2], h1 = i2 + 1 < a.m ? out[i2 + 1] : a.cc2.lo;
              bool s0, s1;
              lkg::Coord c0 = lkg::lut_coords_fast_nb(a.cc2, kf2, h0, s0);
              lkg::Coord c1 = lkg::lut_coords_fast_nb(a.cc2, kf2, h1, s1);
              if (s0 || s1) {
                if (s0) c0 = lkg::lut_coords(a.cc2, ktab2, h0);
                if (s1) c1 = lkg::lut_coords(a.cc2, ktab2, h1);
              }
              nfacc2 = fmaf(h0, 0.0f, fmaf(h1, 0.0f, nfacc2));
              const bool has1 = i2 + 1 < a.m;
              oob2_inputs += (uint32_t)!c0.in + (uint32_t)(has1 && !c1.in);
              r_oob2 |= !c0.in || (has1 && !c1.in);
#pragma unroll
              for (int t = 0; t < 2; t++) {
                const lkg::Coord& c = t ? c1 : c0;
                const float h = t ? h1 : h0;
                if (t == 0 || has1) {
                  const int ii = i2 + t;
                  const bool tab = !(ZS && !c.in);
                  // value table entry (k, l0, ii) of the interleaved small layout (build_small_vt_kernel)
                  const int ent = (c.k * L2 + c.l0) * a.m + ii;
                  const float2 v0 = V2[ent * (a.vp2 ? 2 : 1)];
                  const float2 v1 = a.vp2 ? V2[ent * 2 + 1] : V2[ent + a.m];
                  const float w1 = c.w1, w0 = 1.0f - w1;
                  float2 v = tab ? make_float2(fmaf(w1, v1.x, w0 * v0.x), fmaf(w1, v1.y, w0 * v0.y))
                                 : make_float2(0.f, 0.f);
                  if (SR) {
                    const float bx2 = lkg::silu_fast(ZS ? h : c.xp);
                    const float2 cb = CB2[ii];
                    v = make_float2(fmaf(cb.x, bx2, v.x), fmaf(cb.y, bx2, v.y));
                  }
                  y2 = make_float2(y2.x + v.x, y2.y + v.y);
                }
              }
            }
          }
          float* y2r = a.Y2 + row * a.m2;
          y2r[0] = y2.x;
          if (a.m2 > 1) y2r[1] = y2.y;
          oob2_rows += (uint32_t)r_oob2;
        } else if (a.ksplit == 1) {
          float* yr = a.Y + row * a.m + j0;
          LKG_DCHECK(row >= 0 && row < a.rows && j0 < a.m, "output coordinate out of range");
          if (j0 + 16 <= a.m && (a.m & 3) == 0) {
#pragma unroll
            for (int q = 0; q < 4; q++)
              reinterpret_cast<float4*>(yr)[q] = make_float4(out[4 * q], out[4 * q + 1], out[4 * q + 2], out[4 * q + 3]);
          } else {
#pragma unroll
            for (int q = 0; q < 16; q++)
              if (j0 + q < a.m) yr[q] = out[q];
          }
        }
        if (a.ksplit > 1) {
          // a row's inputs are spread over the splits: the first split to flag the row counts it
          if (cnt & (row_oob >> r)) {
            const uint32_t bit = 1u << (row & 31);
            oob_rows += (uint32_t)((atomicOr(a.rowflags + (row >> 5), bit) & bit) == 0u);
          }
        } else {
          oob_rows += (uint32_t)(cnt & (row_oob >> r));
        }
      }
    }
  }
  // OOB counters (runtime.cpp:216-222) and the non-finite flag (runtime.cpp:172)
  unsigned long long oi = oob_inputs, orow = oob_rows;
  for (int o = 16; o; o >>= 1) {
    oi += __shfl_xor_sync(0xffffffffu, oi, o);
    orow += __shfl_xor_sync(0xffffffffu, orow, o);
  }
  if (lane == 0) {
    if (orow) atomicAdd(a.counters + 0, orow);
    if (oi) atomicAdd(a.counters + 1, oi);
  }
  nonfinite |= !(nfacc == 0.0f);
  if (__any_sync(0xffffffffu, nonfinite) && lane == 0) atomicExch(a.counters + 2, 1ull);
  if (F64) {  // every warp is done with TMEM
    lkg::tmem_fence_before_sync();
    __syncthreads();
    lkg::tmem_fence_after_sync();
    if (warp == 0) lkg::tmem_dealloc(tm_base, kTmCols);
  }
  if (FUSE) {
    unsigned long long oi2 = oob2_inputs, orow2 = oob2_rows;
    for (int o = 16; o; o >>= 1) {
      oi2 += __shfl_xor_sync(0xffffffffu, oi2, o);
      orow2 += __shfl_xor_sync(0xffffffffu, orow2, o);
    }
    if (lane == 0) {
      if (orow2) atomicAdd(a.counters2 + 0, orow2);
      if (oi2) atomicAdd(a.counters2 + 1, oi2);
    }
    nonfinite2 |= !(nfacc2 == 0.0f);
    if (__any_sync(0xffffffffu, nonfinite2) && lane == 0) atomicExch(a.counters2 + 2, 1ull);
  }
}

template <int R, int W, bool ASYM, bool SR, bool ZS, bool F64, bool FUSE = false, int MINB = 1, bool GC = false,
          bool BAL = false, int XB = 1, bool XT = false, int IDPM = 0, bool REC = false, int NSX = 0>
void launch_tiled(cudaStream_t st, const TiledArgs& a, size_t smem, int grid) {
  auto kern = fwd_tiled<R, W, ASYM, SR, ZS, F64, FUSE, MINB, GC, BAL, XB, XT, IDPM, REC, NSX>;
  static bool attr = false;
  if (!attr) {
    LKG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
    static const char* co = getenv("LKG_CARVEOUT");  // experiment hook: shared-memory carveout %
    if (co) LKG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, atoi(co)));
    attr = true;
  }
  kern<<<grid, W * 32, smem, st>>>(a);
}

// The layer's table walk (TileGeom::idp) as a runtime choice over the compiled variants; pair lines
// are never used with codes in global memory.
template <int R, int W, bool ASYM, bool SR, bool ZS, bool F64, bool FUSE = false, int MINB = 1, bool GC = false,
          bool BAL = false, int XB = 1, bool XT = false, int NSX = 0>
void launch_idp(int idp, cudaStream_t st, const TiledArgs& a, size_t smem, int grid, bool rec = false) {
  if constexpr (NSX != 0) {  // the small-batch variant: standard lines only (integer or fp32 lerp)
    if (idp == 2)
      launch_tiled<R, W, ASYM, SR, ZS, F64, FUSE, MINB, GC, BAL, XB, XT, 2, false, NSX>(st, a, smem, grid);
    else
      launch_tiled<R, W, ASYM, SR, ZS, F64, FUSE, MINB, GC, BAL, XB, XT, 0, false, NSX>(st, a, smem, grid);
    return;
  }
  if constexpr (XT) {
    if (rec) {  // coordinate records (coord_pass_kernel) over the standard lines / the GC pair entries
      if constexpr (GC) {
        if (idp == 3) {
          launch_tiled<R, W, ASYM, SR, ZS, F64, FUSE, MINB, GC, BAL, XB, XT, 3, true>(st, a, smem, grid);
          return;
        }
      }
      launch_tiled<R, W, ASYM, SR, ZS, F64, FUSE, MINB, GC, BAL, XB, XT, 2, true>(st, a, smem, grid);
      return;
    }
  }
  if constexpr (GC) {
    if (idp == 3) {  // pair entries in global memory
      launch_tiled<R, W, ASYM, SR, ZS, F64, FUSE, MINB, GC, BAL, XB, XT, 3>(st, a, smem, grid);
      return;
    }
  }
  if (idp == 2) {
    launch_tiled<R, W, ASYM, SR, ZS, F64, FUSE, MINB, GC, BAL, XB, XT, 2>(st, a, smem, grid);
    return;
  }
  if constexpr (!GC) {
    if (idp == 1) {
      launch_tiled<R, W, ASYM, SR, ZS, F64, FUSE, MINB, GC, BAL, XB, XT, 1>(st, a, smem, grid);
      return;
    }
  }
  launch_tiled<R, W, ASYM, SR, ZS, F64, FUSE, MINB, GC, BAL, XB, XT, 0>(st, a, smem, grid);
}


}  // namespace
