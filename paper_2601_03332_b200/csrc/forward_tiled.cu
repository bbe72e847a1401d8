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

// ---------------------------------------------------------------------------------------
// Small-out_dim layers (m <= 8, whole table <= ~200 KB, d <= 256): the entire layer is
// resident in shared memory. Lane = row: each lane walks every input of its row — starting
// at input (lane mod d) so the lanes of a warp read different inputs' tables — and keeps its
// m outputs in registers (no cross-lane reduction). Preferred table (VT): the dequantized
// value table V[i][k][l][MP] = f32(out*spline*(y_min + scale*q)) and CB[i][MP]; fallback for
// larger tables: codes [i][k][l][MP] + P/Q [i][k][MP] + CB.
struct SmallArgs {
  const uint8_t* lut;
  int32_t lut_bytes, p_off, q_off, cb_off, MP;
  const float* X;
  int64_t rows;
  int32_t d, x_blk;
  float* Y;
  int32_t m;
  unsigned long long* counters;
  lkg::CoordConst cc;
  float4 ktab[kMaxKT];
};

// n consecutive floats from shared memory with the widest aligned vector loads
template <int N>
__device__ __forceinline__ void lkg_small_load(const float* p, float (&v)[N]) {
  if constexpr (N % 4 == 0) {
#pragma unroll
    for (int j = 0; j < N; j += 4) {
      const float4 t = *reinterpret_cast<const float4*>(p + j);
      v[j] = t.x, v[j + 1] = t.y, v[j + 2] = t.z, v[j + 3] = t.w;
    }
  } else if constexpr (N % 2 == 0) {
#pragma unroll
    for (int j = 0; j < N; j += 2) {
      const float2 t = *reinterpret_cast<const float2*>(p + j);
      v[j] = t.x, v[j + 1] = t.y;
    }
  } else {
#pragma unroll
    for (int j = 0; j < N; j++) v[j] = p[j];
  }
}

template <bool ASYM, bool SR, bool ZS, bool VT, int MPT, bool VP = false>
__global__ void __launch_bounds__(1024) fwd_small(const __grid_constant__ SmallArgs a) {
  extern __shared__ __align__(128) uint8_t smem[];
  uint8_t* lut = smem;
  float4* ktab = reinterpret_cast<float4*>(smem + ((a.lut_bytes + 15) & ~15));
  float2* kf = reinterpret_cast<float2*>(ktab + kMaxKT);  // compact {T_k, (L-1)/h_k} (coords.cuh)
  const int tid = threadIdx.x, lane = tid & 31;
  // the table arrives by TMA bulk copies issued by one thread (small batches run small blocks, where
  // a per-thread copy loop is a chain of L2 round trips); odd sizes take the loop
  __shared__ __align__(8) uint64_t tbar;
  const bool bulk = (a.lut_bytes & 15) == 0 && (reinterpret_cast<uintptr_t>(a.lut) & 15) == 0;
  if (bulk) {
    if (tid == 0) {
      mbar_init(&tbar, 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      mbar_expect_tx(&tbar, (uint32_t)a.lut_bytes);
      for (int32_t o = 0; o < a.lut_bytes; o += 32768)
        bulk_g2s(lut + o, a.lut + o, (uint32_t)(a.lut_bytes - o < 32768 ? a.lut_bytes - o : 32768), &tbar);
    }
  } else {
    for (int o = tid * 16; o < a.lut_bytes; o += blockDim.x * 16)
      *reinterpret_cast<uint4*>(lut + o) = __ldg(reinterpret_cast<const uint4*>(a.lut + o));
  }
  for (int k = tid; k < a.cc.K; k += blockDim.x) {
    ktab[k] = a.ktab[k];
    kf[k] = make_float2(a.ktab[k].x, a.ktab[k].y);
  }
  __syncthreads();
  if (bulk) mbar_wait(&tbar, 0);
  const float lo = a.cc.lo;
  const int K = a.cc.K, L = a.cc.L, d = a.d, MP = VT ? MPT : a.MP;
  const int64_t x_rs = a.x_blk > 0 ? a.x_blk : d;
  const int i0 = lane % d;
  const float* V = reinterpret_cast<const float*>(lut);
  const float* CBt = reinterpret_cast<const float*>(lut + a.cb_off);
  uint32_t oob_inputs = 0, oob_rows = 0;
  bool nonfinite = false;
  float nfacc = 0.0f;
  // input pairs need 8-byte aligned (i, i+1) in the same row / column block
  const bool pairs = (d % 2 == 0) && (a.x_blk > 0 ? a.x_blk % 2 == 0 : true) &&
                     ((reinterpret_cast<uintptr_t>(a.X) & 7) == 0);
  // Each block owns an equal, 64-aligned row range (a row keeps its lane, hence its input
  // rotation and result bits, under any split): the SMs get equal work, where a grid-stride walk
  // over 1024-row chunks left some SMs 8 chunks and others 6 (configs[1] layer 1).
  const int64_t b_lo = (a.rows * blockIdx.x / gridDim.x) / 64 * 64;
  const int64_t b_hi = blockIdx.x + 1 == gridDim.x ? a.rows : (a.rows * (blockIdx.x + 1) / gridDim.x) / 64 * 64;
  for (int64_t rb = b_lo; rb < b_hi; rb += blockDim.x) {
    const int64_t row = rb + tid;
    if (rb + (tid & ~31) >= b_hi) break;  // this warp has no row left (warp-uniform)
    const bool vrow = row < b_hi;
    float y[8];
#pragma unroll
    for (int j = 0; j < 8; j++) y[j] = 0.0f;
    bool any_oob = false;
    // one input's table walk + base branch for this row (runtime.cpp:192-212)
    auto accum = [&](int i, float x, const lkg::Coord& co) {
      oob_inputs += (uint32_t)!co.in;
      any_oob |= !co.in;
      const bool tab = !(ZS && !co.in);
      float bx = 0.0f;
      if (SR) {
        const float xb = ZS ? x : co.xp;  // clip_x clips the base branch too (runtime.cpp:189)
        bx = lkg::silu_fast(xb);
      }
      const int cell = i * K + co.k;
      const float w1 = co.w1, w0 = 1.0f - w1;
      const float* CB = CBt + i * MP;
      if (VT) {
        // Interleaved value table V[k][l][i] (input fastest, build_small_vt_kernel): the lanes of a
        // load phase walk different inputs (i = lane + t mod d), so their entries sit in distinct
        // bank groups whatever (k, l0) each row selects. VP: each entry also holds the next
        // sample's values (one load); otherwise the next sample is the next line (+d entries).
        // l0 = L-1 comes with w1 = 0, and the table ends with a padding line.
        constexpr int ES = VP ? 2 * MPT : MPT;
        const float* V0 = V + ((int64_t)(co.k * L + co.l0) * d + i) * ES;
        LKG_DCHECK(co.k >= 0 && co.k < K && co.l0 >= 0 && co.l0 < L && i >= 0 && i < d, "value-table index");
        LKG_DCHECK((VP ? ((int64_t)(co.k * L + co.l0) * d + i + 1) * ES
                       : ((int64_t)(co.k * L + co.l0 + 1) * d + i + 1) * ES) * 4 <= a.cb_off,
                   "value-table entry past the table");
        float v0[MPT], v1[MPT], cb[MPT];
        lkg_small_load<MPT>(V0, v0);
        lkg_small_load<MPT>(VP ? V0 + MPT : V0 + d * ES, v1);
        if (SR) lkg_small_load<MPT>(CB, cb);
#pragma unroll
        for (int j = 0; j < MPT; j++) {
          const float v = tab ? fmaf(w1, v1[j], w0 * v0[j]) : 0.0f;
          y[j] += SR ? fmaf(cb[j], bx, v) : v;
        }
      } else {
        const int l1 = min(co.l0 + 1, L - 1);
        const uint8_t* c0 = lut + (cell * L + co.l0) * MP;
        const uint8_t* c1 = lut + (cell * L + l1) * MP;
        const float* P = reinterpret_cast<const float*>(lut + a.p_off) + cell * MP;
        const float* Q = reinterpret_cast<const float*>(lut + a.q_off) + cell * MP;
#pragma unroll
        for (int j = 0; j < 8; j++) {
          if (j < MP) {
            const float q0 = ASYM ? (float)c0[j] : (float)(int8_t)c0[j];
            const float q1 = ASYM ? (float)c1[j] : (float)(int8_t)c1[j];
            float v = 0.0f;
            if (tab) {
              v = P[j] * fmaf(w1, q1, w0 * q0);
              if (ASYM) v += Q[j];
            }
            y[j] += SR ? fmaf(CB[j], bx, v) : v;
          }
        }
      }
    };
    const float* xrow = a.X + row * x_rs;  // this row (row-major layout)
    auto x_ptr = [&](int i) -> const float* {
      if (a.x_blk > 0) {  // blocked all-gather layout [i / x_blk][rows][x_blk]
        const int b = i / a.x_blk;
        return a.X + (int64_t)b * a.rows * a.x_blk + row * x_rs + (i - b * a.x_blk);
      }
      return xrow + i;
    };
    if (pairs && !VT) {
      // inputs in pairs (i even): one 8-byte load, both fast coordinate chains side by side,
      // the exact path once if either needs it
      // the next pair's load is issued one iteration ahead (its latency was the top stall)
      int i = 2 * (lane % (d >> 1));
      float2 xn = make_float2(lo, lo);
      if (vrow) xn = __ldg(reinterpret_cast<const float2*>(x_ptr(i)));
      for (int t = 0; t < d; t += 2, i = (i + 2 == d) ? 0 : i + 2) {
        const float2 xx = xn;
        const int inx = (i + 2 == d) ? 0 : i + 2;
        if (vrow && t + 2 < d) xn = __ldg(reinterpret_cast<const float2*>(x_ptr(inx)));
        bool s0, s1;
        lkg::Coord c0 = lkg::lut_coords_fast_nb(a.cc, kf, xx.x, s0);
        lkg::Coord c1 = lkg::lut_coords_fast_nb(a.cc, kf, xx.y, s1);
        if (s0 || s1) {
          if (s0) c0 = lkg::lut_coords(a.cc, ktab, xx.x);
          if (s1) c1 = lkg::lut_coords(a.cc, ktab, xx.y);
        }
        nfacc = fmaf(xx.x, 0.0f, fmaf(xx.y, 0.0f, nfacc));  // NaN once any input is NaN or inf
        accum(i, xx.x, c0);
        accum(i + 1, xx.y, c1);
      }
    } else if (VT && a.x_blk <= 0 && (d & 1) == 0 && rb + (tid | 31) < b_hi) {
      // the common case of the walk below — row-major input, an even input count, every row of the
      // warp valid — without its per-load layout, row-bound and odd-tail tests (the same inputs in
      // the same order: identical bits)
      auto nxt = [&](int v) { return v + 1 == d ? 0 : v + 1; };
      int i = i0;
      float xa_n = __ldg(xrow + i), xb_n = __ldg(xrow + nxt(i));
      for (int t = 0; t < d; t += 2) {
        const int ia = i, ib = nxt(i);
        const float xa = xa_n, xb = xb_n;
        i = nxt(ib);
        if (t + 2 < d) {
          xa_n = __ldg(xrow + i);
          xb_n = __ldg(xrow + nxt(i));
        }
        bool s0, s1;
        lkg::Coord c0 = lkg::lut_coords_fast_nb(a.cc, kf, xa, s0);
        lkg::Coord c1 = lkg::lut_coords_fast_nb(a.cc, kf, xb, s1);
        if (s0 || s1) {
          if (s0) c0 = lkg::lut_coords(a.cc, ktab, xa);
          if (s1) c1 = lkg::lut_coords(a.cc, ktab, xb);
        }
        nfacc = fmaf(xa, 0.0f, nfacc);  // NaN once any input is NaN or inf
        accum(ia, xa, c0);
        nfacc = fmaf(xb, 0.0f, nfacc);
        accum(ib, xb, c1);
      }
    } else if (VT) {
      // the interleaved value table wants consecutive lanes on consecutive inputs: lane walks
      // i0, i0+1, ... (mod d) two inputs per iteration (two independent coordinate chains), the
      // next pair's x loads one iteration ahead
      auto nxt = [&](int v) { return v + 1 == d ? 0 : v + 1; };
      int i = i0;
      float xa_n = lo, xb_n = lo;
      if (vrow) {
        xa_n = __ldg(x_ptr(i));
        if (d > 1) xb_n = __ldg(x_ptr(nxt(i)));
      }
      for (int t = 0; t < d; t += 2) {
        const int ia = i, ib = nxt(i);
        const float xa = xa_n, xb = xb_n;
        i = nxt(ib);
        if (vrow && t + 2 < d) {
          xa_n = __ldg(x_ptr(i));
          if (t + 3 < d) xb_n = __ldg(x_ptr(nxt(i)));
        }
        const bool two = t + 1 < d;
        bool s0, s1;
        lkg::Coord c0 = lkg::lut_coords_fast_nb(a.cc, kf, xa, s0);
        lkg::Coord c1 = lkg::lut_coords_fast_nb(a.cc, kf, two ? xb : lo, s1);
        if (s0 || s1) {
          if (s0) c0 = lkg::lut_coords(a.cc, ktab, xa);
          if (s1) c1 = lkg::lut_coords(a.cc, ktab, xb);
        }
        nfacc = fmaf(xa, 0.0f, nfacc);  // NaN once any input is NaN or inf
        accum(ia, xa, c0);
        if (two) {
          nfacc = fmaf(xb, 0.0f, nfacc);
          accum(ib, xb, c1);
        }
      }
    } else {
      int i = i0;
      float xn = lo;
      if (vrow) xn = __ldg(x_ptr(i));
      for (int t = 0; t < d; t++, i = (i + 1 == d) ? 0 : i + 1) {
        const float x = xn;
        if (vrow && t + 1 < d) xn = __ldg(x_ptr(i + 1 == d ? 0 : i + 1));
        const lkg::Coord co = lkg::lut_coords_fast(a.cc, ktab, kf, x);
        nfacc = fmaf(x, 0.0f, nfacc);
        accum(i, x, co);
      }
    }
    if (vrow) {
      float* yr = a.Y + row * a.m;
      LKG_DCHECK(row >= 0 && row < a.rows, "small-layer output row out of range");
#pragma unroll
      for (int j = 0; j < 8; j++)
        if (j < a.m) yr[j] = y[j];
      oob_rows += any_oob;
    }
  }
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
}

// Dequantized value table for small layers: V[i][k][l][j] = (f32)(cs * (y_min + scale * q)),
// cs = out*spline (1 for phi), evaluated in f64 like fetch_quant (runtime.cpp:124-128, 202-205).
// Layout: entry (k, l, i) at ((k*L + l)*d + i) * ES floats, ES = MP (vp = 0) or 2*MP (vp = 1: the
// entry also holds sample l+1's values; sample L-1 repeats its own).
__global__ void build_small_vt_kernel(const uint8_t* q, const float* scale, const float* ymin, const float* gains,
                                      float* V, int32_t d, int32_t m, int32_t K, int32_t L, int32_t MP,
                                      int32_t cb_off, int sr, int sym, int vp) {
  const int64_t cell = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t E = (int64_t)d * m;
  if (cell >= E * K) return;
  const int64_t e = cell / K;
  const int k = (int)(cell - e * K);
  const int i = (int)(e / m), j = (int)(e - (int64_t)i * m);
  const double cs = sr ? (double)gains[2 * E + e] * (double)gains[E + e] : 1.0;
  const double ym = ymin[cell], sc = scale[cell];
  const int ES = vp ? 2 * MP : MP;
  for (int l = 0; l < L; l++) {
    const uint8_t b = q[cell * L + l];
    const double qv = sym ? (double)(int8_t)b : (double)b;
    const float v = (float)(cs * (ym + sc * qv));
    float* ent = V + ((int64_t)(k * L + l) * d + i) * ES;
    ent[j] = v;
    if (vp) {
      if (l > 0) ent[j - (int64_t)d * ES + MP] = v;  // the previous sample's "next" slot
      if (l == L - 1) ent[MP + j] = v;
    }
  }
  if (sr && k == 0)
    reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(V) + cb_off)[i * MP + j] =
        (float)((double)gains[2 * E + e] * (double)gains[e]);
}

__global__ void build_small_kernel(const uint8_t* q, const float* scale, const float* ymin, const float* gains,
                                   uint8_t* lut, int32_t d, int32_t m, int32_t K, int32_t L, int32_t MP,
                                   int32_t p_off, int32_t q_off, int32_t cb_off, int sr, int asym) {
  const int64_t cell = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t E = (int64_t)d * m;
  if (cell >= E * K) return;
  const int64_t e = cell / K;
  const int k = (int)(cell - e * K);
  const int i = (int)(e / m), j = (int)(e - (int64_t)i * m);
  for (int l = 0; l < L; l++) lut[((int64_t)(i * K + k) * L + l) * MP + j] = q[cell * L + l];
  const double cs = sr ? (double)gains[2 * E + e] * (double)gains[E + e] : 1.0;
  reinterpret_cast<float*>(lut + p_off)[(i * K + k) * MP + j] = (float)(cs * (double)scale[cell]);
  if (asym) reinterpret_cast<float*>(lut + q_off)[(i * K + k) * MP + j] = (float)(cs * (double)ymin[cell]);
  if (sr && k == 0)
    reinterpret_cast<float*>(lut + cb_off)[i * MP + j] = (float)((double)gains[2 * E + e] * (double)gains[e]);
}

// Reference layout -> tiles (one thread per (edge, segment) cell). idp: 1 = pair lines, 2 = standard
// lines; both store P pre-scaled by 2^-15 (exact) for the integer lerp.
__global__ void build_tiles_kernel(const uint8_t* q, const float* scale, const float* ymin, const float* gains,
                                   uint8_t* tiles, int64_t tile_bytes, int32_t n_ih, int32_t d, int32_t m,
                                   int32_t K, int32_t L, int32_t p_off, int32_t q_off, int32_t cb_off, int sym,
                                   int sr, int asym, int idp) {
  const int64_t cell = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t E = (int64_t)d * m;
  if (cell >= E * K) return;
  const int64_t e = cell / K;
  const int k = (int)(cell - e * K);
  const int i = (int)(e / m), j = (int)(e - (int64_t)i * m);
  const int ih = i / G, il = i % G, jb = j / JB, jl = j % JB;
  uint8_t* t = tiles + ((int64_t)jb * n_ih + ih) * tile_bytes;
  const uint8_t* src = q + cell * L;
  if (idp == 3) {
    for (int l = 0; l < L; l++) {
      uint8_t* ent = t + gce_off(il, k, l, K, L) + (jl >> 1) * 4 + (jl & 1) * 2;
      ent[0] = sym ? (uint8_t)(src[l] ^ 0x80u) : src[l];
      ent[1] = l + 1 < L ? (sym ? (uint8_t)(src[l + 1] ^ 0x80u) : src[l + 1]) : 0;
    }
  } else if (idp == 1) {
    for (int l = 0; l < L; l++) {
      uint8_t* line = t + (int64_t)(k * L + l) * PLINE;
      line[pair_off(il, jl, 0)] = sym ? (uint8_t)(src[l] ^ 0x80u) : src[l];
      line[pair_off(il, jl, 1)] = l + 1 < L ? (sym ? (uint8_t)(src[l + 1] ^ 0x80u) : src[l + 1]) : 0;
    }
  } else {
    for (int l = 0; l < L; l++) t[(k * L + l) * LINE + il * JB + jl] = sym ? (uint8_t)(src[l] ^ 0x80u) : src[l];
  }
  // fused gains in f64 (runtime.cpp:263-273), then one rounding to f32
  const double cs = sr ? (double)gains[2 * E + e] * (double)gains[E + e] : 1.0;
  float* P = reinterpret_cast<float*>(t + p_off + (k * G + il) * PROW) + jl;
  *P = (float)(cs * (double)scale[cell]) * (idp ? 0x1p-15f : 1.0f);
  if (asym) *reinterpret_cast<float*>(t + q_off + (k * G + il) * PROW + jl * 4) = (float)(cs * (double)ymin[cell]);
  if (sr && k == 0)
    *reinterpret_cast<float*>(t + cb_off + il * PROW + jl * 4) = (float)((double)gains[2 * E + e] * (double)gains[e]);
}

// Weight-rounding error of the integer lerp, per output column j: sum over inputs i of
// (max_k |P_kij| * max_l |u_l+1 - u_l|)^2 (one thread per edge; f64 atomics). W1 = round(w1 2^15)
// moves each interpolant by at most that product times 2^-16, independently per input.
//
// acc[m + j] (fp32-accumulation bound): sum over inputs i of the squared largest term edge (i, j) can
// contribute, (max_kl |table value| + |cb| * silu_max)^2 — the scale of output j's partial sums.
__global__ void idp_bound_kernel(const uint8_t* q, const float* scale, const float* ymin, const float* gains,
                                 int32_t d, int32_t m, int32_t K, int32_t L, int sr, int sym, double silu_max,
                                 double* acc) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t E = (int64_t)d * m;
  if (e >= E) return;
  const double cs = sr ? std::fabs((double)gains[2 * E + e] * (double)gains[E + e]) : 1.0;
  double worst = 0.0, vmax = 0.0;
  for (int k = 0; k < K; k++) {
    const uint8_t* c = q + (e * K + k) * L;
    const double sc = (double)scale[e * K + k], ym = sym ? 0.0 : (double)ymin[e * K + k];
    int dq = 0;
    for (int l = 0; l < L; l++) {
      const int a0 = sym ? (int)(int8_t)c[l] : (int)c[l];
      if (l + 1 < L) dq = max(dq, abs((sym ? (int)(int8_t)c[l + 1] : (int)c[l + 1]) - a0));
      vmax = fmax(vmax, cs * std::fabs(ym + sc * a0));
    }
    worst = fmax(worst, cs * std::fabs(sc) * dq);
  }
  atomicAdd(acc + (e % m), worst * worst);
  const double term = vmax + (sr ? std::fabs((double)gains[2 * E + e] * (double)gains[e]) * silu_max : 0.0);
  atomicAdd(acc + m + (e % m), term * term);
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

namespace lkg {

#ifndef LKG_W
#define LKG_W 16
#endif
#ifndef LKG_R
#define LKG_R 2
#endif
static constexpr int kW = LKG_W, kR = LKG_R;    // fp32 mode: 16 warps x 64 rows = 1024-row tiles
static constexpr int kW64 = kW, kR64 = kR;      // f64 mode: same shape, f64 accumulators in TMEM
static constexpr int kSmallMaxBytes = 200 * 1024;
static constexpr double kIdpRss = 1.5e-6;  // IDP weight-rounding bound (build_tiles)
static constexpr double kAcc32Max = 4e-6;  // fp32-accumulation error estimate above which a layer takes f64

bool tiled_eligible(const lkg_layer* L) {
  if (L->float_table.p || L->K > kMaxKT) return false;
  return L->geom.tile_bytes > 0;
}

void build_tiles(lkg_ctx* ctx, lkg_layer* L) {
  TileGeom& gm = L->geom;
  gm = TileGeom{};
  if (L->float_table.p || L->K > kMaxKT) return;
  {  // the in-kernel segment estimate needs uniformly spaced knots (all BASELINE grids are)
    double hmin = 1e300, hmax = 0;
    for (int k = 0; k < L->K; k++) {
      hmin = std::min(hmin, (double)L->knots[k + 1] - L->knots[k]);
      hmax = std::max(hmax, (double)L->knots[k + 1] - L->knots[k]);
    }
    if (hmax > hmin * (1.0 + 1e-4)) return;
  }
  const int d = L->in_dim, m = L->col1 - L->col0, K = L->K, Ls = L->L;
  const bool asym = L->scheme == LKG_SCHEME_ASYMMETRIC, sr = L->value_repr == LKG_REPR_SPLINE_COMPONENT;
  const int64_t cells = (int64_t)d * m * K;
  // Per-layer precision bounds from the codes (idp_bound_kernel): the integer lerp's weight-rounding
  // error, and the scale of the partial sums an fp32 accumulator would carry. fp32 accumulation (d <=
  // 256) rounds every add at the partial sum's ulp: with terms of rms t the error is ~2^-24 t d /
  // sqrt(3) (a random walk of d roundings at |partial| ~ t sqrt(d)); the BASELINE layers sit at 1-2e-6,
  // but a layer with large gains (a 1000-seed fuzz campaign: d = 130, coefficients N(0, 0.3^2), gains
  // up to 2.25 -> 2-4e-5 on a few outputs) does not. Above kAcc32Max the layer takes the f64 (TMEM)
  // accumulators whatever its width, and no fp32-accumulating small-layer kernel.
  double idp_rss = -1.0;
  if (L->q.p) {
    DBuf acc;
    acc.alloc(sizeof(double) * 2 * m);
    LKG_CUDA(cudaMemsetAsync(acc.p, 0, acc.bytes, ctx->stream));
    const int64_t E = (int64_t)d * m;
    auto silu = [](double x) { return x / (1.0 + std::exp(-x)); };
    // base activation range: x' in [t_0, t_K] under clip_x; zero_spline feeds the raw input (taken as
    // up to half a grid width outside)
    const bool zs = L->oob_policy == LKG_OOB_ZERO_SPLINE;
    const double lo = L->knots[0], hi = L->knots[K], ext = zs ? 0.5 * (hi - lo) : 0.0;
    const double silu_max = std::max({std::fabs(silu(lo - ext)), std::fabs(silu(hi + ext)), 0.2785});
    idp_bound_kernel<<<(unsigned)((E + 255) / 256), 256, 0, ctx->stream>>>(
        L->q.as<uint8_t>(), L->scale.as<float>(), L->ymin.as<float>(), L->gains.as<float>(), d, m, K, Ls, sr, !asym,
        silu_max, acc.as<double>());
    LKG_CUDA(cudaGetLastError());
    ctx->launches++;
    std::vector<double> h(2 * m);
    LKG_CUDA(cudaMemcpyAsync(h.data(), acc.p, acc.bytes, cudaMemcpyDeviceToHost, ctx->stream));
    LKG_CUDA(cudaStreamSynchronize(ctx->stream));
    double worst = 0.0, t2 = 0.0;
    for (int j = 0; j < m; j++) {
      worst = std::max(worst, h[j]);
      t2 = std::max(t2, h[m + j]);
    }
    idp_rss = std::sqrt(worst) * 0x1p-16;
    gm.acc32_err = 0x1p-24 * std::sqrt(t2 / 3.0) * std::sqrt((double)d);
    static const char* a64 = getenv("LKG_ACC64");  // test / A-B hook: 1 forces, 0 forbids
    gm.acc64 = a64 ? (a64[0] == '1') : (d <= kFp32MaxD && gm.acc32_err > kAcc32Max);
    static const bool verbose = getenv("LKG_VERBOSE") != nullptr;
    if (verbose)
      fprintf(stderr, "lkg build_tiles %dx%d K%d L%d: idp_rss %.3g acc32_err %.3g acc64 %d\n", d, m, K, Ls, idp_rss,
              gm.acc32_err, gm.acc64);
  }
  // small out_dim: the whole layer in shared memory (fwd_small)
  if (m <= 8 && d <= kFp32MaxD && !gm.acc64) {
    const int MP = m <= 1 ? 1 : (m <= 2 ? 2 : (m <= 4 ? 4 : 8));
    // preferred: dequantized value table V = out*spline*(y_min + scale*q) in f32 (one rounding of
    // the f64 product), so the table walk is two loads and two FMAs per edge
    // interleaved V[k][l][i] (conflict-free lane walk), with the next sample in each entry when
    // that still fits (vp, one load per edge), else a padding line for the next-line read
    int vp = 1;
    int64_t vt = (int64_t)K * Ls * d * 2 * MP * 4;
    if (vt + ((int64_t)d * MP * 4 + 15) / 16 * 16 + kMaxKT * 16 > kSmallMaxBytes) {
      vp = 0;
      vt = ((int64_t)(K * Ls + 1) * d * MP * 4 + 15) / 16 * 16;
    }
    const int64_t vt_total = vt + ((int64_t)d * MP * 4 + 15) / 16 * 16;
    if (vt_total + kMaxKT * 16 <= kSmallMaxBytes) {
      gm.small = 2;
      gm.MP = MP;
      gm.p_off = vp;  // (small == 2: p_off carries the pair flag)
      gm.cb_off = (int32_t)vt;
      gm.tile_bytes = vt_total;
      L->tiles.alloc((size_t)vt_total);
      LKG_CUDA(cudaMemsetAsync(L->tiles.p, 0, L->tiles.bytes, ctx->stream));
      build_small_vt_kernel<<<(unsigned)((cells + 255) / 256), 256, 0, ctx->stream>>>(
          L->q.as<uint8_t>(), L->scale.as<float>(), L->ymin.as<float>(), L->gains.as<float>(),
          L->tiles.as<float>(), d, m, K, Ls, MP, gm.cb_off, sr, !asym, vp);
      LKG_CUDA(cudaGetLastError());
      ctx->launches++;
      return;
    }
    int64_t off = ((int64_t)d * K * Ls * MP + 15) / 16 * 16;
    const int64_t pq = ((int64_t)d * K * MP * 4 + 15) / 16 * 16;
    gm.p_off = (int32_t)off;
    off += pq;
    gm.q_off = (int32_t)off;
    if (asym) off += pq;
    gm.cb_off = (int32_t)off;
    off += ((int64_t)d * MP * 4 + 15) / 16 * 16;
    if (off + kMaxKT * 16 <= kSmallMaxBytes) {
      gm.small = 1;
      gm.MP = MP;
      gm.tile_bytes = off;
      L->tiles.alloc((size_t)off);
      LKG_CUDA(cudaMemsetAsync(L->tiles.p, 0, L->tiles.bytes, ctx->stream));
      build_small_kernel<<<(unsigned)((cells + 255) / 256), 256, 0, ctx->stream>>>(
          L->q.as<uint8_t>(), L->scale.as<float>(), L->ymin.as<float>(), L->gains.as<float>(), L->tiles.as<uint8_t>(),
          d, m, K, Ls, MP, gm.p_off, gm.q_off, gm.cb_off, sr, asym);
      LKG_CUDA(cudaGetLastError());
      ctx->launches++;
      return;
    }
  }
  // Integer-lerp (IDP) walk when its weight rounding stays far inside the parity bar: the 2^-16
  // weight error moves output j by a sum of independent terms whose root-sum-square is at most
  // sqrt(sum_i e_ij^2) 2^-16 (idp_bound_kernel); allowed up to kIdpRss (a 6-sigma tail of that,
  // plus the fp32 accumulation's ~1e-6, stays below 1e-5). LKG_IDP=0 forces the fp32 lerp.
  static const char* idp_env = getenv("LKG_IDP");
  int idp = 0;
  if (!(idp_env && idp_env[0] == '0') && idp_rss >= 0.0) {
    gm.idp_rss = idp_rss;
    idp = gm.idp_rss <= kIdpRss ? 2 : 0;
  }
  const size_t xs_bytes = (size_t)1 * kW * G * (32 * kR + 4) * 4;  // one x buffer (fwd_tiled XB)
  auto layout = [&](int mode) {  // tile offsets for the given code layout; returns the tile bytes
    int64_t o = mode == 3   ? (int64_t)K * Ls * G * GCE
                : mode == 1 ? (int64_t)K * Ls * PLINE
                            : (int64_t)(K * Ls + 1) * LINE;
    gm.p_off = (int32_t)o;
    o += (int64_t)(K + 1) * G * PROW;
    if (asym) {
      gm.q_off = (int32_t)o;
      o += (int64_t)(K + 1) * G * PROW;
    }
    if (sr) {
      gm.cb_off = (int32_t)o;
      o += G * PROW;
    }
    return (o + 127) / 128 * 128;
  };
  static const bool force_gc = getenv("LKG_FORCE_GC") != nullptr;  // test / tuning hook
  // Pair lines (twice the code bytes, no PRMT) only on request (LKG_IDP=1) and where two stage
  // buffers of them fit: measured on configs[1] layer 0 they lose to the standard lines (0.496 vs
  // 0.446 ms), which leave room for the second x buffer and halve the TMA bytes per tile.
  if (idp && idp_env && idp_env[0] == '1' && !force_gc && 2 * layout(1) + xs_bytes + kMaxKT * 32 + 256 <= 227 * 1024)
    idp = 1;
  int64_t off = layout(idp == 1 ? 1 : 0);
  gm.idp = idp;
  gm.codes_global = force_gc || 2 * off + xs_bytes + kMaxKT * 32 + 256 > 227 * 1024;  // codes stay in global (L2)
  if (gm.codes_global && 2 * (off - gm.p_off) + xs_bytes + kMaxKT * 32 + 256 > 227 * 1024) return;  // generic
  // Codes in global memory on the integer-lerp walk: pair entries (twice the code bytes; one 256-bit
  // load of one sector per (row, input) instead of two 16-byte loads from two lines plus 8 PRMT — the
  // walk was L1TEX-bound on sectors) when the device has room for them. LKG_GCPAIR=0 keeps the lines.
  if (gm.codes_global && idp == 2) {
    static const char* gp = getenv("LKG_GCPAIR");
    const int64_t off3 = layout(3);
    size_t mfree = 0, mtotal = 0;
    LKG_CUDA(cudaMemGetInfo(&mfree, &mtotal));
    const size_t need = (size_t)((d + G - 1) / G) * ((m + JB - 1) / JB) * (size_t)off3;
    // Only where a tile's code lines outgrow L1 anyway (configs[4]: 262 KB per tile, measured 162.5 ->
    // 148.9 ms per layer); a tile that L1 holds (configs[2] at L=128: 131 KB) is faster on the lines
    // (0.466 vs 0.532 ms: the doubled bytes halve its L1 hit rate). LKG_GCPAIR=1 forces the entries.
    const bool big = (int64_t)(K * Ls + 1) * LINE > 192 * 1024 || (gp && gp[0] == '1');
    if (!(gp && gp[0] == '0') && big && need + (4ull << 30) <= mfree) {
      idp = 3;
      gm.idp = 3;
      off = off3;
    } else {
      off = layout(0);  // (restores the offsets of the standard lines)
    }
  }
  gm.tile_bytes = off;
  gm.JB = JB;
  gm.IC = G;
  gm.n_ih = (d + G - 1) / G;
  gm.n_jb = (m + JB - 1) / JB;
  L->tiles.alloc((size_t)gm.n_ih * gm.n_jb * off);
  LKG_CUDA(cudaMemsetAsync(L->tiles.p, 0, L->tiles.bytes, ctx->stream));
  build_tiles_kernel<<<(unsigned)((cells + 255) / 256), 256, 0, ctx->stream>>>(
      L->q.as<uint8_t>(), L->scale.as<float>(), L->ymin.as<float>(), L->gains.as<float>(), L->tiles.as<uint8_t>(),
      off, gm.n_ih, d, m, K, Ls, gm.p_off, gm.q_off, gm.cb_off, !asym, sr, asym, gm.idp);
  LKG_CUDA(cudaGetLastError());
  ctx->launches++;
  // Layers above 2 GB of codes (configs[3]/[4]) keep their codes only in the tiles; the reference
  // layout is rebuilt from the tiles on download (download_q_from_tiles).
  const char* lim = getenv("LKG_TILE_ONLY_BYTES");  // test hook: force the tiles-only mode
  if (L->q.bytes > (lim ? strtoull(lim, nullptr, 10) : (2ull << 30))) {
    LKG_CUDA(cudaStreamSynchronize(ctx->stream));
    L->q.release();
  }
}

// Tiles -> reference q layout for input rows [i0, i1) (inverse of build_tiles_kernel's code scatter).
__global__ void tiles_to_q_kernel(const uint8_t* tiles, int64_t tile_bytes, int32_t n_ih, int32_t i0, int32_t i1,
                                  int32_t m, int32_t K, int32_t L, int sym, int idp, uint8_t* q) {
  const int64_t cell = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;  // cell within the chunk
  const int64_t n = (int64_t)(i1 - i0) * m * K;
  if (cell >= n) return;
  const int64_t e = cell / K;
  const int k = (int)(cell - e * K);
  const int i = i0 + (int)(e / m), j = (int)(e % m);
  const uint8_t* t = tiles + ((int64_t)(j / JB) * n_ih + i / G) * tile_bytes;
  for (int l = 0; l < L; l++) {
    const int jl = j % JB;
    const uint8_t b = idp == 3   ? t[gce_off(i % G, k, l, K, L) + (jl >> 1) * 4 + (jl & 1) * 2]
                      : idp == 1 ? t[(int64_t)(k * L + l) * PLINE + pair_off(i % G, jl, 0)]
                                 : t[(k * L + l) * LINE + (i % G) * JB + jl];
    q[cell * L + l] = sym ? (uint8_t)(b ^ 0x80u) : b;
  }
}

void download_q_from_tiles(lkg_ctx* ctx, const lkg_layer* L, uint8_t* host_q) {
  const TileGeom& gm = L->geom;
  if (!L->tiles.p || gm.small) throw Error{LKG_ERR_INVALID_ARG, "layer has no code tiles"};
  const int m = L->col1 - L->col0;
  const int64_t row_bytes = (int64_t)m * L->K * L->L;
  const int rows_per_chunk = (int)std::max<int64_t>(1, (256ll << 20) / row_bytes);
  DBuf tmp;
  tmp.alloc((size_t)rows_per_chunk * row_bytes);
  for (int i0 = 0; i0 < L->in_dim; i0 += rows_per_chunk) {
    const int i1 = std::min(L->in_dim, i0 + rows_per_chunk);
    const int64_t cells = (int64_t)(i1 - i0) * m * L->K;
    tiles_to_q_kernel<<<(unsigned)((cells + 255) / 256), 256, 0, ctx->stream>>>(
        L->tiles.as<uint8_t>(), gm.tile_bytes, gm.n_ih, i0, i1, m, L->K, L->L, L->scheme == LKG_SCHEME_SYMMETRIC,
        gm.idp, tmp.as<uint8_t>());
    LKG_CUDA(cudaGetLastError());
    LKG_CUDA(cudaMemcpyAsync(host_q + (int64_t)i0 * row_bytes, tmp.p, (size_t)(i1 - i0) * row_bytes,
                             cudaMemcpyDeviceToHost, ctx->stream));
  }
  LKG_CUDA(cudaStreamSynchronize(ctx->stream));
}

// Per-layer coordinate constants (coords.cuh), from the artifact's f32 knots.
void fill_coord_const(const lkg_layer* L, CoordConst& c, float4* ktab) {
  c.K = L->K;
  c.L = L->L;
  const bool half_open = L->boundary_mode == LKG_BOUNDARY_HALF_OPEN;
  const float hi = L->knots[L->K];
  c.lo = L->knots[0];
  c.hi_clip = half_open ? std::nextafterf(hi, -INFINITY) : hi;  // runtime.cpp:150-153
  c.inv_h = (float)L->K / (hi - c.lo);
  for (int k = 0; k < L->K; k++) {
    const float t0 = L->knots[k], t1 = L->knots[k + 1];
    ktab[k] = make_float4(t0, (float)(L->L - 1) / (t1 - t0), t1, 0.f);  // coords.cuh layout
  }
  // fp32 z = (x' - t_k) * (L-1)/h carries <= 3 roundings: re-evaluate in f64 within 8x that of a node
  c.z_thr = (float)std::max(8.0 * 0x1p-24 * (L->L - 1), 0x1p-20);
  {  // x' == hi_clip, evaluated exactly as runtime.cpp:176-181
    const double T0 = L->knots[L->K - 1], T1 = L->knots[L->K];
    const double u = ((double)c.hi_clip - T0) / (T1 - T0), zz = u * (double)(L->L - 1);
    int l0 = (int)std::floor(zz);
    l0 = l0 < 0 ? 0 : (l0 > L->L - 1 ? L->L - 1 : l0);
    c.top_l0 = l0;
    const float w = l0 >= L->L - 1 ? 0.0f : (float)(zz - (double)l0);
    c.top_w1 = (w + 1.0f) - 1.0f;  // multiple of 2^-23, as lut_coords returns it
  }
  // lut_coords_fast: the fp32 segment estimate (x' - t_0) * inv_h carries <= 3 roundings
  // (<= 3K 2^-24 segments) plus the knots' own deviation from a uniform grid; both become z
  // distances after scaling by (L-1)/h_k. Coordinates within twice that (plus z_thr) of a node
  // take the exact path.
  double dev = 0.0, hmin = 1e300, hmax = 0.0;
  for (int k = 0; k <= L->K; k++) dev = std::max(dev, std::fabs(((double)L->knots[k] - c.lo) * c.inv_h - k));
  for (int k = 0; k < L->K; k++) {
    hmin = std::min(hmin, (double)L->knots[k + 1] - L->knots[k]);
    hmax = std::max(hmax, (double)L->knots[k + 1] - L->knots[k]);
  }
  const double seg = (hi - (double)c.lo) / L->K;
  const double dz = (dev + 4.0 * L->K * 0x1p-24) * (L->L - 1) * seg / hmin;
  const double thr = 2.0 * dz + c.z_thr;
  c.fast_half = (thr < 1.0 / 16 && hmax < 1.01 * hmin) ? (float)(0.5 - thr) : -1.0f;
}

static int sm_count(int dev) {
  static int sms[64] = {0};
  if (dev < 0 || dev >= 64) return 148;
  if (!sms[dev]) cudaDeviceGetAttribute(&sms[dev], cudaDevAttrMultiProcessorCount, dev);
  return sms[dev] > 0 ? sms[dev] : 148;
}

template <bool ASYM, bool SR, bool ZS, bool VT, int MPT, bool VP = false>
static void launch_small_t(cudaStream_t st, const SmallArgs& a, size_t smem, int grid, int block) {
  auto kern = fwd_small<ASYM, SR, ZS, VT, MPT, VP>;
  static bool attr = false;
  if (!attr) {
    LKG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 224 * 1024));  // (+ the barrier)
    attr = true;
  }
  kern<<<grid, block, smem, st>>>(a);
}

static void launch_forward_small(lkg_ctx* ctx, const lkg_layer* L, const float* X, int64_t rows, int32_t x_blk,
                                 float* Y, int slot) {
  const TileGeom& gm = L->geom;
  SmallArgs a{};
  a.lut = L->tiles.as<uint8_t>();
  a.lut_bytes = (int32_t)gm.tile_bytes;
  a.p_off = gm.p_off;
  a.q_off = gm.q_off;
  a.cb_off = gm.cb_off;
  a.MP = gm.MP;
  a.X = X;
  a.rows = rows;
  a.d = L->in_dim;
  a.x_blk = x_blk;
  a.Y = Y;
  a.m = L->col1 - L->col0;
  a.counters = ctx->counters.as<unsigned long long>() + 4 * slot;
  fill_coord_const(L, a.cc, a.ktab);
  // one resident block per SM (1024 threads x ~47 registers) and one equal row range per block; a
  // small batch takes smaller blocks so that it still spreads over the SMs (a 4096-row batch ran on 4)
  int block = 1024;
  while (block > 128 && rows < (int64_t)sm_count(ctx->device) * block) block >>= 1;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((rows + block - 1) / block, sm_count(ctx->device)));
  const size_t smem = ((gm.tile_bytes + 15) & ~15) + kMaxKT * 16 + kMaxKT * 8;
  const bool asym = L->scheme == LKG_SCHEME_ASYMMETRIC, sr = L->value_repr == LKG_REPR_SPLINE_COMPONENT;
  const bool zs = L->oob_policy == LKG_OOB_ZERO_SPLINE;
  const int sz = (sr << 1) | (int)zs;
  if (gm.small == 2) {  // value table: compile-time padded out_dim, pair entries or not
    const int mp = gm.MP == 1 ? 0 : (gm.MP == 2 ? 1 : (gm.MP == 4 ? 2 : 3));
    switch ((gm.p_off << 4) | (mp << 2) | sz) {
#define CASE(S)                                                                                                  \
  case S:                                                                                                        \
    launch_small_t<false, (S >> 1) & 1, S & 1, true, 1 << ((S >> 2) & 3), ((S >> 4) & 1) != 0>(ctx->stream, a, \
                                                                                        smem, grid, block);     \
    break;
      CASE(0) CASE(1) CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7)
      CASE(8) CASE(9) CASE(10) CASE(11) CASE(12) CASE(13) CASE(14) CASE(15)
      CASE(16) CASE(17) CASE(18) CASE(19) CASE(20) CASE(21) CASE(22) CASE(23)
      CASE(24) CASE(25) CASE(26) CASE(27) CASE(28) CASE(29) CASE(30) CASE(31)
#undef CASE
    }
  } else {
    switch ((asym << 2) | sz) {
#define CASE(S) \
  case S: launch_small_t<(S >> 2) & 1, (S >> 1) & 1, S & 1, false, 8>(ctx->stream, a, smem, grid, block); break;
      CASE(0) CASE(1) CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7)
#undef CASE
    }
  }
  LKG_CUDA(cudaGetLastError());
  ctx->launches++;
}

static size_t tiled_smem(const lkg_layer* L, int W, int R, int ns = LKG_NS, int xb = 1) {
  const int64_t sb = L->geom.tile_bytes - (L->geom.codes_global ? L->geom.p_off : 0);
  // stages, x buffers, ktab, the barrier block (full/fin/xbar: 24 x 8 B), the compact tables kf, kf2
  return ns * sb + (size_t)xb * W * G * (32 * R + 4) * 4 + kMaxKT * 16 + 24 * 8 + 2 * kMaxKT * 8;
}


bool can_fuse(const lkg_layer* L1, const lkg_layer* L2) {
  // Off by default: measured on C2, the fused epilogue (16 coordinates per row at the end of
  // each item, all warps at once) costs 0.11 ms per step against 0.05 ms for the separate
  // fwd_small launch (1.81e12 vs 1.99e12 edge-evals/s).
  // LKG_FUSE=1 re-enables it (kept for the C1-sized chains of SURVEY §8f rank 3).
  static const char* fz = getenv("LKG_FUSE");
  if (!fz || fz[0] != '1') return false;
  const TileGeom &g1 = L1->geom, &g2 = L2->geom;
  if (!g1.tile_bytes || g1.small || g1.codes_global || g1.n_jb != 1 || !g2.tile_bytes || g2.small != 2) return false;
  if (g2.MP != 2) return false;  // the fused epilogue reads the value table as float2 (2 outputs)
  if (L1->in_dim > kFp32MaxD || g1.acc64 || L2->in_dim != L1->col1 - L1->col0 || L2->col1 - L2->col0 > 8) return false;
  if (L1->scheme != L2->scheme || L1->value_repr != L2->value_repr || L1->oob_policy != L2->oob_policy) return false;
  return tiled_smem(L1, kW, kR) + kMaxKT * 16 + ((g2.tile_bytes + 15) & ~15) <= 227 * 1024;
}

// X [rows][d] -> Xt [d][rows] (32x32 tiles through shared memory, both sides coalesced), and the
// base-branch activations St = silu(zs ? x : clamp(x, t_0, hi_clip)) in the same layout (f64, one
// rounding to f32: each element once, instead of once per j-block inside the table walk).
__global__ void transpose_kernel(const float* __restrict__ X, int64_t rows, int32_t d, float* __restrict__ Xt,
                                 float* __restrict__ St, float lo, float hi_clip, int zs, int exact) {
  __shared__ float t[32][33];
  const int64_t r0 = (int64_t)blockIdx.x * 32;
  const int c0 = blockIdx.y * 32;
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {
    const int64_t r = r0 + k;
    const int c = c0 + threadIdx.x;
    if (r < rows && c < d) t[k][threadIdx.x] = X[r * d + c];
  }
  __syncthreads();
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {
    const int c = c0 + k;
    const int64_t r = r0 + threadIdx.x;
    if (r < rows && c < d) {
      const float v = t[threadIdx.x][k];
      Xt[(int64_t)c * rows + r] = v;
      const float xb = zs ? v : fminf(fmaxf(v, lo), hi_clip);
      St[(int64_t)c * rows + r] = exact ? lkg::silu_exact(xb) : lkg::silu_fast(xb);
    }
  }
}

// Coordinate records (REC walk): the per-(row, input) half of the table walk — finite check, mask,
// clip, segment, sample index and integer lerp weight (coords.cuh fast path with its exact fallback,
// i.e. exactly what the walk computes in registers) plus the base activation silu(x') in f64 —
// done ONCE per input element instead of once per j-block, written transposed ([d][ld] with the
// row count padded to 4 for the tensor maps) next to each other:
//   Rt: W1 (bits 0-14, W1 = round(w1 * 2^15); 2^15 moves to the next sample with W1 = 0, the same
//       integer lerp) | code line k*L + l0 (bits 15-27) | out of range (bit 31);
//   St: silu(zero_spline ? x : x').
struct CoordPassArgs {
  lkg::CoordConst cc;
  float4 ktab[kMaxKT];
};

__global__ void coord_pass_kernel(const __grid_constant__ CoordPassArgs c, const float* __restrict__ X, int64_t rows,
                                  int32_t d, int64_t ld, uint32_t* __restrict__ Rt, float* __restrict__ St, int zs,
                                  int exact, unsigned long long* nonfinite) {
  __shared__ float t[32][33];
  __shared__ float4 ktab[kMaxKT];
  __shared__ float2 kf[kMaxKT];
  const int tid = threadIdx.y * 32 + threadIdx.x;
  for (int q = tid; q < c.cc.K; q += 32 * blockDim.y) {
    ktab[q] = c.ktab[q];
    kf[q] = make_float2(c.ktab[q].x, c.ktab[q].y);
  }
  const int64_t r0 = (int64_t)blockIdx.x * 32;
  const int c0 = blockIdx.y * 32;
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {
    const int64_t r = r0 + k;
    const int col = c0 + threadIdx.x;
    if (r < rows && col < d) t[k][threadIdx.x] = X[r * d + col];
  }
  __syncthreads();
  bool bad = false;
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {
    const int col = c0 + k;
    const int64_t r = r0 + threadIdx.x;
    if (r < rows && col < d) {
      const float v = t[threadIdx.x][k];
      bad |= !(fabsf(v) <= 3.402823466e38f);  // runtime.cpp:172 (NaN and inf)
      const lkg::Coord co = lkg::lut_coords_fast(c.cc, ktab, kf, v);
      uint32_t w1 = __float_as_uint(fmaf(co.w1, 32768.0f, 8388608.0f)) - 0x4B000000u;
      int l0 = co.l0;
      if (w1 >= 32768u) {
        w1 = 0u;
        l0 += 1;
      }
      const uint32_t line = (uint32_t)(co.k * c.cc.L + l0);
      Rt[(int64_t)col * ld + r] = w1 | (line << 15) | (co.in ? 0u : 0x80000000u);
      // the walk's own base activation: f64 for the f64-accumulating layers, MUFU otherwise (so a
      // layer keeps its result bits whether or not it takes the coordinate pass, e.g. column shards)
      St[(int64_t)col * ld + r] = exact ? lkg::silu_exact(zs ? v : co.xp) : lkg::silu_fast(zs ? v : co.xp);
    }
  }
  if (__any_sync(0xffffffffu, bad) && threadIdx.x == 0) atomicExch(nonfinite, 1ull);
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no libcuda link dependency)
static void encode_x_map(CUtensorMap* map, const float* Xt, int64_t rows, int d, int box_rows, int box_cols,
                         int64_t ld = 0) {
  typedef CUresult (*Encode)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  static Encode enc = nullptr;
  if (!enc) {
    cudaDriverEntryPointQueryResult q;
    LKG_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&enc), cudaEnableDefault, &q));
    if (!enc || q != cudaDriverEntryPointSuccess) throw Error{LKG_ERR_CUDA, "cuTensorMapEncodeTiled unavailable"};
  }
  const cuuint64_t dims[2] = {(cuuint64_t)rows, (cuuint64_t)d};
  const cuuint64_t strides[1] = {(cuuint64_t)(ld > 0 ? ld : rows) * sizeof(float)};
  const cuuint32_t box[2] = {(cuuint32_t)box_rows, (cuuint32_t)box_cols}, es[2] = {1u, 1u};
  if (enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(Xt), dims, strides, box, es,
          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    throw Error{LKG_ERR_CUDA, "cuTensorMapEncodeTiled failed"};
}

// Y = the f64 sum of the input splits' planes, in split order, rounded once to f32.
__global__ void ksplit_reduce_kernel(const double* __restrict__ part, int64_t n, int32_t S, float* __restrict__ Y) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double v = part[i];
  for (int s = 1; s < S; s++) v += part[(int64_t)s * n + i];
  Y[i] = (float)v;
}

// Input splits per (row tile, j-block) so that the items fill the SMs evenly: the persistent grid
// runs ceil(items / SMs) waves, and a layer with few items (a configs[4] column shard on 8 GPUs:
// 512 items = 3.46 waves on 148 SMs, i.e. 4) loses the unused part of the last one. Splitting the
// inputs S ways makes S times as many items of 1/S the length. LKG_KSPLIT=n forces n (1 = off).
static int choose_ksplit(int64_t items, int sms, int n_ih, int64_t rows, int m) {
  static const char* env = getenv("LKG_KSPLIT");
  // at least 8 tiles per item; the f64 planes bounded at 1 GB
  auto ok = [&](int S) {
    return S == 1 || (S > 1 && n_ih % S == 0 && n_ih / S >= 8 && rows * (int64_t)m * S <= (128ll << 20));
  };
  if (env) {
    const int S = atoi(env);
    return ok(S) ? S : 1;
  }
  auto eff = [&](int S) {
    const int64_t I = items * S, waves = (I + sms - 1) / sms;
    return (double)I / (double)(waves * sms);
  };
  int best = 1;
  double be = eff(1);
  if (be >= 0.93) return 1;
  for (int S = 2; S <= 8; S *= 2) {
    if (!ok(S)) break;
    const double e = eff(S) - 0.01 * S;  // (each split adds an epilogue and a plane of partials)
    if (e > be + 0.03) {
      best = S;
      be = e;
    }
  }
  return best;
}

void launch_forward_tiled(lkg_ctx* ctx, const lkg_layer* L, const float* X, int64_t rows, int32_t x_blk, float* Y,
                          int slot, const lkg_layer* L2, float* Y2) {
  const TileGeom& gm = L->geom;
  if (gm.small) {
    launch_forward_small(ctx, L, X, rows, x_blk, Y, slot);
    return;
  }
  TiledArgs a{};
  a.tiles = L->tiles.as<uint8_t>();
  a.tile_bytes = gm.tile_bytes;
  a.tiles_bytes = (int64_t)L->tiles.bytes;
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
  a.x_vec2 = (x_blk <= 0 ? (L->in_dim % 2 == 0) : (x_blk % 8 == 0));
  fill_coord_const(L, a.cc, a.ktab);
  const bool f64 = L->in_dim > kFp32MaxD || gm.acc64;
  const bool asym = L->scheme == LKG_SCHEME_ASYMMETRIC, sr = L->value_repr == LKG_REPR_SPLINE_COMPONENT;
  const bool zs = L->oob_policy == LKG_OOB_ZERO_SPLINE;
  const int W = f64 ? kW64 : kW, R = f64 ? kR64 : kR;
  const int64_t row_tile = (int64_t)W * 32 * R;
  a.n_rt = (rows + row_tile - 1) / row_tile;
  a.n_items = a.n_rt * gm.n_jb;
  // Balanced rows (fwd_tiled BAL): one-j-block fp32 layers with codes in shared memory. Their grid
  // spreads even a small batch over every SM (>= 64 rows per CTA): a 4096-row configs[1] batch took
  // the time of one whole 1024-row item on each of 4 CTAs.
  const bool bal_mode = !f64 && gm.n_jb == 1 && !gm.codes_global;
  a.ksplit = (!f64 || L2 || rows <= 0) ? 1 : choose_ksplit(a.n_items, sm_count(ctx->device), gm.n_ih, rows, a.m);
  a.n_ihs = gm.n_ih / a.ksplit;
  a.n_items *= a.ksplit;
  if (a.ksplit > 1) {  // f64 planes of partial sums, then the row flags of the OOB row count (zeroed per launch)
    const size_t plane = (size_t)rows * a.m * sizeof(double), flags = (size_t)((rows + 31) / 32) * 4;
    const size_t need = a.ksplit * plane + flags;
    if (ctx->ksp.bytes < need) ctx->ksp.alloc(need);
    a.Ypart = ctx->ksp.as<double>();
    a.rowflags = reinterpret_cast<uint32_t*>(ctx->ksp.as<uint8_t>() + a.ksplit * plane);
    LKG_CUDA(cudaMemsetAsync(a.rowflags, 0, flags, ctx->stream));
  }
  auto reduce_splits = [&] {
    if (a.ksplit <= 1) return;
    const int64_t n = rows * (int64_t)a.m;
    ksplit_reduce_kernel<<<(unsigned)((n + 255) / 256), 256, 0, ctx->stream>>>(a.Ypart, n, a.ksplit, Y);
    LKG_CUDA(cudaGetLastError());
    ctx->launches++;
  };
  const int grid = bal_mode ? (int)std::max<int64_t>(1, std::min<int64_t>((rows + 63) / 64, sm_count(ctx->device)))
                            : (int)std::min<int64_t>(a.n_items, sm_count(ctx->device));
  {  // row tiles per item group (item_coords). Measured on configs[3] layer 1 (1M rows): 4/8/16/32
     // within 1.5% of each other; L2 evict_last/evict_first hints on x/tiles doubled DRAM reads.
    static const char* rg = getenv("LKG_RTG");  // tuning hook
    a.rt_group = rg ? (uint32_t)std::max(1, atoi(rg)) : 8u;
  }
  size_t smem = tiled_smem(L, W, R);
  const int sel = (asym << 2) | (sr << 1) | (int)zs;
  // XT: layers that re-read every x block for many j-blocks take their input transposed once
  // ([d][rows], one extra pass over X) so each warp's x block is a single 2D TMA box in whole
  // bursts: no per-lane copies, no L1 allocation, half the DRAM traffic. Whole row tiles
  // and input tiles only (no padding rows or inputs to keep out of the OOB counts). Measured: C4
  // layer (64 j-blocks) 457.5 -> 445.9 ms incl. the transpose; C3 layer 0 (4 j-blocks) +3% (the
  // transpose outweighs the gain), hence the j-block threshold.
  static const char* xt_env = getenv("LKG_XT");  // LKG_XT=0 disables (A/B hook)
  // codes-in-L2 (GC) layers take XT too when they have f64 accumulators (C5 layer 0: -4.4 % time;
  // the row-major x staging shares L1 with the __ldg code reads there)
  const bool xt_gc_ok = f64;
  // REC: layers with several j-blocks on the integer-lerp walk get their coordinates once per input
  // element from coord_pass_kernel (transposed records + silu, TMA boxes like XT): the walk keeps
  // only the table work. Any row count and input width (the boxes past the ends are zero records,
  // which are in range and hit zero P entries). LKG_REC=0 disables (A/B hook).
  static const char* rec_env = getenv("LKG_REC");
  const int Ls = L->L;
  const bool rec = !(rec_env && rec_env[0] == '0') && (gm.idp == 2 || gm.idp == 3) && (Ls & (Ls - 1)) == 0 && L->K * Ls <= 8192 &&
                   !L2 && x_blk <= 0 && gm.n_jb >= 4 && rows > 0 && rows < (1ll << 31) &&
                   (!gm.codes_global || xt_gc_ok);
  const bool xt = rec || (!(xt_env && xt_env[0] == '0') && (!gm.codes_global || xt_gc_ok) && !L2 && gm.n_jb >= 16 &&
                          x_blk <= 0 && rows % row_tile == 0 && L->in_dim % G == 0 && rows < (1ll << 31));
  if (xt) {
    const int64_t ld = (rows + 3) / 4 * 4;  // 16-byte tensor-map strides
    const size_t xt_elems = (size_t)ld * L->in_dim;
    if (ctx->xt.bytes < 2 * sizeof(float) * xt_elems) ctx->xt.alloc(2 * sizeof(float) * xt_elems);
    float* Xt = ctx->xt.as<float>();
    float* St = Xt + xt_elems;
    const dim3 tgrid((unsigned)((rows + 31) / 32), (unsigned)((L->in_dim + 31) / 32));
    if (rec) {
      CoordPassArgs ca{};
      ca.cc = a.cc;
      for (int k = 0; k < a.cc.K; k++) ca.ktab[k] = a.ktab[k];
      coord_pass_kernel<<<tgrid, dim3(32, 8), 0, ctx->stream>>>(ca, X, rows, L->in_dim, ld,
                                                               reinterpret_cast<uint32_t*>(Xt), St, zs, f64,
                                                               a.counters + 2);
      a.lgL = __builtin_ctz((unsigned)Ls);
    } else {
      transpose_kernel<<<tgrid, dim3(32, 8), 0, ctx->stream>>>(X, rows, L->in_dim, Xt, St, a.cc.lo, a.cc.hi_clip,
                                                               zs, f64);
    }
    LKG_CUDA(cudaGetLastError());
    ctx->launches++;
    encode_x_map(&a.xmap, Xt, rows, L->in_dim, 32 * R, G, ld);
    encode_x_map(&a.smap, St, rows, L->in_dim, 32 * R, G, ld);
    a.X = Xt;
    smem += (size_t)W * G * (32 * R) * 4;  // the silu boxes
    switch (sel) {
#define CASE(S)                                                                                                \
  case S:                                                                                                      \
    if (f64 && gm.codes_global)                                                                                \
      launch_idp<kR64, kW64, (S >> 2) & 1, (S >> 1) & 1, S & 1, true, false, 1, true, false, 1, true>(       \
          gm.idp, ctx->stream, a, smem, grid, rec);                                                                         \
    else if (f64)                                                                                              \
      launch_idp<kR64, kW64, (S >> 2) & 1, (S >> 1) & 1, S & 1, true, false, 1, false, false, 1, true>(      \
          gm.idp, ctx->stream, a, smem, grid, rec);                                                                         \
    else                                                                                                       \
      launch_idp<kR, kW, (S >> 2) & 1, (S >> 1) & 1, S & 1, false, false, 1, false, false, 1, true>(         \
          gm.idp, ctx->stream, a, smem, grid, rec);                                                                         \
    break;
      CASE(0) CASE(1) CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7)
#undef CASE
    }
    LKG_CUDA(cudaGetLastError());
    ctx->launches++;
    reduce_splits();
    return;
  }
  if (gm.codes_global) {
    switch (sel) {
#define CASE(S)                                                                                                \
  case S:                                                                                                      \
    if (f64)                                                                                                   \
      launch_idp<kR64, kW64, (S >> 2) & 1, (S >> 1) & 1, S & 1, true, false, 1, true>(gm.idp, ctx->stream, a, smem, grid); \
    else                                                                                                       \
      launch_idp<kR, kW, (S >> 2) & 1, (S >> 1) & 1, S & 1, false, false, 1, true>(gm.idp, ctx->stream, a, smem, grid);    \
    break;
      CASE(0) CASE(1) CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7)
#undef CASE
    }
    LKG_CUDA(cudaGetLastError());
    ctx->launches++;
    reduce_splits();
    return;
  }
  if (L2) {  // fused chain step: this layer + the small next layer in one launch
    const TileGeom& g2 = L2->geom;
    a.lut2 = L2->tiles.as<uint8_t>();
    a.lut2_bytes = (int32_t)g2.tile_bytes;
    a.p_off2 = g2.p_off;
    a.q_off2 = g2.q_off;
    a.cb_off2 = g2.cb_off;
    a.MP2 = g2.MP;
    a.vp2 = g2.p_off;
    a.m2 = L2->col1 - L2->col0;
    a.Y2 = Y2;
    a.counters2 = ctx->counters.as<unsigned long long>() + 4 * (slot + 1);
    fill_coord_const(L2, a.cc2, a.ktab2);
    smem += kMaxKT * 16 + ((g2.tile_bytes + 15) & ~15);
    switch (sel) {
#define CASE(S) \
  case S: launch_idp<kR, kW, (S >> 2) & 1, (S >> 1) & 1, S & 1, false, true, 1, false, true>(gm.idp, ctx->stream, a, smem, grid); break;
      CASE(0) CASE(1) CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7)
#undef CASE
    }
    LKG_CUDA(cudaGetLastError());
    ctx->launches++;
    return;
  }
  const bool bal = bal_mode;
  // Small batches of a one-j-block layer (serving): with 2 rows per lane a 4096-row configs[1] batch
  // is 64 single-warp CTAs walking 10 tiles each, latency-bound (36 us). One row per lane (R = 1)
  // doubles the warps and halves each one's work per tile; same lane and input order per row, so the
  // same bits (test_balanced_rows_small_batches_bit_identical). LKG_R1=0 disables.
  static const char* r1_env = getenv("LKG_R1");
  const bool r1 = bal && !(r1_env && r1_env[0] == '0') && rows <= (int64_t)64 * sm_count(ctx->device) &&
                  gm.idp != 1 && tiled_smem(L, W, 1, 4) <= 227 * 1024;  // (4 stage buffers: see NSX)
  if (r1) {
    smem = tiled_smem(L, W, 1, 4);
    const int grid1 = (int)std::max<int64_t>(1, std::min<int64_t>((rows + 31) / 32, sm_count(ctx->device)));
    switch (sel) {
#define CASE(S)                                                                                                  \
  case S:                                                                                                        \
    launch_idp<1, kW, (S >> 2) & 1, (S >> 1) & 1, S & 1, false, false, 1, false, true, 1, false, 4>(           \
        gm.idp, ctx->stream, a, smem, grid1);                                                                    \
    break;
      CASE(0) CASE(1) CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7)
#undef CASE
    }
    LKG_CUDA(cudaGetLastError());
    ctx->launches++;
    return;
  }
  // two x buffers only for the int8 one-j-block layers (see fwd_tiled's XB), where they fit
  const bool xb2 = bal && !asym && tiled_smem(L, W, R, LKG_NS, 2) <= 227 * 1024;
  if (xb2) smem = tiled_smem(L, W, R, LKG_NS, 2);
  switch (sel) {
#define CASE(S)                                                                                         \
  case S:                                                                                               \
    if (f64)                                                                                            \
      launch_idp<kR64, kW64, (S >> 2) & 1, (S >> 1) & 1, S & 1, true>(gm.idp, ctx->stream, a, smem, grid);     \
    else if (xb2)                                                                                       \
      launch_idp<kR, kW, (S >> 2) & 1, (S >> 1) & 1, S & 1, false, false, 1, false, true,              \
                   ((S >> 2) & 1) ? 1 : 2>(gm.idp, ctx->stream, a, smem, grid);                                 \
    else if (bal)                                                                                       \
      launch_idp<kR, kW, (S >> 2) & 1, (S >> 1) & 1, S & 1, false, false, 1, false, true>(gm.idp, ctx->stream, a, \
                                                                                         smem, grid);  \
    else                                                                                                \
      launch_idp<kR, kW, (S >> 2) & 1, (S >> 1) & 1, S & 1, false>(gm.idp, ctx->stream, a, smem, grid);        \
    break;
    CASE(0) CASE(1) CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7)
#undef CASE
  }
  LKG_CUDA(cudaGetLastError());
  ctx->launches++;
  reduce_splits();
}

}  // namespace lkg
