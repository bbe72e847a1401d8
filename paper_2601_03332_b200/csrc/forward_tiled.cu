// forward_tiled.cu — K2 on sm_100a, host side and layouts: tile builders, the small-layer kernel
// fwd_small, the coordinate / transpose passes and the dispatch of the table walk fwd_tiled
// (fwd_tiled.cuh; its variants are instantiated in forward_tiled_{xt,gc,rows}.cu).
#include "fwd_tiled.cuh"

namespace {

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

}  // namespace

namespace lkg {

using tiled::kR;
using tiled::kR64;
using tiled::kW;
using tiled::kW64;
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
// (x_blk > 0: X is in the rank-major all-gather layout, element (r, i) at
// X[(i / x_blk) * rows * x_blk + r * x_blk + i % x_blk])
__device__ __forceinline__ int64_t x_index(int64_t r, int c, int64_t rows, int32_t d, int32_t x_blk) {
  if (x_blk <= 0) return r * d + c;
  const int b = c / x_blk;
  return (int64_t)b * rows * x_blk + r * x_blk + (c - b * x_blk);
}

__global__ void transpose_kernel(const float* __restrict__ X, int64_t rows, int32_t d, int32_t x_blk,
                                 float* __restrict__ Xt, float* __restrict__ St, float lo, float hi_clip, int zs,
                                 int exact) {
  __shared__ float t[32][33];
  const int64_t r0 = (int64_t)blockIdx.x * 32;
  const int c0 = blockIdx.y * 32;
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {
    const int64_t r = r0 + k;
    const int c = c0 + threadIdx.x;
    if (r < rows && c < d) t[k][threadIdx.x] = X[x_index(r, c, rows, d, x_blk)];
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

constexpr int kCoordSub = 8;  // 32-row sub-tiles per coord_pass block (32 columns x 256 rows)

__global__ void coord_pass_kernel(const __grid_constant__ CoordPassArgs c, const float* __restrict__ X, int64_t rows,
                                  int32_t d, int32_t x_blk, int64_t ld, uint32_t* __restrict__ Rt,
                                  float* __restrict__ St, int zs, int exact, unsigned long long* nonfinite) {
  __shared__ float t[2][32][33];
  __shared__ float4 ktab[kMaxKT];
  __shared__ float2 kf[kMaxKT];
  const int tid = threadIdx.y * 32 + threadIdx.x;
  for (int q = tid; q < c.cc.K; q += 32 * blockDim.y) {
    ktab[q] = c.ktab[q];
    kf[q] = make_float2(c.ktab[q].x, c.ktab[q].y);
  }
  // a block walks kCoordSub 32x32 sub-tiles down the rows (one barrier each: the tile buffer is
  // double-buffered), so the table staging and the index set-up serve 32 elements per thread, not 4
  const int c0 = blockIdx.y * 32;
  const int64_t rbase = (int64_t)blockIdx.x * 32 * kCoordSub;
  const int lcol = c0 + threadIdx.x;  // the column this thread loads
  bool bad = false;
  for (int sub = 0; sub < kCoordSub; sub++) {
    const int64_t r0 = rbase + 32 * sub;
    if (r0 >= rows) break;
    float(*tb)[33] = t[sub & 1];
    for (int k = threadIdx.y; k < 32; k += blockDim.y) {
      const int64_t r = r0 + k;
      if (r < rows && lcol < d) tb[k][threadIdx.x] = X[x_index(r, lcol, rows, d, x_blk)];
    }
    __syncthreads();
    const int64_t r = r0 + threadIdx.x;
    if (r < rows) {
      uint32_t* rp = Rt + (int64_t)(c0 + threadIdx.y) * ld + r;
      float* sp = St + (int64_t)(c0 + threadIdx.y) * ld + r;
      const int64_t step = (int64_t)blockDim.y * ld;
      for (int k = threadIdx.y; k < 32 && c0 + k < d; k += blockDim.y, rp += step, sp += step) {
        const float v = tb[threadIdx.x][k];
        bad |= !(fabsf(v) <= 3.402823466e38f);  // runtime.cpp:172 (NaN and inf)
        const lkg::Coord co = lkg::lut_coords_fast(c.cc, ktab, kf, v);
        uint32_t w1 = __float_as_uint(fmaf(co.w1, 32768.0f, 8388608.0f)) - 0x4B000000u;
        int l0 = co.l0;
        if (w1 >= 32768u) {
          w1 = 0u;
          l0 += 1;
        }
        const uint32_t line = (uint32_t)(co.k * c.cc.L + l0);
        *rp = w1 | (line << 15) | (co.in ? 0u : 0x80000000u);
        // the walk's own base activation: f64 for the f64-accumulating layers, MUFU otherwise (so a
        // layer keeps its result bits whether or not it takes the coordinate pass, e.g. column shards)
        *sp = exact ? lkg::silu_exact(zs ? v : co.xp) : lkg::silu_fast(zs ? v : co.xp);
      }
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
  static const bool rtg_env = getenv("LKG_RTG") != nullptr;
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
                   !L2 && gm.n_jb >= 4 && rows > 0 && rows < (1ll << 31) &&
                   (!gm.codes_global || xt_gc_ok);
  const bool xt = rec || (!(xt_env && xt_env[0] == '0') && (!gm.codes_global || xt_gc_ok) && !L2 && gm.n_jb >= 16 &&
                          rows % row_tile == 0 && L->in_dim % G == 0 && rows < (1ll << 31));
  if (xt) {
    const int64_t ld = (rows + 3) / 4 * 4;  // 16-byte tensor-map strides
    const size_t xt_elems = (size_t)ld * L->in_dim;
    if (ctx->xt.bytes < 2 * sizeof(float) * xt_elems) ctx->xt.alloc(2 * sizeof(float) * xt_elems);
    float* Xt = ctx->xt.as<float>();
    float* St = Xt + xt_elems;
    const dim3 tgrid((unsigned)((rows + 31) / 32), (unsigned)((L->in_dim + 31) / 32));
    if (rec) {
      const dim3 cgrid((unsigned)((rows + 32 * kCoordSub - 1) / (32 * kCoordSub)), tgrid.y);
      CoordPassArgs ca{};
      ca.cc = a.cc;
      for (int k = 0; k < a.cc.K; k++) ca.ktab[k] = a.ktab[k];
      coord_pass_kernel<<<cgrid, dim3(32, 8), 0, ctx->stream>>>(ca, X, rows, L->in_dim, x_blk, ld,
                                                               reinterpret_cast<uint32_t*>(Xt), St, zs, f64,
                                                               a.counters + 2);
      a.lgL = __builtin_ctz((unsigned)Ls);
    } else {
      transpose_kernel<<<tgrid, dim3(32, 8), 0, ctx->stream>>>(X, rows, L->in_dim, x_blk, Xt, St, a.cc.lo,
                                                               a.cc.hi_clip, zs, f64);
    }
    LKG_CUDA(cudaGetLastError());
    ctx->launches++;
    encode_x_map(&a.xmap, Xt, rows, L->in_dim, 32 * R, G, ld);
    encode_x_map(&a.smap, St, rows, L->in_dim, 32 * R, G, ld);
    a.X = Xt;
    a.x_blk = 0;  // (the passes read the blocked all-gather layout; the walk reads their [d][rows] output)
    // Record walk: wide groups, i.e. the CTAs in flight share ONE j-block's tiles (each tile read from
    // DRAM once per group) and stream their own row tiles' record boxes, which no ordering kept in L2
    // anyway. Measured on configs[3] (1M rows): groups of 8 / 32 / 64 / 128 row tiles 299.5 / 288.3 /
    // 282.8 / 281.6 ms, DRAM 829 -> 592 GB per layer, L2 hit rate 20 -> 38 %.
    if (rec && !rtg_env) a.rt_group = 128u;
    smem += (size_t)W * G * (32 * R) * 4;  // the silu boxes
    tiled::launch_xt(sel, f64, gm.codes_global != 0, gm.idp, ctx->stream, a, smem, grid, rec);
    LKG_CUDA(cudaGetLastError());
    ctx->launches++;
    reduce_splits();
    return;
  }
  if (gm.codes_global) {
    tiled::launch_gc(sel, f64, gm.idp, ctx->stream, a, smem, grid);
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
    tiled::launch_fused(sel, gm.idp, ctx->stream, a, smem, grid);
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
    tiled::launch_r1(sel, gm.idp, ctx->stream, a, smem, grid1);
    LKG_CUDA(cudaGetLastError());
    ctx->launches++;
    return;
  }
  // two x buffers only for the int8 one-j-block layers (see fwd_tiled's XB), where they fit
  const bool xb2 = bal && !asym && tiled_smem(L, W, R, LKG_NS, 2) <= 227 * 1024;
  if (xb2) smem = tiled_smem(L, W, R, LKG_NS, 2);
  tiled::launch_rows(sel, f64, xb2, bal, gm.idp, ctx->stream, a, smem, grid);
  LKG_CUDA(cudaGetLastError());
  ctx->launches++;
  reduce_splits();
}

}  // namespace lkg
