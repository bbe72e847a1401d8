// Instruction-throughput probe for the LUT-forward inner loop on sm_100a.
// Each kernel runs NITER iterations of 8 independent op chains per thread;
// ops/clk/SM = total ops / (max SM cycles) / active SMs. Built and run only
// by tools/microbench/run.sh on the GPU box; not part of the product.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define NITER 4096
#define CHAINS 8

__global__ void k_i2f_u8(uint32_t seed, float* out, long long* cyc) {
  uint32_t v[CHAINS]; float a[CHAINS];
  for (int c = 0; c < CHAINS; c++) { v[c] = seed * (threadIdx.x + c); a[c] = 0.f; }
  long long t0 = clock64();
  for (int it = 0; it < NITER; it++) {
#pragma unroll
    for (int c = 0; c < CHAINS; c++) {
      a[c] += (float)(uint8_t)(v[c] >> 8);   // I2F.U8 .B1
      v[c] += a[c] > 1e30f;                  // keep v loop-variant
    }
  }
  long long t1 = clock64();
  float s = 0; for (int c = 0; c < CHAINS; c++) s += a[c];
  if (s == 1.2345f) out[0] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

// pure conversion rate: 4 byte converts per word, 8 words
__global__ void k_i2f_pure(const uint32_t* in, float* out, long long* cyc) {
  uint32_t v[CHAINS]; float a[CHAINS];
  for (int c = 0; c < CHAINS; c++) { v[c] = in[(threadIdx.x + c) & 255]; a[c] = 0.f; }
  long long t0 = clock64();
  for (int it = 0; it < NITER; it++) {
#pragma unroll
    for (int c = 0; c < CHAINS; c++) {
      float f0 = (float)(uint8_t)(v[c]);
      float f1 = (float)(uint8_t)(v[c] >> 8);
      float f2 = (float)(uint8_t)(v[c] >> 16);
      float f3 = (float)(uint8_t)(v[c] >> 24);
      a[c] = fmaf(f0, f1, a[c]); a[c] = fmaf(f2, f3, a[c]);
      v[c] = v[c] * 1664525u + 1013904223u;
    }
  }
  long long t1 = clock64();
  float s = 0; for (int c = 0; c < CHAINS; c++) s += a[c];
  if (s == 1.2345f) out[0] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__global__ void k_ffma(float seed, float* out, long long* cyc) {
  float a[CHAINS], b = seed, c2 = seed * 0.5f;
  for (int c = 0; c < CHAINS; c++) a[c] = seed + c;
  long long t0 = clock64();
  for (int it = 0; it < NITER; it++) {
#pragma unroll
    for (int c = 0; c < CHAINS; c++) { a[c] = fmaf(a[c], b, c2); a[c] = fmaf(a[c], c2, b); }
  }
  long long t1 = clock64();
  float s = 0; for (int c = 0; c < CHAINS; c++) s += a[c];
  if (s == 1.2345f) out[0] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__device__ __forceinline__ unsigned long long ffma2(unsigned long long a, unsigned long long b, unsigned long long c) {
  unsigned long long d;
  asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}

__global__ void k_ffma2(float seed, float* out, long long* cyc) {
  unsigned long long a[CHAINS], b, c2;
  float2 bb = make_float2(seed, seed * 0.3f), cc = make_float2(seed * 0.5f, seed * 0.7f);
  b = *(unsigned long long*)&bb; c2 = *(unsigned long long*)&cc;
  for (int c = 0; c < CHAINS; c++) { float2 t = make_float2(seed + c, seed - c); a[c] = *(unsigned long long*)&t; }
  long long t0 = clock64();
  for (int it = 0; it < NITER; it++) {
#pragma unroll
    for (int c = 0; c < CHAINS; c++) { a[c] = ffma2(a[c], b, c2); a[c] = ffma2(a[c], c2, b); }
  }
  long long t1 = clock64();
  float s = 0; for (int c = 0; c < CHAINS; c++) { float2 t = *(float2*)&a[c]; s += t.x + t.y; }
  if (s == 1.2345f) out[0] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__global__ void k_prmt(uint32_t seed, float* out, long long* cyc) {
  uint32_t v[CHAINS];
  for (int c = 0; c < CHAINS; c++) v[c] = seed + c;
  long long t0 = clock64();
  for (int it = 0; it < NITER; it++) {
#pragma unroll
    for (int c = 0; c < CHAINS; c++) { v[c] = __byte_perm(v[c], 0x4B000000u, 0x7651); v[c] = __byte_perm(v[c], seed, 0x1054); }
  }
  long long t1 = clock64();
  uint32_t s = 0; for (int c = 0; c < CHAINS; c++) s += v[c];
  if (s == 12345u) out[0] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__global__ void k_dadd(double seed, float* out, long long* cyc) {
  double a[CHAINS], b = seed;
  for (int c = 0; c < CHAINS; c++) a[c] = seed + c;
  long long t0 = clock64();
  for (int it = 0; it < NITER; it++) {
#pragma unroll
    for (int c = 0; c < CHAINS; c++) { a[c] = a[c] + b; a[c] = a[c] - b * 0.5; }
  }
  long long t1 = clock64();
  double s = 0; for (int c = 0; c < CHAINS; c++) s += a[c];
  if (s == 1.2345) out[0] = (float)s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__global__ void k_f2f64(float seed, float* out, long long* cyc) {
  double a[CHAINS]; float f[CHAINS];
  for (int c = 0; c < CHAINS; c++) { a[c] = 0; f[c] = seed + c; }
  long long t0 = clock64();
  for (int it = 0; it < NITER; it++) {
#pragma unroll
    for (int c = 0; c < CHAINS; c++) { a[c] += (double)f[c]; f[c] = f[c] * 1.0001f; }
  }
  long long t1 = clock64();
  double s = 0; for (int c = 0; c < CHAINS; c++) s += a[c];
  if (s == 1.2345) out[0] = (float)s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

// shared-memory load throughput: each lane reads consecutive words (conflict-free)
template <int W>
__global__ void k_lds(float* out, long long* cyc) {
  __shared__ __align__(16) uint32_t sm[8192];
  for (int i = threadIdx.x; i < 8192; i += blockDim.x) sm[i] = i * 2654435761u;
  __syncthreads();
  uint32_t acc = 0;
  int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  long long t0 = clock64();
  for (int it = 0; it < NITER; it++) {
    int base = ((it * 7 + warp * 3) & 31) * 128;   // warp-uniform line
    if (W == 4) { acc += sm[(base + lane) & 8191]; }
    if (W == 8) { uint2 v = *(const uint2*)&sm[(base + lane * 2) & 8190]; acc += v.x ^ v.y; }
    if (W == 16) { uint4 v = *(const uint4*)&sm[(base + lane * 4) & 8188]; acc += v.x ^ v.y ^ v.z ^ v.w; }
    acc = acc * 3u;
  }
  long long t1 = clock64();
  if (acc == 12345u) out[0] = acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

// dp2a (IDP.2A): two 16-bit x 8-bit products + 32-bit accumulate, the integer lerp of the
// IDP table walk (forward_tiled.cu): lo and hi halves of the code word
__device__ __forceinline__ uint32_t dp2a_lo(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d;
  asm volatile("dp2a.lo.u32.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}
__device__ __forceinline__ uint32_t dp2a_hi(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d;
  asm volatile("dp2a.hi.u32.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}

__global__ void k_dp2a(uint32_t seed, float* out, long long* cyc) {
  uint32_t v[CHAINS], w = seed * 7u;
  for (int c = 0; c < CHAINS; c++) v[c] = seed + c;
  long long t0 = clock64();
  for (int it = 0; it < NITER; it++) {
#pragma unroll
    for (int c = 0; c < CHAINS; c++) { v[c] = dp2a_lo(w, v[c], seed); v[c] = dp2a_hi(w, v[c], seed); }
  }
  long long t1 = clock64();
  uint32_t s = 0; for (int c = 0; c < CHAINS; c++) s += v[c];
  if (s == 12345u) out[0] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__global__ void k_imad(uint32_t seed, float* out, long long* cyc) {
  uint32_t v[CHAINS], w = seed * 7u;
  for (int c = 0; c < CHAINS; c++) v[c] = seed + c;
  long long t0 = clock64();
  for (int it = 0; it < NITER; it++) {
#pragma unroll
    for (int c = 0; c < CHAINS; c++) { v[c] = v[c] * w + seed; v[c] = v[c] * seed + w; }
  }
  long long t1 = clock64();
  uint32_t s = 0; for (int c = 0; c < CHAINS; c++) s += v[c];
  if (s == 12345u) out[0] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

// the IDP walk's core per 2 outputs: 2 dp2a (lo, hi) -> FADD2 (magic off) -> FFMA2 (x P) -> FFMA2 (base)
// 5 issue slots; counted as 5 ops per pair
__global__ void k_idp_core(uint32_t seed, float* out, long long* cyc) {
  unsigned long long acc[CHAINS];
  uint32_t v[CHAINS], w = seed * 7u;
  float2 pp = make_float2(1e-3f, 2e-3f), cb = make_float2(0.5f, 0.25f), bx = make_float2(0.1f, 0.1f);
  const float2 mg = make_float2(-12582912.f, -12582912.f);
  for (int c = 0; c < CHAINS; c++) { v[c] = seed + 3 * c; acc[c] = 0; }
  long long t0 = clock64();
  for (int it = 0; it < NITER; it++) {
#pragma unroll
    for (int c = 0; c < CHAINS; c++) {
      const uint32_t r0 = dp2a_lo(w, v[c], 0x4B000000u), r1 = dp2a_hi(w, v[c], 0x4B000000u);
      float2 f = make_float2(__uint_as_float(r0), __uint_as_float(r1));
      f = __fadd2_rn(f, mg);
      float2 a = *(float2*)&acc[c];
      a = __ffma2_rn(pp, f, a);
      a = __ffma2_rn(cb, bx, a);
      acc[c] = *(unsigned long long*)&a;
      v[c] += 0x01010101u;
    }
  }
  long long t1 = clock64();
  float s = 0; for (int c = 0; c < CHAINS; c++) { float2 t = *(float2*)&acc[c]; s += t.x + t.y; }
  if (s == 1.2345f) out[0] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

// the round-1 core per 2 outputs: 4 PRMT + 5 FFMA2 (9 issue slots), counted as 9 ops per pair
__global__ void k_prmt_core(uint32_t seed, float* out, long long* cyc) {
  unsigned long long acc[CHAINS];
  uint32_t v[CHAINS], u[CHAINS];
  const float2 W0 = make_float2(0.3f, 0.3f), W1 = make_float2(0.7f, 0.7f), CA = make_float2(-3e6f, -3e6f),
               CB2 = make_float2(-5e6f, -5e6f), pp = make_float2(1e-3f, 2e-3f), cb = make_float2(0.5f, 0.25f),
               bx = make_float2(0.1f, 0.1f);
  for (int c = 0; c < CHAINS; c++) { v[c] = seed + 3 * c; u[c] = seed * 5 + c; acc[c] = 0; }
  long long t0 = clock64();
  for (int it = 0; it < NITER; it++) {
#pragma unroll
    for (int c = 0; c < CHAINS; c++) {
      const float2 fa = make_float2(__uint_as_float(__byte_perm(v[c], 0x4B000000u, 0x7440)),
                                    __uint_as_float(__byte_perm(v[c], 0x4B000000u, 0x7441)));
      const float2 fb = make_float2(__uint_as_float(__byte_perm(u[c], 0x4B000000u, 0x7440)),
                                    __uint_as_float(__byte_perm(u[c], 0x4B000000u, 0x7441)));
      const float2 a0 = __ffma2_rn(W0, fa, CA), b0 = __ffma2_rn(W1, fb, CB2);
      float2 a = *(float2*)&acc[c];
      a = __ffma2_rn(pp, a0, a);
      a = __ffma2_rn(pp, b0, a);
      a = __ffma2_rn(cb, bx, a);
      acc[c] = *(unsigned long long*)&a;
      v[c] += 0x01010101u;
      u[c] += 0x01010101u;
    }
  }
  long long t1 = clock64();
  float s = 0; for (int c = 0; c < CHAINS; c++) { float2 t = *(float2*)&acc[c]; s += t.x + t.y; }
  if (s == 1.2345f) out[0] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <typename K, typename... A>
void run(const char* name, K kern, int grid, int block, double ops_per_thread_iter, A... args) {
  long long* cyc; float* out;
  cudaMalloc(&cyc, grid * sizeof(long long)); cudaMalloc(&out, 64);
  kern<<<grid, block>>>(args..., out, cyc);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  kern<<<grid, block>>>(args..., out, cyc);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  long long* h = new long long[grid];
  cudaMemcpy(h, cyc, grid * sizeof(long long), cudaMemcpyDeviceToHost);
  long long mx = 0; for (int i = 0; i < grid; i++) mx = h[i] > mx ? h[i] : mx;
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double ops = (double)grid * block * NITER * ops_per_thread_iter;
  int blocks_per_sm = (grid + sms - 1) / sms;
  // per-SM rate: ops of all blocks resident on one SM over the max block cycle count
  double per_sm_clk = (double)block * blocks_per_sm * NITER * ops_per_thread_iter / (double)mx;
  printf("%-12s grid=%d block=%d  %.1f lane-ops/clk/SM   %.3e ops/s (event %.3f ms)  err=%s\n", name, grid, block,
         per_sm_clk, ops / (ms * 1e-3), ms, cudaGetErrorString(cudaGetLastError()));
  delete[] h; cudaFree(cyc); cudaFree(out);
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("SMs=%d clock=%d kHz\n", sms, clk);
  uint32_t* in; cudaMalloc(&in, 1024); cudaMemset(in, 0x37, 1024);
  for (int bps : {4, 8}) {
    int g = sms * bps;
    run("i2f_u8", k_i2f_u8, g, 256, CHAINS * 1.0, 12345u);
    run("i2f_pure", k_i2f_pure, g, 256, CHAINS * 4.0, (const uint32_t*)in);
    run("ffma", k_ffma, g, 256, CHAINS * 2.0, 1.0001f);
    run("ffma2(x2)", k_ffma2, g, 256, CHAINS * 4.0, 1.0001f);
    run("prmt", k_prmt, g, 256, CHAINS * 2.0, 12345u);
    run("dp2a", k_dp2a, g, 256, CHAINS * 2.0, 12345u);
    run("imad", k_imad, g, 256, CHAINS * 2.0, 12345u);
    run("idp_core(5/pair)", k_idp_core, g, 256, CHAINS * 5.0, 12345u);
    run("prmt_core(9/pair)", k_prmt_core, g, 256, CHAINS * 9.0, 12345u);
    run("dadd", k_dadd, g, 256, CHAINS * 2.0, 1.0001);
    run("f2f64+dadd", k_f2f64, g, 256, CHAINS * 1.0, 1.0001f);
    run("lds32", k_lds<4>, g, 256, 1.0);
    run("lds64", k_lds<8>, g, 256, 1.0);
    run("lds128", k_lds<16>, g, 256, 1.0);
  }
  return 0;
}
