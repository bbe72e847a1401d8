/*
 * lk_oracle.c — plain-C restatement of the reference LUT-KAN hot path.
 *
 * TEST INFRASTRUCTURE ONLY (see lk_oracle.h). This is the CHECKER for the CUDA
 * product, never the product: it is loaded only by tests/, smoke() and the CPU
 * baseline legs of bench.py. Every function restates a reference function in the
 * reference's exact f64 operation order (citations are /root/reference paths);
 * it is compiled with -ffp-contract=off so no FMA contraction changes the bits
 * (SURVEY.md Appendix B.3). Parity of this port against the reference itself is
 * pinned by tests/test_oracle.py (against oracle/_ref when it is built, and
 * against the committed golden vectors in tests/golden/ generated from the
 * reference by tests/golden/make_golden.py).
 */
#include "lk_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static __thread char g_err[256];
static int fail(int code, const char* msg) {
  snprintf(g_err, sizeof g_err, "%s", msg);
  return code;
}
const char* ork_last_error(void) { return g_err; }
const char* ork_impl_name(void) { return "port"; }

enum { OK = 0, CONFIG = 1, DIMENSION = 2, NONFINITE = 3, UNSUPPORTED = 4 };

/* ---------------------------------------------------------------- float16 */
/* proj/core/src/float16.cpp:7-42 (round to nearest even, subnormals kept). */
uint16_t ork_f32_to_f16_bits(float f) {
  uint32_t x;
  memcpy(&x, &f, 4);
  uint32_t sign = (x >> 16) & 0x8000u, ex = (x >> 23) & 0xffu, man = x & 0x7fffffu;
  if (ex == 0xffu) return (uint16_t)(sign | 0x7c00u | (man ? 0x200u | (man >> 13) : 0));
  int e = (int)ex - 127 + 15;
  if (e >= 0x1f) return (uint16_t)(sign | 0x7c00u);
  if (e <= 0) {
    if (e < -10) return (uint16_t)sign;
    man |= 0x800000u;
    int sh = 14 - e;
    uint32_t hm = man >> sh, rem = man & ((1u << sh) - 1), half = 1u << (sh - 1);
    if (rem > half || (rem == half && (hm & 1u))) hm++;
    return (uint16_t)(sign | hm);
  }
  uint32_t h = sign | ((uint32_t)e << 10) | (man >> 13), rem = man & 0x1fffu;
  if (rem > 0x1000u || (rem == 0x1000u && (h & 1u))) h++;
  return (uint16_t)h;
}
/* float16.cpp:44-71 */
float ork_f16_bits_to_f32(uint16_t h) {
  uint32_t sign = ((uint32_t)h & 0x8000u) << 16, ex = (h >> 10) & 0x1fu, man = h & 0x3ffu, out;
  if (ex == 0x1fu) out = sign | 0x7f800000u | (man << 13);
  else if (ex == 0) {
    if (man == 0) out = sign;
    else {
      int e = -1;
      do { man <<= 1; e++; } while ((man & 0x400u) == 0);
      out = sign | ((uint32_t)(127 - 15 - e) << 23) | ((man & 0x3ffu) << 13);
    }
  } else out = sign | ((ex - 15 + 127) << 23) | (man << 13);
  float f;
  memcpy(&f, &out, 4);
  return f;
}

/* -------------------------------------------------------------------- rng */
/* proj/core/include/lutkan/rng.hpp:13-58 and src/rng.cpp:7-22. */
typedef struct { uint64_t s[4]; double spare; int has_spare; } rng_t;
static uint64_t rotl(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }
static void rng_init(rng_t* r, uint64_t seed) {
  uint64_t x = seed;
  for (int i = 0; i < 4; i++) {
    x += 0x9e3779b97f4a7c15ull;
    uint64_t z = x;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    r->s[i] = z ^ (z >> 31);
  }
  r->spare = 0.0;
  r->has_spare = 0;
}
static uint64_t rng_u64(rng_t* r) {
  uint64_t* s = r->s;
  uint64_t res = rotl(s[0] + s[3], 23) + s[0], t = s[1] << 17;
  s[2] ^= s[0]; s[3] ^= s[1]; s[1] ^= s[2]; s[0] ^= s[3]; s[2] ^= t; s[3] = rotl(s[3], 45);
  return res;
}
static double rng_uniform(rng_t* r) { return (double)(rng_u64(r) >> 11) * 0x1.0p-53; }
static double rng_uniform_ab(rng_t* r, double lo, double hi) { return lo + (hi - lo) * rng_uniform(r); }
static double rng_normal(rng_t* r) {
  if (r->has_spare) { r->has_spare = 0; return r->spare; }
  double u, v, s;
  do {
    u = 2.0 * rng_uniform(r) - 1.0;
    v = 2.0 * rng_uniform(r) - 1.0;
    s = u * u + v * v;
  } while (s >= 1.0 || s == 0.0);
  double f = sqrt(-2.0 * log(s) / s);
  r->spare = v * f;
  r->has_spare = 1;
  return u * f;
}
static double rng_normal_ms(rng_t* r, double mean, double sd) { return mean + sd * rng_normal(r); }
void ork_rng_uniform(uint64_t seed, int64_t n, double* out) {
  rng_t r; rng_init(&r, seed);
  for (int64_t i = 0; i < n; i++) out[i] = rng_uniform(&r);
}
void ork_rng_normal(uint64_t seed, int64_t n, double* out) {
  rng_t r; rng_init(&r, seed);
  for (int64_t i = 0; i < n; i++) out[i] = rng_normal(&r);
}

/* ----------------------------------------------------------------- spline */
/* KnotGrid extension, proj/core/src/spline.cpp:8-27. ext has K+1+2p entries. */
static int knot_grid(const double* bp, int K, int p, double* ext) {
  if (p < 0) return fail(CONFIG, "degree must be >= 0");
  if (K < 1) return fail(CONFIG, "need at least 2 breakpoints");
  for (int i = 0; i <= K; i++) {
    if (!isfinite(bp[i])) return fail(NONFINITE, "non-finite breakpoint");
    if (i > 0 && !(bp[i - 1] < bp[i])) return fail(CONFIG, "breakpoints must be strictly increasing");
  }
  int n = K + 1;
  double hl = bp[1] - bp[0], hr = bp[n - 1] - bp[n - 2];
  for (int i = 0; i < p; i++) ext[p - 1 - i] = bp[0] - (i + 1) * hl;
  for (int i = 0; i < n; i++) ext[p + i] = bp[i];
  for (int i = 0; i < p; i++) ext[p + n + i] = bp[n - 1] + (i + 1) * hr;
  return OK;
}

/* basis_into, spline.cpp:69-83: all n0 degree-0 indicators, then the recursion. */
static void basis_into(const double* T, int nT, int p, double x, double* buf) {
  int n0 = nT - 1;
  for (int r = 0; r < n0; r++) buf[r] = (T[r] <= x && x < T[r + 1]) ? 1.0 : 0.0;
  for (int q = 1; q <= p; q++) {
    int count = n0 - q;
    for (int r = 0; r < count; r++) {
      double acc = 0.0;
      double d1 = T[r + q] - T[r];
      if (d1 > 0.0) acc += (x - T[r]) / d1 * buf[r];
      double d2 = T[r + q + 1] - T[r + 1];
      if (d2 > 0.0) acc += (T[r + q + 1] - x) / d2 * buf[r + 1];
      buf[r] = acc;
    }
  }
}
static double silu(double x) { return x / (1.0 + exp(-x)); } /* spline.cpp:85 */

int ork_basis_values(const double* bp, int32_t K, int32_t p, double x, double* out) {
  double* ext = (double*)malloc(sizeof(double) * (K + 1 + 2 * p));
  double* buf = (double*)malloc(sizeof(double) * (K + 2 * p + 1));
  int st = knot_grid(bp, K, p, ext);
  if (st == OK) {
    basis_into(ext, K + 1 + 2 * p, p, x, buf);
    memcpy(out, buf, sizeof(double) * (K + p));
  }
  free(ext); free(buf);
  return st;
}

static int check_spec(const ork_spec* s) {
  if (s->in_dim < 1 || s->out_dim < 1) return fail(CONFIG, "layer dims must be >= 1");
  int64_t E = (int64_t)s->in_dim * s->out_dim, R = s->K + s->degree;
  for (int64_t i = 0; i < E * R; i++)
    if (!isfinite(s->coeffs[i])) return fail(NONFINITE, "non-finite spline coefficient");
  for (int64_t e = 0; e < E; e++)
    if (!isfinite(s->base_scale[e]) || !isfinite(s->spline_scale[e]) || !isfinite(s->out_scale[e]))
      return fail(NONFINITE, "non-finite edge scale");
  return OK;
}

/* ------------------------------------------------------------------ pool */
typedef struct { void (*fn)(void*, int64_t, int64_t); void* ctx; int64_t r0, r1; } job_t;
static void* job_run(void* p) { job_t* j = (job_t*)p; j->fn(j->ctx, j->r0, j->r1); return NULL; }
static void run_rows(void (*fn)(void*, int64_t, int64_t), void* ctx, int64_t rows, int nthreads) {
  if (nthreads <= 1 || rows < 2) { fn(ctx, 0, rows); return; }
  if (nthreads > rows) nthreads = (int)rows;
  pthread_t th[256];
  job_t jobs[256];
  if (nthreads > 256) nthreads = 256;
  for (int t = 0; t < nthreads; t++) {
    jobs[t].fn = fn; jobs[t].ctx = ctx;
    jobs[t].r0 = rows * t / nthreads; jobs[t].r1 = rows * (t + 1) / nthreads;
    pthread_create(&th[t], NULL, job_run, &jobs[t]);
  }
  for (int t = 0; t < nthreads; t++) pthread_join(th[t], NULL);
}

/* ---------------------------------------------------------- spline forward */
typedef struct { const ork_spec* s; const double* T; int nT; const double* X; double* Y; int tier; } sf_ctx;

static void spline_rows(void* p, int64_t r0, int64_t r1) {
  sf_ctx* c = (sf_ctx*)p;
  const ork_spec* s = c->s;
  int d = s->in_dim, m = s->out_dim, deg = s->degree, R = s->K + deg;
  double* basis = (double*)malloc(sizeof(double) * (R + deg + 1));
  for (int64_t row = r0; row < r1; row++) {
    const double* x = c->X + row * d;
    double* y = c->Y + row * m;
    if (c->tier == 1) {
      /* forward_optimized, spline.cpp:145-179: y[j] += os*(bs*b + ss*sp), i outer */
      for (int j = 0; j < m; j++) y[j] = 0.0;
      for (int i = 0; i < d; i++) {
        basis_into(c->T, c->nT, deg, x[i], basis);
        double b = silu(x[i]);
        for (int j = 0; j < m; j++) {
          int64_t e = (int64_t)i * m + j;
          const double* cf = s->coeffs + e * R;
          double sp = 0.0;
          for (int r = 0; r < R; r++) sp += cf[r] * basis[r];
          y[j] += s->out_scale[e] * (s->base_scale[e] * b + s->spline_scale[e] * sp);
        }
      }
    } else {
      /* forward_scalar, spline.cpp:129-143: acc over i of eval_edge_phi */
      for (int j = 0; j < m; j++) {
        double acc = 0.0;
        for (int i = 0; i < d; i++) {
          int64_t e = (int64_t)i * m + j;
          double b = silu(x[i]);
          basis_into(c->T, c->nT, deg, x[i], basis);
          const double* cf = s->coeffs + e * R;
          double sp = 0.0;
          for (int r = 0; r < R; r++) sp += cf[r] * basis[r];
          acc += s->out_scale[e] * (s->base_scale[e] * b + s->spline_scale[e] * sp);
        }
        y[j] = acc;
      }
    }
  }
  free(basis);
}

int ork_spline_forward(const ork_spec* s, const double* X, int64_t rows, int32_t tier,
                       int32_t nthreads, double* Y) {
  int st = check_spec(s);
  if (st) return st;
  int nT = s->K + 1 + 2 * s->degree;
  double* T = (double*)malloc(sizeof(double) * nT);
  st = knot_grid(s->breakpoints, s->K, s->degree, T);
  if (st) { free(T); return st; }
  sf_ctx c = {s, T, nT, X, Y, tier};
  run_rows(spline_rows, &c, rows, nthreads);
  free(T);
  return OK;
}

/* ---------------------------------------------------------------- compile */
/* round_half_away (compiler.cpp:77) is std::round == C round(). */
static double round_param(double v, int param_dtype) { /* compiler.cpp:97-101 */
  float f = (float)v;
  if (param_dtype == 1) return (double)ork_f16_bits_to_f32(ork_f32_to_f16_bits(f));
  return (double)f;
}
static void codes_for(const double* v, int n, double scale, double y_min, int lo, int hi, int* q) {
  for (int i = 0; i < n; i++) q[i] = 0; /* compiler.cpp:86-95 */
  if (scale <= 0.0) return;
  for (int i = 0; i < n; i++) {
    double r = round((v[i] - y_min) / scale);
    if (r < lo) r = lo;
    if (r > hi) r = hi;
    q[i] = (int)r;
  }
}

int ork_quantize_segment(const double* v, int32_t n, int32_t scheme, int32_t* q, double* scale,
                         double* y_min) {
  if (n <= 0) return fail(CONFIG, "cannot quantize an empty segment");
  for (int i = 0; i < n; i++)
    if (!isfinite(v[i])) return fail(NONFINITE, "non-finite table value");
  if (scheme == 0) { /* compiler.cpp:105-114 */
    double amax = 0.0;
    for (int i = 0; i < n; i++) amax = fmax(amax, fabs(v[i]));
    *y_min = 0.0;
    *scale = amax / 127.0;
    codes_for(v, n, *scale, 0.0, -127, 127, q);
  } else { /* compiler.cpp:116-128 */
    double lo = v[0], hi = v[0];
    for (int i = 0; i < n; i++) { lo = fmin(lo, v[i]); hi = fmax(hi, v[i]); }
    *y_min = lo;
    *scale = (hi - lo) / 255.0;
    codes_for(v, n, *scale, lo, 0, 255, q);
  }
  return OK;
}

int ork_compile_layer(const ork_spec* s, int32_t L, int32_t scheme, int32_t value_repr,
                      int32_t param_dtype, int32_t boundary_mode, int32_t oob_policy,
                      float* knots, uint8_t* qout, float* scale, float* y_min, float* bsc,
                      float* ssc, float* osc, double* float_table) {
  (void)boundary_mode; (void)oob_policy; /* recorded by the caller; no effect on bytes */
  if (L < 2) return fail(CONFIG, "samples_per_segment must be >= 2"); /* compiler.cpp:10-16 */
  int st = check_spec(s);
  if (st) return st;
  const int K = s->K, p = s->degree, R = K + p, nT = K + 1 + 2 * p;
  const int64_t E = (int64_t)s->in_dim * s->out_dim, npts = (int64_t)K * L;
  double* T = (double*)malloc(sizeof(double) * nT);
  st = knot_grid(s->breakpoints, K, p, T);
  if (st) { free(T); return st; }
  /* build_float_lut, compiler.cpp:29-73: points (right endpoint excluded), basis
   * once per point, s = sum_r c_r b_r from 0.0 in ascending r. */
  double* pts = (double*)malloc(sizeof(double) * npts);
  double* basis = (double*)malloc(sizeof(double) * npts * R);
  double* base = (double*)malloc(sizeof(double) * npts);
  double* buf = (double*)malloc(sizeof(double) * (R + p + 1));
  for (int k = 0; k < K; k++) {
    double t0 = s->breakpoints[k], step = (s->breakpoints[k + 1] - t0) / (double)L;
    for (int l = 0; l < L; l++) pts[(int64_t)k * L + l] = t0 + (double)l * step;
  }
  for (int64_t pi = 0; pi < npts; pi++) {
    basis_into(T, nT, p, pts[pi], buf);
    memcpy(basis + pi * R, buf, sizeof(double) * R);
    base[pi] = value_repr == 0 ? silu(pts[pi]) : 0.0;
  }
  double* vals = (double*)malloc(sizeof(double) * npts);
  int* q = (int*)malloc(sizeof(int) * L);
  for (int64_t e = 0; e < E; e++) {
    const double* c = s->coeffs + e * R;
    for (int64_t pi = 0; pi < npts; pi++) {
      const double* b = basis + pi * R;
      double acc = 0.0;
      for (int r = 0; r < R; r++) acc += c[r] * b[r];
      vals[pi] = value_repr == 0
                     ? s->out_scale[e] * (s->base_scale[e] * base[pi] + s->spline_scale[e] * acc)
                     : acc;
    }
    if (float_table) memcpy(float_table + e * npts, vals, sizeof(double) * npts);
    /* per-cell quantization, compiler.cpp:173-204 */
    for (int k = 0; k < K; k++) {
      const double* seg = vals + (int64_t)k * L;
      double sc, ym, dummy_s, dummy_y;
      for (int l = 0; l < L; l++)
        if (!isfinite(seg[l])) { st = fail(NONFINITE, "non-finite table value"); goto done; }
      ork_quantize_segment(seg, L, scheme, q, &dummy_s, &dummy_y);
      if (scheme == 0) {
        ym = 0.0;
        sc = round_param(dummy_s, param_dtype);
        codes_for(seg, L, sc, ym, -127, 127, q);
      } else {
        ym = round_param(dummy_y, param_dtype);
        double hi = seg[0];
        for (int l = 0; l < L; l++) hi = fmax(hi, seg[l]);
        sc = fmax(round_param((hi - ym) / 255.0, param_dtype), 0.0);
        codes_for(seg, L, sc, ym, 0, 255, q);
      }
      int64_t cell = e * K + k;
      scale[cell] = (float)sc;
      y_min[cell] = (float)ym;
      uint8_t* dst = qout + cell * L;
      for (int l = 0; l < L; l++) dst[l] = scheme == 0 ? (uint8_t)(int8_t)q[l] : (uint8_t)q[l];
    }
  }
  for (int i = 0; i <= K; i++) knots[i] = (float)s->breakpoints[i];
  if (value_repr == 1 && bsc)
    for (int64_t e = 0; e < E; e++) {
      bsc[e] = (float)s->base_scale[e];
      ssc[e] = (float)s->spline_scale[e];
      osc[e] = (float)s->out_scale[e];
    }
done:
  free(T); free(pts); free(basis); free(base); free(buf); free(vals); free(q);
  return st;
}

/* ---------------------------------------------------------------- runtime */
/* LutLayerArtifact::finalize checks, runtime.cpp:11-43. */
static int check_artifact(const ork_artifact* a) {
  if (a->in_dim < 1 || a->out_dim < 1) return fail(CONFIG, "artifact dims must be >= 1");
  if (a->L < 2) return fail(CONFIG, "samples per segment must be >= 2");
  if (a->K < 1) return fail(CONFIG, "artifact needs at least 2 knots");
  for (int i = 0; i <= a->K; i++) {
    if (!isfinite(a->knots[i])) return fail(NONFINITE, "non-finite knot");
    if (i > 0 && !(a->knots[i - 1] < a->knots[i])) return fail(CONFIG, "knots must be strictly increasing");
  }
  if (a->value_repr == 1 && (!a->base_scale || !a->spline_scale || !a->out_scale))
    return fail(DIMENSION, "edge scale arrays must have one entry per edge");
  if (a->value_repr == 0 && (a->base_scale || a->spline_scale || a->out_scale))
    return fail(CONFIG, "phi artifact must not carry edge scale arrays");
  return OK;
}

static double hi_clip_of(const ork_artifact* a) { /* runtime.cpp:150-153 */
  float tK = a->knots[a->K];
  return a->boundary_mode == 0 ? (double)nextafterf(tK, -INFINITY) : (double)tK;
}

static double fetch_cell(const ork_artifact* a, int64_t cell, int l) { /* runtime.cpp:81-88 */
  int64_t off = cell * a->L + l;
  if (a->float_table) return a->float_table[off];
  double q = a->scheme == 0 ? (double)(int8_t)a->q[off] : (double)a->q[off];
  return (double)a->y_min[cell] + (double)a->scale[cell] * q;
}

static void coords1(const ork_artifact* a, double x, int* in, double* xp, int* k, int* l0, int* l1, double* w) {
  double lo = (double)a->knots[0], hi = (double)a->knots[a->K];
  /* in_range runtime.cpp:71-75, safe_clip :45-51, segment_index :53-58 (upper_bound),
   * interp_coords :60-69 */
  *in = a->boundary_mode == 0 ? (lo <= x && x < hi) : (lo <= x && x <= hi);
  double h = hi_clip_of(a), c = x < lo ? lo : (x > h ? h : x);
  *xp = c;
  int kk = 0;
  while (kk + 1 <= a->K && (double)a->knots[kk + 1] <= c) kk++; /* upper_bound - 1 */
  if (kk > a->K - 1) kk = a->K - 1;
  if (kk < 0) kk = 0;
  double t0 = a->knots[kk], t1 = a->knots[kk + 1];
  double u = (c - t0) / (t1 - t0), z = u * (double)(a->L - 1);
  int ll = (int)floor(z);
  if (ll < 0) ll = 0;
  if (ll > a->L - 1) ll = a->L - 1;
  *k = kk; *l0 = ll; *l1 = ll + 1 < a->L - 1 ? ll + 1 : a->L - 1;
  *w = z - (double)ll;
}

int ork_coords(const ork_artifact* a, const double* x, int64_t n, uint8_t* in_range, double* x_clip,
               int32_t* k, int32_t* l0, int32_t* l1, double* w) {
  int st = check_artifact(a);
  if (st) return st;
  for (int64_t i = 0; i < n; i++) {
    int in, kk, a0, a1; double xp, ww;
    coords1(a, x[i], &in, &xp, &kk, &a0, &a1, &ww);
    if (in_range) in_range[i] = (uint8_t)in;
    if (x_clip) x_clip[i] = xp;
    if (k) k[i] = kk;
    if (l0) l0[i] = a0;
    if (l1) l1[i] = a1;
    if (w) w[i] = ww;
  }
  return OK;
}

int ork_eval_value(const ork_artifact* a, int32_t e, double x, double* value, int32_t* was_oob) {
  /* lut_eval_value, runtime.cpp:96-109 */
  int st = check_artifact(a);
  if (st) return st;
  if (!isfinite(x)) return fail(NONFINITE, "non-finite input value");
  if (e < 0 || e >= a->in_dim * a->out_dim) return fail(DIMENSION, "edge index out of range");
  int in, k, l0, l1; double xp, w;
  coords1(a, x, &in, &xp, &k, &l0, &l1, &w);
  int64_t cell = (int64_t)e * a->K + k;
  double v0 = fetch_cell(a, cell, l0), v1 = fetch_cell(a, cell, l1);
  double v = (1.0 - w) * v0 + w * v1;
  if (a->oob_policy == 1 && !in) v = 0.0;
  *value = v;
  if (was_oob) *was_oob = !in;
  return OK;
}

int ork_eval_phi(const ork_artifact* a, int32_t e, double x, double* value) {
  /* lut_eval_phi, runtime.cpp:111-120 */
  double v; int32_t oob;
  int st = ork_eval_value(a, e, x, &v, &oob);
  if (st) return st;
  if (a->value_repr == 0) { *value = v; return OK; }
  double xb = x;
  if (a->oob_policy == 0) {
    double lo = a->knots[0], h = hi_clip_of(a);
    xb = x < lo ? lo : (x > h ? h : x);
  }
  double bx = silu(xb);
  *value = (double)a->out_scale[e] * ((double)a->base_scale[e] * bx + (double)a->spline_scale[e] * v);
  return OK;
}

/* ---------------------------------------------------- artifact container */
/* Not restated in the port: the container is pinned by reference-written fixtures. */
int ork_artifact_save(const ork_artifact* a, const char* path) {
  (void)a; (void)path;
  return fail(99, "artifact I/O is checked against the reference library only");
}
int ork_artifact_load_resave(const char* path, const char* resave_path) {
  (void)path; (void)resave_path;
  return fail(99, "artifact I/O is checked against the reference library only");
}

/* ------------------------------------------------------- eval_accuracy */
typedef struct {
  const ork_spec* s; const ork_artifact* a; const double* X; const double* T; int nT;
  double sum_in, max_in, sum_oob, max_oob;
  uint64_t n_in, n_oob, n_bd, oob_samples;
  int err;
  pthread_mutex_t mu;
} ea_ctx;

/* lut_eval_phi (runtime.cpp:96-120) without the per-call artifact validation. */
static double phi_of(const ork_artifact* a, int64_t e, double x) {
  int in, k, l0, l1; double xp, w;
  coords1(a, x, &in, &xp, &k, &l0, &l1, &w);
  int64_t cell = e * a->K + k;
  double v = (1.0 - w) * fetch_cell(a, cell, l0) + w * fetch_cell(a, cell, l1);
  if (a->oob_policy == 1 && !in) v = 0.0;
  if (a->value_repr == 0) return v;
  double bx = silu(a->oob_policy == 0 ? xp : x);
  return (double)a->out_scale[e] * ((double)a->base_scale[e] * bx + (double)a->spline_scale[e] * v);
}

/* metrics.cpp:44-84, over rows [r0, r1) */
static void eval_rows(void* p, int64_t r0, int64_t r1) {
  ea_ctx* c = (ea_ctx*)p;
  const ork_spec* s = c->s; const ork_artifact* a = c->a;
  int d = s->in_dim, m = s->out_dim, R = s->K + s->degree;
  double lo = (double)a->knots[0], hi = (double)a->knots[a->K];
  double* basis = (double*)malloc(sizeof(double) * (c->nT + 1));
  double sum_in = 0, max_in = 0, sum_oob = 0, max_oob = 0;
  uint64_t n_in = 0, n_oob = 0, n_bd = 0, oob_samples = 0;
  int err = 0;
  for (int64_t row = r0; row < r1 && !err; row++) {
    int any = 0;
    for (int i = 0; i < d; i++) {
      double x = c->X[row * d + i];
      if (!isfinite(x)) { err = NONFINITE; break; }
      int masked = a->boundary_mode == 0 ? !(lo <= x && x < hi) : !(lo <= x && x <= hi);
      any |= masked;
      int interior = lo <= x && x < hi;
      basis_into(c->T, c->nT, s->degree, x, basis);
      double base = silu(x);
      for (int j = 0; j < m; j++) {
        int64_t e = (int64_t)i * m + j;
        double sp = 0.0;
        for (int r = 0; r < R; r++) sp += s->coeffs[e * R + r] * basis[r];
        double ref = s->out_scale[e] * (s->base_scale[e] * base + s->spline_scale[e] * sp);
        double err_ = fabs(phi_of(a, e, x) - ref);
        if (masked) { sum_oob += err_; if (err_ > max_oob) max_oob = err_; n_oob++; }
        else if (interior) { sum_in += err_; if (err_ > max_in) max_in = err_; n_in++; }
        else n_bd++;
      }
    }
    if (any) oob_samples++;
  }
  free(basis);
  pthread_mutex_lock(&c->mu);
  if (err) c->err = err;
  c->sum_in += sum_in; c->sum_oob += sum_oob;
  if (max_in > c->max_in) c->max_in = max_in;
  if (max_oob > c->max_oob) c->max_oob = max_oob;
  c->n_in += n_in; c->n_oob += n_oob; c->n_bd += n_bd; c->oob_samples += oob_samples;
  pthread_mutex_unlock(&c->mu);
}

int ork_eval_accuracy(const ork_spec* s, const ork_artifact* a, const double* X, int64_t rows,
                      int32_t nthreads, double* acc, uint64_t* counts, int32_t* has_oob) {
  int st = check_artifact(a);
  if (st) return st;
  if ((st = check_spec(s))) return st;
  if (s->in_dim != a->in_dim || s->out_dim != a->out_dim) return fail(DIMENSION, "layer and artifact shapes differ");
  int nT = s->K + 1 + 2 * s->degree;
  double* T = (double*)malloc(sizeof(double) * nT);
  if ((st = knot_grid(s->breakpoints, s->K, s->degree, T))) { free(T); return st; }
  ea_ctx c;
  memset(&c, 0, sizeof(c));
  c.s = s; c.a = a; c.X = X; c.T = T; c.nT = nT;
  pthread_mutex_init(&c.mu, NULL);
  run_rows(eval_rows, &c, rows, nthreads);
  pthread_mutex_destroy(&c.mu);
  free(T);
  if (c.err) return fail(c.err, "non-finite input value");
  acc[0] = c.n_in ? c.sum_in / (double)c.n_in : 0.0;
  acc[1] = c.max_in;
  acc[2] = c.n_oob ? c.sum_oob / (double)c.n_oob : 0.0;
  acc[3] = c.n_oob ? c.max_oob : 0.0;
  acc[4] = rows ? (double)c.oob_samples / (double)rows : 0.0;
  *has_oob = c.n_oob > 0;
  /* memory_breakdown, metrics.cpp:8-28 */
  uint64_t E = (uint64_t)a->in_dim * a->out_dim, ps = a->param_dtype ? 2 : 4;
  counts[0] = c.n_in; counts[1] = c.n_oob; counts[2] = c.n_bd; counts[3] = c.oob_samples;
  counts[4] = E * a->K * a->L;
  counts[5] = E * a->K * ps;
  counts[6] = E * a->K * ps;
  counts[7] = (uint64_t)(a->K + 1) * 4;
  counts[8] = a->value_repr ? 3 * E * 4 : 0;
  counts[9] = counts[4] + counts[5] + counts[6] + counts[7] + counts[8];
  counts[10] = 4 * E * (uint64_t)(s->K + s->degree + 3);
  acc[5] = counts[10] ? (double)counts[9] / (double)counts[10] : 0.0;
  return OK;
}

typedef struct {
  const ork_artifact* a; const double* X; double* Y; int tier;
  const double* cb; const double* cs; const double* T;
  uint64_t oob_inputs, oob_samples; int err;
  pthread_mutex_t mu;
} lf_ctx;

static void lut_rows(void* p, int64_t r0, int64_t r1) {
  lf_ctx* c = (lf_ctx*)p;
  const ork_artifact* a = c->a;
  const int d = a->in_dim, m = a->out_dim, L = a->L, K = a->K;
  const int sr = a->value_repr == 1, zs = a->oob_policy == 1, i8 = a->scheme == 0;
  uint64_t oi = 0, os = 0;
  int err = 0;
  if (c->tier == 0 || a->float_table) {
    /* forward_generic, runtime.cpp:225-246 */
    for (int64_t s = r0; s < r1 && !err; s++) {
      const double* x = c->X + s * d;
      double* y = c->Y + s * m;
      int any = 0;
      for (int i = 0; i < d; i++) {
        if (!isfinite(x[i])) { err = 1; break; }
        double lo = a->knots[0], hi = a->knots[K];
        int in = a->boundary_mode == 0 ? (lo <= x[i] && x[i] < hi) : (lo <= x[i] && x[i] <= hi);
        any |= !in;
        oi += !in;
      }
      if (err) break;
      for (int j = 0; j < m; j++) {
        double acc = 0.0;
        for (int i = 0; i < d; i++) {
          double v;
          ork_eval_phi(a, i * m + j, x[i], &v);
          acc += v;
        }
        y[j] = acc;
      }
      os += any;
    }
  } else {
    /* forward_quant<SR,ZS,I8>, runtime.cpp:135-223 */
    const double* T = c->T;
    const double lo = T[0], hi = T[K], hic = hi_clip_of(a), Lm1 = (double)(L - 1);
    const int half_open = a->boundary_mode == 0;
    int64_t* cell0v = (int64_t*)malloc(sizeof(int64_t) * d);
    int* l0v = (int*)malloc(sizeof(int) * d);
    int* l1v = (int*)malloc(sizeof(int) * d);
    double* w0v = (double*)malloc(sizeof(double) * d);
    double* w1v = (double*)malloc(sizeof(double) * d);
    double* bxv = (double*)malloc(sizeof(double) * d);
    for (int64_t s = r0; s < r1 && !err; s++) {
      const double* xr = c->X + s * d;
      double* yr = c->Y + s * m;
      for (int j = 0; j < m; j++) yr[j] = 0.0;
      int row_oob = 0;
      for (int i = 0; i < d; i++) {
        const double x = xr[i];
        if (!isfinite(x)) { err = 1; break; }
        const int in = lo <= x && (half_open ? x < hi : x <= hi);
        row_oob += !in;
        const double xp = x < lo ? lo : (x > hic ? hic : x);
        int k = 0;
        for (int r = 1; r < K; r++) k += xp >= T[r];
        const double u = (xp - T[k]) / (T[k + 1] - T[k]);
        const double z = u * Lm1;
        int l0 = (int)floor(z);
        l0 = l0 < 0 ? 0 : (l0 > L - 1 ? L - 1 : l0);
        const double w1 = z - (double)l0;
        const double mask = (zs && !in) ? 0.0 : 1.0;
        cell0v[i] = (int64_t)i * m * K + k;
        l0v[i] = l0;
        l1v[i] = l0 + 1 < L ? l0 + 1 : L - 1;
        w0v[i] = mask * (1.0 - w1);
        w1v[i] = mask * w1;
        if (sr) bxv[i] = silu(zs ? x : xp);
      }
      if (err) break;
      for (int i = 0; i < d; i++) {
        const int64_t e0 = (int64_t)i * m, cell0 = cell0v[i];
        const int64_t l0 = l0v[i], l1 = l1v[i];
        const double w0m = w0v[i], w1m = w1v[i], bx = sr ? bxv[i] : 0.0;
        for (int j = 0; j < m; j++) {
          const int64_t cell = cell0 + (int64_t)j * K, off = cell * L;
          const double ym = (double)a->y_min[cell], sc = (double)a->scale[cell];
          const double q0 = i8 ? (double)(int8_t)a->q[off + l0] : (double)a->q[off + l0];
          const double q1 = i8 ? (double)(int8_t)a->q[off + l1] : (double)a->q[off + l1];
          const double v0 = ym + sc * q0, v1 = ym + sc * q1;
          const double v = w0m * v0 + w1m * v1;
          if (sr) yr[j] += c->cb[e0 + j] * bx + c->cs[e0 + j] * v;
          else yr[j] += v;
        }
      }
      oi += (uint64_t)row_oob;
      os += row_oob != 0;
    }
    free(cell0v); free(l0v); free(l1v); free(w0v); free(w1v); free(bxv);
  }
  pthread_mutex_lock(&c->mu);
  c->oob_inputs += oi;
  c->oob_samples += os;
  if (err) c->err = 1;
  pthread_mutex_unlock(&c->mu);
}

int ork_lut_forward(const ork_artifact* a, const double* X, int64_t rows, int32_t tier,
                    int32_t nthreads, double* Y, uint64_t* stats) {
  int st = check_artifact(a);
  if (st) return st;
  const int64_t E = (int64_t)a->in_dim * a->out_dim;
  double* cb = NULL; double* cs = NULL;
  double* T = (double*)malloc(sizeof(double) * (a->K + 1));
  for (int i = 0; i <= a->K; i++) T[i] = (double)a->knots[i]; /* knots_f64, runtime.cpp:42 */
  if (a->value_repr == 1) { /* gain fusion, runtime.cpp:263-273 */
    cb = (double*)malloc(sizeof(double) * E);
    cs = (double*)malloc(sizeof(double) * E);
    for (int64_t e = 0; e < E; e++) {
      cb[e] = (double)a->out_scale[e] * (double)a->base_scale[e];
      cs[e] = (double)a->out_scale[e] * (double)a->spline_scale[e];
    }
  }
  lf_ctx c;
  memset(&c, 0, sizeof c);
  c.a = a; c.X = X; c.Y = Y; c.tier = tier; c.cb = cb; c.cs = cs; c.T = T;
  pthread_mutex_init(&c.mu, NULL);
  run_rows(lut_rows, &c, rows, nthreads);
  pthread_mutex_destroy(&c.mu);
  free(cb); free(cs); free(T);
  if (c.err) return fail(NONFINITE, "non-finite input value");
  if (stats) {
    stats[0] = (uint64_t)rows;
    stats[1] = c.oob_samples;
    stats[2] = (uint64_t)rows * (uint64_t)a->in_dim;
    stats[3] = c.oob_inputs;
  }
  return OK;
}

int ork_lut_model_forward(const ork_artifact* chain, int32_t n, const double* X, int64_t rows,
                          int32_t tier, int32_t nthreads, double* Y, uint64_t* stats) {
  /* lut_model_forward_batch, runtime.cpp:298-314 */
  if (n < 1) return fail(CONFIG, "artifact chain is empty");
  for (int l = 1; l < n; l++)
    if (chain[l].in_dim != chain[l - 1].out_dim) return fail(DIMENSION, "artifact chain dimension mismatch");
  const double* cur = X;
  double* buf = NULL;
  for (int l = 0; l < n; l++) {
    double* out = l == n - 1 ? Y : (double*)malloc(sizeof(double) * rows * chain[l].out_dim);
    int st = ork_lut_forward(&chain[l], cur, rows, tier, nthreads, out, stats ? stats + 4 * l : NULL);
    free(buf);
    buf = l == n - 1 ? NULL : out;
    if (st) { free(buf); return st; }
    cur = out;
  }
  return OK;
}

/* ----------------------------------------------------------------- recipes */
/* The BASELINE.json configs, generated with the reference Rng per SURVEY.md §8(d).
 * Pinned recipe: breakpoints lo+(hi-lo)*k/G; one Rng(seed) stream
 * across the layers in order; per edge e=i*m+j: R coeffs N(0,sigma), then
 * base_scale=U(-1,1); spline_scale=out_scale=1. */
typedef struct { int nl; int dims[5]; int G; double lo, hi, sigma; uint64_t seed; } recipe_t;
static int recipe_of(int cfg, recipe_t* r) {
  static const recipe_t R[5] = {
      {2, {2, 5, 1}, 5, -1.0, 1.0, 0.1, 0},
      {2, {78, 16, 2}, 5, -1.0, 1.0, 0.1, 1},
      {2, {64, 64, 1}, 8, -1.0, 1.0, 0.1, 2},
      {3, {1024, 1024, 1024, 10}, 8, -1.0, 1.0, 0.05, 3},
      {2, {4096, 4096, 4096}, 16, -2.0, 2.0, 0.02, 4},
  };
  if (cfg < 1 || cfg > 5) return fail(CONFIG, "unknown config");
  *r = R[cfg - 1];
  return OK;
}

int ork_recipe_layer(int32_t cfg, int32_t layer, double* bp, double* coeffs, double* bs,
                     double* ss, double* os) {
  recipe_t r;
  int st = recipe_of(cfg, &r);
  if (st) return st;
  if (layer < 0 || layer >= r.nl) return fail(DIMENSION, "layer out of range");
  for (int k = 0; k <= r.G; k++) bp[k] = r.lo + (r.hi - r.lo) * (double)k / (double)r.G;
  const int R = r.G + 3;
  rng_t g;
  rng_init(&g, r.seed);
  for (int l = 0; l <= layer; l++) {
    int64_t E = (int64_t)r.dims[l] * r.dims[l + 1];
    for (int64_t e = 0; e < E; e++) {
      for (int q = 0; q < R; q++) {
        double v = rng_normal_ms(&g, 0.0, r.sigma);
        if (l == layer) coeffs[e * R + q] = v;
      }
      double b = rng_uniform_ab(&g, -1.0, 1.0);
      if (l == layer) { bs[e] = b; ss[e] = 1.0; os[e] = 1.0; }
    }
  }
  return OK;
}

/* gen_layer (model_gen.cpp:7-27) */
int ork_gen_layer(uint64_t seed, int32_t d, int32_t m, int32_t segments, int32_t degree, double* bp, double* coeffs,
                  double* bs, double* ss, double* os) {
  if (segments < 1) return fail(CONFIG, "segments must be >= 1");
  for (int k = 0; k <= segments; k++) bp[k] = -1.0 + 2.0 * (double)k / segments;
  rng_t r;
  rng_init(&r, seed);
  int R = segments + degree;
  for (int64_t e = 0; e < (int64_t)d * m; e++) {
    for (int q = 0; q < R; q++) coeffs[e * R + q] = rng_normal_ms(&r, 0.0, 0.1);
    bs[e] = rng_uniform_ab(&r, 0.5, 1.5);
    ss[e] = rng_uniform_ab(&r, 0.5, 1.5);
    os[e] = rng_uniform_ab(&r, 0.5, 1.5);
  }
  return OK;
}

/* gen_inputs (model_gen.cpp:33-45) */
int ork_gen_inputs(uint64_t seed, int64_t n, int64_t dim, double lo, double hi, int32_t clip, double* X) {
  if (!(lo < hi)) return fail(CONFIG, "input range must satisfy lo < hi");
  rng_t r;
  rng_init(&r, seed);
  for (int64_t t = 0; t < n * dim; t++) {
    double x = rng_normal(&r);
    if (clip) x = x < lo ? lo : (hi < x ? hi : x);
    X[t] = x;
  }
  return OK;
}

int ork_recipe_inputs(int32_t cfg, int64_t row0, int64_t rows, float* X) {
  recipe_t r;
  int st = recipe_of(cfg, &r);
  if (st) return st;
  rng_t g;
  rng_init(&g, r.seed ^ 0x5eed5eed5eed5eedull); /* sweep.cpp:25 input salt */
  const int d = r.dims[0];
  const int64_t n0 = row0 * d, n1 = (row0 + rows) * d;
  for (int64_t n = 0; n < n1; n++) {
    double x;
    switch (cfg) {
      case 1: x = rng_uniform_ab(&g, -1.2, 1.2); break;
      case 2: {
        x = rng_normal_ms(&g, 0.0, 0.4);
        if (rng_uniform(&g) < 0.01) {
          int neg = rng_uniform(&g) < 0.5;
          double mag = rng_uniform_ab(&g, 1.5, 4.0);
          x = neg ? -mag : mag;
        }
        break;
      }
      case 3: {
        x = rng_uniform_ab(&g, -1.5, 1.5);
        if (rng_uniform(&g) < 0.005) {
          int k = (int)(rng_uniform(&g) * (double)(r.G + 1));
          x = r.lo + (r.hi - r.lo) * (double)k / (double)r.G;
        }
        break;
      }
      case 4: x = rng_normal_ms(&g, 0.0, 0.5); break;
      default: x = rng_uniform_ab(&g, -2.5, 2.5); break;
    }
    if (n >= n0) X[n - n0] = (float)x;
  }
  return OK;
}
