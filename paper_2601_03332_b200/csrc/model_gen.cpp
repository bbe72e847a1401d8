// model_gen.cpp — host-side support for the hot path: the deterministic generator of
// the reference (rng.hpp:13-58, rng.cpp:7-22 — splitmix64 seeding, xoshiro256++
// stream, Marsaglia polar normals with a cached spare), the synthetic BASELINE
// config recipes (pinned in DESIGN.md §3), and the exact f64
// Cox-de Boor basis used to build compile tables (spline.cpp:8-27, 69-85).
#include <cmath>
#include <cstdint>
#include <stdexcept>
#include <vector>

#include "lkg_internal.h"

namespace lkg {
namespace {

class Xoshiro {
 public:
  explicit Xoshiro(uint64_t seed) {
    uint64_t x = seed;
    for (uint64_t& w : s_) {  // splitmix64
      x += 0x9e3779b97f4a7c15ull;
      uint64_t z = x;
      z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
      z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
      w = z ^ (z >> 31);
    }
  }
  uint64_t next() {
    const uint64_t out = rot(s_[0] + s_[3], 23) + s_[0];
    const uint64_t t = s_[1] << 17;
    s_[2] ^= s_[0];
    s_[3] ^= s_[1];
    s_[1] ^= s_[2];
    s_[0] ^= s_[3];
    s_[2] ^= t;
    s_[3] = rot(s_[3], 45);
    return out;
  }
  double uniform() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }
  double uniform(double lo, double hi) { return lo + (hi - lo) * uniform(); }
  double normal() {
    if (have_) {
      have_ = false;
      return spare_;
    }
    double u, v, s;
    do {
      u = 2.0 * uniform() - 1.0;
      v = 2.0 * uniform() - 1.0;
      s = u * u + v * v;
    } while (s >= 1.0 || s == 0.0);
    const double f = std::sqrt(-2.0 * std::log(s) / s);
    spare_ = v * f;
    have_ = true;
    return u * f;
  }
  double normal(double mean, double sd) { return mean + sd * normal(); }

 private:
  static uint64_t rot(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }
  uint64_t s_[4];
  double spare_ = 0.0;
  bool have_ = false;
};

struct Recipe {
  int n_layers;
  int dims[5];
  int G;
  double lo, hi, sigma;
  uint64_t seed;
};

// BASELINE.json configs[0..4] (C1..C5).
const Recipe kRecipes[5] = {
    {2, {2, 5, 1}, 5, -1.0, 1.0, 0.1, 0},
    {2, {78, 16, 2}, 5, -1.0, 1.0, 0.1, 1},
    {2, {64, 64, 1}, 8, -1.0, 1.0, 0.1, 2},
    {3, {1024, 1024, 1024, 10}, 8, -1.0, 1.0, 0.05, 3},
    {2, {4096, 4096, 4096}, 16, -2.0, 2.0, 0.02, 4},
};

const Recipe& recipe(int cfg) {
  if (cfg < 1 || cfg > 5) throw Error{LKG_ERR_CONFIG, "unknown config " + std::to_string(cfg)};
  return kRecipes[cfg - 1];
}

}  // namespace

int recipe_dims(int cfg, int* n_layers, int* dims, int* G, double* lo, double* hi) {
  const Recipe& r = recipe(cfg);
  *n_layers = r.n_layers;
  for (int l = 0; l <= r.n_layers; l++) dims[l] = r.dims[l];
  *G = r.G;
  *lo = r.lo;
  *hi = r.hi;
  return 0;
}

// One Rng(seed) stream across the layers in order; per edge e = i*m + j: R coeffs
// N(0, sigma), then base_scale = U(-1, 1); spline_scale = out_scale = 1.
void recipe_layer(int cfg, int layer, int col0, int col1, double* bp, double* coeffs, double* bs,
                  double* ss, double* os) {
  const Recipe& r = recipe(cfg);
  if (layer < 0 || layer >= r.n_layers) throw Error{LKG_ERR_DIMENSION, "layer out of range"};
  const int m = r.dims[layer + 1];
  if (col1 <= col0) {
    col0 = 0;
    col1 = m;
  }
  if (col0 < 0 || col1 > m) throw Error{LKG_ERR_DIMENSION, "column range out of range"};
  const int mc = col1 - col0, R = r.G + 3;
  for (int k = 0; k <= r.G; k++) bp[k] = r.lo + (r.hi - r.lo) * static_cast<double>(k) / r.G;
  Xoshiro g(r.seed);
  for (int l = 0; l <= layer; l++) {
    const int64_t d = r.dims[l], ml = r.dims[l + 1];
    const bool keep = l == layer;
    for (int64_t i = 0; i < d; i++)
      for (int64_t j = 0; j < ml; j++) {
        const bool in_cols = keep && j >= col0 && j < col1;
        const int64_t e = i * mc + (j - col0);
        for (int q = 0; q < R; q++) {
          const double v = g.normal(0.0, r.sigma);
          if (in_cols) coeffs[e * R + q] = v;
        }
        const double b = g.uniform(-1.0, 1.0);
        if (in_cols) {
          bs[e] = b;
          ss[e] = 1.0;
          os[e] = 1.0;
        }
      }
  }
}

// gen_layer (model_gen.cpp:7-27): breakpoints -1 + 2k/G, one Rng(seed) stream, per edge R
// coefficients normal(0, 0.1) then base, spline, out scales uniform(0.5, 1.5).
void gen_layer(uint64_t seed, int d, int m, int segments, int degree, double* bp, double* coeffs, double* bs,
               double* ss, double* os) {
  for (int k = 0; k <= segments; k++) bp[k] = -1.0 + 2.0 * static_cast<double>(k) / segments;
  Xoshiro rng(seed);
  const int R = segments + degree;
  const int64_t E = (int64_t)d * m;
  for (int64_t e = 0; e < E; e++) {
    for (int r = 0; r < R; r++) coeffs[e * R + r] = rng.normal(0.0, 0.1);
    bs[e] = rng.uniform(0.5, 1.5);
    ss[e] = rng.uniform(0.5, 1.5);
    os[e] = rng.uniform(0.5, 1.5);
  }
}

// gen_inputs (model_gen.cpp:33-45): standard normals, optionally clamped to [lo, hi].
void gen_inputs(uint64_t seed, int64_t n, int64_t dim, double lo, double hi, bool clip, double* X) {
  Xoshiro rng(seed);
  for (int64_t t = 0; t < n * dim; t++) {
    double x = rng.normal();
    if (clip) x = x < lo ? lo : (hi < x ? hi : x);  // std::clamp
    X[t] = x;
  }
}

void recipe_inputs(int cfg, int64_t row0, int64_t rows, float* X) {
  const Recipe& r = recipe(cfg);
  Xoshiro g(r.seed ^ 0x5eed5eed5eed5eedull);  // input salt, sweep.cpp:25
  const int64_t d = r.dims[0], n0 = row0 * d, n1 = (row0 + rows) * d;
  for (int64_t n = 0; n < n1; n++) {
    double x;
    switch (cfg) {
      case 1: x = g.uniform(-1.2, 1.2); break;
      case 2:  // N(0, 0.4) with 1% +-U(1.5, 4) outliers
        x = g.normal(0.0, 0.4);
        if (g.uniform() < 0.01) {
          const bool neg = g.uniform() < 0.5;
          const double mag = g.uniform(1.5, 4.0);
          x = neg ? -mag : mag;
        }
        break;
      case 3:  // U(-1.5, 1.5) with 0.5% exact knot values
        x = g.uniform(-1.5, 1.5);
        if (g.uniform() < 0.005) {
          const int k = static_cast<int>(g.uniform() * (r.G + 1));
          x = r.lo + (r.hi - r.lo) * static_cast<double>(k) / r.G;
        }
        break;
      case 4: x = g.normal(0.0, 0.5); break;
      default: x = g.uniform(-2.5, 2.5); break;
    }
    if (n >= n0) X[n - n0] = static_cast<float>(x);
  }
}

// KnotGrid extension (spline.cpp:8-27): degree knots each side continuing the end spacing.
void knot_grid(const std::vector<double>& bp, int degree, std::vector<double>& ext) {
  const size_t n = bp.size();
  const double hl = bp[1] - bp[0], hr = bp[n - 1] - bp[n - 2];
  ext.assign(n + 2 * static_cast<size_t>(degree), 0.0);
  for (int i = 0; i < degree; i++) ext[degree - 1 - i] = bp.front() - (i + 1) * hl;
  for (size_t i = 0; i < n; i++) ext[degree + i] = bp[i];
  for (int i = 0; i < degree; i++) ext[degree + n + i] = bp.back() + (i + 1) * hr;
}

// Cox-de Boor with the 0/0 -> 0 guard, every indicator evaluated (spline.cpp:69-83).
void basis_into(const std::vector<double>& T, int degree, double x, double* buf) {
  const int n0 = static_cast<int>(T.size()) - 1;
  for (int r = 0; r < n0; r++) buf[r] = (T[r] <= x && x < T[r + 1]) ? 1.0 : 0.0;
  for (int q = 1; q <= degree; q++)
    for (int r = 0; r < n0 - q; r++) {
      double acc = 0.0;
      const double d1 = T[r + q] - T[r];
      if (d1 > 0.0) acc += (x - T[r]) / d1 * buf[r];
      const double d2 = T[r + q + 1] - T[r + 1];
      if (d2 > 0.0) acc += (T[r + q + 1] - x) / d2 * buf[r + 1];
      buf[r] = acc;
    }
}

double silu_host(double x) { return x / (1.0 + std::exp(-x)); }

}  // namespace lkg
