// ref_capi.cpp — C-ABI adapter over the UNMODIFIED reference library (TEST
// INFRASTRUCTURE ONLY). oracle/Makefile compiles the reference's own sources in
// place from /root/reference/proj/core/src and links them with this file into
// oracle/_ref/liblutkan_ref.so, which exports the lk_oracle.h interface. Every
// function below converts plain arrays into the reference types and calls the
// reference entry point named in its comment; exceptions map to status codes
// (types.hpp:11-39 taxonomy).
#include <algorithm>
#include <cstring>
#include <exception>
#include <memory>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "lutkan/artifact_io.hpp"
#include "lutkan/compiler.hpp"
#include "lutkan/float16.hpp"
#include "lutkan/metrics.hpp"
#include "lutkan/model_gen.hpp"
#include "lutkan/rng.hpp"
#include "lutkan/runtime.hpp"
#include "lutkan/spline.hpp"

extern "C" {
#include "lk_oracle.h"
}

using namespace lutkan;

namespace {
thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const CorruptArchiveError& e) {  // artifact_io.hpp:11-52, statuses as lutkan_b200.h
    g_err = e.what();
    return 10;
  } catch (const CorruptBlobError& e) {
    g_err = e.what();
    return 11;
  } catch (const MissingKeyError& e) {
    g_err = e.what();
    return 12;
  } catch (const ShapeError& e) {
    g_err = e.what();
    return 13;
  } catch (const VersionError& e) {
    g_err = e.what();
    return 14;
  } catch (const EnumError& e) {
    g_err = e.what();
    return 15;
  } catch (const IoError& e) {
    g_err = e.what();
    return 9;
  } catch (const UnsupportedBaseError& e) {
    g_err = e.what();
    return 4;
  } catch (const NonFiniteError& e) {
    g_err = e.what();
    return 3;
  } catch (const DimensionError& e) {
    g_err = e.what();
    return 2;
  } catch (const ConfigError& e) {
    g_err = e.what();
    return 1;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 99;
  }
}

KanLayerSpec to_spec(const ork_spec* s) {
  std::vector<double> bp(s->breakpoints, s->breakpoints + s->K + 1);
  KnotGrid g(std::move(bp), s->degree);
  const int R = g.basis_count();
  const std::size_t E = static_cast<std::size_t>(s->in_dim) * s->out_dim;
  std::vector<EdgeParams> edges(E);
  for (std::size_t e = 0; e < E; e++) {
    edges[e].coeffs.assign(s->coeffs + e * R, s->coeffs + (e + 1) * R);
    edges[e].base_scale = s->base_scale[e];
    edges[e].spline_scale = s->spline_scale[e];
    edges[e].out_scale = s->out_scale[e];
  }
  return KanLayerSpec(s->in_dim, s->out_dim, std::move(g), "silu", std::move(edges));
}

LutLayerArtifact to_artifact(const ork_artifact* a) {
  LutLayerArtifact r;
  r.in_dim = a->in_dim;
  r.out_dim = a->out_dim;
  r.L = a->L;
  r.value_repr = a->value_repr ? ValueRepr::SplineComponent : ValueRepr::Phi;
  r.scheme = a->scheme ? Scheme::Asymmetric : Scheme::Symmetric;
  r.dtype = a->scheme ? Dtype::Uint8 : Dtype::Int8;
  r.param_dtype = a->param_dtype ? ParamDtype::F16 : ParamDtype::F32;
  r.oob.boundary_mode = a->boundary_mode ? BoundaryMode::Closed : BoundaryMode::HalfOpen;
  r.oob.oob_policy = a->oob_policy ? OobPolicy::ZeroSpline : OobPolicy::ClipX;
  r.base_kind = a->value_repr ? "silu" : "";
  const std::size_t E = static_cast<std::size_t>(a->in_dim) * a->out_dim, K = a->K;
  r.knots.assign(a->knots, a->knots + K + 1);
  r.q_table.assign(a->q, a->q + E * K * a->L);
  r.scale.assign(a->scale, a->scale + E * K);
  r.y_min.assign(a->y_min, a->y_min + E * K);
  if (a->base_scale) r.edge_base_scale.assign(a->base_scale, a->base_scale + E);
  if (a->spline_scale) r.edge_spline_scale.assign(a->spline_scale, a->spline_scale + E);
  if (a->out_scale) r.edge_out_scale.assign(a->out_scale, a->out_scale + E);
  if (a->float_table) r.float_table.assign(a->float_table, a->float_table + E * K * a->L);
  r.finalize();
  return r;
}

Matrix to_matrix(const double* X, std::int64_t rows, int cols) {
  Matrix m(static_cast<std::size_t>(rows), static_cast<std::size_t>(cols));
  std::memcpy(m.data.data(), X, sizeof(double) * m.data.size());
  return m;
}

// Row shards over std::threads; the reference functions are pure and re-entrant
// (tests/test_spline.cpp:310-323).
template <class F>
void shard_rows(std::int64_t rows, int nthreads, F&& f) {
  if (nthreads <= 1 || rows < 2) {
    f(0, rows, 0);
    return;
  }
  if (nthreads > rows) nthreads = static_cast<int>(rows);
  std::vector<std::thread> th;
  std::vector<std::exception_ptr> errs(nthreads);
  for (int t = 0; t < nthreads; t++)
    th.emplace_back([&, t] {
      try {
        f(rows * t / nthreads, rows * (t + 1) / nthreads, t);
      } catch (...) {
        errs[t] = std::current_exception();
      }
    });
  for (auto& t : th) t.join();
  for (auto& e : errs)
    if (e) std::rethrow_exception(e);
}

}  // namespace

extern "C" {

const char* ork_last_error(void) { return g_err.c_str(); }
const char* ork_impl_name(void) { return "reference"; }

int ork_compile_layer(const ork_spec* s, int32_t L, int32_t scheme, int32_t value_repr,
                      int32_t param_dtype, int32_t boundary_mode, int32_t oob_policy, float* knots,
                      uint8_t* q, float* scale, float* y_min, float* bs, float* ss, float* os,
                      double* float_table) {
  return guarded([&] {
    QuantConfig cfg;  // compiler.hpp:15-24
    cfg.samples_per_segment = L;
    cfg.scheme = scheme ? Scheme::Asymmetric : Scheme::Symmetric;
    cfg.dtype = scheme ? Dtype::Uint8 : Dtype::Int8;
    cfg.value_repr = value_repr ? ValueRepr::SplineComponent : ValueRepr::Phi;
    cfg.param_dtype = param_dtype ? ParamDtype::F16 : ParamDtype::F32;
    OobConfig oob{boundary_mode ? BoundaryMode::Closed : BoundaryMode::HalfOpen,
                  oob_policy ? OobPolicy::ZeroSpline : OobPolicy::ClipX};
    const KanLayerSpec spec = to_spec(s);
    // compile_layer / compile_layer_debug_float, compiler.cpp:213-233
    const LutLayerArtifact a = float_table ? compile_layer_debug_float(spec, cfg, oob)
                                           : compile_layer(spec, cfg, oob);
    std::memcpy(knots, a.knots.data(), sizeof(float) * a.knots.size());
    std::memcpy(q, a.q_table.data(), a.q_table.size());
    std::memcpy(scale, a.scale.data(), sizeof(float) * a.scale.size());
    std::memcpy(y_min, a.y_min.data(), sizeof(float) * a.y_min.size());
    if (bs && !a.edge_base_scale.empty()) {
      std::memcpy(bs, a.edge_base_scale.data(), sizeof(float) * a.edge_base_scale.size());
      std::memcpy(ss, a.edge_spline_scale.data(), sizeof(float) * a.edge_spline_scale.size());
      std::memcpy(os, a.edge_out_scale.data(), sizeof(float) * a.edge_out_scale.size());
    }
    if (float_table)
      std::memcpy(float_table, a.float_table.data(), sizeof(double) * a.float_table.size());
  });
}

int ork_lut_forward(const ork_artifact* a, const double* X, int64_t rows, int32_t tier,
                    int32_t nthreads, double* Y, uint64_t* stats) {
  return guarded([&] {
    const LutLayerArtifact art = to_artifact(a);
    const Tier t = tier ? Tier::Optimized : Tier::Scalar;
    OobStats total;
    std::vector<OobStats> parts(nthreads > 1 ? nthreads : 1);
    shard_rows(rows, nthreads, [&](std::int64_t r0, std::int64_t r1, int ti) {
      Matrix Xs = to_matrix(X + r0 * a->in_dim, r1 - r0, a->in_dim);
      auto [Ys, st] = lut_layer_forward_batch(art, Xs, t);  // runtime.cpp:250-285
      std::memcpy(Y + r0 * a->out_dim, Ys.data.data(), sizeof(double) * Ys.data.size());
      parts[ti] = st;
    });
    for (auto& p : parts) total.merge(p);  // runtime.hpp:114-119
    if (stats) {
      stats[0] = total.n_samples;
      stats[1] = total.n_oob_samples;
      stats[2] = total.n_inputs;
      stats[3] = total.n_oob_inputs;
    }
  });
}

int ork_lut_model_forward(const ork_artifact* chain, int32_t n, const double* X, int64_t rows,
                          int32_t tier, int32_t nthreads, double* Y, uint64_t* stats) {
  return guarded([&] {
    std::vector<LutLayerArtifact> arts;
    for (int l = 0; l < n; l++) arts.push_back(to_artifact(&chain[l]));
    const Tier t = tier ? Tier::Optimized : Tier::Scalar;
    const int d = n > 0 ? chain[0].in_dim : 0, mo = n > 0 ? chain[n - 1].out_dim : 0;
    std::vector<std::vector<OobStats>> parts(nthreads > 1 ? nthreads : 1);
    shard_rows(rows, nthreads, [&](std::int64_t r0, std::int64_t r1, int ti) {
      Matrix Xs = to_matrix(X + r0 * d, r1 - r0, d);
      ChainBatchResult r = lut_model_forward_batch(arts, Xs, t);  // runtime.cpp:298-314
      std::memcpy(Y + r0 * mo, r.Y.data.data(), sizeof(double) * r.Y.data.size());
      parts[ti] = r.per_layer;
    });
    if (stats)
      for (int l = 0; l < n; l++) {
        OobStats tot;
        for (auto& p : parts)
          if (!p.empty()) tot.merge(p[l]);
        stats[4 * l + 0] = tot.n_samples;
        stats[4 * l + 1] = tot.n_oob_samples;
        stats[4 * l + 2] = tot.n_inputs;
        stats[4 * l + 3] = tot.n_oob_inputs;
      }
  });
}

// A prepared chain forward for timing the reference fairly (bench.py's CPU legs): the artifacts are
// converted and the batch is cut into the per-thread Matrix shards ONCE, outside the timed region —
// what a multi-threaded caller of the reference would hold anyway; a run is then only the threads'
// lut_model_forward_batch calls (runtime.cpp:298-314) and the copy of their results into Y.
struct ChainSession {
  std::vector<LutLayerArtifact> arts;
  std::vector<Matrix> shards;
  std::vector<std::int64_t> row0;
  Tier tier = Tier::Optimized;
  std::int64_t rows = 0;
  int mo = 0;
};

void* ork_chain_session_create(const ork_artifact* chain, int32_t n, const double* X, int64_t rows, int32_t tier,
                               int32_t nthreads) {
  ChainSession* S = nullptr;
  const int rc = guarded([&] {
    auto s = std::make_unique<ChainSession>();
    for (int l = 0; l < n; l++) s->arts.push_back(to_artifact(&chain[l]));
    s->tier = tier ? Tier::Optimized : Tier::Scalar;
    s->rows = rows;
    s->mo = n > 0 ? chain[n - 1].out_dim : 0;
    const int d = n > 0 ? chain[0].in_dim : 0;
    int T = nthreads > 1 ? nthreads : 1;
    if (T > rows) T = rows > 0 ? static_cast<int>(rows) : 1;
    for (int t = 0; t < T; t++) {
      const std::int64_t r0 = rows * t / T, r1 = rows * (t + 1) / T;
      s->row0.push_back(r0);
      s->shards.push_back(to_matrix(X + r0 * d, r1 - r0, d));
    }
    S = s.release();
  });
  return rc == 0 ? S : nullptr;
}

int ork_chain_session_run(void* session, double* Y, uint64_t* stats) {
  return guarded([&] {
    ChainSession* s = static_cast<ChainSession*>(session);
    if (!s) throw std::invalid_argument("null chain session");
    const int T = static_cast<int>(s->shards.size()), n = static_cast<int>(s->arts.size());
    std::vector<std::vector<OobStats>> parts(T);
    shard_rows(T, T, [&](std::int64_t t0, std::int64_t, int) {
      const int t = static_cast<int>(t0);
      ChainBatchResult r = lut_model_forward_batch(s->arts, s->shards[t], s->tier);
      std::memcpy(Y + s->row0[t] * s->mo, r.Y.data.data(), sizeof(double) * r.Y.data.size());
      parts[t] = r.per_layer;
    });
    if (stats)
      for (int l = 0; l < n; l++) {
        OobStats tot;
        for (auto& p : parts)
          if (!p.empty()) tot.merge(p[l]);
        stats[4 * l + 0] = tot.n_samples;
        stats[4 * l + 1] = tot.n_oob_samples;
        stats[4 * l + 2] = tot.n_inputs;
        stats[4 * l + 3] = tot.n_oob_inputs;
      }
  });
}

void ork_chain_session_free(void* session) { delete static_cast<ChainSession*>(session); }

int ork_spline_forward(const ork_spec* s, const double* X, int64_t rows, int32_t tier,
                       int32_t nthreads, double* Y) {
  return guarded([&] {
    const KanLayerSpec spec = to_spec(s);
    const Tier t = tier ? Tier::Optimized : Tier::Scalar;
    shard_rows(rows, nthreads, [&](std::int64_t r0, std::int64_t r1, int) {
      Matrix Xs = to_matrix(X + r0 * s->in_dim, r1 - r0, s->in_dim);
      Matrix Ys = layer_forward_batch(spec, Xs, t);  // spline.cpp:183-187
      std::memcpy(Y + r0 * s->out_dim, Ys.data.data(), sizeof(double) * Ys.data.size());
    });
  });
}

int ork_gen_layer(uint64_t seed, int32_t d, int32_t m, int32_t segments, int32_t degree, double* bp, double* coeffs,
                  double* bs, double* ss, double* os) {
  return guarded([&] {
    const KanLayerSpec s = gen_layer(seed, d, m, segments, degree);  // model_gen.cpp:7-27
    const auto& b = s.grid().breakpoints();
    std::copy(b.begin(), b.end(), bp);
    const auto& c = s.packed_coeffs();
    std::copy(c.begin(), c.end(), coeffs);
    std::copy(s.base_scales().begin(), s.base_scales().end(), bs);
    std::copy(s.spline_scales().begin(), s.spline_scales().end(), ss);
    std::copy(s.out_scales().begin(), s.out_scales().end(), os);
  });
}

int ork_gen_inputs(uint64_t seed, int64_t n, int64_t dim, double lo, double hi, int32_t clip, double* X) {
  return guarded([&] {
    const Matrix M = gen_inputs(seed, static_cast<std::size_t>(n), static_cast<std::size_t>(dim), lo, hi, clip != 0);
    std::copy(M.data.begin(), M.data.end(), X);
  });
}

int ork_artifact_save(const ork_artifact* a, const char* path) {
  return guarded([&] { save_artifact(to_artifact(a), path); });  // artifact_io.cpp:206-219
}

int ork_artifact_load_resave(const char* path, const char* resave_path) {
  return guarded([&] {
    const LutLayerArtifact a = load_artifact(path);  // artifact_io.cpp:221-300
    if (resave_path) save_artifact(a, resave_path);
  });
}

int ork_eval_accuracy(const ork_spec* s, const ork_artifact* a, const double* X, int64_t rows,
                      int32_t nthreads, double* acc, uint64_t* counts, int32_t* has_oob) {
  return guarded([&] {
    const KanLayerSpec spec = to_spec(s);
    const LutLayerArtifact art = to_artifact(a);
    std::vector<EvalReport> parts(nthreads > 1 ? nthreads : 1);
    std::vector<std::int64_t> nrows(parts.size(), 0);
    shard_rows(rows, nthreads, [&](std::int64_t r0, std::int64_t r1, int t) {
      parts[t] = eval_accuracy(spec, art, to_matrix(X + r0 * s->in_dim, r1 - r0, s->in_dim));  // metrics.cpp:30
      nrows[t] = r1 - r0;
    });
    // merge row shards (one shard: the reference's report unchanged)
    double sum_in = 0, sum_oob = 0, max_in = 0, max_oob = 0, oob_rows = 0;
    std::uint64_t n_in = 0, n_oob = 0, n_bd = 0;
    for (std::size_t t = 0; t < parts.size(); t++) {
      const EvalReport& r = parts[t];
      sum_in += r.mae_inrange * static_cast<double>(r.n_inrange_evals);
      n_in += r.n_inrange_evals;
      max_in = std::max(max_in, r.maxabs_inrange);
      if (r.mae_oob) {
        sum_oob += *r.mae_oob * static_cast<double>(r.n_oob_evals);
        max_oob = std::max(max_oob, *r.maxabs_oob);
      }
      n_oob += r.n_oob_evals;
      n_bd += r.n_boundary_evals;
      oob_rows += r.oob_any_frac * static_cast<double>(nrows[t]);
    }
    const EvalReport& r0 = parts[0];
    const bool one = parts.size() == 1;
    acc[0] = one ? r0.mae_inrange : (n_in ? sum_in / static_cast<double>(n_in) : 0.0);
    acc[1] = max_in;
    acc[2] = one ? r0.mae_oob.value_or(0.0) : (n_oob ? sum_oob / static_cast<double>(n_oob) : 0.0);
    acc[3] = n_oob ? max_oob : 0.0;
    acc[4] = one ? r0.oob_any_frac : (rows ? oob_rows / static_cast<double>(rows) : 0.0);
    acc[5] = r0.memory.overhead_ratio;
    *has_oob = n_oob > 0;
    const MemoryBreakdown& mb = r0.memory;
    const std::uint64_t c[11] = {n_in, n_oob, n_bd,
                                 static_cast<std::uint64_t>(acc[4] * static_cast<double>(rows) + 0.5),
                                 mb.q_table_bytes, mb.scale_bytes, mb.y_min_bytes, mb.knots_bytes,
                                 mb.edge_scalar_bytes, mb.total_bytes, mb.float_model_bytes};
    std::memcpy(counts, c, sizeof(c));
  });
}

int ork_coords(const ork_artifact* a, const double* x, int64_t n, uint8_t* in_range_out,
               double* x_clip, int32_t* k, int32_t* l0, int32_t* l1, double* w) {
  return guarded([&] {
    const LutLayerArtifact art = to_artifact(a);
    for (int64_t i = 0; i < n; i++) {
      const double xp = safe_clip(x[i], art.knots, art.oob.boundary_mode);  // runtime.cpp:45
      const int kk = segment_index(art.knots_f64, xp);                      // runtime.cpp:53
      const InterpCoords c = interp_coords(art.knots_f64, kk, xp, art.L);   // runtime.cpp:60
      if (in_range_out) in_range_out[i] = in_range(art, x[i]) ? 1 : 0;     // runtime.cpp:71
      if (x_clip) x_clip[i] = xp;
      if (k) k[i] = kk;
      if (l0) l0[i] = c.l0;
      if (l1) l1[i] = c.l1;
      if (w) w[i] = c.w;
    }
  });
}

int ork_eval_value(const ork_artifact* a, int32_t e, double x, double* value, int32_t* was_oob) {
  return guarded([&] {
    const ValueResult r = lut_eval_value(to_artifact(a), e, x);  // runtime.cpp:96-109
    *value = r.value;
    if (was_oob) *was_oob = r.was_oob;
  });
}

int ork_eval_phi(const ork_artifact* a, int32_t e, double x, double* value) {
  return guarded([&] { *value = lut_eval_phi(to_artifact(a), e, x); });  // runtime.cpp:111-120
}

int ork_basis_values(const double* bp, int32_t K, int32_t degree, double x, double* out) {
  return guarded([&] {
    KnotGrid g(std::vector<double>(bp, bp + K + 1), degree);
    const std::vector<double> b = basis_values(g, x);  // spline.cpp:89-94
    std::memcpy(out, b.data(), sizeof(double) * b.size());
  });
}

int ork_quantize_segment(const double* v, int32_t n, int32_t scheme, int32_t* q, double* scale,
                         double* y_min) {
  return guarded([&] {
    std::vector<double> vals(v, v + n);
    const SegmentQuant sq = scheme ? quantize_segment_asymmetric(vals)  // compiler.cpp:116
                                   : quantize_segment_symmetric(vals);  // compiler.cpp:105
    for (int i = 0; i < n; i++) q[i] = sq.q[i];
    *scale = sq.scale;
    *y_min = sq.y_min;
  });
}

uint16_t ork_f32_to_f16_bits(float f) { return f32_to_f16_bits(f); }
float ork_f16_bits_to_f32(uint16_t h) { return f16_bits_to_f32(h); }

void ork_rng_uniform(uint64_t seed, int64_t n, double* out) {
  Rng r(seed);
  for (int64_t i = 0; i < n; i++) out[i] = r.uniform();
}
void ork_rng_normal(uint64_t seed, int64_t n, double* out) {
  Rng r(seed);
  for (int64_t i = 0; i < n; i++) out[i] = r.normal();
}

// BASELINE config recipes, drawn with the reference Rng class.
namespace {
struct Recipe {
  int nl;
  int dims[5];
  int G;
  double lo, hi, sigma;
  std::uint64_t seed;
};
const Recipe kRecipes[5] = {
    {2, {2, 5, 1}, 5, -1.0, 1.0, 0.1, 0},
    {2, {78, 16, 2}, 5, -1.0, 1.0, 0.1, 1},
    {2, {64, 64, 1}, 8, -1.0, 1.0, 0.1, 2},
    {3, {1024, 1024, 1024, 10}, 8, -1.0, 1.0, 0.05, 3},
    {2, {4096, 4096, 4096}, 16, -2.0, 2.0, 0.02, 4},
};
}  // namespace

int ork_recipe_layer(int32_t cfg, int32_t layer, double* bp, double* coeffs, double* bs,
                     double* ss, double* os) {
  if (cfg < 1 || cfg > 5) {
    g_err = "unknown config";
    return 1;
  }
  const Recipe& r = kRecipes[cfg - 1];
  if (layer < 0 || layer >= r.nl) {
    g_err = "layer out of range";
    return 2;
  }
  for (int k = 0; k <= r.G; k++) bp[k] = r.lo + (r.hi - r.lo) * static_cast<double>(k) / r.G;
  const int R = r.G + 3;
  Rng g(r.seed);
  for (int l = 0; l <= layer; l++) {
    const std::int64_t E = static_cast<std::int64_t>(r.dims[l]) * r.dims[l + 1];
    for (std::int64_t e = 0; e < E; e++) {
      for (int q = 0; q < R; q++) {
        const double v = g.normal(0.0, r.sigma);
        if (l == layer) coeffs[e * R + q] = v;
      }
      const double b = g.uniform(-1.0, 1.0);
      if (l == layer) {
        bs[e] = b;
        ss[e] = 1.0;
        os[e] = 1.0;
      }
    }
  }
  return 0;
}

int ork_recipe_inputs(int32_t cfg, int64_t row0, int64_t rows, float* X) {
  if (cfg < 1 || cfg > 5) {
    g_err = "unknown config";
    return 1;
  }
  const Recipe& r = kRecipes[cfg - 1];
  Rng g(r.seed ^ 0x5eed5eed5eed5eedull);
  const std::int64_t d = r.dims[0], n0 = row0 * d, n1 = (row0 + rows) * d;
  for (std::int64_t n = 0; n < n1; n++) {
    double x;
    switch (cfg) {
      case 1: x = g.uniform(-1.2, 1.2); break;
      case 2:
        x = g.normal(0.0, 0.4);
        if (g.uniform() < 0.01) {
          const bool neg = g.uniform() < 0.5;
          const double mag = g.uniform(1.5, 4.0);
          x = neg ? -mag : mag;
        }
        break;
      case 3:
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
  return 0;
}

}  // extern "C"
