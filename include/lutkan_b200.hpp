// lutkan_b200.hpp — header-only C++ shim that re-exposes the reference hot-path signatures
// (namespace lutkan, /root/reference/proj/core/include/lutkan) on top of the C-ABI in
// lutkan_b200.h. Include it AFTER the reference headers; every function takes and returns the
// reference's own types and throws the reference's own exceptions, so a call site switches
// backend by changing the namespace:
//
//   lutkan::lut_layer_forward_batch(a, X, tier)   ->  lutkan_b200::lut_layer_forward_batch(a, X, tier)
//   lutkan::lut_model_forward_batch(chain, X, t)  ->  lutkan_b200::lut_model_forward_batch(chain, X, t)
//   lutkan::compile_layer(spec, qc, oob)          ->  lutkan_b200::compile_layer(spec, qc, oob)
//   lutkan::layer_forward_batch(spec, X, tier)    ->  lutkan_b200::layer_forward_batch(spec, X, tier)
//   lutkan::eval_accuracy(spec, a, X)             ->  lutkan_b200::eval_accuracy(spec, a, X)
//   lutkan::save_artifact(a, path)                ->  lutkan_b200::save_artifact(a, path)
//   lutkan::load_artifact(path)                   ->  lutkan_b200::load_artifact(path)
//
// Documented differences: activations cross to the device as fp32 (results are widened back to
// f64 in the returned Matrix); Tier is accepted and ignored (one backend, no CPU fallback).
// Device copies of artifacts are cached per Artifact address for the lifetime of the Context;
// every host thread has its own default Context, so concurrent calls are safe as in the reference.
#pragma once

#include <cstdint>
#include <cstring>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "lutkan/artifact_io.hpp"
#include "lutkan/compiler.hpp"
#include "lutkan/metrics.hpp"
#include "lutkan/runtime.hpp"
#include "lutkan/spline.hpp"
#include "lutkan_b200.h"

namespace lutkan_b200 {

// Map a C-ABI status to the reference exception taxonomy (types.hpp:11-39).
inline void check(lkg_status st) {
  if (st == LKG_OK) return;
  const std::string msg = lkg_last_error();
  switch (st) {
    case LKG_ERR_CONFIG: throw lutkan::ConfigError(msg);
    case LKG_ERR_DIMENSION: throw lutkan::DimensionError(msg);
    case LKG_ERR_NON_FINITE: throw lutkan::NonFiniteError(msg);
    case LKG_ERR_UNSUPPORTED_BASE: throw lutkan::UnsupportedBaseError(msg);
    case LKG_ERR_IO: throw lutkan::IoError(msg);  // artifact_io.hpp:11-52
    case LKG_ERR_CORRUPT_ARCHIVE: throw lutkan::CorruptArchiveError(msg);
    case LKG_ERR_CORRUPT_BLOB: throw lutkan::CorruptBlobError(msg);
    case LKG_ERR_MISSING_KEY: throw lutkan::MissingKeyError(msg);
    case LKG_ERR_SHAPE: throw lutkan::ShapeError(msg);
    case LKG_ERR_VERSION: throw lutkan::VersionError(msg);
    case LKG_ERR_ENUM: throw lutkan::EnumError(msg);
    default: throw lutkan::Error("lutkan_b200: " + msg);
  }
}

// One CUDA context (device + stream) and its device-resident artifacts. Not thread-safe: one
// Context per host thread (default_context() is thread_local).
class Context {
 public:
  explicit Context(int device = 0) { check(lkg_ctx_create(device, nullptr, &ctx_)); }
  ~Context() {
    for (auto& kv : layers_) lkg_layer_free(kv.second);
    for (auto& kv : specs_) lkg_spec_free(kv.second);
    lkg_ctx_destroy(ctx_);
  }
  Context(const Context&) = delete;
  Context& operator=(const Context&) = delete;
  lkg_ctx* get() const { return ctx_; }

  // LutLayerArtifact (runtime.hpp:31-63) -> device layer (validated like finalize()). The cache
  // key is the artifact's address plus a fingerprint of its buffers (heap addresses, sizes and a
  // sample of the bytes), so a different artifact that reuses the address is re-uploaded.
  const lkg_layer* layer(const lutkan::LutLayerArtifact& a) {
    const uint64_t fp = fingerprint(a);
    auto it = layers_.find(&a);
    if (it != layers_.end()) {
      if (layer_fp_[&a] == fp) return it->second;
      lkg_layer_free(it->second);
      layers_.erase(it);
    }
    layer_fp_[&a] = fp;
    const lkg_layer_desc d = desc(a);
    lkg_layer* out = nullptr;
    check(lkg_layer_upload(ctx_, &d, &out));
    layers_[&a] = out;
    return out;
  }

  // The artifact's arrays as a C-ABI descriptor (host pointers into `a`).
  static lkg_layer_desc desc(const lutkan::LutLayerArtifact& a) {
    lkg_layer_desc d{};
    d.in_dim = a.in_dim;
    d.out_dim = a.out_dim;
    d.K = static_cast<int32_t>(a.knots.size()) - 1;
    d.L = a.L;
    d.value_repr = static_cast<int32_t>(a.value_repr);
    d.interp = static_cast<int32_t>(a.interp);
    d.scheme = static_cast<int32_t>(a.scheme);
    d.dtype = static_cast<int32_t>(a.dtype);
    d.param_dtype = static_cast<int32_t>(a.param_dtype);
    d.boundary_mode = static_cast<int32_t>(a.oob.boundary_mode);
    d.oob_policy = static_cast<int32_t>(a.oob.oob_policy);
    d.base_kind = a.base_kind.c_str();
    const size_t E = static_cast<size_t>(a.in_dim) * a.out_dim, K = a.knots.size() - 1;
    if (a.q_table.size() != E * K * a.L) throw lutkan::DimensionError("q_table size does not match [E, K, L]");
    if (a.scale.size() != E * K) throw lutkan::DimensionError("scale size does not match [E, K]");
    if (a.y_min.size() != E * K) throw lutkan::DimensionError("y_min size does not match [E, K]");
    d.knots = a.knots.data();
    d.q_table = a.q_table.data();
    d.scale = a.scale.data();
    d.y_min = a.y_min.data();
    d.edge_base_scale = a.edge_base_scale.empty() ? nullptr : a.edge_base_scale.data();
    d.edge_spline_scale = a.edge_spline_scale.empty() ? nullptr : a.edge_spline_scale.data();
    d.edge_out_scale = a.edge_out_scale.empty() ? nullptr : a.edge_out_scale.data();
    d.float_table = a.float_table.empty() ? nullptr : a.float_table.data();
    return d;
  }

  // KanLayerSpec (spline.hpp:35-74) -> device spec (same keying as layer()).
  const lkg_spec* spec(const lutkan::KanLayerSpec& s) {
    const uint64_t fp = fingerprint(s);
    auto it = specs_.find(&s);
    if (it != specs_.end()) {
      if (spec_fp_[&s] == fp) return it->second;
      lkg_spec_free(it->second);
      specs_.erase(it);
    }
    spec_fp_[&s] = fp;
    lkg_spec_desc d{};
    d.in_dim = s.in_dim();
    d.out_dim = s.out_dim();
    d.K = s.grid().segment_count();
    d.degree = s.grid().degree();
    d.base_kind = s.base_kind().c_str();
    d.breakpoints = s.grid().breakpoints().data();
    d.coeffs = s.packed_coeffs().data();
    d.base_scale = s.base_scales().data();
    d.spline_scale = s.spline_scales().data();
    d.out_scale = s.out_scales().data();
    lkg_spec* out = nullptr;
    check(lkg_spec_upload(ctx_, &d, &out));
    specs_[&s] = out;
    return out;
  }

  void forget(const lutkan::LutLayerArtifact& a) {
    auto it = layers_.find(&a);
    if (it != layers_.end()) {
      lkg_layer_free(it->second);
      layers_.erase(it);
    }
  }

 private:
  static uint64_t mix(uint64_t h, uint64_t v) { return (h ^ v) * 0x100000001b3ull; }
  template <class V>
  static uint64_t sample(uint64_t h, const V& v) {
    h = mix(h, reinterpret_cast<uintptr_t>(v.data()));
    h = mix(h, v.size());
    const size_t n = v.size(), step = n > 256 ? n / 256 : 1;
    for (size_t i = 0; i < n; i += step) {
      uint64_t bits = 0;
      std::memcpy(&bits, &v[i], sizeof(v[i]) < 8 ? sizeof(v[i]) : 8);
      h = mix(h, bits);
    }
    return h;
  }
  static uint64_t fingerprint(const lutkan::LutLayerArtifact& a) {
    uint64_t h = 0xcbf29ce484222325ull;
    h = mix(h, (uint64_t)a.in_dim << 32 | (uint32_t)a.out_dim);
    h = mix(h, (uint64_t)a.L << 32 | ((uint32_t)a.scheme << 8) | ((uint32_t)a.value_repr << 4) |
                   ((uint32_t)a.oob.boundary_mode << 2) | (uint32_t)a.oob.oob_policy);
    h = sample(sample(sample(sample(h, a.knots), a.q_table), a.scale), a.y_min);
    h = sample(sample(sample(h, a.edge_base_scale), a.edge_spline_scale), a.edge_out_scale);
    return sample(h, a.float_table);
  }
  static uint64_t fingerprint(const lutkan::KanLayerSpec& s) {
    uint64_t h = mix(0xcbf29ce484222325ull, (uint64_t)s.in_dim() << 32 | (uint32_t)s.out_dim());
    h = sample(sample(h, s.grid().breakpoints()), s.packed_coeffs());
    return sample(sample(sample(h, s.base_scales()), s.spline_scales()), s.out_scales());
  }

  lkg_ctx* ctx_ = nullptr;
  std::map<const void*, lkg_layer*> layers_;
  std::map<const void*, lkg_spec*> specs_;
  std::map<const void*, uint64_t> layer_fp_, spec_fp_;
};

// The default context is PER HOST THREAD: a Context (one lkg_ctx: stream, scratch buffers, OOB
// counters, artifact cache) must never be driven by two threads at once (lutkan_b200.h threading
// contract), so each thread calling the reference-signature functions below gets its own. That
// keeps the reference's guarantee that these functions are pure and safe to call concurrently
// (test_spline.cpp:310-323). A thread's context and its device copies of the
// artifacts it used are released when the thread exits.
inline Context& default_context() {
  static thread_local Context ctx(0);
  return ctx;
}

inline lutkan::OobStats to_stats(const lkg_oob_stats& s) {
  lutkan::OobStats o;
  o.n_samples = s.n_samples;
  o.n_oob_samples = s.n_oob_samples;
  o.n_inputs = s.n_inputs;
  o.n_oob_inputs = s.n_oob_inputs;
  return o;
}

// lut_model_forward_batch (runtime.cpp:298-314).
inline lutkan::ChainBatchResult lut_model_forward_batch(const std::vector<lutkan::LutLayerArtifact>& chain,
                                                        const lutkan::Matrix& X,
                                                        lutkan::Tier = lutkan::Tier::Optimized,
                                                        Context& ctx = default_context()) {
  if (chain.empty()) throw lutkan::ConfigError("artifact chain is empty");
  if (X.cols != static_cast<size_t>(chain.front().in_dim))
    throw lutkan::DimensionError("batch column count does not match artifact in_dim");
  std::vector<const lkg_layer*> dev;
  for (const auto& a : chain) dev.push_back(ctx.layer(a));
  const size_t m = static_cast<size_t>(chain.back().out_dim);
  std::vector<lkg_oob_stats> st(chain.size());
  lutkan::ChainBatchResult r;
  r.Y = lutkan::Matrix(X.rows, m);
  // the f64 rows go to the device as they are and are narrowed there (documented: fp32 activations
  // on the device), the fp32 outputs widened there
  check(lkg_model_forward_host_f64(ctx.get(), dev.data(), static_cast<int32_t>(dev.size()), X.data.data(),
                                   static_cast<int64_t>(X.rows), r.Y.data.data(), st.data()));
  for (const auto& s : st) r.per_layer.push_back(to_stats(s));
  return r;
}

// lut_layer_forward_batch (runtime.cpp:250-285).
inline std::pair<lutkan::Matrix, lutkan::OobStats> lut_layer_forward_batch(
    const lutkan::LutLayerArtifact& a, const lutkan::Matrix& X, lutkan::Tier tier = lutkan::Tier::Optimized,
    Context& ctx = default_context()) {
  if (X.cols != static_cast<size_t>(a.in_dim))
    throw lutkan::DimensionError("batch column count does not match artifact in_dim");
  const lkg_layer* dev = ctx.layer(a);
  lkg_oob_stats st{};
  (void)tier;
  lutkan::Matrix Y(X.rows, static_cast<size_t>(a.out_dim));
  check(lkg_model_forward_host_f64(ctx.get(), &dev, 1, X.data.data(), static_cast<int64_t>(X.rows), Y.data.data(),
                                   &st));
  return {std::move(Y), to_stats(st)};
}

// compile_layer / compile_layer_debug_float (compiler.cpp:213-233): bytes bit-exact with the
// reference; the returned artifact is downloaded and finalized like the reference's.
inline lutkan::LutLayerArtifact compile_layer(const lutkan::KanLayerSpec& spec, const lutkan::QuantConfig& cfg,
                                              const lutkan::OobConfig& oob, bool keep_float = false,
                                              Context& ctx = default_context()) {
  cfg.validate();
  lkg_quant_config qc{cfg.samples_per_segment, static_cast<int32_t>(cfg.scheme), static_cast<int32_t>(cfg.dtype),
                      static_cast<int32_t>(cfg.value_repr), static_cast<int32_t>(cfg.interp),
                      static_cast<int32_t>(cfg.param_dtype)};
  lkg_oob_config oc{static_cast<int32_t>(oob.boundary_mode), static_cast<int32_t>(oob.oob_policy)};
  lkg_layer* dev = nullptr;
  check(lkg_compile_layer(ctx.get(), ctx.spec(spec), &qc, &oc, keep_float ? 1 : 0, &dev));
  std::unique_ptr<lkg_layer, lkg_status (*)(lkg_layer*)> guard(dev, lkg_layer_free);
  lkg_layer_info info{};
  check(lkg_layer_info_get(dev, &info));
  lutkan::LutLayerArtifact a;
  a.in_dim = info.in_dim;
  a.out_dim = info.out_dim;
  a.L = info.L;
  a.value_repr = cfg.value_repr;
  a.interp = cfg.interp;
  a.scheme = cfg.scheme;
  a.dtype = cfg.dtype;
  a.param_dtype = cfg.param_dtype;
  a.oob = oob;
  a.base_kind = cfg.value_repr == lutkan::ValueRepr::SplineComponent ? spec.base_kind() : "";
  const size_t E = static_cast<size_t>(info.in_dim) * info.out_dim, K = info.K;
  a.knots.resize(K + 1);
  a.q_table.resize(E * K * a.L);
  a.scale.resize(E * K);
  a.y_min.resize(E * K);
  const bool sr = cfg.value_repr == lutkan::ValueRepr::SplineComponent;
  if (sr) {
    a.edge_base_scale.resize(E);
    a.edge_spline_scale.resize(E);
    a.edge_out_scale.resize(E);
  }
  if (keep_float) a.float_table.resize(E * K * a.L);
  check(lkg_layer_download(ctx.get(), dev, a.knots.data(), a.q_table.data(), a.scale.data(), a.y_min.data(),
                           sr ? a.edge_base_scale.data() : nullptr, sr ? a.edge_spline_scale.data() : nullptr,
                           sr ? a.edge_out_scale.data() : nullptr, keep_float ? a.float_table.data() : nullptr));
  a.finalize();
  return a;
}

inline std::vector<lutkan::LutLayerArtifact> compile_model(const std::vector<lutkan::KanLayerSpec>& layers,
                                                           const lutkan::QuantConfig& cfg,
                                                           const lutkan::OobConfig& oob,
                                                           Context& ctx = default_context()) {
  if (layers.empty()) throw lutkan::ConfigError("model has no layers");
  for (size_t l = 1; l < layers.size(); l++)
    if (layers[l].in_dim() != layers[l - 1].out_dim())
      throw lutkan::DimensionError("layer shapes do not chain at position " + std::to_string(l));
  std::vector<lutkan::LutLayerArtifact> out;
  for (const auto& s : layers) out.push_back(compile_layer(s, cfg, oob, false, ctx));
  return out;
}

// layer_forward_batch (spline.cpp:183-187) — the same-backend B-spline baseline.
inline lutkan::Matrix layer_forward_batch(const lutkan::KanLayerSpec& spec, const lutkan::Matrix& X,
                                          lutkan::Tier = lutkan::Tier::Optimized,
                                          Context& ctx = default_context()) {
  if (X.cols != static_cast<size_t>(spec.in_dim()))
    throw lutkan::DimensionError("batch column count does not match in_dim");
  std::vector<float> x(X.data.begin(), X.data.end());
  std::vector<float> y(X.rows * static_cast<size_t>(spec.out_dim()));
  check(lkg_spline_forward_host(ctx.get(), ctx.spec(spec), x.data(), static_cast<int64_t>(X.rows), y.data()));
  lutkan::Matrix Y(X.rows, static_cast<size_t>(spec.out_dim()));
  for (size_t i = 0; i < y.size(); i++) Y.data[i] = y[i];
  return Y;
}

// eval_accuracy (metrics.cpp:30-103) on the GPU (f64, the reference's expressions); memory
// accounting by the reference's own memory_breakdown.
inline lutkan::EvalReport eval_accuracy(const lutkan::KanLayerSpec& layer, const lutkan::LutLayerArtifact& a,
                                        const lutkan::Matrix& X, Context& ctx = default_context()) {
  if (layer.in_dim() != a.in_dim || layer.out_dim() != a.out_dim)
    throw lutkan::DimensionError("layer and artifact shapes differ");
  if (X.cols != static_cast<size_t>(layer.in_dim()))
    throw lutkan::DimensionError("input column count does not match in_dim");
  lkg_eval_report r{};  // the Matrix's f64 values, unrounded (eval_accuracy is not a hot path)
  check(lkg_eval_accuracy_host_f64(ctx.get(), ctx.spec(layer), ctx.layer(a), X.data.data(),
                                   static_cast<int64_t>(X.rows), &r));
  lutkan::EvalReport e;
  e.quant.samples_per_segment = a.L;
  e.quant.scheme = a.scheme;
  e.quant.dtype = a.dtype;
  e.quant.value_repr = a.value_repr;
  e.quant.interp = a.interp;
  e.quant.param_dtype = a.param_dtype;
  e.oob = a.oob;
  e.n_samples = X.rows;
  e.mae_inrange = r.mae_inrange;
  e.maxabs_inrange = r.maxabs_inrange;
  if (r.has_oob) {
    e.mae_oob = r.mae_oob;
    e.maxabs_oob = r.maxabs_oob;
  }
  e.oob_any_frac = r.oob_any_frac;
  e.n_inrange_evals = r.n_inrange_evals;
  e.n_oob_evals = r.n_oob_evals;
  e.n_boundary_evals = r.n_boundary_evals;
  e.memory = lutkan::memory_breakdown(a, layer);
  return e;
}

// save_artifact (artifact_io.cpp:206-219): byte-identical archive.
inline void save_artifact(const lutkan::LutLayerArtifact& a, const std::string& path) {
  const lkg_layer_desc d = Context::desc(a);
  check(lkg_artifact_save_desc(&d, path.c_str(), 0));
}

// load_artifact (artifact_io.cpp:221-300): parsed, checked and uploaded by the engine (the
// device copy is what forwards use); the reference's host artifact is returned, finalized.
inline lutkan::LutLayerArtifact load_artifact(const std::string& path, Context& ctx = default_context()) {
  lkg_layer* dev = nullptr;
  check(lkg_artifact_load(ctx.get(), path.c_str(), &dev));
  std::unique_ptr<lkg_layer, lkg_status (*)(lkg_layer*)> guard(dev, lkg_layer_free);
  lkg_layer_info info{};
  check(lkg_layer_info_get(dev, &info));
  lutkan::LutLayerArtifact a;
  a.in_dim = info.in_dim;
  a.out_dim = info.out_dim;
  a.L = info.L;
  a.value_repr = static_cast<lutkan::ValueRepr>(info.value_repr);
  a.scheme = static_cast<lutkan::Scheme>(info.scheme);
  a.dtype = info.scheme ? lutkan::Dtype::Uint8 : lutkan::Dtype::Int8;
  a.param_dtype = static_cast<lutkan::ParamDtype>(info.param_dtype);
  a.oob.boundary_mode = static_cast<lutkan::BoundaryMode>(info.boundary_mode);
  a.oob.oob_policy = static_cast<lutkan::OobPolicy>(info.oob_policy);
  const bool sr = a.value_repr == lutkan::ValueRepr::SplineComponent;
  a.base_kind = lkg_layer_base_kind(dev);
  const size_t E = static_cast<size_t>(info.in_dim) * info.out_dim, K = info.K;
  a.knots.resize(K + 1);
  a.q_table.resize(E * K * a.L);
  a.scale.resize(E * K);
  a.y_min.resize(E * K);
  if (sr) {
    a.edge_base_scale.resize(E);
    a.edge_spline_scale.resize(E);
    a.edge_out_scale.resize(E);
  }
  check(lkg_layer_download(ctx.get(), dev, a.knots.data(), a.q_table.data(), a.scale.data(), a.y_min.data(),
                           sr ? a.edge_base_scale.data() : nullptr, sr ? a.edge_spline_scale.data() : nullptr,
                           sr ? a.edge_out_scale.data() : nullptr, nullptr));
  a.finalize();
  return a;
}

}  // namespace lutkan_b200
