// shim_parity.cpp — the C++ drop-in shim (include/lutkan_b200.hpp) exercised against the
// UNMODIFIED reference library (oracle/_ref/liblutkan_ref.a, built in place from the reference
// sources), in the style of the reference's own tests (tests/test_runtime.cpp,
// tests/test_compiler.cpp). Built by oracle/Makefile (target `shim`) where /root/reference
// exists; run on the GPU box by tests/test_gpu_shim.py. Prints one line per check and exits
// non-zero on the first failure.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <iterator>
#include <string>
#include <thread>
#include <vector>

#include "lutkan/artifact_io.hpp"
#include "lutkan/compiler.hpp"
#include "lutkan/metrics.hpp"
#include "lutkan/model_gen.hpp"
#include "lutkan/runtime.hpp"
#include "lutkan/spline.hpp"
#include "lutkan_b200.hpp"

using namespace lutkan;

static int fails = 0;
#define CHECK(cond, what)                                    \
  do {                                                       \
    if (!(cond)) {                                           \
      std::printf("[FAIL] %s (%s:%d)\n", what, __FILE__, __LINE__); \
      fails++;                                               \
    } else {                                                 \
      std::printf("[PASS] %s\n", what);                      \
    }                                                        \
  } while (0)

static double max_err(const Matrix& a, const Matrix& b) {
  double m = 0;
  for (size_t i = 0; i < a.data.size(); i++) {
    const double d = std::fabs(a.data[i] - b.data[i]);
    const double tol = std::fabs(b.data[i]) > 1.0 ? 1e-5 * std::fabs(b.data[i]) : 1e-5;
    m = std::fmax(m, d / tol * 1e-5);
  }
  return m;
}

int main() {
  // compile parity: bytes identical to lutkan::compile_layer (test_compiler.cpp:269-281 style)
  for (Scheme sch : {Scheme::Symmetric, Scheme::Asymmetric}) {
    QuantConfig cfg;
    cfg.samples_per_segment = 32;
    cfg.scheme = sch;
    cfg.dtype = sch == Scheme::Symmetric ? Dtype::Int8 : Dtype::Uint8;
    const KanLayerSpec layer = gen_layer(11, 24, 12, 8, 3);
    const OobConfig oob{BoundaryMode::HalfOpen, OobPolicy::ZeroSpline};
    const LutLayerArtifact ref = lutkan::compile_layer(layer, cfg, oob);
    const LutLayerArtifact gpu = lutkan_b200::compile_layer(layer, cfg, oob);
    CHECK(ref.q_table == gpu.q_table && ref.scale == gpu.scale && ref.y_min == gpu.y_min &&
              ref.knots == gpu.knots && ref.edge_out_scale == gpu.edge_out_scale,
          sch == Scheme::Symmetric ? "compile_layer bytes (int8 symmetric)" : "compile_layer bytes (uint8 asymmetric)");
    // forward parity on seeded inputs that spill past the domain (test_runtime.cpp:328-344 style)
    const Matrix X = gen_inputs(53, 2000, 24, -1.3, 1.3, false);
    Matrix Xf = X;
    for (double& v : Xf.data) v = static_cast<double>(static_cast<float>(v));
    const auto [yr, sr] = lutkan::lut_layer_forward_batch(ref, Xf, Tier::Optimized);
    const auto [yg, sg] = lutkan_b200::lut_layer_forward_batch(gpu, Xf, Tier::Optimized);
    CHECK(max_err(yg, yr) <= 1e-5, "lut_layer_forward_batch within 1e-5");
    CHECK(sr.n_oob_inputs == sg.n_oob_inputs && sr.n_oob_samples == sg.n_oob_samples && sr.n_samples == sg.n_samples &&
              sr.n_inputs == sg.n_inputs,
          "OobStats identical");
    const Matrix ys_ref = lutkan::layer_forward_batch(layer, Xf, Tier::Optimized);
    const Matrix ys_gpu = lutkan_b200::layer_forward_batch(layer, Xf, Tier::Optimized);
    CHECK(max_err(ys_gpu, ys_ref) <= 1e-5, "layer_forward_batch (spline) within 1e-5");
  }
  // chains and their error behaviour (test_runtime.cpp:256-296 style)
  {
    QuantConfig cfg;
    const std::vector<KanLayerSpec> layers = {gen_layer(7, 10, 8, 8, 3), gen_layer(8, 8, 3, 8, 3)};
    const OobConfig oob{};
    const auto ref = lutkan::compile_model(layers, cfg, oob);
    const auto gpu = lutkan_b200::compile_model(layers, cfg, oob);
    const Matrix X = gen_inputs(9, 500, 10, -1.0, 1.0, true);
    Matrix Xf = X;
    for (double& v : Xf.data) v = static_cast<double>(static_cast<float>(v));
    const auto cr = lutkan::lut_model_forward_batch(ref, Xf, Tier::Optimized);
    const auto cg = lutkan_b200::lut_model_forward_batch(gpu, Xf, Tier::Optimized);
    int agree = 0;
    for (size_t r = 0; r < X.rows; r++) {
      int a = 0, b = 0;
      for (int j = 1; j < 3; j++) {
        if (cr.Y.at(r, j) > cr.Y.at(r, a)) a = j;
        if (cg.Y.at(r, j) > cg.Y.at(r, b)) b = j;
      }
      agree += a == b;
    }
    CHECK(agree == static_cast<int>(X.rows), "lut_model_forward_batch argmax classes identical");
    CHECK(cr.per_layer.size() == cg.per_layer.size() && cr.per_layer[0].n_oob_inputs == cg.per_layer[0].n_oob_inputs,
          "chain per-layer OobStats");
    bool threw = false;
    try {
      lutkan_b200::lut_model_forward_batch({}, Xf);
    } catch (const ConfigError&) {
      threw = true;
    }
    CHECK(threw, "empty chain -> ConfigError");
    threw = false;
    Matrix bad(1, 1);
    bad.at(0, 0) = NAN;
    try {
      lutkan_b200::lut_layer_forward_batch(gpu[0], Matrix(1, 3));
    } catch (const DimensionError&) {
      threw = true;
    }
    CHECK(threw, "column mismatch -> DimensionError");
    threw = false;
    Matrix nf(2, 10);
    nf.at(1, 4) = INFINITY;
    try {
      lutkan_b200::lut_layer_forward_batch(gpu[0], nf);
    } catch (const NonFiniteError&) {
      threw = true;
    }
    CHECK(threw, "non-finite input -> NonFiniteError");
  }
  // concurrency (test_spline.cpp:310-323 "batch forward is safe to call concurrently"):
  // 4 host threads call the three batch entry points at once through their default contexts;
  // every thread's results are bit-identical to a single-threaded call
  {
    QuantConfig cfg;
    const KanLayerSpec layer = gen_sanity_layer(5);
    const std::vector<KanLayerSpec> layers = {gen_layer(7, 10, 8, 8, 3), gen_layer(8, 8, 3, 8, 3)};
    const LutLayerArtifact art = lutkan::compile_layer(layer, cfg, OobConfig{});
    const auto chain = lutkan::compile_model(layers, cfg, OobConfig{});
    Matrix X = gen_inputs(43, 4099, 10, -1.2, 1.2, false);
    for (double& v : X.data) v = static_cast<double>(static_cast<float>(v));
    const auto want_l = lutkan_b200::lut_layer_forward_batch(art, X, Tier::Optimized);
    const auto want_m = lutkan_b200::lut_model_forward_batch(chain, X, Tier::Optimized);
    const Matrix want_s = lutkan_b200::layer_forward_batch(layer, X, Tier::Optimized);
    std::vector<int> ok(4, 0);
    std::vector<std::thread> ts;
    for (int t = 0; t < 4; ++t)
      ts.emplace_back([&, t] {
        int good = 1;
        for (int it = 0; it < 25; it++) {  // interleave many calls per thread
          const auto l = lutkan_b200::lut_layer_forward_batch(art, X, Tier::Optimized);
          const auto m = lutkan_b200::lut_model_forward_batch(chain, X, Tier::Optimized);
          const Matrix sp = lutkan_b200::layer_forward_batch(layer, X, Tier::Optimized);
          good &= l.first.data == want_l.first.data && l.second.n_oob_inputs == want_l.second.n_oob_inputs &&
                  l.second.n_oob_samples == want_l.second.n_oob_samples && l.second.n_samples == want_l.second.n_samples;
          good &= m.Y.data == want_m.Y.data && m.per_layer.size() == want_m.per_layer.size() &&
                  m.per_layer[0].n_oob_inputs == want_m.per_layer[0].n_oob_inputs &&
                  m.per_layer[1].n_oob_inputs == want_m.per_layer[1].n_oob_inputs;
          good &= sp.data == want_s.data;
        }
        ok[t] = good;
      });
    for (auto& t : ts) t.join();
    CHECK(ok[0] && ok[1] && ok[2] && ok[3],
          "4 threads x (lut_layer_forward_batch, lut_model_forward_batch, layer_forward_batch): bit-identical");
  }
  // eval_accuracy and the artifact container through the shim
  {
    QuantConfig cfg;
    cfg.samples_per_segment = 16;
    const KanLayerSpec layer = gen_layer(7, 9, 6, 5, 3);
    const OobConfig oob{BoundaryMode::Closed, OobPolicy::ClipX};
    const LutLayerArtifact art = lutkan::compile_layer(layer, cfg, oob);
    Matrix X = gen_inputs(19, 500, 9, -1.4, 1.4, false);
    for (double& v : X.data) v = static_cast<double>(static_cast<float>(v));
    const EvalReport er = lutkan::eval_accuracy(layer, art, X);
    const EvalReport eg = lutkan_b200::eval_accuracy(layer, art, X);
    CHECK(er.n_inrange_evals == eg.n_inrange_evals && er.n_oob_evals == eg.n_oob_evals &&
              er.n_boundary_evals == eg.n_boundary_evals && er.oob_any_frac == eg.oob_any_frac &&
              er.mae_oob.has_value() == eg.mae_oob.has_value(),
          "eval_accuracy buckets and counts identical");
    CHECK(std::fabs(er.mae_inrange - eg.mae_inrange) <= 1e-12 * er.mae_inrange &&
              std::fabs(er.maxabs_inrange - eg.maxabs_inrange) <= 1e-15 + 1e-12 * er.maxabs_inrange &&
              er.memory.total_bytes == eg.memory.total_bytes,
          "eval_accuracy errors agree (f64)");
    lutkan::save_artifact(art, "/tmp/shim_ref.lut");
    lutkan_b200::save_artifact(art, "/tmp/shim_gpu.lut");
    auto slurp = [](const char* p) {
      std::ifstream f(p, std::ios::binary);
      return std::string((std::istreambuf_iterator<char>(f)), std::istreambuf_iterator<char>());
    };
    CHECK(slurp("/tmp/shim_ref.lut") == slurp("/tmp/shim_gpu.lut"), "save_artifact bytes identical");
    const LutLayerArtifact back = lutkan_b200::load_artifact("/tmp/shim_ref.lut");
    const LutLayerArtifact back_ref = lutkan::load_artifact("/tmp/shim_ref.lut");
    CHECK(back.q_table == back_ref.q_table && back.scale == back_ref.scale && back.knots == back_ref.knots &&
              back.edge_base_scale == back_ref.edge_base_scale && back.base_kind == back_ref.base_kind,
          "load_artifact fields identical");
    {
      std::ofstream f("/tmp/shim_bad.lut", std::ios::binary);
      const std::string raw = slurp("/tmp/shim_ref.lut");
      f << raw.substr(0, raw.size() / 2);
    }
    bool threw = false;
    try {
      lutkan_b200::load_artifact("/tmp/shim_bad.lut");
    } catch (const CorruptArchiveError&) {
      threw = true;
    }
    CHECK(threw, "truncated archive -> CorruptArchiveError");
  }
  std::printf("%s: %d failure(s)\n", fails ? "FAILED" : "OK", fails);
  return fails ? 1 : 0;
}
