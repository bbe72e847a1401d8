// shim_e2e.cpp — end-to-end timing of the path a reference caller takes: configs[1] ("C2", the
// BASELINE recipe layers [78,16,2], int8 symmetric, closed + clip_x) compiled through
// lutkan_b200::compile_model and evaluated with lutkan_b200::lut_model_forward_batch on a
// reference lutkan::Matrix of f64 rows (include/lutkan_b200.hpp: f64 rows to the device, narrowed and
// widened there). Prints one JSON object: edge-evals/s per step, host wall clock, after warm-up.
// Built by oracle/Makefile (target `shim`, needs the reference headers); run by bench.py.
//   shim_e2e [rows] [steps] [warmup]
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "lutkan/compiler.hpp"
#include "lutkan/runtime.hpp"
#include "lutkan/spline.hpp"
#include "lutkan_b200.hpp"

using namespace lutkan;

static KanLayerSpec recipe_spec(int cfg, int layer) {
  int32_t nl = 0, dims[8] = {}, G = 0;
  double lo = 0, hi = 0;
  lutkan_b200::check(lkg_recipe_dims(cfg, &nl, dims, &G, &lo, &hi));
  const int d = dims[layer], m = dims[layer + 1], R = G + 3, E = d * m;
  std::vector<double> bp(G + 1), co((size_t)E * R), bs(E), ss(E), os(E);
  lutkan_b200::check(lkg_recipe_layer(cfg, layer, 0, 0, bp.data(), co.data(), bs.data(), ss.data(), os.data()));
  std::vector<EdgeParams> edges(E);
  for (int e = 0; e < E; e++) {
    edges[e].coeffs.assign(co.begin() + (size_t)e * R, co.begin() + (size_t)(e + 1) * R);
    edges[e].base_scale = bs[e];
    edges[e].spline_scale = ss[e];
    edges[e].out_scale = os[e];
  }
  return KanLayerSpec(d, m, KnotGrid(bp, 3), "silu", edges);
}

int main(int argc, char** argv) {
  const long rows = argc > 1 ? atol(argv[1]) : 1000000;
  const int steps = argc > 2 ? atoi(argv[2]) : 10, warmup = argc > 3 ? atoi(argv[3]) : 3;
  const std::vector<KanLayerSpec> specs = {recipe_spec(2, 0), recipe_spec(2, 1)};
  QuantConfig cfg;  // L = 64, int8 symmetric (the defaults)
  const OobConfig oob{BoundaryMode::Closed, OobPolicy::ClipX};
  const auto chain = lutkan_b200::compile_model(specs, cfg, oob);
  std::vector<float> xf((size_t)rows * 78);
  lutkan_b200::check(lkg_recipe_inputs(2, 0, rows, xf.data()));
  Matrix X(rows, 78);
  for (size_t i = 0; i < xf.size(); i++) X.data[i] = xf[i];
  for (int w = 0; w < warmup; w++) lutkan_b200::lut_model_forward_batch(chain, X, Tier::Optimized);
  double best = 1e30, sum = 0;
  for (int s = 0; s < steps; s++) {
    const auto t0 = std::chrono::steady_clock::now();
    const auto r = lutkan_b200::lut_model_forward_batch(chain, X, Tier::Optimized);
    const double sec = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    sum += sec;
    best = sec < best ? sec : best;
    if (r.Y.rows != (size_t)rows) return 1;
  }
  const double ee = (double)rows * (78 * 16 + 16 * 2), mean = sum / steps;
  // PCIe bytes: the fp32 rows (narrowed on the host) and the fp32 outputs; the caller's f64 Matrix
  // is what the host threads read and write
  std::printf("{\"value\": %.6e, \"unit\": \"edge-evals/s\", \"ms_per_step\": %.4f, \"best_ms\": %.4f, "
              "\"rows\": %ld, \"steps\": %d, \"h2d_bytes_per_step\": %ld, \"d2h_bytes_per_step\": %ld, "
              "\"host_f64_bytes_per_step\": %ld}\n",
              ee / mean, mean * 1e3, best * 1e3, rows, steps, rows * 78 * 4, rows * 2 * 4, rows * (78 + 2) * 8);
  return 0;
}
