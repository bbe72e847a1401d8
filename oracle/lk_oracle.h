/*
 * lk_oracle.h — C-ABI of the CPU ORACLE for the LUT-KAN hot path.
 *
 * TEST INFRASTRUCTURE ONLY. Two libraries export exactly this interface:
 *   oracle/liblk_oracle.so        plain-C restatement of the reference (lk_oracle.c)
 *   oracle/_ref/liblutkan_ref.so  the reference's own C++ sources built in place
 *                                 (oracle/Makefile) behind an adapter (ref_capi.cpp)
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference legs may load either one, and only as the checker or the timed CPU
 * baseline. The product (paper_2601_03332_b200/) never links or calls them.
 *
 * Enum values follow the declaration order in proj/core/include/lutkan/types.hpp:41-49
 * and are identical to the product's lkg_* enums (include/lutkan_b200.h).
 * Status codes: 0 ok, 1 ConfigError, 2 DimensionError, 3 NonFiniteError,
 * 4 UnsupportedBaseError (types.hpp:11-39).
 */
#ifndef LK_ORACLE_H
#define LK_ORACLE_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

/* KanLayerSpec (proj/core/include/lutkan/spline.hpp:35-74) as plain arrays.
 * Edges are input-major: e = i*out_dim + j (spline.hpp:43). R = K + degree. */
typedef struct {
  int32_t in_dim, out_dim, K, degree;
  const double* breakpoints;   /* [K+1] */
  const double* coeffs;        /* [E*R] packed_coeffs (spline.hpp:57-62) */
  const double* base_scale;    /* [E] */
  const double* spline_scale;  /* [E] */
  const double* out_scale;     /* [E] */
} ork_spec;

/* LutLayerArtifact (proj/core/include/lutkan/runtime.hpp:31-63) as plain arrays.
 * dtype is implied by scheme (symmetric<->int8, asymmetric<->uint8, runtime.cpp:19-22). */
typedef struct {
  int32_t in_dim, out_dim, K, L;
  int32_t value_repr;     /* 0 phi, 1 spline_component */
  int32_t scheme;         /* 0 symmetric(int8), 1 asymmetric(uint8) */
  int32_t param_dtype;    /* 0 f32, 1 f16 */
  int32_t boundary_mode;  /* 0 half_open, 1 closed */
  int32_t oob_policy;     /* 0 clip_x, 1 zero_spline */
  const float* knots;     /* [K+1] */
  const uint8_t* q;       /* [E*K*L] */
  const float* scale;     /* [E*K] */
  const float* y_min;     /* [E*K] */
  const float* base_scale;   /* [E] or NULL (phi) */
  const float* spline_scale; /* [E] or NULL */
  const float* out_scale;    /* [E] or NULL */
  const double* float_table; /* [E*K*L] or NULL (debug artifacts) */
} ork_artifact;

const char* ork_last_error(void);
const char* ork_impl_name(void); /* "port" or "reference" */

/* compile_layer / compile_layer_debug_float (compiler.cpp:132-233).
 * Outputs are caller-allocated; gains/float_table may be NULL when not wanted. */
int ork_compile_layer(const ork_spec* spec, int32_t L, int32_t scheme, int32_t value_repr,
                      int32_t param_dtype, int32_t boundary_mode, int32_t oob_policy,
                      float* knots, uint8_t* q, float* scale, float* y_min,
                      float* base_scale, float* spline_scale, float* out_scale,
                      double* float_table);

/* lut_layer_forward_batch (runtime.cpp:250-285); tier 0 scalar, 1 optimized.
 * stats = {n_samples, n_oob_samples, n_inputs, n_oob_inputs} (runtime.hpp:105-120).
 * nthreads > 1 shards rows across std::threads / pthreads (pure functions). */
int ork_lut_forward(const ork_artifact* a, const double* X, int64_t rows, int32_t tier,
                    int32_t nthreads, double* Y, uint64_t* stats);

/* lut_model_forward_batch (runtime.cpp:298-314); stats is [n_layers][4]. */
int ork_lut_model_forward(const ork_artifact* chain, int32_t n_layers, const double* X,
                          int64_t rows, int32_t tier, int32_t nthreads, double* Y,
                          uint64_t* stats);

/* layer_forward_batch (spline.cpp:183-187). */
int ork_spline_forward(const ork_spec* spec, const double* X, int64_t rows, int32_t tier,
                       int32_t nthreads, double* Y);

/* Per-element primitives (runtime.cpp:45-75): in-range flag, clipped x, segment,
 * interpolation coordinates, as the scalar tier computes them. */
int ork_coords(const ork_artifact* a, const double* x, int64_t n, uint8_t* in_range,
               double* x_clip, int32_t* k, int32_t* l0, int32_t* l1, double* w);

/* lut_eval_value / lut_eval_phi (runtime.cpp:96-120). */
int ork_eval_value(const ork_artifact* a, int32_t e, double x, double* value, int32_t* was_oob);
int ork_eval_phi(const ork_artifact* a, int32_t e, double x, double* value);

/* Artifact container (artifact_io.cpp:206-300). REFERENCE LIBRARY ONLY: the port returns 99
 * (its pin is the .lut fixtures under tests/golden/artifacts, written by the reference). Status codes 9..15 follow the
 * IoError family as numbered in include/lutkan_b200.h. load_resave loads path and, when
 * resave_path != NULL, saves the loaded artifact again (a byte-level round trip). */
int ork_artifact_save(const ork_artifact* a, const char* path);
int ork_artifact_load_resave(const char* path, const char* resave_path);

/* eval_accuracy + memory_breakdown (metrics.cpp:8-103).
 * acc    = {mae_inrange, maxabs_inrange, mae_oob, maxabs_oob, oob_any_frac, overhead_ratio}
 * counts = {n_inrange_evals, n_oob_evals, n_boundary_evals, n_oob_samples, q_table_bytes,
 *           scale_bytes, y_min_bytes, knots_bytes, edge_scalar_bytes, total_bytes, float_model_bytes}
 * *has_oob = 1 when the OOB bucket is non-empty (mae_oob/maxabs_oob present).
 * nthreads > 1 shards rows and merges the partial sums (mae then differs in the last bits). */
int ork_eval_accuracy(const ork_spec* spec, const ork_artifact* a, const double* X, int64_t rows,
                      int32_t nthreads, double* acc, uint64_t* counts, int32_t* has_oob);

/* basis_values (spline.cpp:89-94) over KnotGrid(breakpoints, degree). out: [K+degree]. */
int ork_basis_values(const double* breakpoints, int32_t K, int32_t degree, double x, double* out);

/* quantize_segment_symmetric / _asymmetric (compiler.cpp:105-128). */
int ork_quantize_segment(const double* v, int32_t n, int32_t scheme, int32_t* q,
                         double* scale, double* y_min);

/* float16.cpp:7-71 */
uint16_t ork_f32_to_f16_bits(float f);
float ork_f16_bits_to_f32(uint16_t h);

/* Rng (rng.hpp:13-58, rng.cpp:7-22): n draws of uniform() / normal(). */
void ork_rng_uniform(uint64_t seed, int64_t n, double* out);
void ork_rng_normal(uint64_t seed, int64_t n, double* out);

/* gen_layer / gen_inputs (model_gen.cpp:7-45). Outputs caller-allocated: breakpoints [K+1],
 * coeffs [E*(K+degree)], gains [E] x3; X [n*dim]. */
int ork_gen_layer(uint64_t seed, int32_t in_dim, int32_t out_dim, int32_t segments, int32_t degree, double* bp,
                  double* coeffs, double* base_scale, double* spline_scale, double* out_scale);
int ork_gen_inputs(uint64_t seed, int64_t n, int64_t dim, double lo, double hi, int32_t clip, double* X);

/* Synthetic BASELINE configs (SURVEY.md §8d recipe, pinned in DESIGN.md §3).
 * cfg: 1..5. Layer l of the chain for cfg; seed stream continues across layers, so
 * generation always walks layers 0..l. Outputs are caller-allocated [E*R] / [E]. */
int ork_recipe_layer(int32_t cfg, int32_t layer, double* breakpoints, double* coeffs,
                     double* base_scale, double* spline_scale, double* out_scale);
/* Rows [row0, row0+rows) of cfg's fp32 inputs (widened to f64 by the caller if needed). */
int ork_recipe_inputs(int32_t cfg, int64_t row0, int64_t rows, float* X);

#ifdef __cplusplus
}
#endif
#endif
