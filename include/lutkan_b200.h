/*
 * lutkan_b200.h — C-ABI of the B200-native LUT-KAN engine (liblutkan_b200.so).
 *
 * Drop-in boundary for the reference's hot path (namespace lutkan, /root/reference/proj/core):
 *   compile    compile_layer / compile_model / compile_layer_debug_float  (compiler.hpp:67-77)
 *   forward    lut_layer_forward_batch / lut_model_forward_batch          (runtime.hpp:130-148)
 *   baseline   layer_forward_batch (spline, Tier::Optimized)              (spline.hpp:100-101)
 * Plain pointers and sizes only; no C++ or torch types cross this boundary. The
 * C++ shim include/lutkan_b200.hpp re-exposes the reference signatures on top of it,
 * and INTEGRATION.md shows the bindings a maintainer adds.
 *
 * Conventions
 *  - Every function returns lkg_status; on failure lkg_last_error() (thread-local)
 *    holds the message. Codes mirror the reference exception taxonomy
 *    (types.hpp:11-39): CONFIG=ConfigError, DIMENSION=DimensionError,
 *    NON_FINITE=NonFiniteError, UNSUPPORTED_BASE=UnsupportedBaseError.
 *  - Enum values are the declaration order of types.hpp:41-49.
 *  - Layouts are the reference's: edges input-major e = i*out_dim + j (spline.hpp:43),
 *    q_table [E,K,L], scale/y_min [E,K], knots [K+1] (runtime.hpp:31-63).
 *  - Device-resident objects (lkg_layer, lkg_spec) are immutable after creation and
 *    may be shared by contexts on the same device and by any number of host threads.
 *  - Threading contract: ONE lkg_ctx PER HOST THREAD. A context owns one CUDA stream, its
 *    scratch buffers and its OOB counters; all work is stream-ordered on it and a context
 *    must not be driven by two threads at once. Distinct contexts may be driven from
 *    distinct host threads concurrently, which is how the reference's purity and
 *    re-entrancy is kept: the C++ shim (lutkan_b200.hpp) gives every
 *    host thread its own default context.
 *  - Documented differences from the reference: activations are fp32 on the device
 *    (the reference's Matrix is f64; parity inputs are fp32-representable, so segment
 *    indices and OOB masks are bit-exact); Tier is accepted by the C++ shim and
 *    ignored (one backend, no CPU fallback).
 */
#ifndef LUTKAN_B200_H
#define LUTKAN_B200_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  LKG_OK = 0,
  LKG_ERR_CONFIG = 1,           /* lutkan::ConfigError */
  LKG_ERR_DIMENSION = 2,        /* lutkan::DimensionError */
  LKG_ERR_NON_FINITE = 3,       /* lutkan::NonFiniteError */
  LKG_ERR_UNSUPPORTED_BASE = 4, /* lutkan::UnsupportedBaseError */
  LKG_ERR_CUDA = 5,
  LKG_ERR_NCCL = 6,
  LKG_ERR_OOM = 7,
  LKG_ERR_INVALID_ARG = 8,
  /* artifact container I/O (artifact_io.hpp:11-52) */
  LKG_ERR_IO = 9,                /* lutkan::IoError */
  LKG_ERR_CORRUPT_ARCHIVE = 10,  /* lutkan::CorruptArchiveError */
  LKG_ERR_CORRUPT_BLOB = 11,     /* lutkan::CorruptBlobError */
  LKG_ERR_MISSING_KEY = 12,      /* lutkan::MissingKeyError */
  LKG_ERR_SHAPE = 13,            /* lutkan::ShapeError */
  LKG_ERR_VERSION = 14,          /* lutkan::VersionError */
  LKG_ERR_ENUM = 15              /* lutkan::EnumError */
} lkg_status;

enum { LKG_SCHEME_SYMMETRIC = 0, LKG_SCHEME_ASYMMETRIC = 1 };      /* Scheme */
enum { LKG_DTYPE_INT8 = 0, LKG_DTYPE_UINT8 = 1 };                  /* Dtype */
enum { LKG_REPR_PHI = 0, LKG_REPR_SPLINE_COMPONENT = 1 };          /* ValueRepr */
enum { LKG_INTERP_LINEAR = 0 };                                    /* Interp */
enum { LKG_BOUNDARY_HALF_OPEN = 0, LKG_BOUNDARY_CLOSED = 1 };      /* BoundaryMode */
enum { LKG_OOB_CLIP_X = 0, LKG_OOB_ZERO_SPLINE = 1 };              /* OobPolicy */
enum { LKG_PARAM_F32 = 0, LKG_PARAM_F16 = 1 };                     /* ParamDtype */

typedef struct lkg_ctx lkg_ctx;     /* device + stream + scratch (+ NCCL communicator) */
typedef struct lkg_layer lkg_layer; /* device-resident LutLayerArtifact (or a column shard) */
typedef struct lkg_spec lkg_spec;   /* device-resident KanLayerSpec (or a column shard) */

/* OobStats, runtime.hpp:105-120. */
typedef struct {
  uint64_t n_samples, n_oob_samples, n_inputs, n_oob_inputs;
} lkg_oob_stats;

/* EvalReport accuracy fields, metrics.hpp:52-76 (has_oob = 0: mae_oob/maxabs_oob absent). */
typedef struct {
  double mae_inrange, maxabs_inrange, mae_oob, maxabs_oob, oob_any_frac;
  uint64_t n_samples, n_inrange_evals, n_oob_evals, n_boundary_evals, n_oob_samples;
  int32_t has_oob;
} lkg_eval_report;

/* LutLayerArtifact fields (runtime.hpp:31-63), host pointers. Gains are required iff
 * value_repr == spline_component; float_table (debug, [E,K,L] f64) is optional. */
typedef struct {
  int32_t in_dim, out_dim, K, L;
  int32_t value_repr, interp, scheme, dtype, param_dtype, boundary_mode, oob_policy;
  const char* base_kind; /* "silu" for spline_component, "" (or NULL) for phi */
  const float* knots;
  const uint8_t* q_table;
  const float* scale;
  const float* y_min;
  const float* edge_base_scale;
  const float* edge_spline_scale;
  const float* edge_out_scale;
  const double* float_table;
} lkg_layer_desc;

/* KanLayerSpec (spline.hpp:35-74), host pointers: f64 breakpoints [K+1], degree,
 * packed_coeffs [E, K+degree], gains [E] (spline.hpp:57-62). */
typedef struct {
  int32_t in_dim, out_dim, K, degree;
  const char* base_kind; /* only "silu" is registered (spline.cpp:105-108) */
  const double* breakpoints;
  const double* coeffs;
  const double* base_scale;
  const double* spline_scale;
  const double* out_scale;
} lkg_spec_desc;

/* QuantConfig (compiler.hpp:15-24); OobConfig (runtime.hpp:19-22). */
typedef struct {
  int32_t L, scheme, dtype, value_repr, interp, param_dtype;
} lkg_quant_config;
typedef struct {
  int32_t boundary_mode, oob_policy;
} lkg_oob_config;

/* Shape / footprint of a device layer (for reporting and download sizing). */
typedef struct {
  int32_t in_dim, out_dim, K, L, col0, col1, full_out_dim;
  int32_t value_repr, scheme, param_dtype, boundary_mode, oob_policy, has_float_table;
  uint64_t device_bytes;
} lkg_layer_info;

/* ------------------------------------------------------------------ context */
const char* lkg_last_error(void);
const char* lkg_version(void);
/* stream: a cudaStream_t to run on (NULL = create a private non-blocking stream). */
lkg_status lkg_ctx_create(int32_t device, void* stream, lkg_ctx** out);
lkg_status lkg_ctx_destroy(lkg_ctx* ctx);
lkg_status lkg_ctx_synchronize(lkg_ctx* ctx);
void* lkg_ctx_stream(lkg_ctx* ctx);
/* Number of kernels this context has launched so far (for bench's gpu_launches). */
uint64_t lkg_ctx_launch_count(lkg_ctx* ctx);
/* Device workspace the context holds between calls: hidden-activation ping-pong buffers, the
 * transposed-input / coordinate-record buffer of the wide-layer table walk (2 x rows x in_dim x 4 B,
 * e.g. 8.6 GB after a configs[3] batch), the sharded chain's gather buffer and the host entries'
 * staging. Buffers grow on demand and are reused; lkg_ctx_trim synchronizes the stream and frees them
 * (the reference's Matrix temporaries die with each call, runtime.cpp:298-314). */
uint64_t lkg_ctx_workspace_bytes(lkg_ctx* ctx);
lkg_status lkg_ctx_trim(lkg_ctx* ctx);

/* -------------------------------------------------------- artifact (F1, F2) */
/* Validates like LutLayerArtifact::finalize (runtime.cpp:11-43) and uploads. */
lkg_status lkg_layer_upload(lkg_ctx* ctx, const lkg_layer_desc* desc, lkg_layer** out);
/* Column shard: only output columns [col0, col1) of desc (edges (i, j) with j in range),
 * i.e. the strided slice {(i*m + j)*K*L ...} of the reference arrays. */
lkg_status lkg_layer_upload_columns(lkg_ctx* ctx, const lkg_layer_desc* desc, int32_t col0,
                                    int32_t col1, lkg_layer** out);
lkg_status lkg_layer_info_get(const lkg_layer* layer, lkg_layer_info* out);
/* Copies the layer back in the reference layout (sizes from lkg_layer_info: E = in_dim *
 * (col1-col0)). Any output pointer may be NULL. */
/* The layer's base_kind ("" for phi), valid while the layer lives. */
const char* lkg_layer_base_kind(const lkg_layer* layer);
lkg_status lkg_layer_download(lkg_ctx* ctx, const lkg_layer* layer, float* knots, uint8_t* q_table,
                              float* scale, float* y_min, float* edge_base_scale,
                              float* edge_spline_scale, float* edge_out_scale, double* float_table);
lkg_status lkg_layer_free(lkg_layer* layer);

/* ------------------------------------------------------------ compile (CM*) */
lkg_status lkg_spec_upload(lkg_ctx* ctx, const lkg_spec_desc* desc, lkg_spec** out);
lkg_status lkg_spec_upload_columns(lkg_ctx* ctx, const lkg_spec_desc* desc, int32_t col0,
                                   int32_t col1, lkg_spec** out);
/* A spec that already holds only output columns [col0, col0 + desc->out_dim) of a layer whose
 * full width is full_out_dim (each rank of a column-sharded deployment materialises only its
 * own edges). Layers compiled from it are column shards. */
lkg_status lkg_spec_upload_shard(lkg_ctx* ctx, const lkg_spec_desc* desc, int32_t col0, int32_t full_out_dim,
                                 lkg_spec** out);
lkg_status lkg_spec_free(lkg_spec* spec);
/* compile_layer (compiler.cpp:213-216): bytes, scales and y_mins bit-exact with the
 * reference. keep_float != 0 also keeps the f64 float table (compile_layer_debug_float). */
lkg_status lkg_compile_layer(lkg_ctx* ctx, const lkg_spec* spec, const lkg_quant_config* qc,
                             const lkg_oob_config* oob, int32_t keep_float, lkg_layer** out);

/* ----------------------------------------------------------- forward (F4-F15) */
/* lut_layer_forward_batch (runtime.cpp:250-285): X [rows, in_dim] fp32 -> Y [rows, out_dim]
 * fp32 (column shard: [rows, col1-col0]); both DEVICE pointers. If stats != NULL the call
 * synchronizes, fills the layer's OobStats and reports NON_FINITE inputs; if stats == NULL
 * it is asynchronous and counters accumulate until lkg_ctx_collect(). */
lkg_status lkg_layer_forward(lkg_ctx* ctx, const lkg_layer* layer, const float* X, int64_t rows,
                             float* Y, lkg_oob_stats* stats);
/* lut_model_forward_batch (runtime.cpp:298-314): hidden activations stay on the device in
 * fp32; stats (optional) is per layer [n_layers]. Chain checks as the reference. */
lkg_status lkg_model_forward(lkg_ctx* ctx, const lkg_layer* const* chain, int32_t n_layers,
                             const float* X, int64_t rows, float* Y, lkg_oob_stats* stats);
/* Same call with HOST buffers (pinned or pageable): H2D of X, the chain, D2H of Y. */
lkg_status lkg_model_forward_host(lkg_ctx* ctx, const lkg_layer* const* chain, int32_t n_layers,
                                  const float* X_host, int64_t rows, float* Y_host,
                                  lkg_oob_stats* stats);
/* Same call on the reference's own f64 rows (Matrix data, row-major, pageable): host threads narrow
 * X to fp32 row chunk by row chunk into pinned staging while the previous chunk copies and runs; Y is
 * widened back by the same threads. The C++ shim's lut_model_forward_batch / lut_layer_forward_batch
 * go through this entry. */
lkg_status lkg_model_forward_host_f64(lkg_ctx* ctx, const lkg_layer* const* chain, int32_t n_layers,
                                      const double* X_host, int64_t rows, double* Y_host,
                                      lkg_oob_stats* stats);
/* A chain forward captured once as a CUDA graph and replayed: the same launches as
 * lkg_model_forward on the same DEVICE buffers (X, Y and the layers are bound at capture; rows > 0),
 * one cudaGraphLaunch per replay on ctx's stream, asynchronous. For small, latency-bound batches
 * served repeatedly. Creation runs the chain once eagerly (sizes scratch, sets kernel attributes).
 * The graph owns its hidden-activation and transposed-input buffers, so other forwards on ctx
 * (any batch size or width) never invalidate it. OOB statistics of the replays accumulate in ctx
 * like direct calls (lkg_ctx_collect). The layers, X and Y must outlive the graph; replays of one
 * graph are stream-ordered on ctx's stream. */
typedef struct lkg_graph lkg_graph;
lkg_status lkg_graph_create(lkg_ctx* ctx, const lkg_layer* const* chain, int32_t n_layers, const float* X,
                            int64_t rows, float* Y, lkg_graph** out);
lkg_status lkg_graph_launch(lkg_graph* graph);
lkg_status lkg_graph_destroy(lkg_graph* graph);
/* Per-element coordinates exactly as the forward kernels compute them (steps 1-4 of the
 * 5-step pipeline, runtime.cpp:45-75 / 170-190): for x [n] fp32 (device), writes
 * in-range mask, segment index k and sample index l0 (device int32 arrays, any may be NULL).
 * Exposed so segment indices and OOB masks can be checked bit-exactly. */
lkg_status lkg_layer_coords(lkg_ctx* ctx, const lkg_layer* layer, const float* x, int64_t n,
                            int32_t* in_range, int32_t* k, int32_t* l0);
/* Reads and resets the asynchronous OOB counters / non-finite flag of the last
 * n_layers layer slots (slot l = l-th layer of the last chain). */
lkg_status lkg_ctx_collect(lkg_ctx* ctx, lkg_oob_stats* stats, int32_t n_layers);

/* ------------------------------------------------ spline baseline (S1, K3) */
/* layer_forward_batch(spec, X, Tier::Optimized) (spline.cpp:145-187); device pointers. */
lkg_status lkg_spline_forward(lkg_ctx* ctx, const lkg_spec* spec, const float* X, int64_t rows,
                              float* Y);
/* Spline kernel family used by this context's lkg_spline_forward[_host]:
 * LKG_SPLINE_AUTO (default): the tensor-core GEMM form (spline_tc.cu: uniform cubic grids with
 *   K <= 16), else the SIMT table kernel (uniform cubic), else the generic Cox-de Boor kernel;
 * LKG_SPLINE_SIMT: skip the tensor-core form (the SIMT kernels, for the same-GPU comparison). */
enum { LKG_SPLINE_AUTO = 0, LKG_SPLINE_SIMT = 1 };
lkg_status lkg_ctx_set_spline_kernel(lkg_ctx* ctx, int32_t kind);
/* Same with HOST buffers (H2D of X, kernel, D2H of Y; synchronous). */
lkg_status lkg_spline_forward_host(lkg_ctx* ctx, const lkg_spec* spec, const float* X_host, int64_t rows,
                                   float* Y_host);

/* ------------------------------------ artifact container */
/* save_artifact (artifact_io.cpp:206-219): the `.lut` ZIP container (format lutkan/1).
 * mode 0: byte-identical to the reference's file (ZIP64 records only above 4 GiB, an extension);
 * mode 1: stored (method 0) entries; mode 2: parallel-inflate deflate (independently compressed
 * segments forming one valid deflate stream, segment index in a central-directory extra field).
 * The reference reader accepts modes 1 and 2. Column shards cannot be saved (CONFIG). */
lkg_status lkg_artifact_save(lkg_ctx* ctx, const lkg_layer* layer, const char* path, int32_t mode);
/* load_artifact (artifact_io.cpp:221-300) straight into a device layer: the same checks in the
 * same order and the same error classes (IO, CORRUPT_ARCHIVE, CORRUPT_BLOB, MISSING_KEY, SHAPE,
 * VERSION, ENUM, then finalize's CONFIG/DIMENSION/NON_FINITE); ZIP64 archives accepted. */
lkg_status lkg_artifact_load(lkg_ctx* ctx, const char* path, lkg_layer** out);
/* Host-only forms (no GPU needed): save from host arrays (finalize checks first), and the full
 * load validation of a file without an upload (returns the status load would return). */
lkg_status lkg_artifact_save_desc(const lkg_layer_desc* desc, const char* path, int32_t mode);
lkg_status lkg_artifact_check(const char* path);
/* artifact_manifest_json (artifact_io.hpp:66-67, artifact_io.cpp:98-124): the manifest text exactly
 * as save_artifact writes it. Reads only the descriptor's shape and enum fields (no array). Writes
 * at most cap-1 bytes plus a NUL into buf (buf may be NULL to query the length) and the full
 * length into *len. Host-only. */
lkg_status lkg_artifact_manifest(const lkg_layer_desc* desc, char* buf, size_t cap, size_t* len);

/* ---------------------------------------------- element primitives (§8a) */
/* The reference's scalar functions, batched on the device in f64 with the reference's
 * expressions (values identical to the reference's); HOST arrays of n elements, synchronous.
 * safe_clip / segment_index / interp_coords / in_range (runtime.cpp:45-75) of x[n] against the
 * layer's knots (any output may be NULL). */
lkg_status lkg_lut_coords64(lkg_ctx* ctx, const lkg_layer* layer, const double* x, int64_t n, uint8_t* in_range,
                            double* x_clip, int32_t* k, int32_t* l0, int32_t* l1, double* w);
/* lut_eval_value / lut_eval_phi (runtime.cpp:96-120) of edges e[n] at x[n]: NON_FINITE for a
 * non-finite x, DIMENSION for an edge out of range, UNSUPPORTED_BASE for an unknown base kind. */
lkg_status lkg_lut_eval(lkg_ctx* ctx, const lkg_layer* layer, const int32_t* e, const double* x, int64_t n,
                        double* value, uint8_t* was_oob, double* phi);
/* basis_values (spline.cpp:89-94) over KnotGrid(breakpoints[K+1], degree): out [n][K+degree]. */
lkg_status lkg_basis_values(lkg_ctx* ctx, const double* breakpoints, int32_t K, int32_t degree, const double* x,
                            int64_t n, double* out);
/* eval_edge_phi (spline.cpp:96-115) of the spec's edges e[n] at x[n]. */
lkg_status lkg_edge_phi(lkg_ctx* ctx, const lkg_spec* spec, const int32_t* e, const double* x, int64_t n,
                        double* phi);
/* quantize_segment_symmetric / _asymmetric (compiler.cpp:105-128) of nseg segments of L values
 * (v [nseg][L]): codes q [nseg][L], unrounded scale / y_min [nseg]. */
lkg_status lkg_quantize_segments(lkg_ctx* ctx, const double* v, int64_t nseg, int32_t L, int32_t scheme, int32_t* q,
                                 double* scale, double* y_min);

/* ------------------------------------------- accuracy */
/* eval_accuracy(layer, artifact, X) (metrics.cpp:30-103): |lut_eval_phi - eval_edge_phi| over
 * every (sample, input, edge), bucketed in-range / OOB / boundary; f64 on the device with the
 * reference's expressions. spec and layer must be the same (unsharded) shape; X [rows, in_dim]
 * fp32 DEVICE pointer. Synchronous. NON_FINITE if any input is NaN or inf. */
lkg_status lkg_eval_accuracy(lkg_ctx* ctx, const lkg_spec* spec, const lkg_layer* layer, const float* X,
                             int64_t rows, lkg_eval_report* out);
/* Same with a HOST X buffer. */
lkg_status lkg_eval_accuracy_host(lkg_ctx* ctx, const lkg_spec* spec, const lkg_layer* layer,
                                  const float* X_host, int64_t rows, lkg_eval_report* out);
/* Same with a HOST f64 X buffer (the reference's Matrix values, not rounded to fp32): the reports
 * of the sweep driver, whose inputs are gen_inputs' f64 normals (sweep.cpp:87-90). */
lkg_status lkg_eval_accuracy_host_f64(lkg_ctx* ctx, const lkg_spec* spec, const lkg_layer* layer,
                                      const double* X_host, int64_t rows, lkg_eval_report* out);

/* ------------------------------------------------ multi-GPU (column shards) */
/* NCCL communicator for output-column sharding. id: 128 bytes from
 * lkg_nccl_unique_id() on rank 0, broadcast by the host (e.g. torch.distributed). */
lkg_status lkg_nccl_unique_id(uint8_t id_out[128]);
lkg_status lkg_ctx_init_nccl(lkg_ctx* ctx, const uint8_t id[128], int32_t nranks, int32_t rank);
/* One layer forward whose input X is in the rank-major all-gather layout of column shards of
 * width x_blk (element (r, i) at X[(i / x_blk) * rows * x_blk + r * x_blk + i % x_blk]), i.e.
 * ncclAllGather output consumed in place; x_blk == 0 means row-major. Device pointers. */
lkg_status lkg_layer_forward_blocked(lkg_ctx* ctx, const lkg_layer* layer, const float* X, int64_t rows,
                                     int32_t x_blk, float* Y, lkg_oob_stats* stats);
/* Column-sharded chain: every rank holds the column shard [col0, col1) of every layer
 * (equal shards, rank-ordered). X [rows, in_dim] replicated; between layers the local
 * outputs are all-gathered over NCCL (rank-major blocks consumed in place); Y receives the
 * last layer's LOCAL columns [rows, col1-col0]. */
lkg_status lkg_model_forward_sharded(lkg_ctx* ctx, const lkg_layer* const* chain, int32_t n_layers,
                                     const float* X, int64_t rows, float* Y, lkg_oob_stats* stats);

/* ------------------------------------------------------- synthetic configs */
/* The BASELINE.json configs (DESIGN.md §3 recipe; reference Rng, rng.hpp:13-58). cfg 1..5.
 * dims_out receives n_layers+1 widths; returns n_layers in *n_layers. */
lkg_status lkg_recipe_dims(int32_t cfg, int32_t* n_layers, int32_t* dims_out, int32_t* G,
                           double* lo, double* hi);
/* Host-side spec arrays of layer `layer` (caller-allocated: bp [G+1], coeffs [E*(G+3)],
 * gains [E] x3). Restricted to columns [col0, col1) when col1 > col0. */
lkg_status lkg_recipe_layer(int32_t cfg, int32_t layer, int32_t col0, int32_t col1,
                            double* breakpoints, double* coeffs, double* base_scale,
                            double* spline_scale, double* out_scale);
/* gen_layer / gen_inputs (model_gen.cpp:7-45): the reference's generator (breakpoints on [-1, 1],
 * coefficients normal(0, 0.1), gains uniform(0.5, 1.5); inputs standard normal, optionally
 * clamped). Host functions; arrays [K+1], [E*(K+degree)], [E] x3, X [n*dim] f64. */
lkg_status lkg_gen_layer(uint64_t seed, int32_t in_dim, int32_t out_dim, int32_t segments, int32_t degree,
                         double* breakpoints, double* coeffs, double* base_scale, double* spline_scale,
                         double* out_scale);
lkg_status lkg_gen_inputs(uint64_t seed, int64_t n, int64_t dim, double lo, double hi, int32_t clip, double* X);
/* fp32 inputs rows [row0, row0+rows). */
lkg_status lkg_recipe_inputs(int32_t cfg, int64_t row0, int64_t rows, float* X);

#ifdef __cplusplus
}
#endif
#endif
