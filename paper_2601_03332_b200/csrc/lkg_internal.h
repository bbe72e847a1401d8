// lkg_internal.h — internal types of liblutkan_b200.so (not part of the C-ABI).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <utility>
#include <vector>

#include "../../include/lutkan_b200.h"
#include "coords.cuh"

namespace lkg {

// Row splits (host-path chunks, sharded-chain chunks, batch shards) start at multiples of this:
// the kernels walk a row's inputs in a lane-dependent rotation (row mod 32 at most), so a row's
// fp32 accumulation order -- and its last bits -- depend on its position modulo 32. Aligned
// splits keep every row bit-identical to the single-launch result.
constexpr int64_t kRowAlign = 64;

// Thread-local last error (lkg_last_error).
void set_error(const std::string& msg);

struct Error {
  lkg_status code;
  std::string msg;
};

#define LKG_CUDA(call)                                                                   \
  do {                                                                                   \
    cudaError_t e_ = (call);                                                             \
    if (e_ != cudaSuccess)                                                               \
      throw ::lkg::Error{e_ == cudaErrorMemoryAllocation ? LKG_ERR_OOM : LKG_ERR_CUDA,   \
                         std::string(#call) + ": " + cudaGetErrorString(e_)};            \
  } while (0)

// Device buffer owned by a layer/spec/context.
struct DBuf {
  void* p = nullptr;
  size_t bytes = 0;
  DBuf() = default;
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  ~DBuf() { release(); }
  void alloc(size_t n) {
    release();
    if (n) LKG_CUDA(cudaMalloc(&p, n));
    bytes = n;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
  }
  template <class T>
  T* as() const { return static_cast<T*>(p); }
  void swap(DBuf& o) {
    std::swap(p, o.p);
    std::swap(bytes, o.bytes);
  }
};

// Forward-kernel tile geometry chosen at upload time (forward.cu).
struct TileGeom {
  int32_t JB = 0;       // output columns per j-block (codes per lane-load)
  int32_t IC = 0;       // inputs interleaved per 128-byte line
  int32_t n_jb = 0;     // number of j-blocks
  int32_t n_ih = 0;     // number of i-tiles
  int64_t tile_bytes = 0;  // bytes of one (i-tile, j-block) tile, 128-aligned
  int32_t p_off = 0, q_off = 0, cb_off = 0;  // byte offsets inside a tile
  int32_t p_stride = 0;  // bytes between (k, i_lo) rows of the P block
  int32_t small = 0, MP = 0;  // whole-layer-in-smem layout (m <= 8), MP = padded out_dim
  int32_t codes_global = 0;   // tiled layout whose code block is read from global/L2 (GC kernel)
  // Integer-lerp table walk (forward_tiled.cu, IDP): 0 = fp32 magic-float lerp; 1 = pair lines
  // (each code stored next to its successor: one dp2a per output, no byte extraction); 2 = the
  // standard lines, pairs built with one PRMT per 2 outputs. P is stored pre-scaled by 2^-15.
  int32_t idp = 0;
  double idp_rss = 0.0;       // statistical bound of the 2^-16 weight-rounding error (build_tiles)
  // fp32-accumulation error estimate of the layer (build_tiles) and whether it therefore takes the
  // f64 accumulators although d <= 256
  double acc32_err = 0.0;
  int32_t acc64 = 0;
};

}  // namespace lkg

// Device artifact. The reference-layout arrays are kept for download/parity; the
// forward kernels read the tiled copy built by lkg::build_tiles (forward.cu).
struct lkg_layer {
  int device = 0;
  int32_t in_dim = 0, out_dim = 0, K = 0, L = 0;
  int32_t col0 = 0, col1 = 0, full_out_dim = 0;  // column shard [col0, col1) of full_out_dim
  int32_t value_repr = 1, scheme = 0, param_dtype = 0, boundary_mode = 1, oob_policy = 0;
  std::vector<float> knots;  // host copy (K+1), fp32
  std::string base_kind;     // spline_component: as uploaded ("silu" for compiled layers)
  lkg::DBuf q, scale, ymin, gains;  // reference layout: q [E,K,L], scale/ymin [E,K], gains [3][E]
  lkg::DBuf float_table;            // optional [E,K,L] f64
  lkg::DBuf cbcs;                   // fused gains fp32 [2][E]: cb = out*base, cs = out*spline
  lkg::TileGeom geom;
  lkg::DBuf tiles;                  // forward layout
  uint64_t device_bytes() const {
    return q.bytes + scale.bytes + ymin.bytes + gains.bytes + float_table.bytes + cbcs.bytes +
           tiles.bytes;
  }
};

struct lkg_spec {
  int device = 0;
  int32_t in_dim = 0, out_dim = 0, K = 0, degree = 3;
  int32_t col0 = 0, col1 = 0, full_out_dim = 0;
  std::vector<double> breakpoints;  // host f64 [K+1]
  lkg::DBuf coeffs;    // f64 [E,R] (compile)
  lkg::DBuf gains;     // f64 [3][E] base, spline, out (compile)
  lkg::DBuf coeffs32;  // f32 [i][R][j] transposed for the spline forward
  lkg::DBuf gains32;   // f32 [2][E]: out*base, out*spline
  lkg::DBuf spline_tiles;  // spline_tiled.cu layout (uniform cubic grids), built lazily
  lkg::DBuf tc_b;          // spline_tc.cu: the coefficient matrix in UMMA blocks (hi/lo tf32), lazily
  int32_t tc_n_ch = 0;
  double fast_err = -1.0;  // rounding estimate of the fast spline kernels (spline.cu), computed once
  int64_t sp_tile_bytes = 0;
  int32_t sp_n_ih = 0, sp_n_jb = 0;
};

struct lkg_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  uint64_t launches = 0;
  // Per-layer-slot counters: [slot][4] = {n_oob_samples, n_oob_inputs, nonfinite, rows}.
  static constexpr int kSlots = 64;
  lkg::DBuf counters;
  uint64_t rows_seen[kSlots] = {};
  int32_t in_dim_seen[kSlots] = {};
  lkg::DBuf scratch[2];  // hidden activations ping-pong
  lkg::DBuf gather;      // sharded chain: all-gathered hidden activations
  lkg::DBuf hostio;      // device staging for lkg_model_forward_host
  lkg::DBuf xt;          // transposed layer input of the XT table walk (forward_tiled.cu)
  lkg::DBuf ksp;         // input-split partial outputs + row flags (forward_tiled.cu, ksplit)
  void* pin = nullptr;                 // pinned host staging of the f64 host entry (grows)
  size_t pin_bytes = 0;
  cudaStream_t copy_stream = nullptr;  // H2D of the next chunk overlaps the chain on `stream`
  cudaEvent_t ev_copied[2] = {nullptr, nullptr}, ev_done[2] = {nullptr, nullptr};
  cudaStream_t comm_stream = nullptr;  // sharded chain: all-gathers overlap the next chunk's compute
  int32_t spline_kernel = 0;  // LKG_SPLINE_AUTO / LKG_SPLINE_SIMT (lkg_ctx_set_spline_kernel)
  void* nccl = nullptr;  // ncclComm_t
  int32_t nranks = 1, rank = 0;
};

namespace lkg {

// Kernel launch wrappers (forward.cu / compile.cu / spline.cu).
void build_tiles(lkg_ctx* ctx, lkg_layer* L);
bool tiled_eligible(const lkg_layer* L);
void fill_coord_const(const lkg_layer* L, CoordConst& c, float4* ktab);
void launch_forward_tiled(lkg_ctx* ctx, const lkg_layer* L, const float* X, int64_t rows, int32_t x_blk, float* Y,
                          int slot, const lkg_layer* L2 = nullptr, float* Y2 = nullptr);
// True when layer L2 (small out_dim, whole LUT in smem) can run in L1's epilogue (chain fusion).
bool can_fuse(const lkg_layer* L1, const lkg_layer* L2);
// Whole-chain fusion (forward_chain.cu): every layer a small value-table layer, one launch.
bool can_fuse_chain(const lkg_layer* const* chain, int n);
void launch_forward_chain(lkg_ctx* ctx, const lkg_layer* const* chain, int n, const float* X, int64_t rows, float* Y);
// Reference-layout q_table of a layer whose codes live only in its tiles.
void download_q_from_tiles(lkg_ctx* ctx, const lkg_layer* L, uint8_t* host_q);
// One layer forward. X has row stride x_ld and, when x_blk > 0, is stored as rank-major
// column blocks of width x_blk (the NCCL all-gather layout): element (r, i) lives at
// X[(i / x_blk) * rows * x_blk + r * x_blk + i % x_blk]. Y [rows, out_cols] row-major.
void launch_forward(lkg_ctx* ctx, const lkg_layer* L, const float* X, int64_t rows, int32_t x_blk,
                    float* Y, int slot, bool count_oob);
void launch_compile(lkg_ctx* ctx, const lkg_spec* S, const lkg_quant_config* qc, lkg_layer* out,
                    const double* d_basis, const int32_t* d_r0, const double* d_silu, int32_t W,
                    bool keep_float);
void launch_spline(lkg_ctx* ctx, const lkg_spec* S, const float* X, int64_t rows, float* Y,
                   const float* d_ext);
void launch_fuse_gains(lkg_ctx* ctx, lkg_layer* L);
void launch_coords(lkg_ctx* ctx, const lkg_layer* L, const float* x, int64_t n, int32_t* in_range, int32_t* k,
                   int32_t* l0);
void launch_spec_prepare(lkg_ctx* ctx, lkg_spec* S);
void validate_layer_desc(const lkg_layer_desc* d);
// element primitives (elements.cu), device pointers
void launch_coords64(lkg_ctx* ctx, const lkg_layer* L, const double* x, int64_t n, uint8_t* in, double* xc,
                     int32_t* k, int32_t* l0, int32_t* l1, double* w);
void launch_lut_eval(lkg_ctx* ctx, const lkg_layer* L, const int32_t* e, const double* x, int64_t n, double* value,
                     uint8_t* was_oob, double* phi, int* flags);
void launch_basis(lkg_ctx* ctx, const std::vector<double>& bp, int degree, const double* x, int64_t n, double* out);
void launch_edge_phi(lkg_ctx* ctx, const lkg_spec* S, const int32_t* e, const double* x, int64_t n, double* phi,
                     int* flags);
void launch_quantize(lkg_ctx* ctx, const double* v, int64_t nseg, int L, int asym, int32_t* q, double* scale,
                     double* ymin, int* flags);  // finalize checks (runtime.cpp:11-43)
void launch_eval(lkg_ctx* ctx, const lkg_spec* S, const lkg_layer* L, const void* X, bool x_f64, int64_t rows,
                 double* dsum, unsigned long long* u);
bool launch_spline_tiled(lkg_ctx* ctx, const lkg_spec* S, const float* X, int64_t rows, float* Y);
bool launch_spline_tc(lkg_ctx* ctx, const lkg_spec* S, const float* X, int64_t rows, float* Y);

// Host model_gen (model_gen.cpp).
int recipe_dims(int cfg, int* n_layers, int* dims, int* G, double* lo, double* hi);
void recipe_layer(int cfg, int layer, int col0, int col1, double* bp, double* coeffs, double* bs,
                  double* ss, double* os);
void recipe_inputs(int cfg, int64_t row0, int64_t rows, float* X);
void gen_layer(uint64_t seed, int d, int m, int segments, int degree, double* bp, double* coeffs, double* bs,
               double* ss, double* os);
void gen_inputs(uint64_t seed, int64_t n, int64_t dim, double lo, double hi, bool clip, double* X);

// Host Cox-de Boor (bit-exact restatement of spline.cpp:8-27,69-83) for compile tables.
void knot_grid(const std::vector<double>& bp, int degree, std::vector<double>& ext);
void basis_into(const std::vector<double>& T, int degree, double x, double* buf);
double silu_host(double x);

}  // namespace lkg
