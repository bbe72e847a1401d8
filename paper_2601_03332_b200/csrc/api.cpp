// api.cpp — host side of the C-ABI (include/lutkan_b200.h): validation mirroring the
// reference (LutLayerArtifact::finalize runtime.cpp:11-43, QuantConfig::validate
// compiler.cpp:10-16, KnotGrid/KanLayerSpec ctors spline.cpp:8-62, chain checks
// runtime.cpp:298-304 / compiler.cpp:218-228), device residency, stream-ordered
// launches, OOB-counter collection, host<->device entry points and the NCCL column-shard
// chain. Errors map to lkg_status codes with a thread-local message.
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <chrono>
#include <cstring>
#include <memory>
#include <string>
#include <atomic>
#include <thread>
#include <vector>

#include "lkg_internal.h"

// NCCL is resolved lazily with dlopen, and only by the column-shard entry points: the
// process may already hold another libnccl.so.2 (PyTorch bundles its own), and linking
// one at load time would shadow it. RTLD_NOLOAD first reuses whatever is loaded.
#include <dlfcn.h>
#if defined(__SSE2__)
#include <emmintrin.h>
#endif
namespace {
struct NcclApi {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};
const NcclApi& nccl_api() {
  static NcclApi api = [] {
    NcclApi a;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) throw lkg::Error{LKG_ERR_NCCL, std::string("cannot load libnccl.so.2: ") + dlerror()};
    a.GetUniqueId = reinterpret_cast<decltype(a.GetUniqueId)>(dlsym(h, "ncclGetUniqueId"));
    a.CommInitRank = reinterpret_cast<decltype(a.CommInitRank)>(dlsym(h, "ncclCommInitRank"));
    a.CommDestroy = reinterpret_cast<decltype(a.CommDestroy)>(dlsym(h, "ncclCommDestroy"));
    a.AllGather = reinterpret_cast<decltype(a.AllGather)>(dlsym(h, "ncclAllGather"));
    a.GetErrorString = reinterpret_cast<decltype(a.GetErrorString)>(dlsym(h, "ncclGetErrorString"));
    if (!a.GetUniqueId || !a.CommInitRank || !a.CommDestroy || !a.AllGather || !a.GetErrorString)
      throw lkg::Error{LKG_ERR_NCCL, "libnccl.so.2 lacks a required symbol"};
    return a;
  }();
  return api;
}
}  // namespace
#define ncclGetUniqueId nccl_api().GetUniqueId
#define ncclCommInitRank nccl_api().CommInitRank
#define ncclCommDestroy nccl_api().CommDestroy
#define ncclAllGather nccl_api().AllGather
#define ncclGetErrorString nccl_api().GetErrorString

namespace lkg {
namespace {
thread_local std::string g_err;
}
void set_error(const std::string& m) { g_err = m; }
const char* last_error() { return g_err.c_str(); }
}  // namespace lkg

using lkg::DBuf;
using lkg::Error;

namespace {

template <class F>
lkg_status guarded(F&& f) {
  try {
    f();
    return LKG_OK;
  } catch (const Error& e) {
    lkg::set_error(e.msg);
    return e.code;
  } catch (const std::bad_alloc&) {
    lkg::set_error("host allocation failed");
    return LKG_ERR_OOM;
  } catch (const std::exception& e) {
    lkg::set_error(e.what());
    return LKG_ERR_INVALID_ARG;
  }
}

[[noreturn]] void fail(lkg_status c, const std::string& m) { throw Error{c, m}; }

void need(const void* p, const char* what) {
  if (!p) fail(LKG_ERR_INVALID_ARG, std::string("null pointer: ") + what);
}

struct DeviceGuard {
  int prev = 0;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) LKG_CUDA(cudaSetDevice(dev));
  }
  ~DeviceGuard() { cudaSetDevice(prev); }
};

// KnotGrid validation (spline.cpp:8-27)
void check_breakpoints(const std::vector<double>& bp, int degree) {
  if (degree < 0) fail(LKG_ERR_CONFIG, "degree must be >= 0");
  if (bp.size() < 2) fail(LKG_ERR_CONFIG, "need at least 2 breakpoints");
  for (size_t i = 0; i < bp.size(); i++) {
    if (!std::isfinite(bp[i])) fail(LKG_ERR_NON_FINITE, "non-finite breakpoint");
    if (i > 0 && !(bp[i - 1] < bp[i])) fail(LKG_ERR_CONFIG, "breakpoints must be strictly increasing");
  }
}

void check_knots(const float* knots, int K) {
  if (K < 1) fail(LKG_ERR_CONFIG, "artifact needs at least 2 knots");
  for (int i = 0; i <= K; i++) {
    if (!std::isfinite(knots[i])) fail(LKG_ERR_NON_FINITE, "non-finite knot");
    if (i > 0 && !(knots[i - 1] < knots[i])) fail(LKG_ERR_CONFIG, "knots must be strictly increasing");
  }
}

void check_scheme(int scheme, int dtype) {
  if (scheme == LKG_SCHEME_SYMMETRIC && dtype != LKG_DTYPE_INT8)
    fail(LKG_ERR_CONFIG, "symmetric scheme requires int8");
  if (scheme == LKG_SCHEME_ASYMMETRIC && dtype != LKG_DTYPE_UINT8)
    fail(LKG_ERR_CONFIG, "asymmetric scheme requires uint8");
  if (scheme != LKG_SCHEME_SYMMETRIC && scheme != LKG_SCHEME_ASYMMETRIC)
    fail(LKG_ERR_CONFIG, "unknown scheme");
}

// LutLayerArtifact::finalize (runtime.cpp:11-43).
void validate_desc(const lkg_layer_desc* d) {
  need(d, "desc");
  if (d->in_dim < 1 || d->out_dim < 1) fail(LKG_ERR_CONFIG, "artifact dims must be >= 1");
  if (d->L < 2) fail(LKG_ERR_CONFIG, "samples per segment must be >= 2");
  need(d->knots, "knots");
  check_knots(d->knots, d->K);
  check_scheme(d->scheme, d->dtype);
  if (d->interp != LKG_INTERP_LINEAR) fail(LKG_ERR_CONFIG, "unknown interp");
  if (d->boundary_mode != LKG_BOUNDARY_HALF_OPEN && d->boundary_mode != LKG_BOUNDARY_CLOSED)
    fail(LKG_ERR_CONFIG, "unknown boundary_mode");
  if (d->oob_policy != LKG_OOB_CLIP_X && d->oob_policy != LKG_OOB_ZERO_SPLINE)
    fail(LKG_ERR_CONFIG, "unknown oob_policy");
  if (d->param_dtype != LKG_PARAM_F32 && d->param_dtype != LKG_PARAM_F16)
    fail(LKG_ERR_CONFIG, "unknown param_dtype");
  need(d->q_table, "q_table");
  need(d->scale, "scale");
  need(d->y_min, "y_min");
  if (d->value_repr == LKG_REPR_SPLINE_COMPONENT) {
    if (!d->edge_base_scale || !d->edge_spline_scale || !d->edge_out_scale)
      fail(LKG_ERR_DIMENSION, "edge scale arrays must have one entry per edge");
    if (!d->base_kind || !*d->base_kind) fail(LKG_ERR_CONFIG, "spline_component artifact needs a base_kind");
    // finalize accepts any base kind (runtime.cpp:34); the optimized forward evaluates silu
    // whatever it names (runtime.cpp:189) and lut_eval_phi rejects unknown kinds (eval_accuracy)
  } else if (d->value_repr == LKG_REPR_PHI) {
    if (d->edge_base_scale || d->edge_spline_scale || d->edge_out_scale)
      fail(LKG_ERR_CONFIG, "phi artifact must not carry edge scale arrays");
  } else {
    fail(LKG_ERR_CONFIG, "unknown value_repr");
  }
}

}  // namespace
namespace lkg {
void validate_layer_desc(const lkg_layer_desc* d) { validate_desc(d); }
}  // namespace lkg
namespace {

// Strided column slice: for every input row i, columns [c0, c1) of a [d, m, inner] array.
template <class T>
void upload_cols(DBuf& dst, const T* src, int64_t d, int64_t m, int64_t inner, int c0, int c1,
                 cudaStream_t st) {
  const int64_t mc = c1 - c0;
  dst.alloc(sizeof(T) * d * mc * inner);
  if (!dst.bytes) return;
  LKG_CUDA(cudaMemcpy2DAsync(dst.p, sizeof(T) * mc * inner, src + c0 * inner, sizeof(T) * m * inner,
                             sizeof(T) * mc * inner, d, cudaMemcpyHostToDevice, st));
}

void ensure(DBuf& b, size_t bytes) {
  if (b.bytes < bytes) b.alloc(bytes);
}

}  // namespace

// ===================================================================== C-ABI
extern "C" {

const char* lkg_last_error(void) { return lkg::last_error(); }
const char* lkg_version(void) { return "lutkan_b200 0.1 (sm_100a)"; }

lkg_status lkg_ctx_create(int32_t device, void* stream, lkg_ctx** out) {
  return guarded([&] {
    need(out, "out");
    int n = 0;
    LKG_CUDA(cudaGetDeviceCount(&n));
    if (device < 0 || device >= n) fail(LKG_ERR_INVALID_ARG, "no such CUDA device");
    DeviceGuard g(device);
    auto c = std::make_unique<lkg_ctx>();
    c->device = device;
    if (stream) {
      c->stream = static_cast<cudaStream_t>(stream);
    } else {
      LKG_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
      c->own_stream = true;
    }
    c->counters.alloc(sizeof(uint64_t) * 4 * lkg_ctx::kSlots);
    LKG_CUDA(cudaMemsetAsync(c->counters.p, 0, c->counters.bytes, c->stream));
    LKG_CUDA(cudaStreamSynchronize(c->stream));
    *out = c.release();
  });
}

lkg_status lkg_ctx_destroy(lkg_ctx* ctx) {
  return guarded([&] {
    if (!ctx) return;
    DeviceGuard g(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    if (ctx->nccl) ncclCommDestroy(static_cast<ncclComm_t>(ctx->nccl));
    if (ctx->own_stream) cudaStreamDestroy(ctx->stream);
    if (ctx->comm_stream) {
      cudaStreamSynchronize(ctx->comm_stream);
      cudaStreamDestroy(ctx->comm_stream);
    }
    if (ctx->pin) cudaFreeHost(ctx->pin);
    if (ctx->copy_stream) {
      cudaStreamSynchronize(ctx->copy_stream);
      cudaStreamDestroy(ctx->copy_stream);
      for (int b = 0; b < 2; b++) {
        cudaEventDestroy(ctx->ev_copied[b]);
        cudaEventDestroy(ctx->ev_done[b]);
      }
    }
    delete ctx;
  });
}

lkg_status lkg_ctx_synchronize(lkg_ctx* ctx) {
  return guarded([&] {
    need(ctx, "ctx");
    LKG_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

void* lkg_ctx_stream(lkg_ctx* ctx) { return ctx ? ctx->stream : nullptr; }
lkg_status lkg_ctx_set_spline_kernel(lkg_ctx* ctx, int32_t kind) {
  return guarded([&] {
    need(ctx, "ctx");
    if (kind != LKG_SPLINE_AUTO && kind != LKG_SPLINE_SIMT) fail(LKG_ERR_INVALID_ARG, "unknown spline kernel");
    ctx->spline_kernel = kind;
  });
}
uint64_t lkg_ctx_launch_count(lkg_ctx* ctx) { return ctx ? ctx->launches : 0; }
uint64_t lkg_ctx_workspace_bytes(lkg_ctx* ctx) {
  if (!ctx) return 0;
  return ctx->scratch[0].bytes + ctx->scratch[1].bytes + ctx->gather.bytes + ctx->hostio.bytes + ctx->xt.bytes + ctx->ksp.bytes;
}
lkg_status lkg_ctx_trim(lkg_ctx* ctx) {
  return guarded([&] {
    need(ctx, "ctx");
    DeviceGuard g(ctx->device);
    LKG_CUDA(cudaStreamSynchronize(ctx->stream));  // no launch still reads the workspace
    if (ctx->copy_stream) LKG_CUDA(cudaStreamSynchronize(ctx->copy_stream));
    if (ctx->comm_stream) LKG_CUDA(cudaStreamSynchronize(ctx->comm_stream));
    ctx->scratch[0].release();
    ctx->scratch[1].release();
    ctx->gather.release();
    ctx->hostio.release();
    ctx->xt.release();
    ctx->ksp.release();
  });
}

// ------------------------------------------------------------------- layers
static lkg_status upload_impl(lkg_ctx* ctx, const lkg_layer_desc* d, int32_t col0, int32_t col1,
                              lkg_layer** out) {
  return guarded([&] {
    need(ctx, "ctx");
    need(out, "out");
    validate_desc(d);
    if (col0 < 0 || col1 > d->out_dim || col1 <= col0) fail(LKG_ERR_DIMENSION, "bad column range");
    DeviceGuard g(ctx->device);
    auto L = std::make_unique<lkg_layer>();
    L->device = ctx->device;
    L->in_dim = d->in_dim;
    L->out_dim = col1 - col0;
    L->full_out_dim = d->out_dim;
    L->col0 = col0;
    L->col1 = col1;
    L->K = d->K;
    L->L = d->L;
    L->value_repr = d->value_repr;
    L->base_kind = d->value_repr == LKG_REPR_SPLINE_COMPONENT && d->base_kind ? d->base_kind : "";
    L->scheme = d->scheme;
    L->param_dtype = d->param_dtype;
    L->boundary_mode = d->boundary_mode;
    L->oob_policy = d->oob_policy;
    L->knots.assign(d->knots, d->knots + d->K + 1);
    const int64_t din = d->in_dim, m = d->out_dim, K = d->K, Ls = d->L;
    const int64_t E = din * (col1 - col0);
    cudaStream_t st = ctx->stream;
    upload_cols(L->q, d->q_table, din, m, K * Ls, col0, col1, st);
    upload_cols(L->scale, d->scale, din, m, K, col0, col1, st);
    upload_cols(L->ymin, d->y_min, din, m, K, col0, col1, st);
    if (d->float_table) upload_cols(L->float_table, d->float_table, din, m, K * Ls, col0, col1, st);
    if (d->value_repr == LKG_REPR_SPLINE_COMPONENT) {
      L->gains.alloc(sizeof(float) * 3 * E);
      const float* src[3] = {d->edge_base_scale, d->edge_spline_scale, d->edge_out_scale};
      for (int t = 0; t < 3; t++)
        LKG_CUDA(cudaMemcpy2DAsync(L->gains.as<float>() + t * E, sizeof(float) * (col1 - col0),
                                   src[t] + col0, sizeof(float) * m, sizeof(float) * (col1 - col0), din,
                                   cudaMemcpyHostToDevice, st));
    }
    lkg::launch_fuse_gains(ctx, L.get());
    lkg::build_tiles(ctx, L.get());
    LKG_CUDA(cudaStreamSynchronize(st));
    *out = L.release();
  });
}

lkg_status lkg_layer_upload(lkg_ctx* ctx, const lkg_layer_desc* desc, lkg_layer** out) {
  return upload_impl(ctx, desc, 0, desc ? desc->out_dim : 0, out);
}

lkg_status lkg_layer_upload_columns(lkg_ctx* ctx, const lkg_layer_desc* desc, int32_t col0,
                                    int32_t col1, lkg_layer** out) {
  return upload_impl(ctx, desc, col0, col1, out);
}

lkg_status lkg_layer_info_get(const lkg_layer* L, lkg_layer_info* o) {
  return guarded([&] {
    need(L, "layer");
    need(o, "out");
    o->in_dim = L->in_dim;
    o->out_dim = L->out_dim;
    o->K = L->K;
    o->L = L->L;
    o->col0 = L->col0;
    o->col1 = L->col1;
    o->full_out_dim = L->full_out_dim;
    o->value_repr = L->value_repr;
    o->scheme = L->scheme;
    o->param_dtype = L->param_dtype;
    o->boundary_mode = L->boundary_mode;
    o->oob_policy = L->oob_policy;
    o->has_float_table = L->float_table.p != nullptr;
    o->device_bytes = L->device_bytes();
  });
}

const char* lkg_layer_base_kind(const lkg_layer* L) { return L ? L->base_kind.c_str() : ""; }

lkg_status lkg_layer_download(lkg_ctx* ctx, const lkg_layer* L, float* knots, uint8_t* q, float* scale,
                              float* y_min, float* bs, float* ss, float* os, double* ft) {
  return guarded([&] {
    need(ctx, "ctx");
    need(L, "layer");
    DeviceGuard g(ctx->device);
    cudaStream_t st = ctx->stream;
    const int64_t E = (int64_t)L->in_dim * L->out_dim;
    if (knots) std::memcpy(knots, L->knots.data(), sizeof(float) * L->knots.size());
    if (q) {
      if (L->q.p) LKG_CUDA(cudaMemcpyAsync(q, L->q.p, L->q.bytes, cudaMemcpyDeviceToHost, st));
      else lkg::download_q_from_tiles(ctx, L, q);  // large layers keep their codes only in tiles
    }
    if (scale) LKG_CUDA(cudaMemcpyAsync(scale, L->scale.p, L->scale.bytes, cudaMemcpyDeviceToHost, st));
    if (y_min) LKG_CUDA(cudaMemcpyAsync(y_min, L->ymin.p, L->ymin.bytes, cudaMemcpyDeviceToHost, st));
    if (L->gains.p) {
      float* dst[3] = {bs, ss, os};
      for (int t = 0; t < 3; t++)
        if (dst[t])
          LKG_CUDA(cudaMemcpyAsync(dst[t], L->gains.as<float>() + t * E, sizeof(float) * E,
                                   cudaMemcpyDeviceToHost, st));
    }
    if (ft && L->float_table.p)
      LKG_CUDA(cudaMemcpyAsync(ft, L->float_table.p, L->float_table.bytes, cudaMemcpyDeviceToHost, st));
    LKG_CUDA(cudaStreamSynchronize(st));
  });
}

lkg_status lkg_layer_free(lkg_layer* L) {
  return guarded([&] {
    if (!L) return;
    DeviceGuard g(L->device);
    delete L;
  });
}

// -------------------------------------------------------------------- specs
static lkg_status spec_upload_impl(lkg_ctx* ctx, const lkg_spec_desc* d, int32_t col0, int32_t col1,
                                   lkg_spec** out) {
  return guarded([&] {
    need(ctx, "ctx");
    need(out, "out");
    need(d, "desc");
    // KnotGrid (spline.cpp:8-27) and KanLayerSpec (spline.cpp:29-62) validation.
    if (d->degree < 0) fail(LKG_ERR_CONFIG, "degree must be >= 0");
    if (d->K < 1) fail(LKG_ERR_CONFIG, "need at least 2 breakpoints");
    need(d->breakpoints, "breakpoints");
    for (int i = 0; i <= d->K; i++) {
      if (!std::isfinite(d->breakpoints[i])) fail(LKG_ERR_NON_FINITE, "non-finite breakpoint");
      if (i > 0 && !(d->breakpoints[i - 1] < d->breakpoints[i]))
        fail(LKG_ERR_CONFIG, "breakpoints must be strictly increasing");
    }
    if (d->in_dim < 1 || d->out_dim < 1) fail(LKG_ERR_CONFIG, "layer dims must be >= 1");
    if (col0 < 0 || col1 > d->out_dim || col1 <= col0) fail(LKG_ERR_DIMENSION, "bad column range");
    need(d->coeffs, "coeffs");
    need(d->base_scale, "base_scale");
    need(d->spline_scale, "spline_scale");
    need(d->out_scale, "out_scale");
    if (d->base_kind && std::strcmp(d->base_kind, "silu") != 0)
      fail(LKG_ERR_UNSUPPORTED_BASE, std::string("unsupported base kind: \"") + d->base_kind + "\"");
    const int64_t din = d->in_dim, m = d->out_dim, R = d->K + d->degree, mc = col1 - col0;
    for (int64_t i = 0; i < din; i++)
      for (int64_t j = col0; j < col1; j++) {
        const int64_t e = i * m + j;
        for (int64_t r = 0; r < R; r++)
          if (!std::isfinite(d->coeffs[e * R + r])) fail(LKG_ERR_NON_FINITE, "non-finite spline coefficient");
        if (!std::isfinite(d->base_scale[e]) || !std::isfinite(d->spline_scale[e]) ||
            !std::isfinite(d->out_scale[e]))
          fail(LKG_ERR_NON_FINITE, "non-finite edge scale");
      }
    DeviceGuard g(ctx->device);
    auto S = std::make_unique<lkg_spec>();
    S->device = ctx->device;
    S->in_dim = d->in_dim;
    S->out_dim = (int32_t)mc;
    S->full_out_dim = d->out_dim;
    S->col0 = col0;
    S->col1 = col1;
    S->K = d->K;
    S->degree = d->degree;
    S->breakpoints.assign(d->breakpoints, d->breakpoints + d->K + 1);
    cudaStream_t st = ctx->stream;
    upload_cols(S->coeffs, d->coeffs, din, m, R, col0, col1, st);
    const int64_t E = din * mc;
    S->gains.alloc(sizeof(double) * 3 * E);
    const double* src[3] = {d->base_scale, d->spline_scale, d->out_scale};
    for (int t = 0; t < 3; t++)
      LKG_CUDA(cudaMemcpy2DAsync(S->gains.as<double>() + t * E, sizeof(double) * mc, src[t] + col0,
                                 sizeof(double) * m, sizeof(double) * mc, din, cudaMemcpyHostToDevice, st));
    S->col0 = 0;  // device arrays hold only the shard; keep the original range for info
    S->col1 = (int32_t)mc;
    // fp32 spline operands are built lazily by the first lkg_spline_forward (saves memory when a
    // spec is only compiled, e.g. the 33.5M-edge configs[4] layers)
    LKG_CUDA(cudaStreamSynchronize(st));
    *out = S.release();
  });
}

lkg_status lkg_spec_upload(lkg_ctx* ctx, const lkg_spec_desc* desc, lkg_spec** out) {
  return spec_upload_impl(ctx, desc, 0, desc ? desc->out_dim : 0, out);
}
lkg_status lkg_spec_upload_columns(lkg_ctx* ctx, const lkg_spec_desc* desc, int32_t col0, int32_t col1,
                                   lkg_spec** out) {
  return spec_upload_impl(ctx, desc, col0, col1, out);
}
lkg_status lkg_spec_upload_shard(lkg_ctx* ctx, const lkg_spec_desc* desc, int32_t col0, int32_t full_out_dim,
                                 lkg_spec** out) {
  const lkg_status st = spec_upload_impl(ctx, desc, 0, desc ? desc->out_dim : 0, out);
  if (st != LKG_OK) return st;
  return guarded([&] {
    if (col0 < 0 || full_out_dim < col0 + desc->out_dim) {
      lkg_spec_free(*out);
      *out = nullptr;
      fail(LKG_ERR_DIMENSION, "shard columns outside the full layer width");
    }
    (*out)->full_out_dim = full_out_dim;
  });
}
lkg_status lkg_spec_free(lkg_spec* S) {
  return guarded([&] {
    if (!S) return;
    DeviceGuard g(S->device);
    delete S;
  });
}

// ------------------------------------------------------------------ compile
lkg_status lkg_compile_layer(lkg_ctx* ctx, const lkg_spec* S, const lkg_quant_config* qc,
                             const lkg_oob_config* oob, int32_t keep_float, lkg_layer** out) {
  return guarded([&] {
    need(ctx, "ctx");
    need(S, "spec");
    need(qc, "quant config");
    need(oob, "oob config");
    need(out, "out");
    // QuantConfig::validate (compiler.cpp:10-16)
    if (qc->L < 2) fail(LKG_ERR_CONFIG, "samples_per_segment must be >= 2");
    check_scheme(qc->scheme, qc->dtype);
    if (qc->value_repr != LKG_REPR_PHI && qc->value_repr != LKG_REPR_SPLINE_COMPONENT)
      fail(LKG_ERR_CONFIG, "unknown value_repr");
    if (qc->param_dtype != LKG_PARAM_F32 && qc->param_dtype != LKG_PARAM_F16)
      fail(LKG_ERR_CONFIG, "unknown param_dtype");
    if (oob->boundary_mode != LKG_BOUNDARY_HALF_OPEN && oob->boundary_mode != LKG_BOUNDARY_CLOSED)
      fail(LKG_ERR_CONFIG, "unknown boundary_mode");
    if (oob->oob_policy != LKG_OOB_CLIP_X && oob->oob_policy != LKG_OOB_ZERO_SPLINE)
      fail(LKG_ERR_CONFIG, "unknown oob_policy");
    DeviceGuard g(ctx->device);
    const int K = S->K, Ls = qc->L, p = S->degree, R = K + p;
    // Sample points and exact f64 basis windows (build_float_lut, compiler.cpp:29-57).
    std::vector<double> ext;
    lkg::knot_grid(S->breakpoints, p, ext);
    const int64_t npts = (int64_t)K * Ls;
    std::vector<double> full((size_t)npts * R), buf(R + p + 1), silu((size_t)npts, 0.0);
    std::vector<int32_t> first((size_t)npts), last((size_t)npts);
    for (int k = 0; k < K; k++) {
      const double t0 = S->breakpoints[k];
      const double step = (S->breakpoints[k + 1] - t0) / static_cast<double>(Ls);
      for (int l = 0; l < Ls; l++) {
        const int64_t pi = (int64_t)k * Ls + l;
        const double x = t0 + static_cast<double>(l) * step;
        lkg::basis_into(ext, p, x, buf.data());
        std::copy(buf.begin(), buf.begin() + R, full.begin() + pi * R);
        int f = R, la = -1;
        for (int r = 0; r < R; r++)
          if (buf[r] != 0.0) {
            f = std::min(f, r);
            la = r;
          }
        first[pi] = f == R ? 0 : f;
        last[pi] = la < 0 ? 0 : la;
        if (qc->value_repr == LKG_REPR_PHI) silu[pi] = lkg::silu_host(x);
      }
    }
    int W = 1;
    for (int64_t pi = 0; pi < npts; pi++) W = std::max(W, last[pi] - first[pi] + 1);
    std::vector<int32_t> r0((size_t)npts);
    std::vector<double> win((size_t)npts * W, 0.0);
    for (int64_t pi = 0; pi < npts; pi++) {
      int s = std::min(first[pi], R - W);
      r0[pi] = s;
      for (int t = 0; t < W; t++) win[pi * W + t] = full[pi * R + s + t];
    }
    DBuf d_basis, d_r0, d_silu;
    d_basis.alloc(sizeof(double) * win.size());
    d_r0.alloc(sizeof(int32_t) * r0.size());
    d_silu.alloc(sizeof(double) * silu.size());
    cudaStream_t st = ctx->stream;
    LKG_CUDA(cudaMemcpyAsync(d_basis.p, win.data(), d_basis.bytes, cudaMemcpyHostToDevice, st));
    LKG_CUDA(cudaMemcpyAsync(d_r0.p, r0.data(), d_r0.bytes, cudaMemcpyHostToDevice, st));
    LKG_CUDA(cudaMemcpyAsync(d_silu.p, silu.data(), d_silu.bytes, cudaMemcpyHostToDevice, st));

    auto L = std::make_unique<lkg_layer>();
    L->device = ctx->device;
    L->in_dim = S->in_dim;
    L->out_dim = S->col1 - S->col0;
    L->full_out_dim = S->full_out_dim;
    L->col0 = 0;
    L->col1 = L->out_dim;
    L->K = K;
    L->L = Ls;
    L->value_repr = qc->value_repr;
    L->base_kind = qc->value_repr == LKG_REPR_SPLINE_COMPONENT ? "silu" : "";
    L->scheme = qc->scheme;
    L->param_dtype = qc->param_dtype;
    L->boundary_mode = oob->boundary_mode;
    L->oob_policy = oob->oob_policy;
    L->knots.resize(K + 1);
    for (int i = 0; i <= K; i++) L->knots[i] = static_cast<float>(S->breakpoints[i]);
    check_knots(L->knots.data(), K);  // finalize(): f32 knots must stay strictly increasing
    const int64_t E = (int64_t)L->in_dim * L->out_dim;
    L->q.alloc((size_t)E * K * Ls);
    L->scale.alloc(sizeof(float) * E * K);
    L->ymin.alloc(sizeof(float) * E * K);
    if (keep_float) L->float_table.alloc(sizeof(double) * E * K * Ls);
    if (qc->value_repr == LKG_REPR_SPLINE_COMPONENT) L->gains.alloc(sizeof(float) * 3 * E);
    lkg::launch_compile(ctx, S, qc, L.get(), d_basis.as<double>(), d_r0.as<int32_t>(),
                        d_silu.as<double>(), W, keep_float != 0);
    lkg::launch_fuse_gains(ctx, L.get());
    lkg::build_tiles(ctx, L.get());
    LKG_CUDA(cudaStreamSynchronize(st));
    *out = L.release();
  });
}

// ------------------------------------------------------------------ forward
static void reset_slots(lkg_ctx* ctx, int n) {
  LKG_CUDA(cudaMemsetAsync(ctx->counters.p, 0, sizeof(uint64_t) * 4 * n, ctx->stream));
  for (int s = 0; s < n; s++) {
    ctx->rows_seen[s] = 0;
    ctx->in_dim_seen[s] = 0;
  }
}

static void collect_impl(lkg_ctx* ctx, lkg_oob_stats* stats, int n) {
  if (n > lkg_ctx::kSlots) fail(LKG_ERR_INVALID_ARG, "too many layer slots");
  std::vector<uint64_t> h(4 * (size_t)n);
  LKG_CUDA(cudaMemcpyAsync(h.data(), ctx->counters.p, sizeof(uint64_t) * h.size(), cudaMemcpyDeviceToHost,
                           ctx->stream));
  LKG_CUDA(cudaStreamSynchronize(ctx->stream));
  bool nonfinite = false;
  for (int s = 0; s < n; s++) {
    nonfinite |= h[4 * s + 2] != 0;
    if (stats) {
      stats[s].n_samples = ctx->rows_seen[s];
      stats[s].n_oob_samples = h[4 * s + 0];
      stats[s].n_inputs = ctx->rows_seen[s] * (uint64_t)ctx->in_dim_seen[s];
      stats[s].n_oob_inputs = h[4 * s + 1];
    }
  }
  reset_slots(ctx, n);
  if (nonfinite) fail(LKG_ERR_NON_FINITE, "non-finite input value");
}

static void check_chain(const lkg_layer* const* chain, int n) {
  if (n < 1 || !chain) fail(LKG_ERR_CONFIG, "artifact chain is empty");
  if (n > lkg_ctx::kSlots) fail(LKG_ERR_CONFIG, "artifact chain too long");
  for (int l = 0; l < n; l++)
    if (!chain[l]) fail(LKG_ERR_INVALID_ARG, "null layer in chain");
}

static void run_chain(lkg_ctx* ctx, const lkg_layer* const* chain, int n, const float* X, int64_t rows,
                      float* Y) {
  for (int l = 1; l < n; l++)
    if (chain[l]->in_dim != chain[l - 1]->out_dim)
      fail(LKG_ERR_DIMENSION, "artifact chain dimension mismatch between layers " + std::to_string(l - 1) +
                                  " and " + std::to_string(l));
  if (rows > 0 && lkg::can_fuse_chain(chain, n)) {
    // every layer is a small value-table layer: the whole chain in one launch (forward_chain.cu),
    // hidden activations stay in the row's thread
    lkg::launch_forward_chain(ctx, chain, n, X, rows, Y);
    for (int s = 0; s < n; s++) {
      ctx->rows_seen[s] += (uint64_t)rows;
      ctx->in_dim_seen[s] = chain[s]->in_dim;
    }
    return;
  }
  size_t hid = 0;
  for (int l = 0; l + 1 < n; l++) hid = std::max(hid, (size_t)chain[l]->out_dim);
  if (n > 1) {
    ensure(ctx->scratch[0], sizeof(float) * rows * hid);
    ensure(ctx->scratch[1], sizeof(float) * rows * hid);
  }
  const float* cur = X;
  for (int l = 0; l < n; l++) {
    float* dst = l == n - 1 ? Y : ctx->scratch[l & 1].as<float>();
    if (l + 1 < n && rows > 0 && lkg::can_fuse(chain[l], chain[l + 1])) {
      // layer l and the small layer l+1 in one launch; the hidden activations never leave registers
      float* dst2 = l + 1 == n - 1 ? Y : ctx->scratch[(l + 1) & 1].as<float>();
      lkg::launch_forward_tiled(ctx, chain[l], cur, rows, 0, nullptr, l, chain[l + 1], dst2);
      for (int s = l; s <= l + 1; s++) {
        ctx->rows_seen[s] += (uint64_t)rows;
        ctx->in_dim_seen[s] = chain[s]->in_dim;
      }
      cur = dst2;
      l++;
      continue;
    }
    lkg::launch_forward(ctx, chain[l], cur, rows, 0, dst, l, true);
    ctx->rows_seen[l] += (uint64_t)rows;
    ctx->in_dim_seen[l] = chain[l]->in_dim;
    cur = dst;
  }
}

lkg_status lkg_layer_forward(lkg_ctx* ctx, const lkg_layer* L, const float* X, int64_t rows, float* Y,
                             lkg_oob_stats* stats) {
  const lkg_layer* chain[1] = {L};
  return lkg_model_forward(ctx, chain, 1, X, rows, Y, stats);
}

lkg_status lkg_model_forward(lkg_ctx* ctx, const lkg_layer* const* chain, int32_t n, const float* X,
                             int64_t rows, float* Y, lkg_oob_stats* stats) {
  return guarded([&] {
    need(ctx, "ctx");
    check_chain(chain, n);
    if (rows < 0) fail(LKG_ERR_DIMENSION, "negative row count");
    if (rows > 0) {
      need(X, "X");
      need(Y, "Y");
    }
    DeviceGuard g(ctx->device);
    run_chain(ctx, chain, n, X, rows, Y);
    if (stats) collect_impl(ctx, stats, n);
  });
}

// ---------------------------------------------------------------- CUDA graph of a chain forward
struct lkg_graph {
  lkg_ctx* ctx = nullptr;
  cudaGraphExec_t exec = nullptr;
  int32_t n = 0;
  int64_t rows = 0;
  uint64_t kernels = 0;          // launches per replay
  std::vector<int32_t> in_dims;  // per layer slot (OobStats bookkeeping of each replay)
  // The graph's own hidden-activation and transposed-input buffers: the replayed kernels (and the
  // XT tensor map baked into their parameters) keep pointing at these, so later forwards on the
  // same context may grow or free the context's buffers freely.
  lkg::DBuf scratch[2], xt, ksp;
};

// Swaps the graph's buffers into the context for the eager pass and the capture, and back out.
struct GraphBuffers {
  lkg_ctx* ctx;
  lkg_graph* G;
  GraphBuffers(lkg_ctx* c, lkg_graph* g) : ctx(c), G(g) { swap(); }
  ~GraphBuffers() { swap(); }
  void swap() {
    ctx->scratch[0].swap(G->scratch[0]);
    ctx->scratch[1].swap(G->scratch[1]);
    ctx->xt.swap(G->xt);
    ctx->ksp.swap(G->ksp);
  }
};

lkg_status lkg_graph_create(lkg_ctx* ctx, const lkg_layer* const* chain, int32_t n, const float* X, int64_t rows,
                            float* Y, lkg_graph** out) {
  return guarded([&] {
    need(ctx, "ctx");
    need(out, "out");
    *out = nullptr;
    check_chain(chain, n);
    if (rows <= 0) fail(LKG_ERR_DIMENSION, "a captured forward needs at least one row");
    need(X, "X");
    need(Y, "Y");
    DeviceGuard g(ctx->device);
    auto G = std::make_unique<lkg_graph>();
    GraphBuffers own(ctx, G.get());
    // one eager pass first: the graph's buffers sized, kernel attributes set (neither is a stream
    // operation a capture could record), and the chain validated
    run_chain(ctx, chain, n, X, rows, Y);
    LKG_CUDA(cudaStreamSynchronize(ctx->stream));
    reset_slots(ctx, n);
    for (int s = 0; s < n; s++) ctx->rows_seen[s] = 0;
    G->ctx = ctx;
    G->n = n;
    G->rows = rows;
    for (int s = 0; s < n; s++) G->in_dims.push_back(chain[s]->in_dim);
    const uint64_t l0 = ctx->launches;
    cudaGraph_t graph = nullptr;
    LKG_CUDA(cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal));
    try {
      run_chain(ctx, chain, n, X, rows, Y);
    } catch (...) {
      cudaStreamEndCapture(ctx->stream, &graph);
      if (graph) cudaGraphDestroy(graph);
      throw;
    }
    LKG_CUDA(cudaStreamEndCapture(ctx->stream, &graph));
    G->kernels = ctx->launches - l0;
    ctx->launches = l0;
    for (int s = 0; s < n; s++) ctx->rows_seen[s] = 0;  // the capture ran nothing
    const cudaError_t e = cudaGraphInstantiate(&G->exec, graph, 0);
    cudaGraphDestroy(graph);
    LKG_CUDA(e);
    *out = G.release();
  });
}

lkg_status lkg_graph_launch(lkg_graph* G) {
  return guarded([&] {
    need(G, "graph");
    DeviceGuard g(G->ctx->device);
    LKG_CUDA(cudaGraphLaunch(G->exec, G->ctx->stream));
    G->ctx->launches += G->kernels;
    for (int s = 0; s < G->n; s++) {
      G->ctx->rows_seen[s] += (uint64_t)G->rows;
      G->ctx->in_dim_seen[s] = G->in_dims[s];
    }
  });
}

lkg_status lkg_graph_destroy(lkg_graph* G) {
  return guarded([&] {
    if (!G) return;
    DeviceGuard g(G->ctx->device);
    cudaStreamSynchronize(G->ctx->stream);  // no replay still reads the graph's buffers
    if (G->exec) cudaGraphExecDestroy(G->exec);
    delete G;
  });
}

lkg_status lkg_model_forward_host(lkg_ctx* ctx, const lkg_layer* const* chain, int32_t n, const float* Xh,
                                  int64_t rows, float* Yh, lkg_oob_stats* stats) {
  return guarded([&] {
    need(ctx, "ctx");
    check_chain(chain, n);
    if (rows < 0) fail(LKG_ERR_DIMENSION, "negative row count");
    DeviceGuard g(ctx->device);
    const int64_t d = chain[0]->in_dim, mo = chain[n - 1]->out_dim;
    // Row chunks of ~32 MB of X: the H2D copy of chunk c+1 (copy stream) overlaps the chain on
    // chunk c (context stream); two device input buffers, event-ordered.
    // Chunk starts are multiples of kRowAlign rows, so every row keeps its lane phase and the
    // chunked path is bit-identical to one launch.
    const int64_t ch = (std::max<int64_t>(65536, (32ll << 20) / (4 * d)) + lkg::kRowAlign - 1) / lkg::kRowAlign *
                       lkg::kRowAlign;
    const int64_t nch = rows > ch ? (rows + ch - 1) / ch : 1, cr = nch > 1 ? ch : rows;
    const size_t xb = sizeof(float) * cr * d, yb = sizeof(float) * rows * mo;
    const size_t xstride = ((xb + 255) / 256) * 256;
    ensure(ctx->hostio, (nch > 1 ? 2 : 1) * xstride + yb + 256);
    float* dXb[2] = {ctx->hostio.as<float>(), reinterpret_cast<float*>(ctx->hostio.as<char>() + xstride)};
    float* dY = reinterpret_cast<float*>(ctx->hostio.as<char>() + (nch > 1 ? 2 : 1) * xstride);
    if (rows > 0) {
      need(Xh, "X");
      need(Yh, "Y");
    }
    if (nch == 1) {
      if (rows > 0) LKG_CUDA(cudaMemcpyAsync(dXb[0], Xh, xb, cudaMemcpyHostToDevice, ctx->stream));
      run_chain(ctx, chain, n, dXb[0], rows, dY);
    } else {
      if (!ctx->copy_stream) {
        LKG_CUDA(cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking));
        for (int b = 0; b < 2; b++) {
          LKG_CUDA(cudaEventCreateWithFlags(&ctx->ev_copied[b], cudaEventDisableTiming));
          LKG_CUDA(cudaEventCreateWithFlags(&ctx->ev_done[b], cudaEventDisableTiming));
        }
      }
      for (int64_t c = 0; c < nch; c++) {
        const int b = (int)(c & 1);
        const int64_t r0 = c * ch, nr = std::min(ch, rows - r0);
        if (c >= 2) LKG_CUDA(cudaStreamWaitEvent(ctx->copy_stream, ctx->ev_done[b], 0));
        LKG_CUDA(cudaMemcpyAsync(dXb[b], Xh + r0 * d, sizeof(float) * nr * d, cudaMemcpyHostToDevice,
                                 ctx->copy_stream));
        LKG_CUDA(cudaEventRecord(ctx->ev_copied[b], ctx->copy_stream));
        LKG_CUDA(cudaStreamWaitEvent(ctx->stream, ctx->ev_copied[b], 0));
        run_chain(ctx, chain, n, dXb[b], nr, dY + r0 * mo);
        LKG_CUDA(cudaEventRecord(ctx->ev_done[b], ctx->stream));
      }
    }
    if (rows > 0) LKG_CUDA(cudaMemcpyAsync(Yh, dY, yb, cudaMemcpyDeviceToHost, ctx->stream));
    if (stats) collect_impl(ctx, stats, n);
    else LKG_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

// static_cast<float> of n doubles into the pinned staging buffer. The staging is read by the copy
// engine, never by the CPU: streaming (non-temporal) stores skip the write-allocate read of the
// destination lines — the narrowing is bound by host memory bandwidth (measured: 8 and 16 threads take
// the same 12-15 ms per 1M x 78 batch), so a fifth less traffic is a fifth less time.
static void narrow_f64_to_f32(const double* src, float* dst, int64_t n) {
  int64_t e = 0;
#if defined(__SSE2__)
  while (e < n && (reinterpret_cast<uintptr_t>(dst + e) & 15)) {
    dst[e] = static_cast<float>(src[e]);
    e++;
  }
  for (; e + 4 <= n; e += 4) {
    const __m128 lo = _mm_cvtpd_ps(_mm_loadu_pd(src + e)), hi = _mm_cvtpd_ps(_mm_loadu_pd(src + e + 2));
    _mm_stream_ps(dst + e, _mm_movelh_ps(lo, hi));
  }
#endif
  for (; e < n; e++) dst[e] = static_cast<float>(src[e]);
#if defined(__SSE2__)
  _mm_sfence();  // the streaming stores are globally visible before the chunk is reported ready
#endif
}

// The reference's own I/O type: f64 Matrix rows in and out (runtime.hpp:130-148), from pageable
// host memory. Host threads narrow X to fp32 row chunk by row chunk into pinned staging (the
// documented fp32 activations: static_cast<float>), each chunk's H2D (copy stream) and chain (context
// stream) overlap the narrowing of the next; Y comes back through pinned staging and is widened by
// the same threads. Chunk starts are multiples of kRowAlign rows (bit-identical to one launch).
lkg_status lkg_model_forward_host_f64(lkg_ctx* ctx, const lkg_layer* const* chain, int32_t n, const double* Xh,
                                      int64_t rows, double* Yh, lkg_oob_stats* stats) {
  return guarded([&] {
    need(ctx, "ctx");
    check_chain(chain, n);
    if (rows < 0) fail(LKG_ERR_DIMENSION, "negative row count");
    if (rows > 0) {
      need(Xh, "X");
      need(Yh, "Y");
    }
    DeviceGuard g(ctx->device);
    const int64_t d = chain[0]->in_dim, mo = chain[n - 1]->out_dim;
    const int64_t ch = (std::max<int64_t>(65536, (16ll << 20) / (4 * d)) + lkg::kRowAlign - 1) / lkg::kRowAlign *
                       lkg::kRowAlign;
    const int64_t nch = rows > ch ? (rows + ch - 1) / ch : 1, cr = nch > 1 ? ch : rows;
    auto up = [](size_t b) { return (b + 255) / 256 * 256; };
    const size_t xb = up(sizeof(float) * cr * d), yb = up(sizeof(float) * rows * mo);
    ensure(ctx->hostio, 2 * xb + yb + 256);
    float* dX[2] = {ctx->hostio.as<float>(), reinterpret_cast<float*>(ctx->hostio.as<char>() + xb)};
    float* dY = reinterpret_cast<float*>(ctx->hostio.as<char>() + 2 * xb);
    if (ctx->pin_bytes < 2 * xb + yb) {
      if (ctx->pin) LKG_CUDA(cudaFreeHost(ctx->pin));
      ctx->pin = nullptr;
      ctx->pin_bytes = 0;
      LKG_CUDA(cudaMallocHost(&ctx->pin, 2 * xb + yb));
      ctx->pin_bytes = 2 * xb + yb;
    }
    float* hX[2] = {static_cast<float*>(ctx->pin), reinterpret_cast<float*>(static_cast<char*>(ctx->pin) + xb)};
    float* hY = reinterpret_cast<float*>(static_cast<char*>(ctx->pin) + 2 * xb);
    if (!ctx->copy_stream) {
      LKG_CUDA(cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking));
      for (int b = 0; b < 2; b++) {
        LKG_CUDA(cudaEventCreateWithFlags(&ctx->ev_copied[b], cudaEventDisableTiming));
        LKG_CUDA(cudaEventCreateWithFlags(&ctx->ev_done[b], cudaEventDisableTiming));
      }
    }
    static const char* ht_env = getenv("LKG_HOST_THREADS");  // tuning hook
    const int T = ht_env ? std::max(1, atoi(ht_env))
                         : (int)std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
    static const bool verbose = getenv("LKG_VERBOSE") != nullptr;
    const auto t_begin = std::chrono::steady_clock::now();
    auto ms_since = [&] {
      return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_begin).count();
    };
    // host workers: for chunk c, worker t narrows its slice into hX[c & 1] once the H2D of chunk c-2
    // (the previous user of that staging buffer) has completed, then counts itself done
    std::vector<std::atomic<int>> ready((size_t)std::max<int64_t>(nch, 1));
    for (auto& r : ready) r.store(0);
    std::atomic<int64_t> copied_upto{-1};  // chunks whose H2D was enqueued (event recorded)
    std::atomic<bool> abort{false};
    auto worker = [&](int t) {
      for (int64_t c = 0; c < nch && rows > 0 && !abort.load(); c++) {
        const int b = (int)(c & 1);
        const int64_t r0 = c * ch, nr = std::min(cr, rows - r0), ne = nr * d;
        if (c >= 2) {
          while (copied_upto.load(std::memory_order_acquire) < c - 2 && !abort.load()) std::this_thread::yield();
          if (cudaEventSynchronize(ctx->ev_copied[b]) != cudaSuccess) abort.store(true);
        }
        const int64_t e0 = ne * t / T, e1 = ne * (t + 1) / T;
        const double* src = Xh + r0 * d;
        float* dst = hX[b];
        narrow_f64_to_f32(src + e0, dst + e0, e1 - e0);
        ready[(size_t)c].fetch_add(1, std::memory_order_release);
      }
    };
    std::vector<std::thread> pool;
    for (int t = 0; t < T; t++) pool.emplace_back(worker, t);
    try {
      for (int64_t c = 0; c < nch && rows > 0; c++) {
        const int b = (int)(c & 1);
        const int64_t r0 = c * ch, nr = std::min(cr, rows - r0);
        while (ready[(size_t)c].load(std::memory_order_acquire) < T) std::this_thread::yield();
        if (c >= 2) LKG_CUDA(cudaStreamWaitEvent(ctx->copy_stream, ctx->ev_done[b], 0));
        LKG_CUDA(cudaMemcpyAsync(dX[b], hX[b], sizeof(float) * nr * d, cudaMemcpyHostToDevice, ctx->copy_stream));
        LKG_CUDA(cudaEventRecord(ctx->ev_copied[b], ctx->copy_stream));
        copied_upto.store(c, std::memory_order_release);
        LKG_CUDA(cudaStreamWaitEvent(ctx->stream, ctx->ev_copied[b], 0));
        run_chain(ctx, chain, n, dX[b], nr, dY + r0 * mo);
        LKG_CUDA(cudaEventRecord(ctx->ev_done[b], ctx->stream));
      }
    } catch (...) {
      abort.store(true);
      copied_upto.store(nch);
      for (auto& th : pool) th.join();
      throw;
    }
    for (auto& th : pool) th.join();
    const double t_enq = ms_since();
    if (abort.load()) fail(LKG_ERR_CUDA, "host staging of the f64 input failed");
    if (rows > 0) LKG_CUDA(cudaMemcpyAsync(hY, dY, sizeof(float) * rows * mo, cudaMemcpyDeviceToHost, ctx->stream));
    if (stats) collect_impl(ctx, stats, n);
    else LKG_CUDA(cudaStreamSynchronize(ctx->stream));
    const double t_sync = ms_since();
    if (verbose)
      fprintf(stderr, "lkg host_f64: %lld rows, %d threads, %lld chunks: enqueued %.2f ms, synced %.2f ms\n",
              (long long)rows, T, (long long)nch, t_enq, t_sync);
    if (rows > 0) {
      const int64_t ny = rows * mo;
      std::vector<std::thread> wid;
      for (int t = 0; t < T; t++)
        wid.emplace_back([&, t] {
          for (int64_t e = ny * t / T; e < ny * (t + 1) / T; e++) Yh[e] = static_cast<double>(hY[e]);
        });
      for (auto& th : wid) th.join();
    }
  });
}

lkg_status lkg_layer_forward_blocked(lkg_ctx* ctx, const lkg_layer* L, const float* X, int64_t rows, int32_t x_blk,
                                     float* Y, lkg_oob_stats* stats) {
  return guarded([&] {
    need(ctx, "ctx");
    need(L, "layer");
    if (rows < 0) fail(LKG_ERR_DIMENSION, "negative row count");
    if (x_blk < 0 || (x_blk > 0 && L->in_dim % x_blk != 0))
      fail(LKG_ERR_DIMENSION, "block width must divide in_dim");
    if (rows > 0) {
      need(X, "X");
      need(Y, "Y");
    }
    DeviceGuard g(ctx->device);
    lkg::launch_forward(ctx, L, X, rows, x_blk, Y, 0, true);
    ctx->rows_seen[0] += (uint64_t)rows;
    ctx->in_dim_seen[0] = L->in_dim;
    if (stats) collect_impl(ctx, stats, 1);
  });
}

lkg_status lkg_layer_coords(lkg_ctx* ctx, const lkg_layer* L, const float* x, int64_t n, int32_t* in_range,
                            int32_t* k, int32_t* l0) {
  return guarded([&] {
    need(ctx, "ctx");
    need(L, "layer");
    if (n < 0) fail(LKG_ERR_DIMENSION, "negative count");
    if (n > 0) need(x, "x");
    DeviceGuard g(ctx->device);
    lkg::launch_coords(ctx, L, x, n, in_range, k, l0);
    LKG_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

lkg_status lkg_ctx_collect(lkg_ctx* ctx, lkg_oob_stats* stats, int32_t n) {
  return guarded([&] {
    need(ctx, "ctx");
    DeviceGuard g(ctx->device);
    collect_impl(ctx, stats, n);
  });
}

lkg_status lkg_spline_forward(lkg_ctx* ctx, const lkg_spec* S, const float* X, int64_t rows, float* Y) {
  return guarded([&] {
    need(ctx, "ctx");
    need(S, "spec");
    if (rows < 0) fail(LKG_ERR_DIMENSION, "negative row count");
    if (rows == 0) return;
    need(X, "X");
    need(Y, "Y");
    DeviceGuard g(ctx->device);
    lkg::launch_spline(ctx, S, X, rows, Y, nullptr);
  });
}

lkg_status lkg_spline_forward_host(lkg_ctx* ctx, const lkg_spec* S, const float* Xh, int64_t rows, float* Yh) {
  return guarded([&] {
    need(ctx, "ctx");
    need(S, "spec");
    if (rows < 0) fail(LKG_ERR_DIMENSION, "negative row count");
    if (rows == 0) return;
    need(Xh, "X");
    need(Yh, "Y");
    DeviceGuard g(ctx->device);
    const size_t xb = sizeof(float) * rows * S->in_dim, yb = sizeof(float) * rows * (S->col1 - S->col0);
    ensure(ctx->hostio, xb + yb + 256);
    float* dX = ctx->hostio.as<float>();
    float* dY = reinterpret_cast<float*>(ctx->hostio.as<char>() + ((xb + 255) / 256) * 256);
    LKG_CUDA(cudaMemcpyAsync(dX, Xh, xb, cudaMemcpyHostToDevice, ctx->stream));
    lkg::launch_spline(ctx, S, dX, rows, dY, nullptr);
    LKG_CUDA(cudaMemcpyAsync(Yh, dY, yb, cudaMemcpyDeviceToHost, ctx->stream));
    LKG_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

// ---------------------------------------------------------------- element primitives
// Host arrays in and out (these are per-element utilities; the copies are small next to a batch).
extern "C++" {
namespace {
struct Staging {
  lkg::DBuf buf;
  size_t off = 0;
  template <class T>
  T* take(size_t n) {  // 256-byte aligned slices of one device allocation
    T* p = reinterpret_cast<T*>(buf.as<char>() + off);
    off += (sizeof(T) * n + 255) / 256 * 256;
    return p;
  }
};
size_t slice(size_t bytes) { return (bytes + 255) / 256 * 256; }
void h2d(void* d, const void* h, size_t b, cudaStream_t st) {
  if (b) LKG_CUDA(cudaMemcpyAsync(d, h, b, cudaMemcpyHostToDevice, st));
}
void d2h(void* h, const void* d, size_t b, cudaStream_t st) {
  if (h && b) LKG_CUDA(cudaMemcpyAsync(h, d, b, cudaMemcpyDeviceToHost, st));
}
}  // namespace
}  // extern "C++"

lkg_status lkg_lut_coords64(lkg_ctx* ctx, const lkg_layer* L, const double* x, int64_t n, uint8_t* in_range,
                            double* x_clip, int32_t* k, int32_t* l0, int32_t* l1, double* w) {
  return guarded([&] {
    need(ctx, "ctx");
    need(L, "layer");
    if (n < 0) fail(LKG_ERR_DIMENSION, "negative element count");
    if (n == 0) return;
    need(x, "x");
    DeviceGuard g(ctx->device);
    Staging s;
    s.buf.alloc(slice(8 * n) * 3 + slice(n) + slice(4 * n) * 3);
    double* dx = s.take<double>(n);
    double* dxc = s.take<double>(n);
    double* dw = s.take<double>(n);
    uint8_t* din = s.take<uint8_t>(n);
    int32_t* dk = s.take<int32_t>(n);
    int32_t* dl0 = s.take<int32_t>(n);
    int32_t* dl1 = s.take<int32_t>(n);
    h2d(dx, x, 8 * n, ctx->stream);
    lkg::launch_coords64(ctx, L, dx, n, din, dxc, dk, dl0, dl1, dw);
    d2h(in_range, din, n, ctx->stream);
    d2h(x_clip, dxc, 8 * n, ctx->stream);
    d2h(k, dk, 4 * n, ctx->stream);
    d2h(l0, dl0, 4 * n, ctx->stream);
    d2h(l1, dl1, 4 * n, ctx->stream);
    d2h(w, dw, 8 * n, ctx->stream);
    LKG_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

lkg_status lkg_lut_eval(lkg_ctx* ctx, const lkg_layer* L, const int32_t* e, const double* x, int64_t n,
                        double* value, uint8_t* was_oob, double* phi) {
  return guarded([&] {
    need(ctx, "ctx");
    need(L, "layer");
    if (n < 0) fail(LKG_ERR_DIMENSION, "negative element count");
    if (n == 0) return;
    need(e, "e");
    need(x, "x");
    if (L->value_repr == LKG_REPR_SPLINE_COMPONENT && L->base_kind != "silu")  // base_fn, spline.cpp:105-108
      fail(LKG_ERR_UNSUPPORTED_BASE, "unsupported base kind: \"" + L->base_kind + "\"");
    DeviceGuard g(ctx->device);
    Staging s;
    s.buf.alloc(slice(8 * n) * 3 + slice(4 * n) + slice(n) + 256);
    double* dx = s.take<double>(n);
    double* dv = s.take<double>(n);
    double* dp = s.take<double>(n);
    int32_t* de = s.take<int32_t>(n);
    uint8_t* doob = s.take<uint8_t>(n);
    int* flags = s.take<int>(2);
    LKG_CUDA(cudaMemsetAsync(flags, 0, 8, ctx->stream));
    h2d(dx, x, 8 * n, ctx->stream);
    h2d(de, e, 4 * n, ctx->stream);
    lkg::launch_lut_eval(ctx, L, de, dx, n, dv, doob, dp, flags);
    int hf[2];
    d2h(hf, flags, 8, ctx->stream);
    LKG_CUDA(cudaStreamSynchronize(ctx->stream));
    if (hf[0]) fail(LKG_ERR_NON_FINITE, "non-finite input value");  // runtime.cpp:97 (checked first)
    if (hf[1]) fail(LKG_ERR_DIMENSION, "edge index out of range");
    d2h(value, dv, 8 * n, ctx->stream);
    d2h(was_oob, doob, n, ctx->stream);
    d2h(phi, dp, 8 * n, ctx->stream);
    LKG_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

lkg_status lkg_basis_values(lkg_ctx* ctx, const double* bp, int32_t K, int32_t degree, const double* x, int64_t n,
                            double* out) {
  return guarded([&] {
    need(ctx, "ctx");
    need(bp, "breakpoints");
    if (n < 0) fail(LKG_ERR_DIMENSION, "negative element count");
    if (K < 1) fail(LKG_ERR_CONFIG, "need at least 2 breakpoints");
    std::vector<double> b(bp, bp + K + 1);
    check_breakpoints(b, degree);
    if (n == 0) return;
    need(x, "x");
    need(out, "out");
    DeviceGuard g(ctx->device);
    const int64_t R = K + degree;
    Staging s;
    s.buf.alloc(slice(8 * n) + slice(8 * n * R));
    double* dx = s.take<double>(n);
    double* dout = s.take<double>(n * R);
    h2d(dx, x, 8 * n, ctx->stream);
    lkg::launch_basis(ctx, b, degree, dx, n, dout);
    d2h(out, dout, 8 * n * R, ctx->stream);
    LKG_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

lkg_status lkg_edge_phi(lkg_ctx* ctx, const lkg_spec* S, const int32_t* e, const double* x, int64_t n, double* phi) {
  return guarded([&] {
    need(ctx, "ctx");
    need(S, "spec");
    if (n < 0) fail(LKG_ERR_DIMENSION, "negative element count");
    if (n == 0) return;
    need(e, "e");
    need(x, "x");
    need(phi, "phi");
    DeviceGuard g(ctx->device);
    Staging s;
    s.buf.alloc(slice(8 * n) * 2 + slice(4 * n) + 256);
    double* dx = s.take<double>(n);
    double* dp = s.take<double>(n);
    int32_t* de = s.take<int32_t>(n);
    int* flags = s.take<int>(2);
    LKG_CUDA(cudaMemsetAsync(flags, 0, 8, ctx->stream));
    h2d(dx, x, 8 * n, ctx->stream);
    h2d(de, e, 4 * n, ctx->stream);
    lkg::launch_edge_phi(ctx, S, de, dx, n, dp, flags);
    int hf[2];
    d2h(hf, flags, 8, ctx->stream);
    LKG_CUDA(cudaStreamSynchronize(ctx->stream));
    if (hf[1]) fail(LKG_ERR_DIMENSION, "edge index out of range");
    d2h(phi, dp, 8 * n, ctx->stream);
    LKG_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

lkg_status lkg_quantize_segments(lkg_ctx* ctx, const double* v, int64_t nseg, int32_t L, int32_t scheme, int32_t* q,
                                 double* scale, double* y_min) {
  return guarded([&] {
    need(ctx, "ctx");
    if (nseg < 0) fail(LKG_ERR_DIMENSION, "negative segment count");
    if (L < 1) fail(LKG_ERR_CONFIG, "cannot quantize an empty segment");  // compiler.cpp:80
    if (scheme != LKG_SCHEME_SYMMETRIC && scheme != LKG_SCHEME_ASYMMETRIC) fail(LKG_ERR_CONFIG, "unknown scheme");
    if (nseg == 0) return;
    need(v, "values");
    DeviceGuard g(ctx->device);
    const int64_t n = nseg * L;
    Staging s;
    s.buf.alloc(slice(8 * n) + slice(4 * n) + slice(8 * nseg) * 2 + 256);
    double* dv = s.take<double>(n);
    int32_t* dq = s.take<int32_t>(n);
    double* ds = s.take<double>(nseg);
    double* dy = s.take<double>(nseg);
    int* flags = s.take<int>(2);
    LKG_CUDA(cudaMemsetAsync(flags, 0, 8, ctx->stream));
    h2d(dv, v, 8 * n, ctx->stream);
    lkg::launch_quantize(ctx, dv, nseg, L, scheme == LKG_SCHEME_ASYMMETRIC, dq, ds, dy, flags);
    int hf[2];
    d2h(hf, flags, 8, ctx->stream);
    LKG_CUDA(cudaStreamSynchronize(ctx->stream));
    if (hf[0]) fail(LKG_ERR_NON_FINITE, "non-finite table value");
    d2h(q, dq, 4 * n, ctx->stream);
    d2h(scale, ds, 8 * nseg, ctx->stream);
    d2h(y_min, dy, 8 * nseg, ctx->stream);
    LKG_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

// ---------------------------------------------------------------- eval_accuracy
static void eval_impl(lkg_ctx* ctx, const lkg_spec* S, const lkg_layer* L, const void* X, bool x_f64,
                      int64_t rows, lkg_eval_report* out) {
  // metrics.cpp:32-35
  if (S->in_dim != L->in_dim || S->col1 - S->col0 != L->col1 - L->col0 || S->col0 != L->col0)
    fail(LKG_ERR_DIMENSION, "layer and artifact shapes differ");
  if (L->value_repr == LKG_REPR_SPLINE_COMPONENT && L->base_kind != "silu")  // base_fn, spline.cpp:105-108
    fail(LKG_ERR_UNSUPPORTED_BASE, "unsupported base kind: \"" + L->base_kind + "\"");
  lkg_eval_report r{};
  r.n_samples = (uint64_t)rows;
  if (rows > 0) {
    lkg::DBuf acc;
    acc.alloc(2 * sizeof(double) + 8 * sizeof(unsigned long long));
    LKG_CUDA(cudaMemsetAsync(acc.p, 0, acc.bytes, ctx->stream));
    double* dsum = acc.as<double>();
    unsigned long long* u = reinterpret_cast<unsigned long long*>(dsum + 2);
    lkg::launch_eval(ctx, S, L, X, x_f64, rows, dsum, u);
    double hs[2];
    unsigned long long hu[8];
    LKG_CUDA(cudaMemcpyAsync(hs, dsum, sizeof(hs), cudaMemcpyDeviceToHost, ctx->stream));
    LKG_CUDA(cudaMemcpyAsync(hu, u, sizeof(hu), cudaMemcpyDeviceToHost, ctx->stream));
    LKG_CUDA(cudaStreamSynchronize(ctx->stream));
    if (hu[6]) fail(LKG_ERR_NON_FINITE, "non-finite input value");
    double mx[2];
    memcpy(mx, hu, sizeof(mx));
    r.n_inrange_evals = hu[2];
    r.n_oob_evals = hu[3];
    r.n_boundary_evals = hu[4];
    r.n_oob_samples = hu[5];
    r.mae_inrange = hu[2] ? hs[0] / (double)hu[2] : 0.0;
    r.maxabs_inrange = mx[0];
    r.has_oob = hu[3] > 0;
    r.mae_oob = hu[3] ? hs[1] / (double)hu[3] : 0.0;
    r.maxabs_oob = hu[3] ? mx[1] : 0.0;
    r.oob_any_frac = (double)hu[5] / (double)rows;
  }
  *out = r;
}

lkg_status lkg_eval_accuracy(lkg_ctx* ctx, const lkg_spec* S, const lkg_layer* L, const float* X, int64_t rows,
                             lkg_eval_report* out) {
  return guarded([&] {
    need(ctx, "ctx");
    need(S, "spec");
    need(L, "layer");
    need(out, "out");
    if (rows < 0) fail(LKG_ERR_DIMENSION, "negative row count");
    if (rows > 0) need(X, "X");
    DeviceGuard g(ctx->device);
    eval_impl(ctx, S, L, X, false, rows, out);
  });
}

lkg_status lkg_eval_accuracy_host(lkg_ctx* ctx, const lkg_spec* S, const lkg_layer* L, const float* Xh,
                                  int64_t rows, lkg_eval_report* out) {
  return guarded([&] {
    need(ctx, "ctx");
    need(S, "spec");
    need(L, "layer");
    need(out, "out");
    if (rows < 0) fail(LKG_ERR_DIMENSION, "negative row count");
    if (rows > 0) need(Xh, "X");
    DeviceGuard g(ctx->device);
    const size_t xb = sizeof(float) * rows * S->in_dim;
    ensure(ctx->hostio, xb + 256);
    float* dX = ctx->hostio.as<float>();
    if (rows > 0) LKG_CUDA(cudaMemcpyAsync(dX, Xh, xb, cudaMemcpyHostToDevice, ctx->stream));
    eval_impl(ctx, S, L, dX, false, rows, out);
  });
}

lkg_status lkg_eval_accuracy_host_f64(lkg_ctx* ctx, const lkg_spec* S, const lkg_layer* L, const double* Xh,
                                      int64_t rows, lkg_eval_report* out) {
  return guarded([&] {
    need(ctx, "ctx");
    need(S, "spec");
    need(L, "layer");
    need(out, "out");
    if (rows < 0) fail(LKG_ERR_DIMENSION, "negative row count");
    if (rows > 0) need(Xh, "X");
    DeviceGuard g(ctx->device);
    const size_t xb = sizeof(double) * rows * S->in_dim;
    ensure(ctx->hostio, xb + 256);
    double* dX = ctx->hostio.as<double>();
    if (rows > 0) LKG_CUDA(cudaMemcpyAsync(dX, Xh, xb, cudaMemcpyHostToDevice, ctx->stream));
    eval_impl(ctx, S, L, dX, true, rows, out);
  });
}

// ---------------------------------------------------------------- multi-GPU
lkg_status lkg_nccl_unique_id(uint8_t id_out[128]) {
  return guarded([&] {
    need(id_out, "id");
    ncclUniqueId id;
    if (ncclGetUniqueId(&id) != ncclSuccess) fail(LKG_ERR_NCCL, "ncclGetUniqueId failed");
    std::memcpy(id_out, id.internal, 128);
  });
}

lkg_status lkg_ctx_init_nccl(lkg_ctx* ctx, const uint8_t id[128], int32_t nranks, int32_t rank) {
  return guarded([&] {
    need(ctx, "ctx");
    need(id, "id");
    if (nranks < 1 || rank < 0 || rank >= nranks) fail(LKG_ERR_INVALID_ARG, "bad rank/nranks");
    DeviceGuard g(ctx->device);
    ncclUniqueId uid;
    std::memcpy(uid.internal, id, 128);
    ncclComm_t comm;
    const ncclResult_t r = ncclCommInitRank(&comm, nranks, uid, rank);
    if (r != ncclSuccess) fail(LKG_ERR_NCCL, std::string("ncclCommInitRank: ") + ncclGetErrorString(r));
    if (ctx->nccl) ncclCommDestroy(static_cast<ncclComm_t>(ctx->nccl));
    ctx->nccl = comm;
    ctx->nranks = nranks;
    ctx->rank = rank;
  });
}

lkg_status lkg_model_forward_sharded(lkg_ctx* ctx, const lkg_layer* const* chain, int32_t n, const float* X,
                                     int64_t rows, float* Y, lkg_oob_stats* stats) {
  return guarded([&] {
    need(ctx, "ctx");
    check_chain(chain, n);
    if (rows < 0) fail(LKG_ERR_DIMENSION, "negative row count");
    const int G = ctx->nranks;
    if (G > 1 && !ctx->nccl) fail(LKG_ERR_NCCL, "context has no NCCL communicator");
    for (int l = 0; l < n; l++) {
      if (chain[l]->out_dim * G != chain[l]->full_out_dim)
        fail(LKG_ERR_DIMENSION, "column shards must split out_dim evenly across ranks");
      if (l > 0 && chain[l]->in_dim != chain[l - 1]->full_out_dim)
        fail(LKG_ERR_DIMENSION, "artifact chain dimension mismatch between layers " + std::to_string(l - 1) +
                                    " and " + std::to_string(l));
    }
    DeviceGuard g(ctx->device);
    size_t loc = 0, full = 0;
    for (int l = 0; l + 1 < n; l++) {
      loc = std::max(loc, (size_t)chain[l]->out_dim);
      full = std::max(full, (size_t)chain[l]->full_out_dim);
    }
    if (n > 1) {
      ensure(ctx->scratch[0], sizeof(float) * rows * loc);
      ensure(ctx->gather, sizeof(float) * rows * full);
    }
    // Row chunks pipeline the exchange: chunk c of layer l is all-gathered on the
    // communication stream while layer l computes chunk c+1, and layer l+1 starts on chunk c as
    // soon as its gather lands. Per chunk the gathered activations are rank-major blocks
    // [G][rows_c][m_l] (ncclAllGather's layout), consumed in place by the next layer.
    // Chunk c owns a FIXED region of scratch (rows from r0 at the widest local width) and of the
    // gather buffer (at the widest full width) in every layer: layer l+1's chunk c then only
    // touches memory whose last users (layer l's chunk-c kernel and gather) it already waits on,
    // whatever the widths (a region packed by each layer's own width let a widening layer
    // overwrite chunks c+1.. of the previous layer while their gathers were in flight).
    static const char* chunk_env = getenv("LKG_SHARD_CHUNKS");
    int nch = chunk_env ? atoi(chunk_env) : (G > 1 && rows >= 8192 ? 4 : 1);
    nch = (int)std::max<int64_t>(1, std::min<int64_t>(nch, std::max<int64_t>(rows, 1)));
    const int64_t rc = ((rows + nch - 1) / nch + lkg::kRowAlign - 1) / lkg::kRowAlign * lkg::kRowAlign;
    if (nch > 1 && n > 1 && !ctx->comm_stream)
      LKG_CUDA(cudaStreamCreateWithFlags(&ctx->comm_stream, cudaStreamNonBlocking));
    cudaStream_t cs = nch > 1 ? ctx->comm_stream : ctx->stream;
    std::vector<cudaEvent_t> events;
    auto new_event = [&]() {
      cudaEvent_t e;
      LKG_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      events.push_back(e);
      return e;
    };
    std::vector<cudaEvent_t> gathered(nch, nullptr), prev_gathered(nch, nullptr);
    for (int l = 0; l < n; l++) {
      const bool last = l == n - 1;
      const int64_t m_l = chain[l]->out_dim, m_prev = l ? chain[l - 1]->out_dim : 0;
      for (int c = 0; c < nch; c++) {
        const int64_t r0 = c * rc, rn = std::min(rc, rows - r0);
        if (rn <= 0) break;
        const float* in = l == 0 ? X + r0 * chain[0]->in_dim : ctx->gather.as<float>() + (int64_t)G * r0 * (int64_t)full;
        if (l > 0 && nch > 1) LKG_CUDA(cudaStreamWaitEvent(ctx->stream, prev_gathered[c], 0));
        float* dst = last ? Y + r0 * m_l : ctx->scratch[0].as<float>() + r0 * (int64_t)loc;
        lkg::launch_forward(ctx, chain[l], in, rn, l == 0 ? 0 : (int32_t)m_prev, dst, l, true);
        if (last) continue;
        if (nch > 1) {
          const cudaEvent_t done = new_event();
          LKG_CUDA(cudaEventRecord(done, ctx->stream));
          LKG_CUDA(cudaStreamWaitEvent(cs, done, 0));
        }
        float* gdst = ctx->gather.as<float>() + (int64_t)G * r0 * (int64_t)full;
        const size_t cnt = (size_t)rn * m_l;
        if (ctx->nccl) {
          const ncclResult_t r = ncclAllGather(dst, gdst, cnt, ncclFloat, static_cast<ncclComm_t>(ctx->nccl), cs);
          if (r != ncclSuccess) fail(LKG_ERR_NCCL, std::string("ncclAllGather: ") + ncclGetErrorString(r));
        } else {
          LKG_CUDA(cudaMemcpyAsync(gdst, dst, sizeof(float) * cnt, cudaMemcpyDeviceToDevice, cs));
        }
        if (nch > 1) {
          gathered[c] = new_event();
          LKG_CUDA(cudaEventRecord(gathered[c], cs));
        }
      }
      ctx->rows_seen[l] += (uint64_t)rows;
      ctx->in_dim_seen[l] = chain[l]->in_dim;
      prev_gathered.swap(gathered);
    }
    if (nch > 1 && n > 1) {  // the caller's stream sees every gather (and nothing outlives the call)
      const cudaEvent_t tail = new_event();
      LKG_CUDA(cudaEventRecord(tail, cs));
      LKG_CUDA(cudaStreamWaitEvent(ctx->stream, tail, 0));
    }
    for (cudaEvent_t e : events) cudaEventDestroy(e);
    if (stats) collect_impl(ctx, stats, n);
  });
}

// ------------------------------------------------------------------ recipes
lkg_status lkg_recipe_dims(int32_t cfg, int32_t* n_layers, int32_t* dims, int32_t* G, double* lo, double* hi) {
  return guarded([&] {
    need(n_layers, "n_layers");
    need(dims, "dims");
    int nl = 0, g = 0, d[5];
    double a = 0, b = 0;
    lkg::recipe_dims(cfg, &nl, d, &g, &a, &b);
    *n_layers = nl;
    for (int i = 0; i <= nl; i++) dims[i] = d[i];
    if (G) *G = g;
    if (lo) *lo = a;
    if (hi) *hi = b;
  });
}

lkg_status lkg_recipe_layer(int32_t cfg, int32_t layer, int32_t col0, int32_t col1, double* bp, double* coeffs,
                            double* bs, double* ss, double* os) {
  return guarded([&] {
    need(bp, "breakpoints");
    need(coeffs, "coeffs");
    need(bs, "base_scale");
    need(ss, "spline_scale");
    need(os, "out_scale");
    lkg::recipe_layer(cfg, layer, col0, col1, bp, coeffs, bs, ss, os);
  });
}

lkg_status lkg_gen_layer(uint64_t seed, int32_t in_dim, int32_t out_dim, int32_t segments, int32_t degree,
                         double* bp, double* coeffs, double* bs, double* ss, double* os) {
  return guarded([&] {
    if (segments < 1) fail(LKG_ERR_CONFIG, "segments must be >= 1");  // model_gen.cpp:8
    if (degree < 0) fail(LKG_ERR_CONFIG, "degree must be >= 0");
    if (in_dim < 1 || out_dim < 1) fail(LKG_ERR_CONFIG, "layer dims must be >= 1");
    need(bp, "breakpoints");
    need(coeffs, "coeffs");
    need(bs, "base_scale");
    need(ss, "spline_scale");
    need(os, "out_scale");
    lkg::gen_layer(seed, in_dim, out_dim, segments, degree, bp, coeffs, bs, ss, os);
  });
}

lkg_status lkg_gen_inputs(uint64_t seed, int64_t n, int64_t dim, double lo, double hi, int32_t clip, double* X) {
  return guarded([&] {
    if (!(lo < hi)) fail(LKG_ERR_CONFIG, "input range must satisfy lo < hi");  // model_gen.cpp:35
    if (n < 0 || dim < 0) fail(LKG_ERR_DIMENSION, "negative size");
    if (n * dim > 0) need(X, "X");
    lkg::gen_inputs(seed, n, dim, lo, hi, clip != 0, X);
  });
}

lkg_status lkg_recipe_inputs(int32_t cfg, int64_t row0, int64_t rows, float* X) {
  return guarded([&] {
    if (rows > 0) need(X, "X");
    if (row0 < 0 || rows < 0) fail(LKG_ERR_DIMENSION, "negative row range");
    lkg::recipe_inputs(cfg, row0, rows, X);
  });
}

}  // extern "C"
