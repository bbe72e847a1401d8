/* c_abi_demo.c — the drop-in boundary from plain C (no C++, no Python): compile a recipe layer
 * on the GPU, run a batch forward from host buffers, round-trip it through a .lut file, and
 * check the loaded layer gives the same outputs. Built by tests/test_capi.py (gcc, C11) against
 * include/lutkan_b200.h and liblutkan_b200.so; run on the B200 by tests/test_gpu_shim.py. */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "lutkan_b200.h"

#define CHECK(call)                                                          \
  do {                                                                       \
    lkg_status st_ = (call);                                                 \
    if (st_ != LKG_OK) {                                                     \
      fprintf(stderr, "%s -> %d: %s\n", #call, (int)st_, lkg_last_error());  \
      return 1;                                                              \
    }                                                                        \
  } while (0)

int main(int argc, char** argv) {
  const char* path = argc > 1 ? argv[1] : "/tmp/c_abi_demo.lut";
  int32_t n_layers = 0, dims[8], G = 0;
  double lo = 0, hi = 0;
  CHECK(lkg_recipe_dims(2, &n_layers, dims, &G, &lo, &hi)); /* configs[1]: [78, 16, 2] */
  const int d = dims[0], m = dims[1], K = G, R = G + 3;
  const int64_t E = (int64_t)d * m, rows = 4096;
  double* bp = malloc(sizeof(double) * (K + 1));
  double* coeffs = malloc(sizeof(double) * E * R);
  double* gains = malloc(sizeof(double) * 3 * E);
  CHECK(lkg_recipe_layer(2, 0, 0, 0, bp, coeffs, gains, gains + E, gains + 2 * E));

  lkg_ctx* ctx = NULL;
  CHECK(lkg_ctx_create(0, NULL, &ctx));
  lkg_spec_desc sd;
  memset(&sd, 0, sizeof(sd));
  sd.in_dim = d;
  sd.out_dim = m;
  sd.K = K;
  sd.degree = 3;
  sd.base_kind = "silu";
  sd.breakpoints = bp;
  sd.coeffs = coeffs;
  sd.base_scale = gains;
  sd.spline_scale = gains + E;
  sd.out_scale = gains + 2 * E;
  lkg_spec* spec = NULL;
  CHECK(lkg_spec_upload(ctx, &sd, &spec));
  lkg_quant_config qc = {64, LKG_SCHEME_SYMMETRIC, LKG_DTYPE_INT8, LKG_REPR_SPLINE_COMPONENT, LKG_INTERP_LINEAR,
                         LKG_PARAM_F32};
  lkg_oob_config oc = {LKG_BOUNDARY_CLOSED, LKG_OOB_CLIP_X};
  lkg_layer* layer = NULL;
  CHECK(lkg_compile_layer(ctx, spec, &qc, &oc, 0, &layer));

  float* X = malloc(sizeof(float) * rows * d);
  float* Y = malloc(sizeof(float) * rows * m);
  float* Y2 = malloc(sizeof(float) * rows * m);
  CHECK(lkg_recipe_inputs(2, 0, rows, X));
  lkg_oob_stats st;
  const lkg_layer* chain[1] = {layer};
  CHECK(lkg_model_forward_host(ctx, chain, 1, X, rows, Y, &st));

  CHECK(lkg_artifact_save(ctx, layer, path, 0));
  lkg_layer* loaded = NULL;
  CHECK(lkg_artifact_load(ctx, path, &loaded));
  const lkg_layer* chain2[1] = {loaded};
  lkg_oob_stats st2;
  CHECK(lkg_model_forward_host(ctx, chain2, 1, X, rows, Y2, &st2));
  int same = memcmp(Y, Y2, sizeof(float) * rows * m) == 0 && st.n_oob_inputs == st2.n_oob_inputs;

  /* the C-ABI reports errors as status codes: a wrong-width batch */
  lkg_status bad = lkg_layer_forward(ctx, layer, X, rows, NULL, NULL);
  printf("c_abi_demo: rows %lld, oob inputs %llu of %llu, y[0][0] %.6f, reload identical %d, null-Y status %d\n",
         (long long)rows, (unsigned long long)st.n_oob_inputs, (unsigned long long)st.n_inputs, Y[0], same,
         (int)bad);
  lkg_layer_free(loaded);
  lkg_layer_free(layer);
  lkg_spec_free(spec);
  lkg_ctx_destroy(ctx);
  free(bp);
  free(coeffs);
  free(gains);
  free(X);
  free(Y);
  free(Y2);
  return same && bad != LKG_OK ? 0 : 2;
}
