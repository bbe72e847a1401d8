// forward_tiled_xt.cu — fwd_tiled variants (see fwd_tiled.cuh)
#include "fwd_tiled.cuh"

namespace lkg {
namespace tiled {

// transposed-input / coordinate-record variants (XT, REC)
void launch_xt(int sel, bool f64, bool gc, int idp, cudaStream_t st, const TiledArgs& a, size_t smem, int grid, bool rec) {
  switch (sel) {
#define CASE(S)                                                                                               \
  case S:                                                                                                     \
    if (f64 && gc)                                                                                            \
      launch_idp<kR64, kW64, (S >> 2) & 1, (S >> 1) & 1, S & 1, true, false, 1, true, false, 1, true>(idp, st, a, smem, \
                                                                                                    grid, rec); \
    else if (f64)                                                                                             \
      launch_idp<kR64, kW64, (S >> 2) & 1, (S >> 1) & 1, S & 1, true, false, 1, false, false, 1, true>(idp, st, a,     \
                                                                                                     smem, grid, rec); \
    else                                                                                                      \
      launch_idp<kR, kW, (S >> 2) & 1, (S >> 1) & 1, S & 1, false, false, 1, false, false, 1, true>(idp, st, a, smem,  \
                                                                                                  grid, rec);  \
    break;
    CASE(0) CASE(1) CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7)
#undef CASE
  }
}

}  // namespace tiled
}  // namespace lkg
