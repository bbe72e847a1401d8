// forward_tiled_gc.cu — fwd_tiled variants (see fwd_tiled.cuh)
#include "fwd_tiled.cuh"

namespace lkg {
namespace tiled {

// codes-in-global variants on row-major input (GC)
void launch_gc(int sel, bool f64, int idp, cudaStream_t st, const TiledArgs& a, size_t smem, int grid) {
  switch (sel) {
#define CASE(S)                                                                                                  \
  case S:                                                                                                        \
    if (f64)                                                                                                     \
      launch_idp<kR64, kW64, (S >> 2) & 1, (S >> 1) & 1, S & 1, true, false, 1, true>(idp, st, a, smem, grid);   \
    else                                                                                                         \
      launch_idp<kR, kW, (S >> 2) & 1, (S >> 1) & 1, S & 1, false, false, 1, true>(idp, st, a, smem, grid);      \
    break;
    CASE(0) CASE(1) CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7)
#undef CASE
  }
}

}  // namespace tiled
}  // namespace lkg
