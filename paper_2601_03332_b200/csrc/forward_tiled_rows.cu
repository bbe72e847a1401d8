// forward_tiled_rows.cu — fwd_tiled variants (see fwd_tiled.cuh)
#include "fwd_tiled.cuh"

namespace lkg {
namespace tiled {

// row-major variants with codes in shared memory: the epilogue-fused chain step, the small-batch
// walk (one row per lane, 4 stages), balanced rows with one or two x buffers, whole-item walks
void launch_fused(int sel, int idp, cudaStream_t st, const TiledArgs& a, size_t smem, int grid) {
  switch (sel) {
#define CASE(S) \
  case S: launch_idp<kR, kW, (S >> 2) & 1, (S >> 1) & 1, S & 1, false, true, 1, false, true>(idp, st, a, smem, grid); break;
    CASE(0) CASE(1) CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7)
#undef CASE
  }
}

void launch_r1(int sel, int idp, cudaStream_t st, const TiledArgs& a, size_t smem, int grid) {
  switch (sel) {
#define CASE(S)                                                                                                       \
  case S:                                                                                                             \
    launch_idp<1, kW, (S >> 2) & 1, (S >> 1) & 1, S & 1, false, false, 1, false, true, 1, false, 4>(idp, st, a, smem, \
                                                                                                   grid);            \
    break;
    CASE(0) CASE(1) CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7)
#undef CASE
  }
}

void launch_rows(int sel, bool f64, bool xb2, bool bal, int idp, cudaStream_t st, const TiledArgs& a, size_t smem,
                 int grid) {
  switch (sel) {
#define CASE(S)                                                                                                  \
  case S:                                                                                                        \
    if (f64)                                                                                                     \
      launch_idp<kR64, kW64, (S >> 2) & 1, (S >> 1) & 1, S & 1, true>(idp, st, a, smem, grid);                   \
    else if (xb2)                                                                                                \
      launch_idp<kR, kW, (S >> 2) & 1, (S >> 1) & 1, S & 1, false, false, 1, false, true, ((S >> 2) & 1) ? 1 : 2>( \
          idp, st, a, smem, grid);                                                                               \
    else if (bal)                                                                                                \
      launch_idp<kR, kW, (S >> 2) & 1, (S >> 1) & 1, S & 1, false, false, 1, false, true>(idp, st, a, smem, grid); \
    else                                                                                                         \
      launch_idp<kR, kW, (S >> 2) & 1, (S >> 1) & 1, S & 1, false>(idp, st, a, smem, grid);                      \
    break;
    CASE(0) CASE(1) CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7)
#undef CASE
  }
}

}  // namespace tiled
}  // namespace lkg
