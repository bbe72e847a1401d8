// checks.cuh — device-side bounds assertions of the forward kernels.
#pragma once
#include <cstdio>

// LKG_CHECKS builds (tools/gpu/checks.sh) compile device-side bounds assertions into the table
// walks: every shared-memory table index, staged-tile address, TMEM column and output coordinate is
// checked against its allocation and the kernel traps with a message on the first violation.
// (compute-sanitizer is closed on the GPU pool; these asserts plus canary buffers and repeat-launch
// bit-identity tests are the memory/race evidence.)
#ifdef LKG_CHECKS
#define LKG_DCHECK(cond, what)                                                                          \
  do {                                                                                                  \
    if (!(cond)) {                                                                                      \
      printf("LKG_CHECKS %s:%d block %d thread %d: %s\n", __FILE__, __LINE__, blockIdx.x, threadIdx.x, \
             what);                                                                                     \
      __trap();                                                                                         \
    }                                                                                                   \
  } while (0)
#else
#define LKG_DCHECK(cond, what) \
  do {                         \
  } while (0)
#endif
