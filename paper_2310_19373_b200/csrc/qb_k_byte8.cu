// Table-load byte-packed threshold kernels (QB_VARIANT_BYTE8): the row-bound 11-bit pass of qb_coarse8.cuh with
// its packed table words read from the kernel parameters (no patched module), one instantiation per
// chunk length of the large-block geometry with at least two outer bits.
#include "qb_coarse8.cuh"
#include "qb_registry.h"

namespace qb {

#define QB_B8(L)                                                                                            \
  LFn {                                                                                                     \
    L, coarse8s_kernel<BIG_B1, BIG_B2, QB_COARSE_B1, QB_COARSE_B2, L, TPB, true, 1, true>, finalize_kernel<BIG_BE, L, TPB> \
  }
static const LFn kByte8[] = {QB_B8(12), QB_B8(13), QB_B8(14), QB_B8(16), QB_B8(18), QB_B8(20), QB_B8(22)};

const LFn* byte8_fns(int* count) {
  *count = (int)(sizeof(kByte8) / sizeof(kByte8[0]));
  return kByte8;
}

}  // namespace qb
