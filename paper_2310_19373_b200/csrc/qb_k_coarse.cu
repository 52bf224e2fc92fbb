// Instantiations of the coarse-filter search kernel (large-block geometry).
#include "qb_coarse.cuh"
#include "qb_registry.h"

namespace qb {

#define QB_C(L) \
  LFn { L, coarse_kernel<BIG_B1, BIG_B2, QB_COARSE_B1, QB_COARSE_B2, L, TPB>, finalize_kernel<BIG_BE, L, TPB> }
static const LFn kCoarse[] = {QB_C(10), QB_C(11), QB_C(12), QB_C(13), QB_C(14),
                              QB_C(16), QB_C(18), QB_C(20), QB_C(22)};

const LFn* coarse_fns(int* count) {
  *count = (int)(sizeof(kCoarse) / sizeof(kCoarse[0]));
  return kCoarse;
}

}  // namespace qb
