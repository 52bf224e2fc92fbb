// Instantiations of the tensor-core coarse-filter search kernel (large-block geometry).
#include "qb_registry.h"
#include "qb_tc.cuh"

namespace qb {

#define QB_TC(L) \
  LFn { L, tc_kernel<BIG_B1, BIG_B2, L>, finalize_kernel<BIG_BE, L, TPB> }
static const LFn kTc[] = {QB_TC(14), QB_TC(16), QB_TC(18), QB_TC(20), QB_TC(22)};

const LFn* tc_fns(int* count) {
  *count = (int)(sizeof(kTc) / sizeof(kTc[0]));
  return kTc;
}

}  // namespace qb
