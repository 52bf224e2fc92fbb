// Instantiations of the batch kernels: one CTA per instance (indexed by block bits B), and the
// warp-per-instance kernel for 12 <= n <= 17.
#include "qb_batch.cuh"
#include "qb_registry.h"

namespace qb {

static const BatchFn kBatch[] = {nullptr,
                                 batch_kernel<0, 1>, batch_kernel<1, 1>, batch_kernel<1, 2>, batch_kernel<2, 2>,
                                 batch_kernel<2, 3>, batch_kernel<3, 3>, batch_kernel<3, 4>, batch_kernel<4, 4>,
                                 batch_kernel<4, 5>, batch_kernel<5, 5>};

const BatchFn* batch_fns(int* count) {
  *count = (int)(sizeof(kBatch) / sizeof(kBatch[0]));
  return kBatch;
}

BatchFn batch_warp_fn(int* warps, int* nmin, int* nmax) {
  *warps = BATCHW_WARPS;
  *nmin = 12;
  *nmax = BATCHW_NMAX;
  return batch_warp_kernel;
}

}  // namespace qb
