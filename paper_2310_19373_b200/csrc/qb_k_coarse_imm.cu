// Patched-immediate coarse search kernels (QB_VARIANT_IMM), compiled to a standalone cubin that is
// embedded in libqubrute_b200.so.  Their coarse table words are placeholder immediates
// (QB_IMM_PH | index, qb_coarse.cuh); the host patches a copy of this cubin with an instance's
// table and loads it with cudaLibraryLoadData (qb_api.cu, imm_module).  Kernel names are the
// mangled qb::coarse_kernel<BIG_B1, BIG_B2, QB_COARSE_B1, QB_COARSE_B2, L, TPB, true>.
#include "qb_coarse.cuh"
#include "qb_registry.h"

namespace qb {

// one cubin per chunk length (-DQB_IMM_L=<L>): each instance load patches and loads only the kernel it runs
#ifndef QB_IMM_L
#error "build with -DQB_IMM_L=<chunk length>"
#endif
template __global__ void coarse_kernel<BIG_B1, BIG_B2, QB_COARSE_B1, QB_COARSE_B2, QB_IMM_L, TPB, true>(
    const __grid_constant__ TableParams);

}  // namespace qb
