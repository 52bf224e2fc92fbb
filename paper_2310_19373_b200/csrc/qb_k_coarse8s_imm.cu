// Super-block byte-packed threshold search kernels (QB_VARIANT_IMM8S, qb_coarse8.cuh), one standalone
// cubin per chunk length (-DQB_IMM_L=<L>), embedded in libqubrute_b200.so (see qb_k_coarse_imm.cu).
// Kernel names: qb::coarse8s_kernel<BIG_B1, BIG_B2, QB_COARSE_B1, QB_COARSE_B2, L, TPB>.
#include "qb_coarse8.cuh"
#include "qb_registry.h"

namespace qb {

#ifndef QB_IMM_L
#error "build with -DQB_IMM_L=<chunk length>"
#endif
template __global__ void coarse8s_kernel<BIG_B1, BIG_B2, QB_COARSE_B1, QB_COARSE_B2, QB_IMM_L, TPB>(
    const __grid_constant__ TableParams);

}  // namespace qb
