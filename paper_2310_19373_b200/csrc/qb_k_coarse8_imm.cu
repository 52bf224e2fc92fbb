// Byte-packed threshold search kernels (QB_VARIANT_IMM8, qb_coarse8.cuh), compiled to one standalone
// cubin per chunk length (-DQB_IMM_L=<L>) and embedded in libqubrute_b200.so like the 16-bit ones
// (qb_k_coarse_imm.cu).  Kernel names: qb::coarse8_kernel<BIG_B1, BIG_B2, QB_COARSE_B1, QB_COARSE_B2, L, TPB>.
#include "qb_coarse8.cuh"
#include "qb_registry.h"

namespace qb {

#ifndef QB_IMM_L
#error "build with -DQB_IMM_L=<chunk length>"
#endif
template __global__ void coarse8_kernel<BIG_B1, BIG_B2, QB_COARSE_B1, QB_COARSE_B2, QB_IMM_L, TPB>(
    const __grid_constant__ TableParams);

}  // namespace qb
