// Byte-packed threshold search kernels (qb_coarse8.cuh), compiled to one standalone cubin per chunk
// length (-DQB_IMM_L=<L>) and form (-DQB_IMM8_SUPER=0/1/2: 10-bit blocks, 11-bit or 12-bit super-blocks;
// -DQB_IMM8_APPROX=0/1: exact row terms or the row-bound form), embedded in libqubrute_b200.so like the
// 16-bit ones (qb_k_coarse_imm.cu).  Kernel names:
// qb::coarse8_kernel<BIG_B1, BIG_B2, QB_COARSE_B1, QB_COARSE_B2, L, TPB, APPROX> and
// qb::coarse8s_kernel<..., L, TPB, APPROX, NX> (NX = extra image bits).
#include "qb_coarse8.cuh"
#include "qb_registry.h"

namespace qb {

#ifndef QB_IMM_L
#error "build with -DQB_IMM_L=<chunk length>"
#endif
#ifndef QB_IMM8_SUPER
#define QB_IMM8_SUPER 0
#endif
#ifndef QB_IMM8_APPROX
#define QB_IMM8_APPROX 0
#endif
#if QB_IMM8_SUPER
template __global__ void coarse8s_kernel<BIG_B1, BIG_B2, QB_COARSE_B1, QB_COARSE_B2, QB_IMM_L, TPB, QB_IMM8_APPROX != 0,
                                         QB_IMM8_SUPER>(const __grid_constant__ TableParams);
#else
template __global__ void coarse8_kernel<BIG_B1, BIG_B2, QB_COARSE_B1, QB_COARSE_B2, QB_IMM_L, TPB, QB_IMM8_APPROX != 0>(
    const __grid_constant__ TableParams);
#endif

}  // namespace qb
