// Microbenchmark: TMEM -> register read throughput (tcgen05.ld 32x32b.x32, with/without .pack::16b)
// per SM, 4 warps per CTA, CTAS CTAs per SM.  build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tmem_bw tools/tmem_bw.cu
#include <cstdio>
#include "../paper_2310_19373_b200/csrc/qb_tc_ptx.cuh"
using namespace qb::tc;

template <bool PACK, int COLS>
__global__ void __launch_bounds__(128) tmem_read(int iters, unsigned* out) {
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) tmem_alloc<COLS>(&tbase);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t t = tbase + ((uint32_t)(warp * 32) << 16);
  unsigned acc = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < COLS; c += (PACK ? 64 : 32)) {
      uint32_t r[32];
      if (PACK) tmem_ld32_pack16(t + c, r);
      else tmem_ld32(t + c, r);
      tmem_wait_ld();
#pragma unroll
      for (int i = 0; i < 32; i += 2) acc = __vimin3_u16x2(acc, r[i], r[i + 1]);
    }
  }
  out[blockIdx.x * 128 + threadIdx.x] = acc;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<COLS>(tbase);
}

template <bool PACK, int COLS>
void run(int ctas_per_sm, unsigned* d) {
  const int grid = 148 * ctas_per_sm, iters = 2000;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  tmem_read<PACK, COLS><<<grid, 128>>>(10, d);
  cudaEventRecord(a);
  tmem_read<PACK, COLS><<<grid, 128>>>(iters, d);
  cudaEventRecord(b);
  cudaError_t e = cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  // columns read per SM: ctas * 128 lanes * COLS * iters; a 32-bit cell = one f16 state (unpacked)
  const double cells = (double)grid * 128 * COLS * iters;
  printf("pack=%d cols=%d ctas/SM=%d: %.3f ms, %.1f cells/clk/SM (@1.965 GHz) %s\n", PACK, COLS, ctas_per_sm, ms,
         cells / (ms * 1e-3) / 148 / 1.965e9, e == cudaSuccess ? "" : cudaGetErrorString(e));
}

int main() {
  unsigned* d;
  cudaMalloc(&d, 148 * 4 * 128 * 4);
  run<false, 128>(1, d);
  run<false, 128>(2, d);
  run<false, 128>(4, d);
  run<true, 128>(1, d);
  run<true, 128>(2, d);
  run<true, 128>(4, d);
  run<true, 256>(2, d);
  return 0;
}
