// Microbenchmark: tcgen05.mma (kind::f16, M=128, K=16, f16 accumulate, SS operands) latency from
// issue to the commit's mbarrier completion, single CTA, for N = 64 / 128 / 256, and the time per
// MMA when 8 are issued back to back before one commit.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tc_lat tools/tc_lat.cu
#include <cstdio>
#include "../paper_2310_19373_b200/csrc/qb_tc_ptx.cuh"
using namespace qb::tc;

template <int N>
__global__ void lat(long long* out) {
  __shared__ __align__(1024) uint8_t sA[128 * 32];
  __shared__ __align__(1024) uint8_t sB[256 * 32];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int t = threadIdx.x;
  for (int i = t; i < 128 * 32 / 4; i += 128) reinterpret_cast<uint32_t*>(sA)[i] = 0x3c003c00u;
  for (int i = t; i < 256 * 32 / 4; i += 128) reinterpret_cast<uint32_t*>(sB)[i] = 0x3c003c00u;
  fence_async_smem();
  if (t < 32) tmem_alloc<256>(&tbase);
  if (t == 0) mbar_init(&bar, 1);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (t == 0) {
    const uint64_t ad = smem_desc(smem_u32(sA), 128, 256), bd = smem_desc(smem_u32(sB), 128, 256);
    const uint32_t id = idesc_f16_f16(128, N);
    uint32_t ph = 0;
    long long single = 0, batch = 0;
    for (int rep = 0; rep < 20; ++rep) {
      long long t0 = clock64();
      mma_f16(tbase, ad, bd, id, 0);
      mma_commit(&bar);
      mbar_wait(&bar, ph);
      ph ^= 1;
      long long t1 = clock64();
      for (int k = 0; k < 8; ++k) mma_f16(tbase, ad, bd, id, 0);
      mma_commit(&bar);
      mbar_wait(&bar, ph);
      ph ^= 1;
      long long t2 = clock64();
      if (rep >= 4) single += t1 - t0, batch += t2 - t1;
    }
    out[0] = single / 16;
    out[1] = batch / 16;
  }
  tc_fence_before();
  __syncthreads();
  if (t < 32) tmem_dealloc<256>(tbase);
}

template <int N>
void run(long long* d) {
  lat<N><<<1, 128>>>(d);
  long long h[2];
  cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
  printf("N=%d: single MMA issue->commit wait %lld clk; 8 back-to-back + commit %lld clk (%.1f / MMA)\n", N, h[0],
         h[1], h[1] / 8.0);
}

int main() {
  long long* d;
  cudaMalloc(&d, 16);
  run<64>(d);
  run<128>(d);
  run<256>(d);
  return 0;
}
