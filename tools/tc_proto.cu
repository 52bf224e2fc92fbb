// Prototype check of the tcgen05 building blocks used by the tensor-core coarse pass
// (qb_tc_ptx.cuh): one kind::f16 MMA (M=128, N, K=16) from K-major SWIZZLE_NONE shared-memory
// operands into TMEM, f16 and f32 accumulators, read back with and without .pack::16b.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tc_proto tools/tc_proto.cu
#include <cuda_fp16.h>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>
#include "../paper_2310_19373_b200/csrc/qb_tc_ptx.cuh"

__host__ __device__ constexpr uint32_t off32(int r, int k) {
  return (uint32_t)((r >> 3) * 512 + (k >> 3) * 128 + (r & 7) * 16 + (k & 7) * 2);
}

using namespace qb::tc;

template <int N, bool F16ACC>
__global__ void mma_test(const uint16_t* A, const uint16_t* B, uint32_t* out_raw, uint32_t* out_pack) {
  __shared__ __align__(1024) uint8_t sA[128 * 32];
  __shared__ __align__(1024) uint8_t sB[N * 32];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int t = threadIdx.x, warp = t >> 5;
  for (int k = 0; k < 16; ++k) *reinterpret_cast<uint16_t*>(sA + operand_offset(t, k)) = A[t * 16 + k];
  for (int r = t; r < N; r += 128)
    for (int k = 0; k < 16; ++k) *reinterpret_cast<uint16_t*>(sB + operand_offset(r, k)) = B[r * 16 + k];
  fence_async_smem();
  if (warp == 0) tmem_alloc<(N < 32 ? 32 : N)>(&tbase);
  if (t == 0) mbar_init(&bar, 1);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t taddr = tbase;
  if (t == 0) {
    const uint64_t ad = smem_desc(smem_u32(sA), 128, 256), bd = smem_desc(smem_u32(sB), 128, 256);
    mma_f16(taddr, ad, bd, F16ACC ? idesc_f16_f16(128, N) : idesc_f16_f32(128, N), 0);
    mma_commit(&bar);
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  const uint32_t lane_addr = taddr + ((uint32_t)(warp * 32) << 16);
  for (int c = 0; c < N; c += 32) {
    uint32_t r[32];
    tmem_ld32(lane_addr + c, r);
    tmem_wait_ld();
    for (int i = 0; i < 32; ++i) out_raw[t * N + c + i] = r[i];
  }
  for (int c = 0; c < N; c += 64) {
    uint32_t r[32];
    tmem_ld32_pack16(lane_addr + c, r);
    tmem_wait_ld();
    for (int i = 0; i < 32; ++i) out_pack[t * (N / 2) + c / 2 + i] = r[i];
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<(N < 32 ? 32 : N)>(taddr);
}


// K = 32 (two kind::f16 K-steps), fp32 accumulators, the operand layout of qb_tc.cuh
__global__ void mma_k32(const uint16_t* A, const uint16_t* B, uint32_t* out) {
  __shared__ __align__(1024) uint8_t sA[128 * 64];
  __shared__ __align__(1024) uint8_t sB[128 * 64];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int t = threadIdx.x, warp = t >> 5;
  for (int k = 0; k < 32; ++k) {
    *reinterpret_cast<uint16_t*>(sA + off32(t, k)) = A[t * 32 + k];
    *reinterpret_cast<uint16_t*>(sB + off32(t, k)) = B[t * 32 + k];
  }
  fence_async_smem();
  if (warp == 0) tmem_alloc<128>(&tbase);
  if (t == 0) mbar_init(&bar, 1);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (t == 0) {
    const uint64_t ad = smem_desc(smem_u32(sA), 128, 512), bd = smem_desc(smem_u32(sB), 128, 512);
    mma_f16(tbase, ad, bd, idesc_f16_f32(128, 128), 0);
    mma_f16(tbase, ad + 16, bd + 16, idesc_f16_f32(128, 128), 1);
    mma_commit(&bar);
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  for (int c = 0; c < 128; c += 32) {
    uint32_t r[32];
    tmem_ld32(tbase + ((uint32_t)(warp * 32) << 16) + c, r);
    tmem_wait_ld();
    for (int i = 0; i < 32; ++i) out[t * 128 + c + i] = r[i];
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<128>(tbase);
}

static float u2f(uint32_t u) {
  float f;
  memcpy(&f, &u, 4);
  return f;
}
static uint16_t h(float x) {
  __half v = __float2half_rn(x);
  return *reinterpret_cast<uint16_t*>(&v);
}
static float fh(uint16_t b) {
  __half v;
  *reinterpret_cast<uint16_t*>(&v) = b;
  return __half2float(v);
}

template <int N, bool F16ACC>
static int run(int range) {
  std::vector<uint16_t> A(128 * 16), B(N * 16);
  std::vector<int> Ai(128 * 16), Bi(N * 16);
  srand(7 + N);
  for (int i = 0; i < 128 * 16; ++i) Ai[i] = rand() % (2 * range + 1) - range, A[i] = h((float)Ai[i]);
  for (int i = 0; i < N * 16; ++i) Bi[i] = rand() % (2 * range + 1) - range, B[i] = h((float)Bi[i]);
  uint16_t *dA, *dB;
  uint32_t *dr, *dp;
  cudaMalloc(&dA, A.size() * 2);
  cudaMalloc(&dB, B.size() * 2);
  cudaMalloc(&dr, 128 * N * 4);
  cudaMalloc(&dp, 128 * N * 2);
  cudaMemcpy(dA, A.data(), A.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 2, cudaMemcpyHostToDevice);
  mma_test<N, F16ACC><<<1, 128>>>(dA, dB, dr, dp);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("N=%d f16acc=%d: CUDA error %s\n", N, F16ACC, cudaGetErrorString(e));
    return 1;
  }
  std::vector<uint32_t> raw(128 * N), pk(128 * N / 2);
  cudaMemcpy(raw.data(), dr, raw.size() * 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(pk.data(), dp, pk.size() * 4, cudaMemcpyDeviceToHost);
  int bad_raw = 0, bad_pack = 0;
  for (int m = 0; m < 128; ++m)
    for (int n = 0; n < N; ++n) {
      int ref = 0;
      for (int k = 0; k < 16; ++k) ref += Ai[m * 16 + k] * Bi[n * 16 + k];
      const uint32_t r = raw[m * N + n];
      const float got = F16ACC ? fh((uint16_t)(r & 0xffff)) : u2f(r);
      if (got != (float)ref) {
        if (bad_raw < 4) printf("  raw mismatch m=%d n=%d ref=%d raw=%08x\n", m, n, ref, r);
        ++bad_raw;
      }
      if (F16ACC) {
        const uint32_t p = pk[m * (N / 2) + n / 2];
        const uint16_t b = (n & 1) ? (uint16_t)(p >> 16) : (uint16_t)(p & 0xffff);
        if (fh(b) != (float)ref) {
          if (bad_pack < 4) printf("  pack mismatch m=%d n=%d ref=%d word=%08x\n", m, n, ref, p);
          ++bad_pack;
        }
      }
    }
  printf("N=%d f16acc=%d range=%d: raw mismatches %d, pack mismatches %d; raw[0][0..3] = %08x %08x %08x %08x\n", N,
         F16ACC, range, bad_raw, bad_pack, raw[0], raw[1], raw[2], raw[3]);
  cudaFree(dA);
  cudaFree(dB);
  cudaFree(dr);
  cudaFree(dp);
  return bad_raw + bad_pack ? 1 : 0;
}


// the qb_tc.cuh pair encoding with random fields (hc in [-100, 100], Tc' and O anywhere in their
// ranges): every TMEM cell must equal the exact integer dot product bit for bit
static int run_pairs(int seed) {
  srand(seed);
  std::vector<uint16_t> A(128 * 32, 0), B(128 * 32, 0);
  std::vector<long long> Ai(128 * 32, 0), Bi(128 * 32, 0);
  auto setA = [&](int r, int k, long long v) { Ai[r * 32 + k] = v; A[r * 32 + k] = h((float)v); };
  auto setB = [&](int r, int k, long long v) { Bi[r * 32 + k] = v; B[r * 32 + k] = h((float)v); };
  for (int r = 0; r < 128; ++r) {
    const int O = rand() % 1025;
    for (int i = 0; i < 10; ++i) {
      const int hc = rand() % 201 - 100;
      setA(r, i, hc);
      setA(r, 16 + i, hc);
    }
    setA(r, 10, 1); setA(r, 11, O); setA(r, 12, 2048);
    setA(r, 26, 2048); setA(r, 27, O);
  }
  for (int p = 0; p < 128; ++p) {
    const int zl = (p * 37 + seed) & 511, zh = zl + 512;
    for (int i = 0; i < 10; ++i) {
      setB(p, i, (zl >> i) & 1);
      setB(p, 16 + i, 2048 * ((zh >> i) & 1));
    }
    setB(p, 10, rand() % 1024); setB(p, 11, 1); setB(p, 12, 4096);
    setB(p, 26, rand() % 1024); setB(p, 27, 2048);
  }
  uint16_t *dA, *dB;
  uint32_t* d;
  cudaMalloc(&dA, A.size() * 2);
  cudaMalloc(&dB, B.size() * 2);
  cudaMalloc(&d, 128 * 128 * 4);
  cudaMemcpy(dA, A.data(), A.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 2, cudaMemcpyHostToDevice);
  mma_k32<<<1, 128>>>(dA, dB, d);
  cudaError_t e = cudaDeviceSynchronize();
  std::vector<uint32_t> out(128 * 128);
  cudaMemcpy(out.data(), d, out.size() * 4, cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int m = 0; m < 128; ++m)
    for (int n = 0; n < 128; ++n) {
      long long ref = 0;
      for (int k = 0; k < 32; ++k) ref += Ai[m * 32 + k] * Bi[n * 32 + k];
      if ((double)u2f(out[m * 128 + n]) != (double)ref) {
        if (bad < 4) printf("  k32 mismatch m=%d n=%d ref=%lld got=%.1f\n", m, n, ref, u2f(out[m * 128 + n]));
        ++bad;
      }
    }
  printf("K=32 pair encoding seed %d: %s, %d mismatches\n", seed, e == cudaSuccess ? "ok" : cudaGetErrorString(e), bad);
  cudaFree(dA);
  cudaFree(dB);
  cudaFree(d);
  return bad ? 1 : 0;
}

int main() {
  int bad = 0;
  bad |= run<128, false>(8);
  bad |= run<128, true>(8);
  bad |= run<256, true>(8);
  bad |= run<64, true>(3);
  for (int sd = 1; sd <= 8; ++sd) bad |= run_pairs(sd);
  printf(bad ? "FAIL\n" : "ALL OK\n");
  return bad;
}
