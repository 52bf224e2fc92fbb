// Which pipe does an instruction use?  Interleave it 1:1 with a reference instruction of a known pipe
// and measure warp-instructions per SM per clock (CUDA events x nvidia-smi-sampled clock, like
// tools/alu_peaks.py).  Two instructions on different pipes (each 1 per 2 clk per SMSP) reach ~4/SM/clk;
// on the same pipe ~2/SM/clk.  Kernels: K0 IMAD+IMAD (heavy+heavy), K1 IMAD+VIMNMX3 (heavy+ALU),
// K2 IMAD+HADD2, K3 VIMNMX3+HADD2, K4 IMAD+HMNMX2, K5 VIMNMX3+HMNMX2, K6 HADD2 alone, K7 HMNMX2 alone,
// K8 FADD+IMAD, K9 HADD2+FADD.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/pipe_probe tools/pipe_probe.cu
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>

constexpr int CH = 12, ITERS = 4096, TPB = 512;

__device__ __forceinline__ unsigned imad(unsigned a, unsigned b, unsigned c) {
  unsigned r;
  asm volatile("mad.lo.u32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(c));
  return r;
}
__device__ __forceinline__ unsigned vmin3(unsigned a, unsigned b, unsigned c) {
  unsigned r;
  asm volatile("{ .reg .b32 t; min.u16x2 t, %1, %2; min.u16x2 %0, t, %3; }" : "=r"(r) : "r"(a), "r"(b), "r"(c));
  return r;
}
__device__ __forceinline__ unsigned hadd2(unsigned a, unsigned b) {
  unsigned r;
  asm volatile("add.rn.f16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
  return r;
}
__device__ __forceinline__ unsigned hmin2(unsigned a, unsigned b) {
  unsigned r;
  asm volatile("min.f16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
  return r;
}
__device__ __forceinline__ float fadd(float a, float b) {
  float r;
  asm volatile("add.rn.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b));
  return r;
}

template <int K>
__global__ void __launch_bounds__(TPB, 2) kern(unsigned* out, unsigned seed) {
  unsigned x[CH], y[CH];
  float f[CH];
#pragma unroll
  for (int i = 0; i < CH; i++) {
    x[i] = threadIdx.x * (i + 3) + seed;
    y[i] = 0x3c003c00u + i;  // half2 (1, 1)
    f[i] = (float)(threadIdx.x + i);
  }
  const unsigned one = seed | 1u;
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int i = 0; i < CH; i++) {
      const int j = (i + 1) % CH, k = (i + 5) % CH;
      if constexpr (K == 0) { x[i] = imad(x[i], one, x[j]); y[i] = imad(y[i], one, y[k]); }
      if constexpr (K == 1) { x[i] = imad(x[i], one, x[j]); y[i] = vmin3(y[i], y[j], y[k]); }
      if constexpr (K == 2) { x[i] = imad(x[i], one, x[j]); y[i] = hadd2(y[i], y[k]); }
      if constexpr (K == 3) { x[i] = vmin3(x[i], x[j], x[k]); y[i] = hadd2(y[i], y[k]); }
      if constexpr (K == 4) { x[i] = imad(x[i], one, x[j]); y[i] = hmin2(y[i], y[k]); }
      if constexpr (K == 5) { x[i] = vmin3(x[i], x[j], x[k]); y[i] = hmin2(y[i], y[k]); }
      if constexpr (K == 6) { x[i] = hadd2(x[i], x[j]); y[i] = hadd2(y[i], y[k]); }
      if constexpr (K == 7) { x[i] = hmin2(x[i], x[j]); y[i] = hmin2(y[i], y[k]); }
      if constexpr (K == 8) { f[i] = fadd(f[i], f[j]); x[i] = imad(x[i], one, x[j]); }
      if constexpr (K == 9) { f[i] = fadd(f[i], f[j]); y[i] = hadd2(y[i], y[k]); }
      // the patched-immediate coarse pass's mix: adds on the FMA-heavy pipe with an immediate table
      // word, VIMNMX3 folds, fused VIADDMNMX with an immediate (K10: 2:1:1, K11: 2:1:2)
      if constexpr (K == 10 || K == 11) {
        unsigned c0, c1;
        asm volatile("mad.lo.u32 %0, %1, %2, 0x12340001;" : "=r"(c0) : "r"(x[j]), "r"(one));
        asm volatile("mad.lo.u32 %0, %1, %2, 0x12340002;" : "=r"(c1) : "r"(x[k]), "r"(one));
        y[i] = vmin3(y[i], c0, c1);
        x[i] = __viaddmin_u16x2(x[(i + 3) % CH], 0x12340003u, x[i]);
        if constexpr (K == 11) f[i] = __uint_as_float(__viaddmin_u16x2(x[(i + 7) % CH], 0x12340004u, __float_as_uint(f[i])));
      }
    }
  }
  unsigned acc = 0;
#pragma unroll
  for (int i = 0; i < CH; i++) acc += x[i] ^ y[i] ^ __float_as_uint(f[i]);
  out[blockIdx.x * TPB + threadIdx.x] = acc;
}

template <int K>
void run(int sms, unsigned* d, int launches) {
  const int grid = 2 * sms;
  kern<K><<<grid, TPB>>>(d, 1);
  cudaDeviceSynchronize();
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int r = 0; r < launches; r++) kern<K><<<grid, TPB>>>(d, 1);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double per_i = K == 10 ? 4.0 : K == 11 ? 5.0 : 2.0;
  const double instr = per_i * CH * ITERS * (double)TPB * grid / 32.0;  // warp-instructions per launch
  printf("{\"kernel\": %d, \"ms_per_launch\": %.5f, \"warp_instr_per_s\": %.5e, \"sms\": %d}\n", K, ms / launches,
         instr / (ms / launches * 1e-3), sms);
}

int main(int argc, char** argv) {
  const int k = argc > 1 ? atoi(argv[1]) : 0, launches = argc > 2 ? atoi(argv[2]) : 200;
  cudaDeviceProp prop;
  cudaGetDeviceProperties(&prop, 0);
  unsigned* d;
  cudaMalloc(&d, sizeof(unsigned) * prop.multiProcessorCount * 2 * TPB);
  switch (k) {
    case 0: run<0>(prop.multiProcessorCount, d, launches); break;
    case 1: run<1>(prop.multiProcessorCount, d, launches); break;
    case 2: run<2>(prop.multiProcessorCount, d, launches); break;
    case 3: run<3>(prop.multiProcessorCount, d, launches); break;
    case 4: run<4>(prop.multiProcessorCount, d, launches); break;
    case 5: run<5>(prop.multiProcessorCount, d, launches); break;
    case 6: run<6>(prop.multiProcessorCount, d, launches); break;
    case 7: run<7>(prop.multiProcessorCount, d, launches); break;
    case 8: run<8>(prop.multiProcessorCount, d, launches); break;
    case 9: run<9>(prop.multiProcessorCount, d, launches); break;
    case 10: run<10>(prop.multiProcessorCount, d, launches); break;
    case 11: run<11>(prop.multiProcessorCount, d, launches); break;
  }
  return 0;
}
