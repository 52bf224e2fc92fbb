// ALU-pipe peak microbenchmarks for the roofline denominators.
//
// MEASURED_PEAKS.json only carries HBM and bf16-GEMM peaks; the Gray-code traversal is
// ALU-bound, so this measures the issue-limited throughput of the instructions the traversal
// kernels are built from (FADD, FADD2, FFMA, FMNMX3, DADD, IADD3, VIMNMX3) and of the
// FADD2 + FMNMX3 + LDCU.128 mix of the table kernel's inner loop.
//
// Each kernel keeps 16 independent dependency chains per thread, 2 CTAs x 512 threads per SM
// (32 warps/SM), ~2-5 ms per launch.  Reported per kernel: lane-ops/s from CUDA events over the
// launch (many back-to-back launches); tools/alu_peaks.py runs one kernel per process while
// nvidia-smi samples the SM clock and converts to per-SM-per-clock figures with the sampled clock.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/alu_peaks tools/alu_peaks.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>

#define CK(x)                                                                                 \
  do {                                                                                        \
    cudaError_t e = (x);                                                                      \
    if (e != cudaSuccess) {                                                                   \
      fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__);       \
      return 1;                                                                               \
    }                                                                                         \
  } while (0)

constexpr int CH = 16;
constexpr int ITERS = 8192;
constexpr int TPB = 512;

__device__ __forceinline__ long long clk() {
  long long c;
  asm volatile("mov.u64 %0, %%clock64;" : "=l"(c));
  return c;
}

enum { K_FADD, K_FADD2, K_FFMA, K_FMNMX3, K_DADD, K_IADD3, K_VIMNMX3, K_MIX, K_VIADD16, K_VMIN3_16, K_MIX16, K_ISSUE, K_NK };
static const char* NAMES[K_NK] = {"fadd", "fadd2", "ffma", "fmnmx3", "dadd", "iadd3", "vimnmx3",
                                  "mix_fadd2_fmnmx3_ldcu128", "viadd_16x2", "vimnmx3_s16x2",
                                  "mix16_viadd2_vimnmx3_ldcu128", "issue_fadd_iadd3"};
// lane-operations per instruction: FADD2 / IADD3 = 2 adds, FMNMX3 / VIMNMX3 = 2 two-input mins,
// MIX counts states (one FADD2 + one FMNMX3 per 2 states)
static const double OPS[K_NK] = {1, 2, 1, 2, 1, 2, 2, 2, 2, 4, 2, 1};
// MIX16 per iteration: 8 VIADD.16x2 (16 states) + 4 VIMNMX3.S16x2; counted as 8 "instructions" of 2 states
static const int INSTR_PER_ITER[K_NK] = {CH, CH / 2, CH, CH, CH, CH, CH, CH / 2, CH, CH, CH / 2, 2 * CH};

struct Tab {
  float t[2048];
};

template <int K>
__global__ void __launch_bounds__(TPB, 2) kern(const __grid_constant__ Tab tab, float* out, long long* cyc) {
  const long long t0 = clk();
  float acc = 0.f;
  if constexpr (K == K_DADD) {
    double d[CH];
#pragma unroll
    for (int i = 0; i < CH; i++) d[i] = threadIdx.x + i;
    for (int it = 0; it < ITERS; it++)
#pragma unroll
      for (int i = 0; i < CH; i++) asm volatile("add.rn.f64 %0, %0, %1;" : "+d"(d[i]) : "d"(d[(i + 1) % CH]));
#pragma unroll
    for (int i = 0; i < CH; i++) acc += (float)d[i];
  } else if constexpr (K == K_VIADD16 || K == K_VMIN3_16 || K == K_MIX16) {
    unsigned v[CH];
#pragma unroll
    for (int i = 0; i < CH; i++) v[i] = threadIdx.x * (i + 3);
    for (int it = 0; it < ITERS; it++) {
      if constexpr (K == K_VIADD16) {
#pragma unroll
        for (int i = 0; i < CH; i++) asm volatile("add.s16x2 %0, %0, %1;" : "+r"(v[i]) : "r"(v[(i + 1) % CH]));
      } else if constexpr (K == K_VMIN3_16) {
#pragma unroll
        for (int i = 0; i < CH; i++)
          asm volatile("{ .reg .b32 t; min.s16x2 t, %0, %1; min.s16x2 %0, t, %2; }" : "+r"(v[i]) : "r"(v[(i + 1) % CH]), "r"(v[(i + 2) % CH]));
      } else {
        // packed-int16 table loop: c = B pair + T pair (constant bank), acc = min3(acc, c0, c1)
        const int base = (it & 1) * 1024;
#pragma unroll
        for (int i = 0; i < CH; i += 4) {
          const uint4 t = *reinterpret_cast<const uint4*>(&tab.t[base + 2 * i]);
          unsigned c0, c1;
          asm("add.s16x2 %0, %1, %2;" : "=r"(c0) : "r"(v[i]), "r"(t.x));
          asm("add.s16x2 %0, %1, %2;" : "=r"(c1) : "r"(v[i + 1]), "r"(t.y));
          asm volatile("{ .reg .b32 m; min.s16x2 m, %0, %1; min.s16x2 %0, m, %2; }" : "+r"(v[i + 2]) : "r"(c0), "r"(c1));
          asm("add.s16x2 %0, %1, %2;" : "=r"(c0) : "r"(v[i + 1]), "r"(t.z));
          asm("add.s16x2 %0, %1, %2;" : "=r"(c1) : "r"(v[i]), "r"(t.w));
          asm volatile("{ .reg .b32 m; min.s16x2 m, %0, %1; min.s16x2 %0, m, %2; }" : "+r"(v[i + 3]) : "r"(c0), "r"(c1));
        }
      }
    }
#pragma unroll
    for (int i = 0; i < CH; i++) acc += (float)(v[i] & 0xffff);
  } else if constexpr (K == K_ISSUE) {
    // issue-slot peak: every iteration issues one FADD (FMA pipes) and one IADD3 (ALU pipe) per chain,
    // independent pipes, so the SMSP can issue up to one instruction per clock
    float f[CH];
    int v[CH];
#pragma unroll
    for (int i = 0; i < CH; i++) {
      f[i] = threadIdx.x * 0.5f + i;
      v[i] = threadIdx.x * (i + 3);
    }
    for (int it = 0; it < ITERS; it++) {
#pragma unroll
      for (int i = 0; i < CH; i++) {
        asm volatile("add.rn.f32 %0, %0, %1;" : "+f"(f[i]) : "f"(f[(i + 1) % CH]));
        asm volatile("{ .reg .s32 t; add.s32 t, %0, %1; add.s32 %0, t, %2; }" : "+r"(v[i]) : "r"(v[(i + 1) % CH]), "r"(v[(i + 2) % CH]));
      }
    }
#pragma unroll
    for (int i = 0; i < CH; i++) acc += f[i] + (float)v[i];
  } else if constexpr (K == K_IADD3 || K == K_VIMNMX3) {
    int v[CH];
#pragma unroll
    for (int i = 0; i < CH; i++) v[i] = threadIdx.x * (i + 3);
    for (int it = 0; it < ITERS; it++) {
#pragma unroll
      for (int i = 0; i < CH; i++) {
        if constexpr (K == K_IADD3)
          asm volatile("{ .reg .s32 t; add.s32 t, %0, %1; add.s32 %0, t, %2; }" : "+r"(v[i]) : "r"(v[(i + 1) % CH]), "r"(v[(i + 2) % CH]));
        else
          asm volatile("{ .reg .s32 t; min.s32 t, %0, %1; min.s32 %0, t, %2; }" : "+r"(v[i]) : "r"(v[(i + 1) % CH]), "r"(v[(i + 2) % CH]));
      }
    }
#pragma unroll
    for (int i = 0; i < CH; i++) acc += (float)v[i];
  } else {
    float f[CH];
#pragma unroll
    for (int i = 0; i < CH; i++) f[i] = threadIdx.x * 0.5f + i;
    for (int it = 0; it < ITERS; it++) {
      if constexpr (K == K_FADD) {
#pragma unroll
        for (int i = 0; i < CH; i++) asm volatile("add.rn.f32 %0, %0, %1;" : "+f"(f[i]) : "f"(f[(i + 1) % CH]));
      } else if constexpr (K == K_FFMA) {
#pragma unroll
        for (int i = 0; i < CH; i++)
          asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(f[i]) : "f"(f[(i + 1) % CH]), "f"(f[(i + 3) % CH]));
      } else if constexpr (K == K_FMNMX3) {
#pragma unroll
        for (int i = 0; i < CH; i++)
          asm volatile("min.f32 %0, %0, %1, %2;" : "+f"(f[i]) : "f"(f[(i + 1) % CH]), "f"(f[(i + 2) % CH]));
      } else if constexpr (K == K_FADD2) {
#pragma unroll
        for (int i = 0; i < CH; i += 2) {
          float2 a = make_float2(f[i], f[i + 1]);
          a = __fadd2_rn(a, make_float2(f[(i + 2) % CH], f[(i + 3) % CH]));
          f[i] = a.x;
          f[i + 1] = a.y;
        }
      } else if constexpr (K == K_MIX) {
        // table-kernel inner loop: cand = B pair + T pair (constant bank), acc = min3(acc, cand)
        const int base = (it & 1) * 1024;
#pragma unroll
        for (int i = 0; i < CH; i += 2) {
          const float2 t = *reinterpret_cast<const float2*>(&tab.t[base + 2 * i]);
          const float2 c = __fadd2_rn(make_float2(f[i], f[(i + 5) % CH]), t);
          f[i + 1] = fminf(fminf(f[i + 1], c.x), c.y);
        }
      }
    }
#pragma unroll
    for (int i = 0; i < CH; i++) acc += f[i];
  }
  const long long t1 = clk();
  out[blockIdx.x * TPB + threadIdx.x] = acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int K>
int run(int sms, float* dout, long long* dcyc, const Tab& tab, int launches) {
  const int grid = sms * 2;
  kern<K><<<grid, TPB>>>(tab, dout, dcyc);
  CK(cudaDeviceSynchronize());
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  // back to back for `launches` launches (long enough for nvidia-smi to sample the SM clock)
  cudaEventRecord(e0);
  for (int rep = 0; rep < launches; rep++) kern<K><<<grid, TPB>>>(tab, dout, dcyc);
  cudaEventRecord(e1);
  CK(cudaEventSynchronize(e1));
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double per_launch_ms = ms / launches;
  const double instr = (double)ITERS * INSTR_PER_ITER[K] * TPB * grid;  // thread-instructions per launch
  printf("{\"kernel\": \"%s\", \"launches\": %d, \"ms_per_launch\": %.5f, \"thread_instr_per_launch\": %.6e, "
         "\"lane_ops_per_instr\": %.1f, \"lane_ops_per_s\": %.5e, \"warp_instr_per_s\": %.5e, \"sms\": %d}\n",
         NAMES[K], launches, per_launch_ms, instr, OPS[K], instr * OPS[K] / (per_launch_ms * 1e-3),
         instr / 32.0 / (per_launch_ms * 1e-3), sms);
  fflush(stdout);
  return 0;
}

int main(int argc, char** argv) {
  if (argc < 2) {
    printf("usage: alu_peaks <kernel index 0..%d> [launches]\n", K_NK - 1);
    for (int k = 0; k < K_NK; k++) printf("  %d %s\n", k, NAMES[k]);
    return 2;
  }
  const int k = atoi(argv[1]);
  const int launches = argc > 2 ? atoi(argv[2]) : 400;
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, 0));
  const int sms = prop.multiProcessorCount;
  float* dout;
  long long* dcyc;
  CK(cudaMalloc(&dout, sizeof(float) * sms * 2 * TPB));
  CK(cudaMalloc(&dcyc, sizeof(long long) * sms * 2));
  static Tab tab;
  for (int i = 0; i < 2048; i++) tab.t[i] = (float)(i % 97) - 40.f;
  switch (k) {
    case K_FADD: return run<K_FADD>(sms, dout, dcyc, tab, launches);
    case K_FADD2: return run<K_FADD2>(sms, dout, dcyc, tab, launches);
    case K_FFMA: return run<K_FFMA>(sms, dout, dcyc, tab, launches);
    case K_FMNMX3: return run<K_FMNMX3>(sms, dout, dcyc, tab, launches);
    case K_DADD: return run<K_DADD>(sms, dout, dcyc, tab, launches);
    case K_IADD3: return run<K_IADD3>(sms, dout, dcyc, tab, launches);
    case K_VIMNMX3: return run<K_VIMNMX3>(sms, dout, dcyc, tab, launches);
    case K_MIX: return run<K_MIX>(sms, dout, dcyc, tab, launches);
    case K_VIADD16: return run<K_VIADD16>(sms, dout, dcyc, tab, launches);
    case K_VMIN3_16: return run<K_VMIN3_16>(sms, dout, dcyc, tab, launches);
    case K_MIX16: return run<K_MIX16>(sms, dout, dcyc, tab, launches);
    case K_ISSUE: return run<K_ISSUE>(sms, dout, dcyc, tab, launches);
  }
  return 2;
}
