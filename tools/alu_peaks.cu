// ALU-pipe peak microbenchmarks for the roofline denominators.
//
// MEASURED_PEAKS.json only carries HBM and bf16-GEMM peaks; the Gray-code
// traversal is ALU-bound, so this measures the issue-limited throughput of the
// instructions the traversal kernels are built from (FADD, FADD2, FMNMX3,
// DADD, DSETP, IADD3, IMAD, VIMNMX3, plus the FADD2+FMNMX3+LDCU mix of the
// blocked-table inner loop).
//
// Each kernel runs many independent dependency chains per thread so latency is
// hidden; throughput is reported both as lane-ops per SM per clock (from
// %clock64 deltas, frequency-independent) and as lane-ops per second (from CUDA
// events over the whole launch).  Output: one JSON object on stdout.
//
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o alu_peaks alu_peaks.cu
#include <cstdio>
#include <cstdint>
#include <cstring>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); return 1; } } while (0)

constexpr int CH = 16;       // independent chains per thread
constexpr int ITERS = 4096;  // loop trips

__device__ __forceinline__ long long clk() { long long c; asm volatile("mov.u64 %0, %%clock64;" : "=l"(c)); return c; }

struct Cyc { unsigned long long cycles; unsigned long long ops; };

// OP kinds
enum { K_FADD, K_FADD2, K_FMNMX3, K_DADD, K_DSETP_OR, K_IADD3, K_IMAD, K_VIMNMX3, K_MIX_TABLE, K_FFMA, K_NK };
static const char* NAMES[K_NK] = {"fadd", "fadd2", "fmnmx3", "dadd", "dsetp_or", "iadd3", "imad",
                                  "vimnmx3", "mix_fadd2_fmnmx3_ldcu", "ffma"};
// lane-ops per instruction (FADD2 does 2 adds; FMNMX3 / VIMNMX3 count as 2 two-input mins)
static const int OPS_PER_INSTR[K_NK] = {1, 2, 2, 1, 1, 1, 1, 2, 2, 1};

struct Tab { float t[2048]; };

template <int K>
__global__ void __launch_bounds__(256) kern(const __grid_constant__ Tab tab, float* out, Cyc* cyc, float seed) {
  long long t0 = clk();
  float f[CH]; double d[CH]; int iv[CH];
#pragma unroll
  for (int i = 0; i < CH; i++) { f[i] = seed * (i + 1) + threadIdx.x; d[i] = f[i]; iv[i] = (int)f[i]; }
  unsigned pred_acc = 0;
  for (int it = 0; it < ITERS; it++) {
    if constexpr (K == K_FADD) {
#pragma unroll
      for (int i = 0; i < CH; i++) asm volatile("add.rn.f32 %0, %0, %1;" : "+f"(f[i]) : "f"(f[(i + 1) % CH]));
    } else if constexpr (K == K_FFMA) {
#pragma unroll
      for (int i = 0; i < CH; i++) asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(f[i]) : "f"(f[(i + 1) % CH]), "f"(f[(i + 3) % CH]));
    } else if constexpr (K == K_FADD2) {
#pragma unroll
      for (int i = 0; i < CH; i += 2) {
        unsigned long long a, b;
        asm volatile("mov.b64 %0, {%1,%2};" : "=l"(a) : "f"(f[i]), "f"(f[i + 1]));
        asm volatile("mov.b64 %0, {%1,%2};" : "=l"(b) : "f"(f[(i + 2) % CH]), "f"(f[(i + 3) % CH]));
        asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(a) : "l"(b));
        asm volatile("mov.b64 {%0,%1}, %2;" : "=f"(f[i]), "=f"(f[i + 1]) : "l"(a));
      }
    } else if constexpr (K == K_FMNMX3) {
#pragma unroll
      for (int i = 0; i < CH; i++) asm volatile("min.f32 %0, %0, %1, %2;" : "+f"(f[i]) : "f"(f[(i + 1) % CH]), "f"(f[(i + 2) % CH]));
    } else if constexpr (K == K_DADD) {
#pragma unroll
      for (int i = 0; i < CH; i++) asm volatile("add.rn.f64 %0, %0, %1;" : "+d"(d[i]) : "d"(d[(i + 1) % CH]));
    } else if constexpr (K == K_DSETP_OR) {
#pragma unroll
      for (int i = 0; i < CH; i++)
        asm volatile("{ .reg .pred p; setp.lt.f64 p, %1, %2; selp.u32 %0, 1, %0, p; }" : "+r"(pred_acc) : "d"(d[i]), "d"(d[(i + it) % CH]));
    } else if constexpr (K == K_IADD3) {
#pragma unroll
      for (int i = 0; i < CH; i++) asm volatile("add.s32 %0, %0, %1;" : "+r"(iv[i]) : "r"(iv[(i + 1) % CH]));
    } else if constexpr (K == K_IMAD) {
#pragma unroll
      for (int i = 0; i < CH; i++) asm volatile("mad.lo.s32 %0, %0, %1, %2;" : "+r"(iv[i]) : "r"(iv[(i + 1) % CH]), "r"(iv[(i + 5) % CH]));
    } else if constexpr (K == K_VIMNMX3) {
#pragma unroll
      for (int i = 0; i < CH; i++) asm volatile("{ .reg .s32 t; min.s32 t, %0, %1; min.s32 %0, t, %2; }" : "+r"(iv[i]) : "r"(iv[(i + 1) % CH]), "r"(iv[(i + 2) % CH]));
    } else if constexpr (K == K_MIX_TABLE) {
      // the blocked-table inner loop: cand = B_pair + T_pair (uniform/const operand), acc = min3(acc, cand.x, cand.y)
      const int base = (it & 1) * 1024;
#pragma unroll
      for (int i = 0; i < CH; i += 2) {
        unsigned long long a, c, tt;
        float t0f = tab.t[base + 2 * i], t1f = tab.t[base + 2 * i + 1];
        asm volatile("mov.b64 %0, {%1,%2};" : "=l"(a) : "f"(f[i]), "f"(f[i + 1]));
        asm volatile("mov.b64 %0, {%1,%2};" : "=l"(tt) : "f"(t0f), "f"(t1f));
        asm volatile("add.rn.f32x2 %0, %1, %2;" : "=l"(c) : "l"(a), "l"(tt));
        float cx, cy;
        asm volatile("mov.b64 {%0,%1}, %2;" : "=f"(cx), "=f"(cy) : "l"(c));
        asm volatile("min.f32 %0, %0, %1, %2;" : "+f"(f[i + 1]) : "f"(cx), "f"(cy));
      }
    }
  }
  long long t1 = clk();
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < CH; i++) s += f[i] + (float)d[i] + (float)iv[i];
  s += (float)pred_acc;
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) { cyc[blockIdx.x].cycles = (unsigned long long)(t1 - t0); }
}

template <int K>
int run(int sms, int blocks_per_sm, float* dout, Cyc* dcyc, const Tab& tab, int first) {
  int grid = sms * blocks_per_sm;
  kern<K><<<grid, 256>>>(tab, dout, dcyc, 1.0f);  // warm-up
  CK(cudaDeviceSynchronize());
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  kern<K><<<grid, 256>>>(tab, dout, dcyc, 1.0f);
  cudaEventRecord(e1);
  CK(cudaEventSynchronize(e1));
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  Cyc* h = new Cyc[grid];
  CK(cudaMemcpy(h, dcyc, sizeof(Cyc) * grid, cudaMemcpyDeviceToHost));
  double mean_cyc = 0; unsigned long long maxc = 0;
  for (int i = 0; i < grid; i++) { mean_cyc += h[i].cycles; if (h[i].cycles > maxc) maxc = h[i].cycles; }
  mean_cyc /= grid;
  delete[] h;
  // instructions issued per thread in the timed loop
  int instr_per_iter = (K == K_FADD2 || K == K_MIX_TABLE) ? CH / 2 : CH;
  double lane_ops_per_block = (double)ITERS * instr_per_iter * OPS_PER_INSTR[K] * 256.0;
  // per-SM per-clock: blocks co-resident per SM each took mean_cyc cycles
  double lane_ops_per_sm_clk = lane_ops_per_block * blocks_per_sm / (double)maxc;
  double warp_instr_per_sm_clk = (double)ITERS * instr_per_iter * 8.0 * blocks_per_sm / (double)maxc;
  double ops_per_s = lane_ops_per_block * grid / (ms * 1e-3);
  printf("%s\"%s\": {\"lane_ops_per_sm_clk\": %.2f, \"warp_instr_per_sm_clk\": %.3f, \"lane_ops_per_s\": %.4e, "
         "\"ms\": %.4f, \"mean_cycles\": %.0f, \"max_cycles\": %llu, \"implied_mhz\": %.0f}",
         first ? "" : ", ", NAMES[K], lane_ops_per_sm_clk, warp_instr_per_sm_clk, ops_per_s, ms, mean_cyc, maxc,
         (double)maxc / (ms * 1e3));
  fflush(stdout);
  return 0;
}

int main() {
  int dev = 0; cudaDeviceProp prop; CK(cudaGetDeviceProperties(&prop, dev));
  int sms = prop.multiProcessorCount;
  int bps = 4;  // 4 x 256 threads = 32 warps per SM
  float* dout; Cyc* dcyc;
  CK(cudaMalloc(&dout, sizeof(float) * sms * bps * 256));
  CK(cudaMalloc(&dcyc, sizeof(Cyc) * sms * bps));
  static Tab tab; for (int i = 0; i < 2048; i++) tab.t[i] = (float)(i % 97) - 40.f;
  printf("{\"gpu\": \"%s\", \"sms\": %d, \"threads_per_sm\": %d, \"chains_per_thread\": %d, \"results\": {", prop.name, sms, bps * 256, CH);
  run<K_FADD>(sms, bps, dout, dcyc, tab, 1);
  run<K_FFMA>(sms, bps, dout, dcyc, tab, 0);
  run<K_FADD2>(sms, bps, dout, dcyc, tab, 0);
  run<K_FMNMX3>(sms, bps, dout, dcyc, tab, 0);
  run<K_DADD>(sms, bps, dout, dcyc, tab, 0);
  run<K_DSETP_OR>(sms, bps, dout, dcyc, tab, 0);
  run<K_IADD3>(sms, bps, dout, dcyc, tab, 0);
  run<K_IMAD>(sms, bps, dout, dcyc, tab, 0);
  run<K_VIMNMX3>(sms, bps, dout, dcyc, tab, 0);
  run<K_MIX_TABLE>(sms, bps, dout, dcyc, tab, 0);
  printf("}}\n");
  return 0;
}
