// Field-walk traversal kernel (QB_VARIANT_FIELDWALK): the per-step form of Alg. 1
// (reference _kernels.py:63-74) on sm_100a.
//
// Each thread walks its chunk's 2^L free-bit states in reflected Gray order.  Every step
// flips bit l = ctz(t), applies Eq. 3 (v += s_l * f_l, with f_l = Q_ll + sum_j Q~_lj x_j the
// local field) and then the row/column update f_j += s_l * Q~_lj of every local field.  All
// L fields live in registers.  The walk is built from 64-step units unrolled at compile time
// (flip bit and, except for bit 5, direction are constants; field rows are constant-bank
// pairs added with FADD2); the flips of bits >= 6 dispatch to one compile-time branch per
// bit.  Minima are reported per 1024-state block (bits 0..9), the same blocks as the table
// kernel, so tie keys, per-chunk minima, finalize and collect kernels are shared.
//
// Values are the same exact integers as the table kernel (Q scaled by 2^e, all |partial
// sums| < 2^24, quantized with every free bit counted as a block bit).
#pragma once
#include "qb_table.cuh"

namespace qb {

constexpr int FW_UB = 6;   // unrolled unit: 2^6 steps
constexpr int FW_RB = 10;  // reporting block: 2^10 states (= table kernel block)

// flip bit ELL with compile-time sign SG
template <int L, int ELL, int SG>
__device__ __forceinline__ void fw_flip_c(const TableParams& p, float& v, float (&f)[L]) {
  v = (SG > 0) ? v + f[ELL] : v - f[ELL];
#pragma unroll
  for (int jj = 0; jj + 1 < L; jj += 2) {
    const float2 q = *reinterpret_cast<const float2*>(&p.Qs[ELL][jj]);
    const float2 r = (SG > 0) ? __fadd2_rn(make_float2(f[jj], f[jj + 1]), q)
                              : __fadd2_rn(make_float2(f[jj], f[jj + 1]), make_float2(-q.x, -q.y));
    f[jj] = r.x;
    f[jj + 1] = r.y;
  }
  if constexpr (L & 1) f[L - 1] = (SG > 0) ? f[L - 1] + p.Qs[ELL][L - 1] : f[L - 1] - p.Qs[ELL][L - 1];
}

// flip bit ELL with a runtime sign (one per 32 steps or rarer)
template <int L, int ELL>
__device__ __forceinline__ void fw_flip_r(const TableParams& p, float sg, float& v, float (&f)[L]) {
  v = fmaf(sg, f[ELL], v);
#pragma unroll
  for (int jj = 0; jj < L; ++jj) f[jj] = fmaf(sg, p.Qs[ELL][jj], f[jj]);
}

template <int L, int ELL>
__device__ __forceinline__ void fw_flip_dispatch(const TableParams& p, int ell, float sg, float& v, float (&f)[L]) {
  if constexpr (ELL < L) {
    if (ell == ELL) fw_flip_r<L, ELL>(p, sg, v, f);
    else fw_flip_dispatch<L, ELL + 1>(p, ell, sg, v, f);
  }
}

__host__ __device__ constexpr int fw_ctz(int k) { return (k & 1) ? 0 : 1 + fw_ctz(k >> 1); }

// Steps T .. 2^FW_UB - 1 of a unit.  Direction of bit l at step t: new bit = 1 ^ bit(l+1) of t;
// for l = FW_UB-1 that bit lies outside the unit (bit 6 of the counter), passed as sg5.
template <int L, int T>
__device__ __forceinline__ void fw_unit_steps(const TableParams& p, float sg5, float& v, float& m, float (&f)[L]) {
  if constexpr (T < (1 << FW_UB)) {
    constexpr int ELL = fw_ctz(T);
    if constexpr (ELL + 1 < FW_UB) {
      constexpr int SG = ((T >> (ELL + 1)) & 1) ? -1 : 1;
      fw_flip_c<L, ELL, SG>(p, v, f);
    } else {
      fw_flip_r<L, ELL>(p, sg5, v, f);
    }
    m = fminf(m, v);
    fw_unit_steps<L, T + 1>(p, sg5, v, m, f);
  }
}

template <int L, int TPB>
__global__ void __launch_bounds__(TPB, QB_MINB) fieldwalk_kernel(const __grid_constant__ TableParams p) {
  static_assert(L > FW_RB, "field walk needs free bits above the reporting block");
  constexpr int LO = L - FW_RB;
  constexpr int NF = L - FW_RB;
  Rec best{LLONG_MAX, ~0ull, 0ull, 0u, 0u};
  const unsigned long long nchunks = p.chunk_end - p.chunk_begin;
  const int lane = threadIdx.x & 31;
  for (;;) {
    unsigned long long base = 0;
    if (lane == 0) base = atomicAdd(p.work, 32ull);
    base = __shfl_sync(0xffffffffu, base, 0);
    if (base >= nchunks) break;
    const unsigned long long ci = base + lane;
    if (ci >= nchunks) continue;
    const unsigned long long c = p.chunk_begin + ci;
    const unsigned long long s = chunk_prefix(p, c);
    long long V0;
    float f[L];
    {
      float H[FW_RB], F[NF];
      base_eval<FW_RB, L>(p, s << L, L, V0, H, F);
#pragma unroll
      for (int i = 0; i < FW_RB; ++i) f[i] = H[i] + p.d[i];
#pragma unroll
      for (int k2 = 0; k2 < NF; ++k2) f[FW_RB + k2] = F[k2] + p.d[FW_RB + k2];
    }
    int dir;
    const unsigned long long key_hi = chunk_key(p, s, dir);
    float v = 0.f;  // running value relative to the chunk start
    long long cmin = LLONG_MAX;
    // walk counter t = (j << 10) | (q << 6) | r; the flip at t = j<<10 (j > 0) is bit 10 + ctz(j),
    // at t = q<<6 (q > 0) bit 6 + ctz(q), else bit ctz(r)
    for (unsigned int j = 0; j < (1u << LO); ++j) {
      if (j) {
        const int r = __ffs(j) - 1;
        fw_flip_dispatch<L, FW_RB>(p, FW_RB + r, ((j >> (r + 1)) & 1u) ? -1.f : 1.f, v, f);
      }
      float m = v;
#pragma unroll 1
      for (unsigned int q = 0; q < (1u << (FW_RB - FW_UB)); ++q) {
        if (q) {
          const int r = __ffs(q) - 1;
          // bit 6 + r; its direction bit (r + 7) may be bit 10 = j & 1
          const unsigned int tq = (q | (j << (FW_RB - FW_UB)));
          fw_flip_dispatch<L, FW_UB>(p, FW_UB + r, ((tq >> (r + 1)) & 1u) ? -1.f : 1.f, v, f);
          m = fminf(m, v);
        }
        fw_unit_steps<L, 1>(p, (q & 1u) ? -1.f : 1.f, v, m, f);
      }
      const long long val = V0 + (long long)m;
      cmin = min(cmin, val);
      if (val <= best.val) {
        const unsigned long long K = block_key(p, key_hi, dir, j, LO);
        if (val < best.val || K < best.K) best = Rec{val, K, c, j, 0u};
      }
    }
    if (p.mode == MODE_SEARCH_RECORD) p.chunk_min[ci] = cmin;
  }
  search_epilogue<FW_RB, L, TPB>(p, best);
}

}  // namespace qb
