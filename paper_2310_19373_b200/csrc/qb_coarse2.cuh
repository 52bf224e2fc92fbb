// Super-block coarse kernel (QB_VARIANT_IMM2): the patched-immediate coarse pass over 11 bits.
//
// Same chunks, blocks, tie keys, certified filter and records as coarse_kernel (qb_coarse.cuh), but
// the coarse image covers the B = 10 table bits AND the first outer bit B: one coarse evaluation
// handles the two blocks that differ only in bit B (2048 states), so the per-block setup (field
// rounding, packed subset sums, outer flip, loop control: ~140 instructions) is paid once per 2048
// states instead of per 1024.  The outer Gray walk runs over bits B+1 .. L-1 only.
//
//   coarse value of (z, b):  sum_{i<B} z_i hc_i + b * hc_B + Tc11(z | b << B)
//   hc_B = rint(F_B 2^-s),   Tc11(z | b << B) = rint((T(z) + b (q_BB + sum_{i<B} z_i q_iB)) 2^-s)
//
// The 1024 words of Tc11 (two 16-bit fields each, biased as in the 10-bit pass) are instruction
// immediates, patched into a copy of the cubin per instance (qb_api.cu imm_kernel).  The 32 rows
// u = (b, bits 6..9) are walked in reflected Gray order, so rows 0..15 of the walk are the b = 0
// block and rows 16..31 the b = 1 block: each block gets its own certified bound
// (11 + 1)/2 coarse units, and a block that survives is re-evaluated exactly by the fp32 table
// (block_min) from its own base (V, H) or (V + q_BB + F_B, H + q_.B).  Original block index of
// half b in super-block j': j = 2 j' + (b ^ (j' & 1)) (reflected Gray code), so keys, records and
// finalize_kernel see exactly the blocks of the 10-bit walk.
#pragma once
#include "qb_coarse.cuh"

#ifndef QB_IMM2_FUSED
#define QB_IMM2_FUSED 12  // super-block pass: pairs per row (after the first two) folded by VIADDMNMX (ALU pipe)
#endif

namespace qb {

// Coarse minima of the two halves of a super-block, in coarse units: out[b] for b = 0, 1.
template <int NP>
__device__ __forceinline__ void coarse2_super_min(const TableParams& p, const float (&H)[BMAX], float FB, int (&out)[2]) {
  constexpr int CB2 = 6, B2 = CB2, NU = 32;  // w = bits 0..5 (32 pairs), u = bits 6..9 + bit B
  static_assert(NP == 1 << (CB2 - 1), "32 pairs per row");
  int hc[BMAX];
#pragma unroll
  for (int i = 0; i < BMAX; ++i) hc[i] = __float2int_rn(H[i] * p.coarse_scale);
  unsigned Bw2[NP];
  Bw2[0] = (unsigned)CB + ((unsigned)(CB + hc[0]) << 16);
#pragma unroll
  for (int i = 1; i < B2; ++i) {
    const unsigned d = (unsigned)hc[i] * 0x10001u;
#pragma unroll
    for (int m = 0; m < (1 << (i - 1)); ++m) Bw2[m + (1 << (i - 1))] = Bw2[m] + d;
  }
  unsigned du[5];
#pragma unroll
  for (int i = 0; i < 4; ++i) du[i] = (unsigned)hc[B2 + i] * 0x10001u;
  du[4] = (unsigned)__float2int_rn(FB * p.coarse_scale) * 0x10001u;
  const unsigned one = p.imm_one;
  unsigned a2 = (unsigned)(2 * CB) * 0x10001u;
  unsigned rmin2[2] = {0u, 0u};
#pragma unroll
  for (int g = 0; g < NU; g += 2) {
    unsigned r2[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int gg = g + h, u = gg ^ (gg >> 1);
      if (gg) {
        const int i = (gg & 1) ? 0 : (gg & 2) ? 1 : (gg & 4) ? 2 : (gg & 8) ? 3 : 4;  // ctz(gg), gg < 32
        a2 = ((u >> i) & 1) ? a2 + du[i] : a2 - du[i];
      }
      const unsigned ph = QB_IMM_PH | (unsigned)(u * NP);
      unsigned acc[2] = {add_fma_pipe(Bw2[0], one, ph | 0u), add_fma_pipe(Bw2[1], one, ph | 1u)};
      unsigned pend = 0u;
      int npend = 0, nfold = 0;
#pragma unroll
      for (int m = 2; m < NP; ++m) {
        const int q = m - 2;
        const bool fused = ((q + 1) * QB_IMM2_FUSED) / (NP - 2) > (q * QB_IMM2_FUSED) / (NP - 2);
        if (fused) {
          acc[nfold & 1] = __viaddmin_u16x2(Bw2[m], ph | m, acc[nfold & 1]);
          ++nfold;
        } else {
          const unsigned c = add_fma_pipe(Bw2[m], one, ph | m);
          if (npend == 0) {
            pend = c;
            npend = 1;
          } else {
            acc[nfold & 1] = umin3(acc[nfold & 1], pend, c);
            ++nfold;
            npend = 0;
          }
        }
      }
      if (npend) acc[0] = umin2(acc[0], pend);
      r2[h] = umin2(acc[0], acc[1]) + a2;
    }
    const int half = g >= 16;  // Gray order over 5 bits: the top bit (b) is 0 for g < 16
    rmin2[half] = (g == 0 || g == 16) ? umin2(r2[0], r2[1]) : umin3(rmin2[half], r2[0], r2[1]);
  }
#pragma unroll
  for (int b = 0; b < 2; ++b) out[b] = (int)min(rmin2[b] & 0xffffu, rmin2[b] >> 16) - 4 * CB;
}

template <int B1, int B2, int L, int TPB>
__global__ void __launch_bounds__(TPB, QB_COARSE_MINB) coarse2_kernel(const __grid_constant__ TableParams p) {
  constexpr int B = B1 + B2;
  static_assert(B == BMAX, "super-blocks extend the 10-bit table blocks");
  static_assert(L >= B + 2, "needs at least one walked outer bit besides bit B");
  constexpr int LO = L - B;        // outer bits of the 10-bit walk (block index j has LO bits)
  constexpr int LS = LO - 1;       // walked bits B+1 .. L-1 (super-block index j')
  constexpr int NF = LO;
  Rec best{LLONG_MAX, ~0ull, 0ull, 0u, 0u};
  const unsigned long long nchunks = p.chunk_end - p.chunk_begin;
  const int lane = threadIdx.x & 31;
  const long long slack = (long long)(B + 2) << p.coarse_shift >> 1;  // (11+1)/2 coarse units, quantized
  const bool coarse_exact = p.coarse_shift == 0;

  for (;;) {
    unsigned long long base = 0;
    if (lane == 0) base = atomicAdd(p.work, 32ull);
    base = __shfl_sync(0xffffffffu, base, 0);
    if (base >= nchunks) break;
    const unsigned long long ci = base + lane;
    if (ci >= nchunks) continue;
    const unsigned long long c = p.chunk_begin + ci;
    const unsigned long long s = chunk_prefix(p, c);
    long long V;
    float H[B], F[NF];
    {
      ChunkStart<B, NF> cs0 = chunk_start_ool<B, L>(p, s);
      V = cs0.V;
#pragma unroll
      for (int i = 0; i < B; ++i) H[i] = cs0.H[i];
#pragma unroll
      for (int m = 0; m < NF; ++m) F[m] = cs0.F[m];
    }
    int dir;
    const unsigned long long key_hi = chunk_key(p, s, dir);
    long long cmin = LLONG_MAX, skip_min = LLONG_MAX;
    long long thr = min(best.val, gbest_dec(__ldcg(p.gbest)));
    if constexpr (LO <= QB_SEED_MAX_LO) thr = min(thr, p.seed_val);
    long long lim = thr > LLONG_MAX - slack ? LLONG_MAX : thr + slack;
    for (unsigned int jp = 0; jp < (1u << LS); ++jp) {
      if (jp) {
        const int r = __ffs(jp) - 1;
        const float sg = ((jp >> (r + 1)) & 1u) ? -1.f : 1.f;
        outer_flip<B, L, B + 1>(p, B + 1 + r, sg, V, H, F);
      }
      int cm[2];
      coarse2_super_min<32>(p, H, F[0], cm);
      const long long cb0 = V + ((long long)cm[0] << p.coarse_shift), cb1 = V + ((long long)cm[1] << p.coarse_shift);
#pragma unroll 1
      for (int t = 0; t < 2; ++t) {
        const int b = t ^ (int)(jp & 1u);  // half evaluated in original block order j = 2 jp + t
        const long long cb = b ? cb1 : cb0;
        long long val;
        if (coarse_exact) {
          val = cb;
        } else {
          if (cb > lim) {
            skip_min = min(skip_min, cb);
            continue;
          }
          // exact fp32 table evaluation from the half's own base: (V, H) or (V + q_BB + F_B, H + q_.B)
          float Hb[B];
#pragma unroll
          for (int i = 0; i < B; ++i) Hb[i] = b ? H[i] + p.Qs[B][i] : H[i];
          const long long Vb = b ? V + (long long)(p.d[B] + F[0]) : V;
          val = Vb + (long long)block_min<B1, B2, 0, NF>(p, Hb, F);
        }
        cmin = min(cmin, val);
        if (val <= best.val) {
          const unsigned int j = 2u * jp + (unsigned)t;
          const unsigned long long K = block_key(p, key_hi, dir, j, LO);
          if (val < best.val || K < best.K) best = Rec{val, K, c, j, 0u};
          if (val < thr) {
            thr = val;
            lim = val + slack;
            atomicMax(p.gbest, gbest_enc(val));
          }
        }
      }
    }
    if (skip_min != LLONG_MAX) cmin = min(cmin, skip_min - slack);
    if (p.mode == MODE_SEARCH_RECORD) p.chunk_min[ci] = cmin;
  }
  const Rec r = cta_reduce<TPB>(best);
  if (threadIdx.x == 0) p.cta_out[blockIdx.x] = r;
}

}  // namespace qb
