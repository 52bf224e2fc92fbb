// Coarse-filter traversal kernel (default for large chunks): packed int16 block pass + exact
// fp32 re-evaluation of the blocks that could beat or tie the running best.
//
// Same chunks, outer Gray walk (Eq. 3 field updates), blocks and tie keys as the table kernel
// (qb_table.cuh).  Each 1024-state block is first evaluated in a coarse integer image:
//     hc_i = rint(H_i * 2^-s),  Tc(z) = rint(T(z) * 2^-s),  C(z) = sum_{i in z} hc_i + Tc(z)
// with two states per 32-bit register (biased 16-bit fields, see below): one 32-bit add forms a
// pair of candidates, VIMNMX3.U16x2 folds two pairs into the running pair-minimum — about one
// instruction per state, table operands from uniform registers.  s is chosen on the host so
// that every coarse component fits a biased 15-bit field.  Each hc_i and Tc(z) carries at most half a coarse unit of rounding, so
//     exact(z) >= (C(z) - (B+1)/2) * 2^s      (certified lower bound, quantized units)
// A block whose bound exceeds the thread's best value cannot contain a better or tied state and is
// skipped; otherwise its exact minimum comes from the fp32 table evaluation (rare after the first
// blocks of a thread).  When s = 0 the coarse image is exact and no re-evaluation is needed.
// The per-chunk minima written for the certified collect pass are lower bounds (exact for
// evaluated blocks, the coarse bound for skipped ones), which keeps that pass complete.
// Two of the 16 table rows (QB_LDC_MASK) load their table words per lane and fold with the fused
// VIADDMNMX.U16x2, which trades issue slots for ALU-pipe work, and the
// pruning threshold starts from a host-found attained value (p.seed_val, whole-space searches).
#pragma once
#include "qb_table.cuh"


namespace qb {

// Packed coarse pairs: two 16-bit fields per 32-bit register, each biased by 2^14 so that a
// plain 32-bit add of two packed values (both fields in [0, 2^15)) never carries between fields.
// The adds are ordinary VIADD / IADD3 that take the table operand straight from a uniform register
// (LDCU.128 = 8 states, broadcast through the operand path, not replicated per lane), and
// VIMNMX3.U16x2 folds two candidate pairs into the running pair-minimum (4 states per min).
constexpr int CB = QB_PACKED_ROWS ? (1 << 13) : (1 << 14);  // field bias of Bw and Tc components
#ifndef QB_SEED_MAX_LO
#define QB_SEED_MAX_LO 30  // chunks of up to 2^LO blocks start from the host seed value (all; measured D -23%, E -0.2%)
#endif
#ifndef QB_LDC_MASK
#define QB_LDC_MASK 0x4040  // table rows u (bit u) taking the per-lane LDC + VIADDMNMX path (measured)
#endif
#ifndef QB_IMM_FUSED
#define QB_IMM_FUSED 14  // patched-immediate pass: of the 30 pairs after the first two per row, those folded by the fused VIADDMNMX (ALU pipe); measured 10: 31.6, 12: 30.1, 14: 29.7, 16: 30.3 ms (n=40)
#endif
#ifndef QB_EXACT_NOINLINE
#define QB_EXACT_NOINLINE 0  // 1: long chunks call the exact re-evaluation out of line (won 52 -> 41 ms before the host seed; inline measured 33.99 -> 33.70 ms since)
#endif

// exact fp32 re-evaluation of one block, out of line (rare path: keeps its 64 live table-loop
// registers out of the coarse loop's allocation).  The fields travel by value: passing their
// address would pin H in local memory and cost a store on every outer flip (measured 5 STL/block).
template <int B>
struct FieldVec {
  float h[B];
};
template <int B1, int B2>
__device__ __noinline__ float exact_block_min_ool(const TableParams& p, const FieldVec<B1 + B2> hv) {
  float H[B1 + B2], F[1] = {0.f};  // block_min<.., SB = 0, ..> never reads the outer fields
#pragma unroll
  for (int i = 0; i < B1 + B2; ++i) H[i] = hv.h[i];
  return block_min<B1, B2, 0, 1>(p, H, F);
}

__device__ __forceinline__ unsigned umin2(unsigned a, unsigned b) {
  unsigned r;
  asm("min.u16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
  return r;
}
__device__ __forceinline__ unsigned umin3(unsigned a, unsigned b, unsigned c) { return umin2(umin2(a, b), c); }

// a + imm on the FMA pipe (IMAD with an opaque multiplier of 1): the pass splits its adds between
// the FMA pipe (this) and the ALU pipe (fused VIADDMNMX) so neither pipe limits the issue rate
__device__ __forceinline__ unsigned add_fma_pipe(unsigned a, unsigned one, unsigned imm) {
  unsigned r;
  asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(one), "r"(imm));
  return r;
}

// Coarse minimum over the 2^B states of a block, in coarse units (exact integer arithmetic).
// IMM: the table words are instruction immediates (patched per instance) instead of constant-bank
// loads.  Integer adds run on the FMA-heavy pipe (IMAD) or the ALU pipe, each one warp-instruction
// per 2 cycles per SMSP, so the pass balances the two: per row of 32 pairs, QB_IMM_FUSED pairs fold
// through the fused VIADDMNMX (ALU) and the rest are IMAD adds (FMA-heavy) folded by VIMNMX3 (ALU).
template <int B1, int B2, bool IMM = false>
__device__ __forceinline__ int coarse_block_min(const TableParams& p, const float (&H)[B1 + B2]) {
  constexpr int B = B1 + B2, NU = 1 << B1, NP = 1 << (B2 - 1);
  static_assert(B2 >= 3, "pairs of w, four pairs per table load");
  int hc[B];
#pragma unroll
  for (int i = 0; i < B; ++i) hc[i] = __float2int_rn(H[i] * p.coarse_scale);
  // Bw2[m] = (Bw(2m) + 2^14) | (Bw(2m+1) + 2^14) << 16, Bw(w) = sum_{i in w} hc_i
  unsigned Bw2[NP];
  Bw2[0] = (unsigned)CB + ((unsigned)(CB + hc[0]) << 16);
#pragma unroll
  for (int i = 1; i < B2; ++i) {
    const unsigned d = (unsigned)hc[i] * 0x10001u;  // adds hc_i to both fields (no carry: fields stay in range)
#pragma unroll
    for (int m = 0; m < (1 << (i - 1)); ++m) Bw2[m + (1 << (i - 1))] = Bw2[m] + d;
  }
#if QB_PACKED_ROWS
  // A2[u] = (A_u + 2^14) in both fields; candidate fields (Bw + 2^13) + (Tc + 2^13) + (A + 2^14) stay in
  // [0, 2^16): rows are folded packed and unpacked once per block
  unsigned A2[NU];
  A2[0] = (unsigned)(2 * CB) * 0x10001u;
#pragma unroll
  for (int i = 0; i < B1; ++i) {
    const unsigned d = (unsigned)hc[B2 + i] * 0x10001u;
#pragma unroll
    for (int u = 0; u < (1 << i); ++u) A2[u + (1 << i)] = A2[u] + d;
  }
  unsigned rmin2 = 0u;
  if constexpr (IMM) {
    const unsigned one = p.imm_one;
    // rows in reflected Gray order of u: each row's A2 is the previous one +- one packed field, so the
    // 16 A2 values are never live at once (16 registers fewer than the table-load path)
    unsigned du[B1];
#pragma unroll
    for (int i = 0; i < B1; ++i) du[i] = (unsigned)hc[B2 + i] * 0x10001u;
    unsigned a2 = (unsigned)(2 * CB) * 0x10001u;
#pragma unroll
    for (int g = 0; g < NU; g += 2) {
      unsigned r2[2];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int gg = g + h, u = gg ^ (gg >> 1);
        if (gg) {
          const int i = (gg & 1) ? 0 : (gg & 2) ? 1 : (gg & 4) ? 2 : 3;  // ctz(gg), gg < 16
          a2 = ((u >> i) & 1) ? a2 + du[i] : a2 - du[i];
        }
        const unsigned ph = QB_IMM_PH | (unsigned)(u * NP);
        // the first two pairs (FMA-pipe adds) start two accumulators; of the remaining NP - 2 pairs,
        // QB_IMM_FUSED (spread evenly) fold through VIADDMNMX and the rest are FMA-pipe adds folded two
        // at a time by VIMNMX3, alternating between the accumulators
        unsigned acc[2] = {add_fma_pipe(Bw2[0], one, ph | 0u), add_fma_pipe(Bw2[1], one, ph | 1u)};
        unsigned pend = 0u;
        int npend = 0, nfold = 0;
#pragma unroll
        for (int m = 2; m < NP; ++m) {
          const int q = m - 2;
          const bool fused = ((q + 1) * QB_IMM_FUSED) / (NP - 2) > (q * QB_IMM_FUSED) / (NP - 2);
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
      rmin2 = (g == 0) ? umin2(r2[0], r2[1]) : umin3(rmin2, r2[0], r2[1]);
    }
    return (int)min(rmin2 & 0xffffu, rmin2 >> 16) - 4 * CB;
  } else {
#pragma unroll
  for (int u = 0; u < NU; u += 2) {
    unsigned r2[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      unsigned acc2 = 0u;
      if constexpr (QB_LDC_MASK != 0) {
        if ((QB_LDC_MASK >> (u + h)) & 1) {
          // per-lane table loads (LDC) feeding fused add+min (VIADDMNMX.U16x2, GPR operands only):
          // fewer issue slots per state than the uniform path, at the cost of the ALU pipe
          unsigned a0 = 0xffffffffu, a1 = 0xffffffffu;
#pragma unroll
          for (int m = 0; m < NP; m += 4) {
            const uint4 t = *reinterpret_cast<const uint4*>(&p.Tc2[(u + h) * NP + m]);
            a0 = __viaddmin_u16x2(Bw2[m], t.x, a0);
            a1 = __viaddmin_u16x2(Bw2[m + 1], t.y, a1);
            a0 = __viaddmin_u16x2(Bw2[m + 2], t.z, a0);
            a1 = __viaddmin_u16x2(Bw2[m + 3], t.w, a1);
          }
          r2[h] = umin2(a0, a1) + A2[u + h];
          continue;
        }
      }
#pragma unroll
      for (int m = 0; m < NP; m += 4) {
        const uint4 t = *reinterpret_cast<const uint4*>(&p.Tc2[(u + h) * NP + m]);
        const unsigned c0 = Bw2[m] + t.x, c1 = Bw2[m + 1] + t.y;
        const unsigned c2 = Bw2[m + 2] + t.z, c3 = Bw2[m + 3] + t.w;
        acc2 = (m == 0) ? umin2(c0, c1) : umin3(acc2, c0, c1);
        acc2 = umin3(acc2, c2, c3);
      }
      r2[h] = acc2 + A2[u + h];
    }
    rmin2 = (u == 0) ? umin2(r2[0], r2[1]) : umin3(rmin2, r2[0], r2[1]);
  }
  return (int)min(rmin2 & 0xffffu, rmin2 >> 16) - 4 * CB;
  }
#else
  // A[u] = sum_{i in u} hc_{B2+i} - 2^15 (removes the two field biases of a candidate)
  int A[NU];
  A[0] = -2 * CB;
#pragma unroll
  for (int i = 0; i < B1; ++i)
#pragma unroll
    for (int u = 0; u < (1 << i); ++u) A[u + (1 << i)] = A[u] + hc[B2 + i];
  int rmin = 0;
#pragma unroll
  for (int u = 0; u < NU; u += 2) {
    int r[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      unsigned acc2 = 0u;
#pragma unroll
      for (int m = 0; m < NP; m += 4) {
        const uint4 t = *reinterpret_cast<const uint4*>(&p.Tc2[(u + h) * NP + m]);
        const unsigned c0 = Bw2[m] + t.x, c1 = Bw2[m + 1] + t.y;
        const unsigned c2 = Bw2[m + 2] + t.z, c3 = Bw2[m + 3] + t.w;
        acc2 = (m == 0) ? umin2(c0, c1) : umin3(acc2, c0, c1);
        acc2 = umin3(acc2, c2, c3);
      }
      r[h] = (int)min(acc2 & 0xffffu, acc2 >> 16) + A[u + h];
    }
    rmin = (u == 0) ? min(r[0], r[1]) : min(min(rmin, r[0]), r[1]);
  }
  return rmin;
#endif
}

// (B1, B2): the fp32 table split used by the exact fallback; (CB1, CB2): the coarse pass's own split
// of the same B table bits (both index the table as z = (u << B2) | w over the same bits).
#ifndef QB_COARSE_MINB
#define QB_COARSE_MINB 4  // 128 registers: fewer uniform-register spills beat the fifth CTA (measured)
#endif

#ifndef QB_CHUNK_START_NOINLINE
#define QB_CHUNK_START_NOINLINE 1  // chunk-start evaluation out of line: keeps the hot loop's code compact (measured -0.5%)
#endif
template <int B, int NF>
struct ChunkStart {
  long long V;
  float H[B];
  float F[NF];
};
template <int B, int L>
__device__ __noinline__ ChunkStart<B, ((L - B) > 0 ? (L - B) : 1)> chunk_start_ool(const TableParams& p,
                                                                             unsigned long long s) {
  ChunkStart<B, ((L - B) > 0 ? (L - B) : 1)> r;
  base_eval<B, L>(p, s << L, L, r.V, r.H, r.F);
  return r;
}

template <int B1, int B2, int CB1, int CB2, int L, int TPB, bool IMM = false>
__global__ void __launch_bounds__(TPB, QB_COARSE_MINB) coarse_kernel(const __grid_constant__ TableParams p) {
  constexpr int B = B1 + B2;
  static_assert(CB1 + CB2 == B, "coarse split must cover the table bits");
  constexpr int LO = L - B;
  constexpr int NF = (L - B) > 0 ? (L - B) : 1;
  Rec best{LLONG_MAX, ~0ull, 0ull, 0u, 0u};
  const unsigned long long nchunks = p.chunk_end - p.chunk_begin;
  const int lane = threadIdx.x & 31;
  const long long slack = (long long)(B + 1) << p.coarse_shift >> 1;  // (B+1)/2 coarse units, quantized
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
#if QB_CHUNK_START_NOINLINE
    {
      ChunkStart<B, NF> cs0 = chunk_start_ool<B, L>(p, s);
      V = cs0.V;
#pragma unroll
      for (int i = 0; i < B; ++i) H[i] = cs0.H[i];
#pragma unroll
      for (int m = 0; m < NF; ++m) F[m] = cs0.F[m];
    }
#else
    base_eval<B, L>(p, s << L, L, V, H, F);
#endif
    int dir;
    const unsigned long long key_hi = chunk_key(p, s, dir);
    long long cmin = LLONG_MAX, skip_min = LLONG_MAX;  // skip_min: least coarse value of a pruned block
    // pruning threshold: the better of this thread's best and the device-wide best so far (any
    // block whose bound exceeds a value some state attains holds neither a minimiser nor a tie)
    long long thr = min(best.val, gbest_dec(__ldcg(p.gbest)));
    // short chunks: start from an attained value found on the host (greedy descent), so the first
    // blocks of every thread are already filtered (pruning stays exact: that state's own block is
    // never skipped, so it and its ties are still found)
    if constexpr (LO <= QB_SEED_MAX_LO) thr = min(thr, p.seed_val);
    long long lim = thr > LLONG_MAX - slack ? LLONG_MAX : thr + slack;  // prune when the coarse value exceeds it
    for (unsigned int j = 0; j < (1u << LO); ++j) {
      if (j) {
        const int r = __ffs(j) - 1;
        const float sg = ((j >> (r + 1)) & 1u) ? -1.f : 1.f;
        outer_flip<B, L, B>(p, B + r, sg, V, H, F);
      }
      // device-wide best: short chunks (<= 64 blocks) refresh it every block, long chunks only at
      // the chunk start (measured: the per-block load costs ~5% at 1024 blocks per chunk)
      long long gb = LLONG_MAX;
      if constexpr (LO <= 6) gb = gbest_dec(__ldcg(p.gbest));
      const long long cb = V + ((long long)coarse_block_min<CB1, CB2, IMM>(p, H) << p.coarse_shift);
      if constexpr (LO <= 6) {
        thr = min(thr, gb);
        lim = thr > LLONG_MAX - slack ? LLONG_MAX : thr + slack;
      }
      long long val;
      if (coarse_exact) {
        val = cb;
      } else {
        if (cb > lim) {  // bound cb - slack > thr: no state of this block can beat or tie the best value seen
          skip_min = min(skip_min, cb);
          continue;
        }
        // short chunks (<= 64 blocks) re-evaluate often enough that inlining wins; long chunks call
        // out of line so the coarse loop keeps the registers
        if constexpr (QB_EXACT_NOINLINE && LO > 6) {
          FieldVec<B> hv;
#pragma unroll
          for (int i = 0; i < B; ++i) hv.h[i] = H[i];
          val = V + (long long)exact_block_min_ool<B1, B2>(p, hv);
        } else {
          val = V + (long long)block_min<B1, B2, 0, NF>(p, H, F);
        }
      }
      cmin = min(cmin, val);
      if (val <= best.val) {
        const unsigned long long K = block_key(p, key_hi, dir, j, LO);
        if (val < best.val || K < best.K) best = Rec{val, K, c, j, 0u};
        if (val < thr) {
          thr = val;
          lim = val + slack;
          atomicMax(p.gbest, gbest_enc(val));
        }
      }
    }
    if (skip_min != LLONG_MAX) cmin = min(cmin, skip_min - slack);  // pruned blocks contribute their bound
    if (p.mode == MODE_SEARCH_RECORD) p.chunk_min[ci] = cmin;
  }
  // records only: the reduction runs as finalize_kernel (see there for why not in this tail)
  const Rec r = cta_reduce<TPB>(best);
  if (threadIdx.x == 0) p.cta_out[blockIdx.x] = r;
}

}  // namespace qb
