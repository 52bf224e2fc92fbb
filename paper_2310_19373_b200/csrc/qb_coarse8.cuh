// Byte-packed threshold kernels: the coarse pass with FOUR states per 32-bit register.
//   QB_VARIANT_IMM8 / IMM8S          exact row terms, 10-bit blocks / 11-bit super-blocks (patched immediates)
//   QB_VARIANT_IMM8A / IMM8AS / AQ   the row-bound form (coarse8_block_and, APPROX), 10 / 11 / 12-bit blocks;
//                                    IMM8AS is AUTO's search kernel for long or repeated solves
//   QB_VARIANT_BYTE8                 IMM8AS with its table words in the kernel parameters (qb_k_byte8.cu)
// AUTO runs them optimistically: coarse8_give_up() stops a run whose blocks fail the test too often, and the
// host repeats the solve with a tighter kernel (qb_api.cu).
//
// Same chunks, outer Gray walk, blocks, tie keys, exact re-evaluation and records as coarse_kernel
// (qb_coarse.cuh).  What changes is the coarse test of a 1024-state block.  The 16-bit pass forms the
// block's coarse MINIMUM (two states per register, packed u16 min) and compares it with the pruning
// limit.  The only thing the search needs from it is the comparison, so this pass forms, for every
// state z of the block, the byte
//
//     f(z) = base + sum_{i in z} hc_i + Tc8(z),     base = 127 - Lc
//
// where hc_i = rint(H_i / U), Tc8(z) = rint(T(z) / U) (coarse unit U quantized units, any real U >= 1) and Lc is
// the block's own limit in coarse units, Lc = floor((lim - V) / U): bit 7 of f(z) is CLEAR exactly when the
// state's coarse value is <= the limit.  Four states share a register (w = 4q .. 4q+3), the adds are
// plain 32-bit adds, and one LOP3 ANDs two result registers into an accumulator: the block holds a
// state under the limit iff some byte of the AND has bit 7 clear.  Every state's coarse value is
// still formed and tested -- one add per four states plus half a LOP3, against one add per two states
// plus a packed min in the 16-bit pass.
//
// Range (host, quantize(): c8_rneg / the choice of U): with X(z) = sum hc_i z_i + Tc8(z) in [-Rneg, Rpos]
// over every state and every reachable field vector, and Rneg + Rpos <= 127, the limit is clamped to
// Lc in [-Rneg - 1, -1].  Lc >= 0 means z = 0 (coarse value 0) is under the limit: the block is
// re-evaluated without looking at the bytes.  Lc < -Rneg - 1 means no state can be under it, and the
// clamped test (nothing <= -Rneg - 1) says the same.  So base lies in [128, 128 + Rneg], every byte in
// [128 - Rneg, 128 + Rneg + Rpos] = [1, 255]: no byte ever wraps or carries into its neighbour, and adding
// a replicated or packed signed constant modulo 2^32 adds it to every byte exactly.
//
// Certified bound: as in the 16-bit pass, exact(z) >= V + (C(z) - (B+1)/2 - 0.02) U (the 0.02 covers the float
// rounding of H_i fl(1/U)), and lim = thr + slack
// (+ 2 Eq on the recording search, see below), so a block with no byte under the limit holds neither a
// better state nor a tie.  Rows u (4 bits) run in reflected Gray order; a row's A_u (replicated in the
// four bytes) is either added by a 3-input IADD3 together with the table immediate (ALU pipe) or by two
// IMADs (FMA-heavy pipe): QB_IMM8_LAZY of the 16 registers of a row take the IADD3 form so that the two
// integer pipes carry equal work (the LOP3 folds are ALU work as well).
//
// Recording search (MODE_SEARCH_RECORD, the certified collect path): the 16-bit kernel records a lower
// bound for each pruned block.  This pass has no block minimum to record; instead its limit includes
// the collect margin (lim = thr + slack + theta_add), so a pruned block holds no state within theta_add
// of any value attained so far -- in particular none within theta_add of the final minimum -- and
// contributes nothing to the chunk minimum.
#pragma once
#include "qb_coarse.cuh"

#ifndef QB_IMM8_LAZY
#define QB_IMM8_LAZY 9  // of the 16 registers of a row, those whose A_u + table add is one IADD3 (ALU pipe); measured n=40: 8: 25.4, 9: 22.7, 10: 23.2, 11: 23.1, 12: 24.2 ms
#endif
#ifndef QB_IMM8_ABORT_ALLOWANCE
#define QB_IMM8_ABORT_ALLOWANCE (1ull << 16)  // exact re-evaluations allowed before the optimistic run may give up (start-up transient)
#endif
#ifndef QB_IMM8_MINB
#define QB_IMM8_MINB 4
#endif

namespace qb {

// a + b on the FMA-heavy pipe (IMAD with an opaque multiplier of 1), both operands in registers
__device__ __forceinline__ unsigned add_fma_reg(unsigned a, unsigned one, unsigned b) {
  unsigned r;
  asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(one), "r"(b));
  return r;
}

// A block's limit in coarse units: an integer >= floor(d / U) for d = lim - V (quantized units), from
// the float product d * fl(1/U).  Its relative error is below 2^-22, i.e. below 2^-10 units wherever the
// limit matters (|d / U| < 2^12; beyond that the limit is clamped or the block passes outright), so adding
// 2^-10 before the floor never under-estimates it; over-estimating only passes more blocks.
__device__ __forceinline__ int coarse8_limit(long long d, float inv_unit) {
  return __float2int_rd(fmaf((float)d, inv_unit, 0.0009765625f));
}

// AUTO's optimistic run (p.c8_abort_shift >= 0), checked every 64 blocks of a long chunk: the thread adds the
// blocks it re-evaluated exactly since its last report to the device-wide count work[6] and gives up
// (work[7] = 1) when that count exceeds the allowed rate -- 1 in 2^shift of the blocks walked so far, estimated
// as this thread's own progress times the resident threads -- plus a start-up allowance.
__device__ __forceinline__ bool coarse8_give_up(const TableParams& p, unsigned& npass, unsigned long long my_blocks,
                                                unsigned long long nthreads) {
  if (p.c8_abort_shift < 0) return false;
  if (npass) {
    atomicAdd(p.work + 6, (unsigned long long)npass);
    npass = 0;
  }
  if (__ldcg(p.work + 6) <= ((my_blocks * nthreads) >> p.c8_abort_shift) + QB_IMM8_ABORT_ALLOWANCE) return false;
  p.work[7] = 1ull;
  return true;
}

// AND of the bytes f(z) of a block (four per register); see the file header.  NX > 0 (super-blocks): the
// rows also run over the first NX outer bits (fields FX[t] = F_{B+t}): 16 << NX rows, and out[part] collects
// the rows of the 10-bit block whose bits B.. have the value `part`.
//
// APPROX (QB_VARIANT_IMM8A / IMM8AS / IMM8AQ, the "row-bound" form): every row uses the SAME row term, the least
// one, amin = sum_{i in row bits} min(hc_i, 0) <= A_u, folded into the base.  A state's byte is then a lower
// bound of its coarse value (low by A_u - amin >= 0), so the test stays certified -- a block with no byte
// under the limit still holds no state under it -- but passes more blocks to the exact evaluation.  In
// exchange a row costs one 2-input add per register instead of a 3-input IADD3 or two IMADs, and the
// per-row A_u chain disappears.  The adds are written plainly: ptxas issues about a fifth of them as IADD3
// (ALU pipe) and the rest as VIADD, which measured faster than any explicit IMAD / IADD3 split (n=40 super-
// blocks: 15.5 ms against 15.9 ms for 12 IMAD + 4 IADD3 per row, 16.9 / 17.2 / 17.6 ms for 3 / 5 / 6 IADD3; forcing
// one or two more IADD3 per row on top of ptxas's split: 15.9 / 15.8 ms).
// TABLE: the packed table words come from the kernel parameters (p.Tc8w, LDCU.128 into uniform registers, one load
// per 16 states) instead of patched immediates: no module to patch and load, about 14% more instructions.
template <int CB1, int CB2, int NX, bool APPROX = false, bool TABLE = false>
__device__ __forceinline__ void coarse8_block_and(const TableParams& p, const float (&H)[CB1 + CB2],
                                                  const float (&FX)[NX > 0 ? NX : 1], int base,
                                                  unsigned (&out)[1 << NX]) {
  constexpr int B = CB1 + CB2, UB = CB1 + NX, NU = 1 << UB, NQ = 1 << (CB2 - 2), NP = 1 << NX;
  static_assert(CB2 >= 3 && CB1 >= 1 && UB <= 6, "four w states per register, at least two registers per row");
  static_assert(APPROX || NX <= 1, "two extra row bits are built for the row-bound form only");
  static_assert(!TABLE || (APPROX && NX == 1), "the table-load form exists for the row-bound 11-bit pass");
  int hc[B];
#pragma unroll
  for (int i = 0; i < B; ++i) hc[i] = __float2int_rn(H[i] * p.c8_scale);
  if constexpr (APPROX) {
    int amin = 0;
#pragma unroll
    for (int i = 0; i < CB1; ++i) amin += min(hc[CB2 + i], 0);
#pragma unroll
    for (int t = 0; t < NX; ++t) amin += min(__float2int_rn(FX[t] * p.c8_scale), 0);
    // X4[q] byte j = base + amin + sum_{i in w} hc_i, w = 4q + j
    unsigned X4[NQ];
    X4[0] = (unsigned)(base + amin) * 0x01010101u + (unsigned)hc[0] * 0x01000100u + (unsigned)hc[1] * 0x01010000u;
#pragma unroll
    for (int i = 2; i < CB2; ++i) {
      const unsigned d = (unsigned)hc[i] * 0x01010101u;
#pragma unroll
      for (int m = 0; m < (1 << (i - 2)); ++m) X4[m + (1 << (i - 2))] = X4[m] + d;
    }
    unsigned acc[NP][2];
#pragma unroll
    for (int h = 0; h < NP; ++h) acc[h][0] = acc[h][1] = 0xffffffffu;
#pragma unroll
    for (int u = 0; u < NU; ++u) {
      const int part = u >> CB1;
      const unsigned ph = QB_IMM_PH | (unsigned)(u * NQ);
      unsigned r[NQ];
#pragma unroll
      for (int q = 0; q < NQ; ++q) r[q] = X4[q] + (TABLE ? p.Tc8w[u * NQ + q] : (ph | (unsigned)q));
#pragma unroll
      for (int q = 0; q < NQ; q += 2) acc[part][(q >> 1) & 1] &= r[q] & r[q + 1];
    }
#pragma unroll
    for (int h = 0; h < NP; ++h) out[h] = acc[h][0] & acc[h][1];
    return;
  }
  const unsigned one = p.imm_one;
  // X4[q] byte j = base + sum_{i in w} hc_i, w = 4q + j
  unsigned X4[NQ];
  X4[0] = (unsigned)base * 0x01010101u + (unsigned)hc[0] * 0x01000100u + (unsigned)hc[1] * 0x01010000u;
#pragma unroll
  for (int i = 2; i < CB2; ++i) {
    const unsigned d = (unsigned)hc[i] * 0x01010101u;
#pragma unroll
    for (int m = 0; m < (1 << (i - 2)); ++m) X4[m + (1 << (i - 2))] = X4[m] + d;
  }
  unsigned du[UB];
#pragma unroll
  for (int i = 0; i < CB1; ++i) du[i] = (unsigned)hc[CB2 + i] * 0x01010101u;
  if constexpr (NX > 0) du[CB1] = (unsigned)__float2int_rn(FX[0] * p.c8_scale) * 0x01010101u;
  unsigned a4 = 0u;
  unsigned acc[2][2] = {{0xffffffffu, 0xffffffffu}, {0xffffffffu, 0xffffffffu}};
#pragma unroll
  for (int g = 0; g < NU; ++g) {
    const int u = g ^ (g >> 1);
    const int half = NX > 0 ? (g >> CB1) : 0;  // reflected Gray order: the top row bit is 0 for the first half
    if (g) {
      const int i = (g & 1) ? 0 : (g & 2) ? 1 : (g & 4) ? 2 : (g & 8) ? 3 : 4;  // ctz(g), g < 32
      a4 = ((u >> i) & 1) ? a4 + du[i] : a4 - du[i];
    }
    const unsigned ph = QB_IMM_PH | (unsigned)(u * NQ);
    unsigned r[NQ];
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      const bool lazy = ((q + 1) * QB_IMM8_LAZY) / NQ > (q * QB_IMM8_LAZY) / NQ;
      if (g == 0) r[q] = add_fma_pipe(X4[q], one, ph | q);             // A_0 = 0
      else if (lazy) r[q] = X4[q] + a4 + (ph | (unsigned)q);           // IADD3 (ALU pipe)
      else r[q] = add_fma_pipe(add_fma_reg(X4[q], one, a4), one, ph | q);  // two IMADs (FMA-heavy pipe)
    }
#pragma unroll
    for (int q = 0; q < NQ; q += 2) acc[half][(q >> 1) & 1] &= r[q] & r[q + 1];
  }
  out[0] = acc[0][0] & acc[0][1];
  if constexpr (NX > 0) out[1] = acc[1][0] & acc[1][1];
}

template <int B1, int B2, int CB1, int CB2, int L, int TPB, bool APPROX = false>
__global__ void __launch_bounds__(TPB, QB_IMM8_MINB) coarse8_kernel(const __grid_constant__ TableParams p) {
  constexpr int B = B1 + B2;
  static_assert(CB1 + CB2 == B, "coarse split must cover the table bits");
  constexpr int LO = L - B;
  constexpr int NF = (L - B) > 0 ? (L - B) : 1;
  Rec best{LLONG_MAX, ~0ull, 0ull, 0u, 0u};
  const unsigned long long nchunks = p.chunk_end - p.chunk_begin;
  const int lane = threadIdx.x & 31;
  // (B+1)/2 coarse units (+ float rounding), quantized; the recording search adds the collect margin (file header)
  const long long slack = p.c8_slack + (p.mode == MODE_SEARCH_RECORD ? p.theta_add : 0ll);
  const float inv_unit = p.c8_scale;
  const int lc_min = -p.c8_rneg - 1;

  bool quit = false;
  unsigned long long my_chunks = 0;
  const unsigned long long nthreads = (unsigned long long)gridDim.x * TPB;
  for (;;) {
    if (__any_sync(0xffffffffu, quit)) break;  // a lane gave up inside its chunk (below): the whole warp stops
    unsigned long long base = 0, passed = 0;
    if (lane == 0) {
      base = atomicAdd(p.work, 32ull);
      passed = __ldcg(p.work + 6);
    }
    base = __shfl_sync(0xffffffffu, base, 0);
    if (base >= nchunks) break;
    if (p.c8_abort_shift >= 0) {
      // AUTO's optimistic run: too many blocks are failing the byte test for it to pay (warp-uniform decision)
      passed = __shfl_sync(0xffffffffu, passed, 0);
      if (passed > ((base << LO) >> p.c8_abort_shift) + QB_IMM8_ABORT_ALLOWANCE) {
        if (lane == 0) p.work[7] = 1ull;
        break;
      }
    }
    const unsigned long long ci = base + lane;
    if (ci >= nchunks) continue;
    unsigned npass = 0;
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
    long long cmin = LLONG_MAX;
    long long thr = min(min(best.val, gbest_dec(__ldcg(p.gbest))), p.seed_val);
    for (unsigned int j = 0; j < (1u << LO); ++j) {
      if (j) {
        const int r = __ffs(j) - 1;
        const float sg = ((j >> (r + 1)) & 1u) ? -1.f : 1.f;
        outer_flip<B, L, B>(p, B + r, sg, V, H, F);
      }
      // device-wide best: refreshed every block in short chunks, every 64 blocks in long ones
      if (LO <= 6 || (j & 63u) == 0u) {
        thr = min(thr, gbest_dec(__ldcg(p.gbest)));
        if (LO > 6 && coarse8_give_up(p, npass, (my_chunks << LO) + j, nthreads)) {
          quit = true;
          break;
        }
      }
      // the block's limit in coarse units relative to its base; no limit yet: everything passes
      const int lrel = thr > LLONG_MAX - slack ? 0 : coarse8_limit(thr + slack - V, inv_unit);
      const int lc = min(max(lrel, lc_min), -1);
      unsigned a[1];
      const float nofx[1] = {0.f};
      coarse8_block_and<CB1, CB2, 0, APPROX>(p, H, nofx, 127 - lc, a);
      if (lrel < 0 && (a[0] & 0x80808080u) == 0x80808080u) continue;  // no state of the block is under the limit
      ++npass;
      const long long val = V + (long long)block_min<B1, B2, 0, NF>(p, H, F);
      cmin = min(cmin, val);
      if (val <= best.val) {
        const unsigned long long K = block_key(p, key_hi, dir, j, LO);
        if (val < best.val || K < best.K) best = Rec{val, K, c, j, 0u};
        if (val < thr) {
          thr = val;
          atomicMax(p.gbest, gbest_enc(val));
        }
      }
    }
    if (p.mode == MODE_SEARCH_RECORD) p.chunk_min[ci] = cmin;
    if (npass) atomicAdd(p.work + 6, (unsigned long long)npass);
    ++my_chunks;
  }
  // records only: the reduction runs as finalize_kernel (qb_table.cuh)
  const Rec r = cta_reduce<TPB>(best);
  if (threadIdx.x == 0) p.cta_out[blockIdx.x] = r;
}

// Super-block forms (QB_VARIANT_IMM8S / IMM8AS: NX = 1; IMM8AQ: NX = 2): the byte image also covers the first NX
// outer bits B .. B+NX-1, as in coarse2_kernel (qb_coarse2.cuh): one pass tests the 2^NX blocks that differ only
// in those bits against the same limit (relative to the base V of the block with those bits 0), the outer
// Gray walk runs over bits B+NX .. L-1, and each block that holds a byte under the limit is re-evaluated
// exactly from its own base, in original block order j = (j' << NX) + t: block j has bits B.. equal to the low
// NX bits of the reflected Gray code of j, so keys, records and finalize_kernel see the blocks of the 10-bit
// walk.  Certified bound: (10 + NX + 1)/2 coarse units (in c8_slack).
template <int B1, int B2, int CB1, int CB2, int L, int TPB, bool APPROX = false, int NX = 1, bool TABLE = false>
__global__ void __launch_bounds__(TPB, QB_IMM8_MINB) coarse8s_kernel(const __grid_constant__ TableParams p) {
  constexpr int B = B1 + B2;
  static_assert(CB1 + CB2 == B && B == BMAX, "super-blocks extend the 10-bit table blocks");
  static_assert(NX >= 1 && NX <= 2 && L >= B + NX + 1, "needs at least one walked outer bit besides the image bits");
  constexpr int LO = L - B;    // outer bits of the 10-bit walk (block index j has LO bits)
  constexpr int LS = LO - NX;  // walked bits B+NX .. L-1 (super-block index j')
  constexpr int NF = LO;
  Rec best{LLONG_MAX, ~0ull, 0ull, 0u, 0u};
  const unsigned long long nchunks = p.chunk_end - p.chunk_begin;
  const int lane = threadIdx.x & 31;
  const long long slack = p.c8_slack + (p.mode == MODE_SEARCH_RECORD ? p.theta_add : 0ll);
  const float inv_unit = p.c8_scale;
  const int lc_min = -p.c8_rneg - 1;

  bool quit = false;
  unsigned long long my_chunks = 0;
  const unsigned long long nthreads = (unsigned long long)gridDim.x * TPB;
  for (;;) {
    if (__any_sync(0xffffffffu, quit)) break;  // a lane gave up inside its chunk (below): the whole warp stops
    unsigned long long base = 0, passed = 0;
    if (lane == 0) {
      base = atomicAdd(p.work, 32ull);
      passed = __ldcg(p.work + 6);
    }
    base = __shfl_sync(0xffffffffu, base, 0);
    if (base >= nchunks) break;
    if (p.c8_abort_shift >= 0) {
      // AUTO's optimistic run: too many blocks are failing the byte test for it to pay (warp-uniform decision)
      passed = __shfl_sync(0xffffffffu, passed, 0);
      if (passed > ((base << LO) >> p.c8_abort_shift) + QB_IMM8_ABORT_ALLOWANCE) {
        if (lane == 0) p.work[7] = 1ull;
        break;
      }
    }
    const unsigned long long ci = base + lane;
    if (ci >= nchunks) continue;
    unsigned npass = 0;
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
    long long cmin = LLONG_MAX;
    long long thr = min(min(best.val, gbest_dec(__ldcg(p.gbest))), p.seed_val);
    for (unsigned int jp = 0; jp < (1u << LS); ++jp) {
      if (jp) {
        const int r = __ffs(jp) - 1;
        const float sg = ((jp >> (r + 1)) & 1u) ? -1.f : 1.f;
        outer_flip<B, L, B + NX>(p, B + NX + r, sg, V, H, F);
      }
      if (LS <= 5 || (jp & 31u) == 0u) {
        thr = min(thr, gbest_dec(__ldcg(p.gbest)));
        if (LS > 5 && coarse8_give_up(p, npass, (my_chunks << LO) + ((unsigned long long)jp << NX), nthreads)) {
          quit = true;
          break;
        }
      }
      const int lrel = thr > LLONG_MAX - slack ? 0 : coarse8_limit(thr + slack - V, inv_unit);
      const int lc = min(max(lrel, lc_min), -1);
      unsigned a[1 << NX];
      float FX[NX];
#pragma unroll
      for (int t = 0; t < NX; ++t) FX[t] = F[t];
      coarse8_block_and<CB1, CB2, NX, APPROX, TABLE>(p, H, FX, 127 - lc, a);
      unsigned all = a[0];
#pragma unroll
      for (int h = 1; h < (1 << NX); ++h) all &= a[h];
      if (lrel < 0 && (all & 0x80808080u) == 0x80808080u) continue;  // no block holds a state under the limit
#pragma unroll 1
      for (int t = 0; t < (1 << NX); ++t) {
        // block j = (jp << NX) + t of the 10-bit walk: its bits B.. are the low NX bits of gray(j)
        const unsigned int j = (jp << NX) + (unsigned)t;
        const int part = (int)((j ^ (j >> 1)) & ((1u << NX) - 1u));
        unsigned ap = a[0];
#pragma unroll
        for (int h = 1; h < (1 << NX); ++h) ap = (part == h) ? a[h] : ap;
        if (lrel < 0 && (ap & 0x80808080u) == 0x80808080u) continue;
        ++npass;
        // exact fp32 table evaluation from the block's own base
        float Hb[B];
#pragma unroll
        for (int i = 0; i < B; ++i) {
          float h = H[i];
#pragma unroll
          for (int e = 0; e < NX; ++e) h += ((part >> e) & 1) ? p.Qs[B + e][i] : 0.f;
          Hb[i] = h;
        }
        float dv = 0.f;
#pragma unroll
        for (int e = 0; e < NX; ++e) {
          if (!((part >> e) & 1)) continue;
          dv += p.d[B + e] + F[e];
#pragma unroll
          for (int e2 = e + 1; e2 < NX; ++e2) dv += ((part >> e2) & 1) ? p.Qs[B + e][B + e2] : 0.f;
        }
        const long long val = V + (long long)dv + (long long)block_min<B1, B2, 0, NF>(p, Hb, F);
        cmin = min(cmin, val);
        if (val <= best.val) {
          const unsigned long long K = block_key(p, key_hi, dir, j, LO);
          if (val < best.val || K < best.K) best = Rec{val, K, c, j, 0u};
          if (val < thr) {
            thr = val;
            atomicMax(p.gbest, gbest_enc(val));
          }
        }
      }
    }
    if (p.mode == MODE_SEARCH_RECORD) p.chunk_min[ci] = cmin;
    if (npass) atomicAdd(p.work + 6, (unsigned long long)npass);
    ++my_chunks;
  }
  const Rec r = cta_reduce<TPB>(best);
  if (threadIdx.x == 0) p.cta_out[blockIdx.x] = r;
}

}  // namespace qb
