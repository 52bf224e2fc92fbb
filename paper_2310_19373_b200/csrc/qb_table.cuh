// Blocked Gray-walk traversal kernel ("table" variant) for sm_100a.
//
// One thread owns one chunk at a time: the states whose top k bits equal the chunk
// prefix s.  Inside the chunk the L free bits are split into B inner bits and
// LO = L - B outer bits:
//
//   * outer bits are walked in reflected Gray order, one flip per block: bit
//     l = B + __ffs(j) - 1, direction from bit l+1 of j (Alg. 1 / reference
//     _kernels.py:63-71).  The flip applies Eq. 3, dV = s_l (Q_ll + F_l), and the
//     row update of the local fields H (inner bits) and F (outer bits), all in
//     registers with compile-time indices (one switch case per outer bit);
//   * the 2^B inner states of a block are evaluated from a per-instance table:
//         f(outer, z) = V + sum_{i<B} z_i H_i + T(z),   z = (u << B2) | w
//     computed as min_u [ A_u + min_w (Bw_w + T(u,w)) ] with A/Bw subset sums of H.
//     Each state costs one packed add (FADD2 on two states, T pair from the constant
//     bank via LDCU.128) and half a 3-input min (FMNMX3).
//
// Arithmetic is exact: the host scales Q by 2^e into integers whose partial sums stay
// below 2^24 in magnitude, so every fp32 add is an exact integer add; block bases V
// are int64.  When Q * 2^e is not integral the search is a certified filter and the
// host re-evaluates the near-minimal candidates exactly (qb_api.cu).
#pragma once
#include "qb_common.cuh"

#ifndef QB_PREFIX_UNROLL
#define QB_PREFIX_UNROLL 1  // unroll of the chunk-start evaluation loop over prefix bits
#endif

namespace qb {

__device__ __forceinline__ float2 add_f32x2(float2 a, float2 b) { return __fadd2_rn(a, b); }

// Chunk-start / block-base ("prefix") evaluation.  For the state x with its B inner bits
// treated as zero: V = f(x & ~innermask) (int64, exact), H_i = sum_{q>=B} x_q Qs[i][q] for the
// inner bits, F_m = sum_{q>=B} x_q Qs[B+m][q] for the outer free bits.  Only bits q >= q_start
// may be set (q_start = L at a chunk start, B for an arbitrary block).  All loops are uniform
// across the warp so the Qs[.][q] operands are warp-uniform constant-bank loads.
template <int B, int L>
__device__ __forceinline__ void base_eval(const TableParams& p, unsigned long long x, int q_start, long long& V,
                                          float (&H)[B], float (&F)[(L - B) > 0 ? (L - B) : 1]) {
#pragma unroll
  for (int i = 0; i < B; ++i) H[i] = 0.f;
#pragma unroll
  for (int m = 0; m < ((L - B) > 0 ? (L - B) : 1); ++m) F[m] = 0.f;
  V = 0;
  constexpr int kUnroll = QB_PREFIX_UNROLL;
#pragma unroll kUnroll
  for (int q = q_start; q < p.n; ++q) {
    const float xq = ((x >> q) & 1ull) ? 1.f : 0.f;
#pragma unroll
    for (int i = 0; i < B; ++i) H[i] = fmaf(xq, p.Qs[i][q], H[i]);
#pragma unroll
    for (int m = 0; m < L - B; ++m) F[m] = fmaf(xq, p.Qs[B + m][q], F[m]);
    float row = p.d[q];
    for (int r = q + 1; r < p.n; ++r) row = fmaf(((x >> r) & 1ull) ? 1.f : 0.f, p.Qs[q][r], row);
    V += (long long)(xq * row);
  }
}

// Outer flip of bit ELL (compile-time in each branch; runtime `ell` selects it) with sign
// sg = +-1: Eq. 3 value update, then the row/column update of every local field (H: table bits,
// F: bits [B, L)).  Linear if-chain from the lowest outer bit: ctz(j) is 0 half the time.
template <int B, int L, int ELL>
__device__ __forceinline__ void outer_flip(const TableParams& p, int ell, float sg, long long& V, float (&H)[B],
                                           float (&F)[(L - B) > 0 ? (L - B) : 1]) {
  if constexpr (ELL < L) {
    if (ell == ELL) {
      V += (long long)(sg * (p.d[ELL] + F[ELL - B]));
#pragma unroll
      for (int i = 0; i < B; ++i) H[i] = fmaf(sg, p.Qs[ELL][i], H[i]);  // row ELL (Qs symmetric): vector loads
#pragma unroll
      for (int m = 0; m < L - B; ++m) F[m] = fmaf(sg, p.Qs[ELL][B + m], F[m]);
    } else {
      outer_flip<B, L, ELL + 1>(p, ell, sg, V, H, F);
    }
  }
}

__host__ __device__ constexpr int ctz_c(int k) { return (k & 1) ? 0 : 1 + ctz_c(k >> 1); }

// S[m] = base + sum_{i : bit i of m} h[i] for m < 2^NB; S[m + 2^i] = S[m] + h[i], pairs via FADD2
template <int NB>
__device__ __forceinline__ void subset_sums(float* S, float base, const float* h) {
  S[0] = base;
  if constexpr (NB > 0) {
    S[1] = base + h[0];
#pragma unroll
    for (int i = 1; i < NB; ++i) {
#pragma unroll
      for (int m = 0; m < (1 << i); m += 2) {
        const float2 r = __fadd2_rn(make_float2(S[m], S[m + 1]), make_float2(h[i], h[i]));
        S[m + (1 << i)] = r.x;
        S[m + 1 + (1 << i)] = r.y;
      }
    }
  }
}

// Minimum over the 2^(B+SB) states of a super-block, relative to its base value V (all block
// bits zero).  The B table bits are split into u (B1 high) and w (B2 low):
//     f(u, w) = V + A_u + Bw_w + T(u, w)
// with A / Bw subset sums of the fields H.  Per state: half an FADD2 (two states, T pair from the
// constant bank through uniform registers), half an FMNMX3, and a quarter of an LDCU.128.
template <int B1, int B2, int SB, int NF>
__device__ __forceinline__ float block_min_p1(const TableParams& p, const float (&H)[B1 + B2], const float (&F)[NF]) {
  constexpr int B = B1 + B2, NU = 1 << B1, NW = 1 << B2, P = 1 << SB;
  static_assert(B2 >= 1, "inner low part needs at least one bit");
  float rmin = 0.f;
#pragma unroll
  for (int s = 0; s < P; ++s) {
    float hs[B];
#pragma unroll
    for (int i = 0; i < B; ++i) {
      float h = H[i];
#pragma unroll
      for (int t = 0; t < SB; ++t)
        if ((s >> t) & 1) h += p.Qs[i][B + t];
      hs[i] = h;
    }
    float dl = 0.f;
#pragma unroll
    for (int t = 0; t < SB; ++t) {
      if (!((s >> t) & 1)) continue;
      dl += p.d[B + t] + F[t];
#pragma unroll
      for (int t2 = t + 1; t2 < SB; ++t2)
        if ((s >> t2) & 1) dl += p.Qs[B + t][B + t2];
    }
    // subset sums: Bw over the w bits, A over the u bits (independent adds, no serial chain);
    // from the second bit on, pairs of sums are extended with one packed FADD2
    float Bw[NW];
    subset_sums<B2>(Bw, 0.f, hs);
    float A[NU];
    subset_sums<B1>(A, dl, hs + B2);
#pragma unroll
    for (int kk = 0; kk < NU; kk += 2) {
      float ru[2];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        if (kk + h >= NU) { ru[h] = ru[0]; continue; }
        const int u = kk + h;
        float acc = 0.f;
#pragma unroll
        for (int w = 0; w < NW; w += 2) {
          const float2 t = *reinterpret_cast<const float2*>(&p.T[u * NW + w]);
          const float2 c = add_f32x2(make_float2(Bw[w], Bw[w + 1]), t);
          acc = (w == 0) ? fminf(c.x, c.y) : fminf(fminf(acc, c.x), c.y);
        }
        ru[h] = acc + A[u];
      }
      rmin = (s == 0 && kk == 0) ? fminf(ru[0], ru[1]) : fminf(fminf(rmin, ru[0]), ru[1]);
    }
  }
  return rmin;
}

template <int B1, int B2, int SB, int NF>
__device__ __forceinline__ float block_min(const TableParams& p, const float (&H)[B1 + B2], const float (&F)[NF]) {
  static_assert(SB == 0, "sub-block table sharing was measured slower (register spills) and is not built");
  return block_min_p1<B1, B2, SB, NF>(p, H, F);
}

// Every state of super-block j of chunk prefix s, evaluated directly from its base (finalize and
// collect; rare).  Calls fn(z_block, value) for the 2^(B+SB) states, z_block = (sub << B) | z.
template <int B, int SB, int L, class Fn>
__device__ __forceinline__ void for_block_states(const TableParams& p, unsigned long long xo, int lane, int lanes,
                                                 Fn&& fn) {
  constexpr int NF = (L - B) > 0 ? (L - B) : 1;
#pragma unroll 1
  for (int sb = 0; sb < (1 << SB); ++sb) {
    long long V;
    float H[B], F[NF];
    base_eval<B, L>(p, xo | ((unsigned long long)sb << B), B, V, H, F);
#pragma unroll 1
    for (unsigned int z = lane; z < (1u << B); z += lanes) {
      float r = p.T[z];
#pragma unroll
      for (int i = 0; i < B; ++i)
        if ((z >> i) & 1u) r += H[i];
      fn(((unsigned int)sb << B) | z, V + (long long)r);
    }
  }
}

// End of every search kernel (table, coarse, field walk): publish this CTA's record; the last CTA
// to finish reduces all records and writes p.final_out (the former separate finalize launch).
// Exact search (MODE_SEARCH): it also re-evaluates the winning block with all its threads and
// picks the lowest-key minimiser inside it.  Recording search (MODE_SEARCH_RECORD, the certified
// collect path): only the minimum value is needed (the collect pass reads it as its threshold).
template <int B, int L, int TPB>
__device__ __noinline__ void search_final(const TableParams& p);

template <int B, int L, int TPB>
__device__ __noinline__ void search_tail(const TableParams& p, const Rec r) {
  __shared__ int last;
  if (threadIdx.x == 0) {
    p.cta_out[blockIdx.x] = r;
    __threadfence();  // the record is visible device-wide before the count that announces it
    last = atomicAdd(p.done, 1ull) == (unsigned long long)gridDim.x - 1ull;
  }
  __syncthreads();
  if (last) search_final<B, L, TPB>(p);
}

template <int B, int L, int TPB>
__device__ __forceinline__ void search_epilogue(const TableParams& p, const Rec& mine) {
  search_tail<B, L, TPB>(p, cta_reduce<TPB>(mine));
}

// The last CTA's work: reduce every CTA record, then (exact search) rescan the winning block.
template <int B, int L, int TPB>
__device__ __noinline__ void search_final(const TableParams& p) {
  __threadfence();
  Rec best{LLONG_MAX, ~0ull, 0ull, 0u, 0u};
  for (int i = threadIdx.x; i < p.nrec; i += TPB) {
    Rec o;
    o.val = __ldcg(&p.cta_out[i].val);
    o.K = __ldcg(&p.cta_out[i].K);
    o.c = __ldcg(&p.cta_out[i].c);
    o.j = __ldcg(&p.cta_out[i].j);
    o.pad = 0u;
    if (rec_less(o, best)) best = o;
  }
  best = cta_reduce<TPB>(best);
  __shared__ Rec win;
  if (threadIdx.x == 0) win = best;
  __syncthreads();
  best = win;
  if (best.val == LLONG_MAX || p.mode != MODE_SEARCH) {
    if (threadIdx.x == 0)
      *p.final_out = FinalOut{best.val, ~0ull, 0ull, best.c, best.j, best.val != LLONG_MAX ? 1 : 0};
    return;
  }
  const unsigned long long s = chunk_prefix(p, best.c);
  int dir;
  (void)chunk_key(p, s, dir);
  const unsigned long long xo = (s << L) | ((unsigned long long)(best.j ^ (best.j >> 1)) << B);
  unsigned int bk = ~0u, bz = 0u;
  const unsigned int jj = best.j;
  const long long target = best.val;
  for_block_states<B, 0, L>(p, xo, threadIdx.x, TPB, [&](unsigned int zb, long long val) {
    if (val == target) {
      const unsigned int kin = inner_key(p, dir, jj, zb, B);
      if (kin < bk) { bk = kin; bz = zb; }
    }
  });
  // (key, state) minimum over the CTA; keys are unique within the block, so the state follows its key
  const unsigned long long kz = ((unsigned long long)bk << 32) | bz;
  unsigned long long m = kz;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) m = min(m, __shfl_xor_sync(0xffffffffu, m, off));
  __shared__ unsigned long long wmin[TPB / 32];
  if ((threadIdx.x & 31) == 0) wmin[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < TPB / 32; ++w) m = min(m, wmin[w]);
    const unsigned int k = (unsigned int)(m >> 32), z = (unsigned int)(m & 0xffffffffu);
    *p.final_out = FinalOut{best.val, (best.K << B) | k, xo | z, best.c, best.j, k != ~0u ? 1 : 0};
  }
}

// The same reduction as a one-CTA launch after a search kernel that only writes its records (the
// coarse kernel: any code in its tail, even an out-of-line call, changes ptxas's integer-add pipe
// split in the hot loop -- IADD3 on the ALU pipe vs VIADD on the FMA pipe -- measured 36 -> 39 ms).
template <int B, int L, int TPB>
__global__ void __launch_bounds__(TPB) finalize_kernel(const __grid_constant__ TableParams p) {
  search_final<B, L, TPB>(p);
}

// ---- certified-filter collect pass (float path / all-minimisers), three small launches:
// 1. chunks whose recorded minimum is <= theta -> chunk_list
template <int B1, int B2, int SB, int L>
__global__ void __launch_bounds__(256) collect_mark_kernel(const __grid_constant__ TableParams p) {
  const unsigned long long nchunks = p.chunk_end - p.chunk_begin;
  const long long theta = collect_theta(p);
  for (unsigned long long ci = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; ci < nchunks;
       ci += (unsigned long long)gridDim.x * blockDim.x) {
    if (p.chunk_min[ci] <= theta) {
      const unsigned long long idx = atomicAdd(&p.counts[0], 1ull);
      if (idx < p.list_cap) p.chunk_list[idx] = ci;
    }
  }
}

// 2. one thread per (listed chunk, block): block base by direct evaluation, table block minimum,
//    blocks <= theta -> block_list
template <int B1, int B2, int SB, int L>
__global__ void __launch_bounds__(128) collect_blocks_kernel(const __grid_constant__ TableParams p) {
  constexpr int B = B1 + B2, BE = B + SB, LO = L - BE;
  constexpr int NF = (L - B) > 0 ? (L - B) : 1;
  const unsigned long long nlisted = min(p.counts[0], p.list_cap);
  const long long theta = collect_theta(p);
  const unsigned long long total = nlisted << LO;
  for (unsigned long long g = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; g < total;
       g += (unsigned long long)gridDim.x * blockDim.x) {
    const unsigned long long ci = p.chunk_list[g >> LO];
    const unsigned int j = (unsigned int)(g & ((1ull << LO) - 1ull));
    const unsigned long long s = chunk_prefix(p, p.chunk_begin + ci);
    const unsigned long long xo = (s << L) | ((unsigned long long)(j ^ (j >> 1)) << BE);
    long long V;
    float H[B], F[NF];
    base_eval<B, L>(p, xo, B, V, H, F);
    if (V + (long long)block_min<B1, B2, SB, NF>(p, H, F) <= theta) {
      const unsigned long long idx = atomicAdd(&p.counts[1], 1ull);
      if (idx < p.list_cap) p.block_list[idx] = (ci << 32) | j;
    }
  }
}

// 3. one warp per listed block: every state <= theta -> cand
template <int B1, int B2, int SB, int L>
__global__ void __launch_bounds__(128) collect_states_kernel(const __grid_constant__ TableParams p) {
  constexpr int B = B1 + B2, BE = B + SB;
  const unsigned long long nblocks = min(p.counts[1], p.list_cap);
  const long long theta = collect_theta(p);
  const int lane = threadIdx.x & 31;
  for (unsigned long long w = ((unsigned long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < nblocks;
       w += ((unsigned long long)gridDim.x * blockDim.x) >> 5) {
    const unsigned long long e = p.block_list[w];
    const unsigned long long ci = e >> 32;
    const unsigned int j = (unsigned int)(e & 0xffffffffu);
    const unsigned long long s = chunk_prefix(p, p.chunk_begin + ci);
    const unsigned long long xo = (s << L) | ((unsigned long long)(j ^ (j >> 1)) << BE);
    // overflow path (MODE_REDUCE_*): exact fp64 value of every candidate, lexicographic (value, key) minimum;
    // each lane keeps its own minimum over the block and the warp issues ONE atomic per block (a massively
    // tied instance has 10^9 candidates: one atomic each on a single word took seconds)
    unsigned long long lane_min = ~0ull;
    const unsigned long long best_vk = (p.mode == MODE_REDUCE_KEY) ? __ldcg(&p.red[0]) : 0ull;
    for_block_states<B, SB, L>(p, xo, lane, 32, [&](unsigned int zb, long long val) {
      if (val > theta) return;
      const unsigned long long x = xo | zb;
      if (p.mode == MODE_COLLECT) {
        const unsigned long long idx = atomicAdd(p.cand_count, 1ull);
        if (idx < p.cand_cap) p.cand[idx] = x;
      } else {
        const unsigned long long vk = ordered_f64(eval_upper_dev(p.coeffs64, p.n, x));
        if (p.mode == MODE_REDUCE_VALUE) lane_min = min(lane_min, vk);
        else if (vk == best_vk) lane_min = min(lane_min, state_tie_key(x, p.n, p.m_tie, p.rule));
      }
    });
    if (p.mode != MODE_COLLECT) {
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) lane_min = min(lane_min, __shfl_xor_sync(0xffffffffu, lane_min, off));
      if (lane == 0 && lane_min != ~0ull) atomicMin(&p.red[p.mode == MODE_REDUCE_VALUE ? 0 : 1], lane_min);
    }
  }
}

template <int B1, int B2, int SB, int L, int TPB>
__global__ void __launch_bounds__(TPB, QB_MINB) table_kernel(const __grid_constant__ TableParams p) {
  constexpr int B = B1 + B2;
  constexpr int BE = B + SB;
  constexpr int LO = L - BE;
  constexpr int NF = (L - B) > 0 ? (L - B) : 1;
  static_assert(LO >= 0, "block bits exceed chunk bits");
  Rec best{LLONG_MAX, ~0ull, 0ull, 0u, 0u};
  const unsigned long long nchunks = p.chunk_end - p.chunk_begin;
  const int lane = threadIdx.x & 31;
  // Work distribution: 32 consecutive chunks per warp from a global counter (one atomic per 32
  // chunks), so all SMs finish within one chunk of each other.
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
    base_eval<B, L>(p, s << L, L, V, H, F);
    int dir;
    const unsigned long long key_hi = chunk_key(p, s, dir);
    long long cmin = LLONG_MAX;
    for (unsigned int j = 0; j < (1u << LO); ++j) {
      if (j) {
        const int r = __ffs(j) - 1;
        const float sg = ((j >> (r + 1)) & 1u) ? -1.f : 1.f;
        outer_flip<B, L, BE>(p, BE + r, sg, V, H, F);
      }
      const float rm = block_min<B1, B2, SB, NF>(p, H, F);
      const long long val = V + (long long)rm;
      cmin = min(cmin, val);
      if (val <= best.val) {
        const unsigned long long K = block_key(p, key_hi, dir, j, LO);
        if (val < best.val || K < best.K) best = Rec{val, K, c, j, 0u};
      }
    }
    if (p.mode == MODE_SEARCH_RECORD) p.chunk_min[ci] = cmin;
  }
  search_epilogue<B1 + B2, L, TPB>(p, best);
}

// Standalone chunk-start ("prefix") evaluation for the qb_prefix_eval test hook: runs the very
// base_eval<B, L> the traversal uses and converts back to coefficient units (x 2^-e).
template <int B1, int B2, int SB, int L>
__global__ void prefix_eval_kernel(const __grid_constant__ TableParams p, double* vals, double* fields, int e) {
  constexpr int B = B1 + B2;
  constexpr int NF = (L - B) > 0 ? (L - B) : 1;
  const unsigned long long idx = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x;
  const unsigned long long c = p.chunk_begin + idx;
  if (c >= p.chunk_end) return;
  const unsigned long long s = chunk_prefix(p, c);
  long long V;
  float H[B], F[NF];
  base_eval<B, L>(p, s << L, L, V, H, F);
  vals[idx] = ldexp((double)V, -e);
#pragma unroll
  for (int i = 0; i < B; ++i) fields[idx * L + i] = ldexp((double)(H[i] + p.d[i]), -e);
#pragma unroll
  for (int m = 0; m < L - B; ++m) fields[idx * L + B + m] = ldexp((double)(F[m] + p.d[B + m]), -e);
}

}  // namespace qb
