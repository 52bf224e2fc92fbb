// Batch kernel (BASELINE config C: 4096 independent n=16 instances): one CTA per instance.
//
// Everything for an instance happens inside its CTA, so the host only copies the
// coefficients in and the answers out:
//   1. quantization (same rule as the single-instance planner, qb_api.cu quantize()):
//      scale 2^e so every partial sum the CTA forms in fp32 stays below 2^24, exactness
//      check, error bound Eq;
//   2. inner table T over the B low bits, in shared memory;
//   3. search: thread t owns prefixes c = t, t + blockDim, ... of the k = n - B high bits;
//      one block of 2^B states per prefix, evaluated with the same FADD2/FMNMX3 table
//      scheme as the single-instance kernel (T pairs from shared memory, broadcast);
//   4. certified candidate set: every state within 2*Eq of the quantized minimum (all
//      exact ties when Eq = 0) is appended to a shared-memory list;
//   5. the candidates are re-evaluated in fp64 in the reference's eval_upper order
//      (_kernels.py:12-20, explicit __dmul_rn/__dadd_rn so no FMA contraction) and the
//      lowest (value, global Gray rank) one is the answer (solve_incremental's rule).
// A candidate-list overflow (massively tied instance) is flagged; the host re-solves that
// instance on the single-instance path.
#pragma once
#include "qb_common.cuh"
#include "qb_table.cuh"
#include "qb_batch_params.h"

#ifndef QB_BATCH_MINB
#define QB_BATCH_MINB 0  // 0: launch bounds on the block size only.  Measured (config C window): 86-102 regs
                         // 0.138-0.148 ms; 64 regs (4 x 256-thread CTAs/SM) 0.158 ms; 80 regs 0.158 ms
#endif

namespace qb {

__device__ __forceinline__ float2 batch_add2(float2 a, float2 b) { return __fadd2_rn(a, b); }

__device__ __forceinline__ float4 lds128(unsigned addr) {
  float4 v;
  asm("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(addr));
  return v;
}
__device__ __forceinline__ float2 lds64(unsigned addr) {
  float2 v;
  asm("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"(addr));
  return v;
}

// min over the 2^B states of one block, table from shared memory (broadcast LDS.128).  sT is a
// shared-space byte address made opaque by the caller each iteration, so ptxas cannot hoist all
// 2^B table loads out of the chunk loop into (spilled) registers.
template <int B1, int B2>
__device__ __forceinline__ float batch_block_min(unsigned sT, const float (&H)[B1 + B2]) {
  constexpr int NU = 1 << B1, NW = 1 << B2;
  float Bw[NW];
  subset_sums<B2>(Bw, 0.f, H);
  float A[NU];
  subset_sums<B1>(A, 0.f, H + B2);
  float rmin = 0.f;
#pragma unroll
  for (int u = 0; u < NU; ++u) {
    float acc = 0.f;
    if constexpr (NW >= 4) {
#pragma unroll
      for (int w = 0; w < NW; w += 4) {
        const float4 t4 = lds128(sT + 4u * (u * NW + w));
        const float2 c0 = batch_add2(make_float2(Bw[w], Bw[w + 1]), make_float2(t4.x, t4.y));
        const float2 c1 = batch_add2(make_float2(Bw[w + 2], Bw[w + 3]), make_float2(t4.z, t4.w));
        acc = (w == 0) ? fminf(c0.x, c0.y) : fminf(fminf(acc, c0.x), c0.y);
        acc = fminf(fminf(acc, c1.x), c1.y);
      }
    } else {
      const float2 t = lds64(sT + 4u * (u * NW));
      const float2 c = batch_add2(make_float2(Bw[0], Bw[1]), t);
      acc = fminf(c.x, c.y);
    }
    const float r = acc + A[u];
    rmin = (u == 0) ? r : fminf(rmin, r);
  }
  return rmin;
}

// Block base for prefix c (bits >= B): V = f(c << B) exactly, H_i = sum_{q>=B} x_q Qs[i][q].
template <int B>
__device__ __forceinline__ void batch_base(const float (*sQ)[BATCH_NMAX + 1], int n, unsigned long long x,
                                           long long& V, float (&H)[B]) {
#pragma unroll
  for (int i = 0; i < B; ++i) H[i] = 0.f;
  V = 0;
  for (int q = B; q < n; ++q) {
    const float xq = ((x >> q) & 1ull) ? 1.f : 0.f;
#pragma unroll
    for (int i = 0; i < B; ++i) H[i] = fmaf(xq, sQ[i][q], H[i]);
    float row = sQ[q][q];
    for (int r = q + 1; r < n; ++r) row = fmaf(((x >> r) & 1ull) ? 1.f : 0.f, sQ[q][r], row);
    V += (long long)(xq * row);
  }
}

// Append every state of block c whose value is <= theta.  Thread tid owns z = tid | (r << LB): the low
// LB bits are fixed (their field sum is formed once), the high B - LB bits are walked in reflected
// Gray order, so each state costs one field add, one table load and the compare (exact: integers
// below 2^24 in fp32, any summation order).
template <int B, int LB>
__device__ __forceinline__ void batch_enumerate(const float* sT, const float (&H)[B], long long V, long long theta,
                                                unsigned int c, int tid, unsigned long long* scand, int* scount) {
  if constexpr (B <= LB) {
    if (tid < (1 << B)) {
      float r = sT[tid];
#pragma unroll
      for (int i = 0; i < B; ++i)
        if ((tid >> i) & 1) r += H[i];
      if (V + (long long)r <= theta) {
        const int idx = atomicAdd(scount, 1);
        if (idx < BATCH_CAP) scand[idx] = ((unsigned long long)c << B) | (unsigned)tid;
      }
    }
  } else {
    constexpr int HB = B - LB;
    float lows = 0.f;
#pragma unroll
    for (int i = 0; i < LB; ++i)
      if ((tid >> i) & 1) lows += H[i];
    float hs = 0.f;
    unsigned r = 0;
#pragma unroll
    for (int g = 0; g < (1 << HB); ++g) {
      if (g) {
        const int bit = (g & 1) ? 0 : (g & 2) ? 1 : (g & 4) ? 2 : (g & 8) ? 3 : 4;  // ctz(g), g < 32
        r ^= 1u << bit;
        hs += ((r >> bit) & 1u) ? H[LB + bit] : -H[LB + bit];
      }
      const unsigned z = (unsigned)tid | (r << LB);
      const float v = sT[z] + (lows + hs);
      if (V + (long long)v <= theta) {
        const int idx = atomicAdd(scount, 1);
        if (idx < BATCH_CAP) scand[idx] = ((unsigned long long)c << B) | z;
      }
    }
  }
}

template <int B1, int B2>
#if QB_BATCH_MINB > 0
__global__ void __launch_bounds__(BATCH_TPB_MAX, QB_BATCH_MINB) batch_kernel(const BatchParams bp) {
#else
__global__ void __launch_bounds__(BATCH_TPB_MAX) batch_kernel(const BatchParams bp) {
#endif
  constexpr int B = B1 + B2;
  constexpr int NT = 1 << B;
  constexpr int CHUNK_CAP = 32;
  constexpr int CHMIN_CAP = 256;
  __shared__ double sC[BATCH_NMAX][BATCH_NMAX + 1];  // folded fp64 coefficients, symmetric copy
  __shared__ float sQ[BATCH_NMAX][BATCH_NMAX + 1];   // quantized: diagonal on the diagonal, symmetric off
  __shared__ __align__(16) float sT[NT];
  __shared__ double sred[BATCH_TPB_MAX / 32];
  __shared__ int sflag[3];                           // [0]: not integral, [1]: not exact, [2]: not finite
  __shared__ unsigned long long scand[BATCH_CAP];
  __shared__ unsigned int schunk[CHUNK_CAP];
  __shared__ long long schmin[CHMIN_CAP];  // per-chunk block minima of the search (chunks <= CHMIN_CAP)
  __shared__ int scount, schunks;
  __shared__ Rec sbest;
  const int n = bp.n;
  const int tid = threadIdx.x, nth = blockDim.x;
  const int ntri = n * (n + 1) / 2;
  const int lane = tid & 31, warp = tid >> 5;

  // ---- 0. load (folded by the host for the packed formats; folded here for the dense one) into
  //         shared memory: one pass over global memory.  Rows are dealt to warps and columns to
  //         lanes (n <= 24 < 32), so no index needs an integer division.  The same pass gathers
  //         what the quantization needs: nonzero count, integrality, r_in and the row sums.
  const int nwarps = (nth + 31) / 32;
  if (tid == 0) { sflag[0] = sflag[1] = sflag[2] = 0; scount = 0; schunks = 0; }
  __syncthreads();
  double part_rin = 0.0;
  int nnz = 0;
  for (int i = warp; i < n; i += nwarps) {
    const int j = i + lane;
    if (j >= n) continue;
    double v;
    if (bp.fmt == BATCH_DENSE_F64) {
      const double* C = static_cast<const double*>(bp.coeffs) + (size_t)blockIdx.x * n * n;
      const double a = C[i * n + j], b = (i == j) ? 0.0 : C[j * n + i];
      if (!isfinite(a) || !isfinite(b)) sflag[2] = 1;  // reported to the host as QB_E_ARG
      v = (i == j) ? a : __dadd_rn(a, b);
    } else {
      const int pidx = i * n - i * (i - 1) / 2 + (j - i);  // packed upper triangle, row-major
      v = bp.fmt == BATCH_UPPER_F32 ? (double)static_cast<const float*>(bp.coeffs)[(size_t)blockIdx.x * ntri + pidx]
                                    : static_cast<const double*>(bp.coeffs)[(size_t)blockIdx.x * ntri + pidx];
      if (!isfinite(v)) sflag[2] = 1;
    }
    sC[i][j] = v;
    sC[j][i] = v;
    if (v != 0.0) ++nnz;
    if (floor(v) != v) sflag[0] = 1;
    if (i < B) part_rin += fabs(v);  // r_in: every upper entry in a row of the block bits
  }
  __syncthreads();
  if (sflag[2]) {  // every coefficient is read here, so the host needs no pass over the batch
    if (tid == 0) bp.out[blockIdx.x] = BatchOut{0ull, 0.0, 3, 0};
    return;
  }

  // ---- 1. quantization: bound M = max(r_in, max row abs sum), as in qb_api.cu quantize()
  double part_row = 0.0;
  if (tid < n) {
    for (int j = 0; j < n; ++j) part_row += fabs(sC[tid][j]);
  }
  auto block_sum = [&](double v) {
    for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    __syncthreads();
    if (lane == 0) sred[warp] = v;
    __syncthreads();
    double t = 0.0;
    for (int w = 0; w < nwarps; ++w) t += sred[w];
    return t;
  };
  auto block_max = [&](double v) {
    for (int off = 16; off > 0; off >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, off));
    __syncthreads();
    if (lane == 0) sred[warp] = v;
    __syncthreads();
    double t = 0.0;
    for (int w = 0; w < nwarps; ++w) t = fmax(t, sred[w]);
    return t;
  };
  const double r_in = block_sum(part_rin);
  const double rmax = block_max(part_row);
  const double nnz_all = block_sum((double)nnz);
  const double M = fmax(r_in, rmax);
  const double LIM = 16777215.0;
  int e = 0;
  if (!(M == 0.0 || (sflag[0] == 0 && M <= LIM))) e = (int)floor(log2(LIM / M));
  for (int guard = 0; guard < 8; ++guard) {  // retry with e-1 if rounding pushed a sum over the bound
    double prin = 0.0, prow = 0.0;
    bool inexact = false;
    for (int i = warp; i < n; i += nwarps) {
      const int j = lane;
      if (j >= n) continue;
      const double x = ldexp(sC[i][j], e), q = nearbyint(x);
      sQ[i][j] = (float)q;
      if (j >= i && i < B) prin += fabs(q);
      if (j >= i && x != q) inexact = true;
    }
    __syncthreads();
    if (tid < n)
      for (int j = 0; j < n; ++j) prow += fabs((double)sQ[tid][j]);
    const double ok_in = block_sum(prin), ok_row = block_max(prow);
    if (fmax(ok_in, ok_row) <= LIM) {
      if (inexact) sflag[1] = 1;
      break;
    }
    --e;
  }
  __syncthreads();
  const bool exact = sflag[1] == 0;
  const long long Eq = exact ? 0 : (long long)((nnz_all + 1.0) / 2.0) + 1;
  // ---- 2. inner table T(z) = sum_{i<=j<B} q_ij z_i z_j
  if constexpr (B1 == 5 && B2 == 5) {
    // split z = (u, w), 5 bits each: T(u, w) = Tw(w) + Tu(u) + sum_{i<5} w_i G_i(u) with
    // G_i(u) = sum_{5<=j<10} u_j q_ij.  Warp 0 fills Tw; then thread t owns row u = t & 31 and a
    // contiguous w range, walked in reflected Gray order (one add per entry for the cross term).
    __shared__ float sTw[32];
    if (tid < 32) {
      float t = 0.f;
      for (int i = 0; i < 5; ++i) {
        if (!((tid >> i) & 1)) continue;
        t += sQ[i][i];
        for (int j = i + 1; j < 5; ++j)
          if ((tid >> j) & 1) t += sQ[i][j];
      }
      sTw[tid] = t;
    }
    __syncthreads();
    const int u = tid & 31, groups = nth >> 5;  // nth in {32, 64, 128, 256}
    const int wspan = 32 / groups, w0 = (tid >> 5) * wspan;
    float tu = 0.f, G[5];
#pragma unroll
    for (int i = 0; i < 5; ++i) G[i] = 0.f;
    for (int a = 0; a < 5; ++a) {
      if (!((u >> a) & 1)) continue;
      tu += sQ[5 + a][5 + a];
      for (int c2 = a + 1; c2 < 5; ++c2)
        if ((u >> c2) & 1) tu += sQ[5 + a][5 + c2];
#pragma unroll
      for (int i = 0; i < 5; ++i) G[i] += sQ[i][5 + a];
    }
    // cross term of the range start w0, then Gray steps over the low log2(wspan) bits of w
    float cross = 0.f;
#pragma unroll
    for (int i = 0; i < 5; ++i)
      if ((w0 >> i) & 1) cross += G[i];
    int w = w0;
    for (int g = 0; g < wspan; ++g) {
      if (g) {
        const int bit = __ffs(g) - 1;
        w ^= 1 << bit;
        float gi = G[0];
#pragma unroll
        for (int i = 1; i < 5; ++i)
          if (bit == i) gi = G[i];
        cross += ((w >> bit) & 1) ? gi : -gi;
      }
      sT[(u << 5) | w] = sTw[w] + tu + cross;
    }
    __syncthreads();
  } else {
    // doubling: T[z + 2^b] = T[z] + q_bb + sum_{i<b} z_i q_ib   (O(B) per entry; B < 10: n < 10)
    if (tid == 0) sT[0] = 0.f;
    __syncthreads();
#pragma unroll 1
    for (int b = 0; b < B; ++b) {
      for (int z = tid; z < (1 << b); z += nth) {
        float t = sT[z] + sQ[b][b];
        for (int i = 0; i < b; ++i) t = fmaf(((z >> i) & 1) ? 1.f : 0.f, sQ[i][b], t);
        sT[z + (1 << b)] = t;
      }
      __syncthreads();
    }
  }

  // ---- 3. search
  const int k = n - B;
  const unsigned int chunks = 1u << k;
  long long tmin = LLONG_MAX;
  Rec best{LLONG_MAX, ~0ull, 0ull, 0u, 0u};
  for (unsigned int c = tid; c < chunks; c += nth) {
    long long V;
    float H[B];
    batch_base<B>(sQ, n, (unsigned long long)c << B, V, H);
    unsigned tp = (unsigned)__cvta_generic_to_shared(sT);
    asm volatile("" : "+r"(tp));  // opaque per iteration: keeps ptxas from hoisting all 2^B table loads
    const long long val = V + (long long)batch_block_min<B1, B2>(tp, H);
    tmin = min(tmin, val);
    if (chunks <= CHMIN_CAP) schmin[c] = val;  // the collect pass below lists from these
    const unsigned long long K = ginv64(c);  // global Gray rank >> B (one block per chunk)
    if (val < best.val || (val == best.val && K < best.K)) best = Rec{val, K, c, 0u, 0u};
  }
  best = cta_reduce<BATCH_TPB_MAX>(best, (nth + 31) / 32);
  if (tid == 0) sbest = best;
  __syncthreads();
  const long long theta = sbest.val + 2 * Eq;

  // ---- 4. certified candidates: list the chunks whose block minimum is <= theta (from the minima
  //         the search stored, or recomputed for more than CHMIN_CAP chunks), then the whole CTA
  //         enumerates those blocks' states in parallel
  if (chunks <= CHMIN_CAP) {
    for (unsigned int c = tid; c < chunks; c += nth) {
      if (schmin[c] > theta) continue;
      const int idx = atomicAdd(&schunks, 1);
      if (idx < CHUNK_CAP) schunk[idx] = c;
    }
  } else if (tmin <= theta) {
    for (unsigned int c = tid; c < chunks; c += nth) {
      long long V;
      float H[B];
      batch_base<B>(sQ, n, (unsigned long long)c << B, V, H);
      unsigned tp = (unsigned)__cvta_generic_to_shared(sT);
      asm volatile("" : "+r"(tp));
      if (V + (long long)batch_block_min<B1, B2>(tp, H) > theta) continue;
      const int idx = atomicAdd(&schunks, 1);
      if (idx < CHUNK_CAP) schunk[idx] = c;
    }
  }
  __syncthreads();
  const int nch = min(schunks, CHUNK_CAP);
  for (int t = 0; t < nch; ++t) {
    const unsigned int c = schunk[t];
    long long V;
    float H[B];
    batch_base<B>(sQ, n, (unsigned long long)c << B, V, H);
    // thread tid owns the states z = tid + nth * r; nth is a power of two (32..256)
    switch (nth) {
      case 32: batch_enumerate<B, 5>(sT, H, V, theta, c, tid, scand, &scount); break;
      case 64: batch_enumerate<B, 6>(sT, H, V, theta, c, tid, scand, &scount); break;
      case 128: batch_enumerate<B, 7>(sT, H, V, theta, c, tid, scand, &scount); break;
      default: batch_enumerate<B, 8>(sT, H, V, theta, c, tid, scand, &scount); break;
    }
  }
  __syncthreads();

  // ---- 5. exact re-evaluation (reference eval_upper order) and tie rule, one warp
  if (warp == 0) {
    const int cnt = scount;
    BatchOut o{0ull, 0.0, 0, cnt};
    if (cnt > BATCH_CAP || schunks > CHUNK_CAP) {
      o.status = 1;
    } else if (cnt == 0) {
      o.status = 2;
    } else {
      double bv = 0.0;
      unsigned long long bx = 0, bk = ~0ull;
      bool have = false;
      for (int t = lane; t < cnt; t += 32) {
        const unsigned long long x = scand[t];
        // eval_upper over the set bits only, in the reference's (i, j) order (bit-identical, see
        // eval_upper_set_bits below)
        double acc = 0.0;
        for (unsigned long long xi = x; xi; xi &= xi - 1) {
          const int i = __ffsll((long long)xi) - 1;
          for (unsigned long long xj = xi; xj; xj &= xj - 1) acc = __dadd_rn(acc, sC[i][__ffsll((long long)xj) - 1]);
        }
        const unsigned long long key = ginv64(x);
        if (!have || acc < bv || (acc == bv && key < bk)) { bv = acc; bx = x; bk = key; have = true; }
      }
      for (int off = 16; off > 0; off >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, bv, off);
        const unsigned long long ox = __shfl_xor_sync(0xffffffffu, bx, off);
        const unsigned long long ok = __shfl_xor_sync(0xffffffffu, bk, off);
        const int oh = __shfl_xor_sync(0xffffffffu, (int)have, off);
        if (oh && (!have || ov < bv || (ov == bv && ok < bk))) { bv = ov; bx = ox; bk = ok; have = true; }
      }
      o.x = bx;
      o.value = bv;
    }
    if (lane == 0) bp.out[blockIdx.x] = o;
  }
}

}  // namespace qb

// ---------------------------------------------------------------------------------------------
// Warp-per-instance batch kernel (12 <= n <= BATCHW_NMAX): the whole instance lives in one warp and
// its slice of shared memory, so no phase needs a CTA barrier (__syncwarp only) and the 4 warps of a
// CTA (different instances) hide each other's latencies.  Same arithmetic, tie rule and outputs as
// batch_kernel: quantization as qb_api.cu quantize(), 5+5-bit table, one 1024-state block per chunk
// (2^(n-10) chunks, at most 32 per lane), certified candidates re-evaluated in fp64 in eval_upper
// order (_kernels.py:12-20), lowest (value, global Gray rank) wins (solver.py:118-136).
namespace qb {

constexpr int BATCHW_WARPS = 4;
constexpr int BATCHW_NMAX = 17;
constexpr int BATCHW_PER_LANE = 4;  // chunks per lane: 2^(n-10) / 32 <= 4 for n <= 17

__device__ __forceinline__ int packed_row(int i, int n) { return i * n - i * (i - 1) / 2; }

// eval_upper (_kernels.py:12-20) of a 0/1 vector over the packed upper triangle, adding only the terms
// with x_i = x_j = 1, in the reference's (i, j) order.  Bit-identical to adding every term: the skipped
// products are +-0.0, the running sum starts at +0.0 and can never become -0.0 under round-to-nearest
// (x + (-x) = +0.0), and adding +-0.0 to any other value returns it unchanged.
__device__ __forceinline__ double eval_upper_set_bits(const double* sCp, int n, unsigned long long x) {
  double acc = 0.0;
  for (unsigned long long xi = x; xi; xi &= xi - 1) {
    const int i = __ffsll((long long)xi) - 1;
    const double* row = sCp + packed_row(i, n) - i;  // row[j] = c_ij for j >= i
    for (unsigned long long xj = xi; xj; xj &= xj - 1) acc = __dadd_rn(acc, row[__ffsll((long long)xj) - 1]);
  }
  return acc;
}

__global__ void __launch_bounds__(BATCHW_WARPS * 32) batch_warp_kernel(const BatchParams bp) {
  constexpr int B1 = 5, B2 = 5, B = 10, NT = 1 << B;
  __shared__ __align__(16) float sTa[BATCHW_WARPS][NT];
  __shared__ float sQa[BATCHW_WARPS][BATCH_NMAX][BATCH_NMAX + 1];
  __shared__ double sCa[BATCHW_WARPS][BATCHW_NMAX * (BATCHW_NMAX + 1) / 2];
  __shared__ float sTwa[BATCHW_WARPS][32];
  __shared__ unsigned long long scanda[BATCHW_WARPS][BATCH_CAP];
  __shared__ unsigned int schunka[BATCHW_WARPS][32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int inst = blockIdx.x * BATCHW_WARPS + warp;
  if (inst >= bp.count) return;  // the whole warp leaves together
  const unsigned FULL = 0xffffffffu;
  float* sT = sTa[warp];
  float (*sQ)[BATCH_NMAX + 1] = sQa[warp];
  double* sC = sCa[warp];
  const int n = bp.n, ntri = n * (n + 1) / 2;

  // ---- 0. load (packed upper triangle; the dense fp64 format is folded here) + statistics
  bool bad = false, nonint = false;
  double part_rin = 0.0;
  int nnz = 0;
  for (int i = 0; i < n; ++i) {
    const int j = i + lane;
    if (j >= n) continue;
    double v;
    if (bp.fmt == BATCH_DENSE_F64) {
      const double* C = static_cast<const double*>(bp.coeffs) + (size_t)inst * n * n;
      const double a = C[i * n + j], b2 = (i == j) ? 0.0 : C[j * n + i];
      bad |= !isfinite(a) || !isfinite(b2);
      v = (i == j) ? a : __dadd_rn(a, b2);
    } else {
      const size_t pidx = (size_t)inst * ntri + packed_row(i, n) + (j - i);
      v = bp.fmt == BATCH_UPPER_F32 ? (double)static_cast<const float*>(bp.coeffs)[pidx]
                                    : static_cast<const double*>(bp.coeffs)[pidx];
      bad |= !isfinite(v);
    }
    sC[packed_row(i, n) + (j - i)] = v;
    if (v != 0.0) ++nnz;
    nonint |= floor(v) != v;
    if (i < B) part_rin += fabs(v);
  }
  if (__any_sync(FULL, bad)) {
    if (lane == 0) bp.out[inst] = BatchOut{0ull, 0.0, 3, 0};
    return;
  }
  __syncwarp();
  auto cget = [&](int i, int j) { return i <= j ? sC[packed_row(i, n) + (j - i)] : sC[packed_row(j, n) + (i - j)]; };
  auto wsum = [&](double v) {
    for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(FULL, v, off);
    return v;
  };
  auto wmax = [&](double v) {
    for (int off = 16; off > 0; off >>= 1) v = fmax(v, __shfl_xor_sync(FULL, v, off));
    return v;
  };
  // ---- 1. quantization (same rule as quantize() / batch_kernel)
  double part_row = 0.0;
  if (lane < n)
    for (int j = 0; j < n; ++j) part_row += fabs(cget(lane, j));
  const double r_in = wsum(part_rin), rmax = wmax(part_row);
  int nnz_all = nnz;
  for (int off = 16; off > 0; off >>= 1) nnz_all += __shfl_xor_sync(FULL, nnz_all, off);
  const bool integral = !__any_sync(FULL, nonint);
  const double M = fmax(r_in, rmax);
  const double LIM = 16777215.0;
  int e = 0;
  if (!(M == 0.0 || (integral && M <= LIM))) e = (int)floor(log2(LIM / M));
  bool exact = true;
  for (int guard = 0; guard < 8; ++guard) {
    double prin = 0.0;
    bool inexact = false;
    if (lane < n) {
      for (int i = 0; i < n; ++i) {
        const double x = ldexp(cget(i, lane), e), q = nearbyint(x);
        sQ[i][lane] = (float)q;
        if (lane >= i && i < B) prin += fabs(q);
        if (lane >= i && x != q) inexact = true;
      }
    }
    __syncwarp();
    double prow = 0.0;
    if (lane < n)
      for (int j = 0; j < n; ++j) prow += fabs((double)sQ[lane][j]);
    const double ok_in = wsum(prin), ok_row = wmax(prow);
    if (fmax(ok_in, ok_row) <= LIM) {
      exact = !__any_sync(FULL, inexact);
      break;
    }
    --e;
    __syncwarp();
  }
  const long long Eq = exact ? 0 : (long long)((nnz_all + 1) / 2) + 1;

  // ---- 2. table: T(u, w) = Tw(w) + Tu(u) + sum_{i<5} w_i G_i(u); lane u writes row u
  {
    float tw = 0.f;
    for (int i = 0; i < 5; ++i) {
      if (!((lane >> i) & 1)) continue;
      tw += sQ[i][i];
      for (int j = i + 1; j < 5; ++j)
        if ((lane >> j) & 1) tw += sQ[i][j];
    }
    sTwa[warp][lane] = tw;
    const int u = lane;
    float tu = 0.f, G[5];
#pragma unroll
    for (int i = 0; i < 5; ++i) G[i] = 0.f;
    for (int a = 0; a < 5; ++a) {
      if (!((u >> a) & 1)) continue;
      tu += sQ[5 + a][5 + a];
      for (int c2 = a + 1; c2 < 5; ++c2)
        if ((u >> c2) & 1) tu += sQ[5 + a][5 + c2];
#pragma unroll
      for (int i = 0; i < 5; ++i) G[i] += sQ[i][5 + a];
    }
    __syncwarp();
    float cross = 0.f;
    int w = 0;
#pragma unroll
    for (int g = 0; g < 32; ++g) {
      if (g) {
        const int bit = (g & 1) ? 0 : (g & 2) ? 1 : (g & 4) ? 2 : (g & 8) ? 3 : 4;  // ctz(g)
        w ^= 1 << bit;
        cross += ((w >> bit) & 1) ? G[bit] : -G[bit];
      }
      sT[(u << 5) | w] = sTwa[warp][w] + tu + cross;
    }
  }
  __syncwarp();

  // ---- 3. search: chunk c = lane + 32 t, one 1024-state block each
  const unsigned int chunks = 1u << (n - B);
  long long vals[BATCHW_PER_LANE];
  long long bestv = LLONG_MAX;
  unsigned long long bestk = ~0ull;
#pragma unroll
  for (int t = 0; t < BATCHW_PER_LANE; ++t) {
    vals[t] = LLONG_MAX;
    const unsigned int c = (unsigned)lane + 32u * t;
    if (c >= chunks) continue;
    long long V;
    float H[B];
    batch_base<B>(sQ, n, (unsigned long long)c << B, V, H);
    unsigned tp = (unsigned)__cvta_generic_to_shared(sT);
    asm volatile("" : "+r"(tp));
    const long long val = V + (long long)batch_block_min<B1, B2>(tp, H);
    vals[t] = val;
    const unsigned long long K = ginv64(c);
    if (val < bestv || (val == bestv && K < bestk)) { bestv = val; bestk = K; }
  }
  for (int off = 16; off > 0; off >>= 1) {
    const long long ov = __shfl_xor_sync(FULL, bestv, off);
    const unsigned long long ok = __shfl_xor_sync(FULL, bestk, off);
    if (ov < bestv || (ov == bestv && ok < bestk)) { bestv = ov; bestk = ok; }
  }
  const long long theta = bestv + 2 * Eq;

  // ---- 4. certified candidates: blocks with minimum <= theta (ballot append), then their states
  int nch = 0;
#pragma unroll
  for (int t = 0; t < BATCHW_PER_LANE; ++t) {
    const bool hit = vals[t] <= theta;
    const unsigned m = __ballot_sync(FULL, hit);
    const int pos = nch + __popc(m & ((1u << lane) - 1u));
    if (hit && pos < 32) schunka[warp][pos] = (unsigned)lane + 32u * t;
    nch += __popc(m);
  }
  __syncwarp();
  int cnt = 0;
  if (nch <= 32) {
    for (int t = 0; t < nch; ++t) {
      const unsigned int c = schunka[warp][t];
      long long V;
      float H[B];
      batch_base<B>(sQ, n, (unsigned long long)c << B, V, H);
      float lows = 0.f;
#pragma unroll
      for (int i = 0; i < 5; ++i)
        if ((lane >> i) & 1) lows += H[i];
      float hs = 0.f;
      unsigned r = 0;
#pragma unroll
      for (int g = 0; g < 32; ++g) {
        if (g) {
          const int bit = (g & 1) ? 0 : (g & 2) ? 1 : (g & 4) ? 2 : (g & 8) ? 3 : 4;
          r ^= 1u << bit;
          hs += ((r >> bit) & 1u) ? H[5 + bit] : -H[5 + bit];
        }
        const unsigned z = (unsigned)lane | (r << 5);
        const bool hit = V + (long long)(sT[z] + (lows + hs)) <= theta;
        const unsigned m = __ballot_sync(FULL, hit);
        const int pos = cnt + __popc(m & ((1u << lane) - 1u));
        if (hit && pos < BATCH_CAP) scanda[warp][pos] = ((unsigned long long)c << B) | z;
        cnt += __popc(m);
      }
    }
  }
  __syncwarp();

  // ---- 5. exact re-evaluation in eval_upper order, lowest (value, global Gray rank)
  BatchOut o{0ull, 0.0, 0, cnt};
  if (nch > 32 || cnt > BATCH_CAP) {
    o.status = 1;
  } else if (cnt == 0) {
    o.status = 2;
  } else {
    double bv = 0.0;
    unsigned long long bx = 0, bk = ~0ull;
    bool have = false;
    if (lane < cnt) {
      const unsigned long long x = scanda[warp][lane];
      const double acc = eval_upper_set_bits(sC, n, x);
      bv = acc;
      bx = x;
      bk = ginv64(x);
      have = true;
    }
    for (int off = 16; off > 0; off >>= 1) {
      const double ov = __shfl_xor_sync(FULL, bv, off);
      const unsigned long long ox = __shfl_xor_sync(FULL, bx, off);
      const unsigned long long ok = __shfl_xor_sync(FULL, bk, off);
      const int oh = __shfl_xor_sync(FULL, (int)have, off);
      if (oh && (!have || ov < bv || (ov == bv && ok < bk))) { bv = ov; bx = ox; bk = ok; have = true; }
    }
    o.x = bx;
    o.value = bv;
  }
  if (lane == 0) bp.out[inst] = o;
}

}  // namespace qb
