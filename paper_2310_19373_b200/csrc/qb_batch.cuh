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

template <int B1, int B2>
__global__ void __launch_bounds__(BATCH_TPB_MAX) batch_kernel(const BatchParams bp) {
  constexpr int B = B1 + B2;
  constexpr int NT = 1 << B;
  constexpr int CHUNK_CAP = 32;
  __shared__ double sC[BATCH_NMAX][BATCH_NMAX + 1];  // folded fp64 coefficients, symmetric copy
  __shared__ float sQ[BATCH_NMAX][BATCH_NMAX + 1];   // quantized: diagonal on the diagonal, symmetric off
  __shared__ __align__(16) float sT[NT];
  __shared__ double sred[BATCH_TPB_MAX / 32];
  __shared__ int sflag[3];                           // [0]: not integral, [1]: not exact, [2]: not finite
  __shared__ unsigned long long scand[BATCH_CAP];
  __shared__ unsigned int schunk[CHUNK_CAP];
  __shared__ int scount, schunks;
  __shared__ Rec sbest;
  const int n = bp.n;
  const int tid = threadIdx.x, nth = blockDim.x;
  const int ntri = n * (n + 1) / 2;
  const int lane = tid & 31, warp = tid >> 5;

  // ---- 0. load (folded by the host for the packed formats; folded here for the dense one) into
  //         shared memory: one pass over global memory
  if (tid == 0) { sflag[0] = sflag[1] = sflag[2] = 0; scount = 0; schunks = 0; }
  __syncthreads();
  if (bp.fmt == BATCH_DENSE_F64) {
    const double* C = static_cast<const double*>(bp.coeffs) + (size_t)blockIdx.x * n * n;
    for (int idx = tid; idx < n * n; idx += nth) {
      const int i = idx / n, j = idx % n;
      if (j < i) continue;
      const double a = C[idx], b = (i == j) ? 0.0 : C[j * n + i];
      if (!isfinite(a) || !isfinite(b)) sflag[2] = 1;  // reported to the host as QB_E_ARG
      const double v = (i == j) ? a : __dadd_rn(a, b);
      sC[i][j] = v;
      sC[j][i] = v;
    }
  } else {
    for (int p = tid; p < ntri; p += nth) {
      // row i of the packed upper triangle starts at i*n - i*(i-1)/2
      int i = 0;
      while ((i + 1) * n - (i + 1) * i / 2 <= p) ++i;
      const int j = i + (p - (i * n - i * (i - 1) / 2));
      const double v = bp.fmt == BATCH_UPPER_F32 ? (double)static_cast<const float*>(bp.coeffs)[(size_t)blockIdx.x * ntri + p]
                                                 : static_cast<const double*>(bp.coeffs)[(size_t)blockIdx.x * ntri + p];
      if (!isfinite(v)) sflag[2] = 1;
      sC[i][j] = v;
      sC[j][i] = v;
    }
  }
  __syncthreads();
  if (sflag[2]) {  // every coefficient is read here, so the host needs no pass over the batch
    if (tid == 0) bp.out[blockIdx.x] = BatchOut{0ull, 0.0, 3, 0};
    return;
  }

  // ---- 1. quantization: bound M = max(r_in, max row abs sum), as in qb_api.cu quantize()
  double part_rin = 0.0, part_row = 0.0;
  int nnz = 0;
  for (int idx = tid; idx < n * n; idx += nth) {
    const int i = idx / n, j = idx % n;
    if (j < i) continue;
    const double v = sC[i][j];
    if (v != 0.0) ++nnz;
    if (floor(v) != v) sflag[0] = 1;
    if (i < B) part_rin += fabs(v);  // r_in: every upper entry in a row of the block bits
  }
  if (tid < n) {
    for (int j = 0; j < n; ++j) part_row += fabs(sC[tid][j]);
  }
  auto block_sum = [&](double v) {
    for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    __syncthreads();
    if (lane == 0) sred[warp] = v;
    __syncthreads();
    double t = 0.0;
    for (int w = 0; w < (nth + 31) / 32; ++w) t += sred[w];
    return t;
  };
  auto block_max = [&](double v) {
    for (int off = 16; off > 0; off >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, off));
    __syncthreads();
    if (lane == 0) sred[warp] = v;
    __syncthreads();
    double t = 0.0;
    for (int w = 0; w < (nth + 31) / 32; ++w) t = fmax(t, sred[w]);
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
    for (int idx = tid; idx < n * n; idx += nth) {
      const int i = idx / n, j = idx % n;
      const double q = nearbyint(ldexp(sC[i][j], e));
      sQ[i][j] = (float)q;
      if (j >= i && i < B) prin += fabs(q);
    }
    __syncthreads();
    if (tid < n)
      for (int j = 0; j < n; ++j) prow += fabs((double)sQ[tid][j]);
    const double ok_in = block_sum(prin), ok_row = block_max(prow);
    if (fmax(ok_in, ok_row) <= LIM) break;
    --e;
  }
  for (int idx = tid; idx < n * n; idx += nth) {
    const int i = idx / n, j = idx % n;
    if (j >= i && ldexp(sC[i][j], e) != (double)sQ[i][j]) sflag[1] = 1;
  }
  // ---- 2. inner table by doubling: T[z + 2^b] = T[z] + q_bb + sum_{i<b} z_i q_ib   (O(B) per entry)
  if (tid == 0) sT[0] = 0.f;
  __syncthreads();
  const bool exact = sflag[1] == 0;
  const long long Eq = exact ? 0 : (long long)((nnz_all + 1.0) / 2.0) + 1;
#pragma unroll 1
  for (int b = 0; b < B; ++b) {
    for (int z = tid; z < (1 << b); z += nth) {
      float t = sT[z] + sQ[b][b];
      for (int i = 0; i < b; ++i) t = fmaf(((z >> i) & 1) ? 1.f : 0.f, sQ[i][b], t);
      sT[z + (1 << b)] = t;
    }
    __syncthreads();
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
    const unsigned long long K = ginv64(c);  // global Gray rank >> B (one block per chunk)
    if (val < best.val || (val == best.val && K < best.K)) best = Rec{val, K, c, 0u, 0u};
  }
  best = cta_reduce<BATCH_TPB_MAX>(best, (nth + 31) / 32);
  if (tid == 0) sbest = best;
  __syncthreads();
  const long long theta = sbest.val + 2 * Eq;

  // ---- 4. certified candidates: list the chunks whose block minimum is <= theta, then the whole
  //         CTA enumerates those blocks' states in parallel
  if (tmin <= theta) {
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
    for (unsigned int z = tid; z < (unsigned int)NT; z += nth) {
      float r = sT[z];
#pragma unroll
      for (int i = 0; i < B; ++i)
        if ((z >> i) & 1u) r += H[i];
      if (V + (long long)r <= theta) {
        const int idx = atomicAdd(&scount, 1);
        if (idx < BATCH_CAP) scand[idx] = ((unsigned long long)c << B) | z;
      }
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
        double acc = 0.0;
        for (int i = 0; i < n; ++i) {
          const double xi = (double)((x >> i) & 1ull);
          for (int j = i; j < n; ++j) {
            const double xj = (double)((x >> j) & 1ull);
            acc = __dadd_rn(acc, __dmul_rn(__dmul_rn(sC[i][j], xi), xj));
          }
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
