// Tensor-core coarse-filter traversal kernel (QB_VARIANT_TC): the coarse block pass of
// qb_coarse.cuh with the 2^B candidate values of every block formed by tcgen05.mma.
//
// Same chunks, outer Gray walk (Eq. 3 field updates), blocks, certified bound, exact fallback and
// tie keys as the coarse kernel.  What changes is who forms the coarse image
//     C(z) = sum_{i<B} z_i hc_i + Tc(z),   hc_i = rint(H_i 2^-s),  Tc(z) = rint(T(z) 2^-s)
// of the 1024 states z of a block: one CTA stacks the fields of the 128 blocks its 128 worker
// threads are on (one block per thread) into A [128 x 16] f16 (hc_0..hc_9, 1, 0...) and multiplies
// it by the per-instance constant Z [1024 x 16] f16 (row z: the bits of z, Tc(z) + beta, 0...):
//     D = A Z^T  ->  D[thread, z] = C_thread(z) + beta
// in M=128 x N=TC_TILE_N x K=16 MMAs with f16 accumulators in TMEM.  The host picks s so that
// every partial sum of every product row lies in [-2048, 2048]: all f16 arithmetic is exact
// integer arithmetic, whatever the tensor core's summation order, and beta makes every D >= 0 so
// the f16 bit patterns order like u16.  Each thread then reads its own TMEM lane (.pack::16b: two
// states per register) and folds it with VIMNMX3.U16x2 (four states per instruction).  Each
// state's coarse value is still formed (by the tensor core) and compared (by the thread).
//
// Roles: four warps, one chunk per thread (CTA-wide rounds of 128 chunks so the rows advance in
// lockstep); thread 0 also issues the MMAs (a dedicated issuer warp would put a third warp on some
// SM sub-partition and cap the registers).  Pipelines (mbarriers):
//   bar_a[2]     warps -> issuer: A rows of batch g written (double-buffered by g & 1)
//   bar_full[2]  MMA -> warps: tile in TMEM buffer b done (tcgen05.commit)
//   bar_empty[2] warps -> issuer: TMEM buffer b read back (one arrival per warp)
// TMEM: 2 TC_TILE_N columns per CTA = two tile buffers; 512 / (2 TC_TILE_N) CTAs per SM.
#pragma once
#include <cuda_fp16.h>
#ifdef QB_TC_TRACE
#include <cstdio>
#endif
#include "qb_coarse.cuh"
#include "qb_tc_ptx.cuh"

namespace qb {


__device__ __forceinline__ void named_bar_sync(int id, int count) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}

__device__ __forceinline__ uint32_t pack_f16x2(float a, float b) {
  const __half2 h = __floats2half2_rn(a, b);
  return *reinterpret_cast<const uint32_t*>(&h);
}

// A row of one block: hc_0..hc_{B-1}, 1, zeros (K = 16) into the operand tile at row r
template <int B>
__device__ __forceinline__ void tc_write_row(uint8_t* a_tile, int r, const float (&H)[B], float scale, bool active) {
  static_assert(B == 10, "row layout assumes 10 table bits (K = 16)");
  float h[B];
#pragma unroll
  for (int i = 0; i < B; ++i) h[i] = active ? rintf(H[i] * scale) : 0.f;
  uint4 lo, hi;
  lo.x = pack_f16x2(h[0], h[1]);
  lo.y = pack_f16x2(h[2], h[3]);
  lo.z = pack_f16x2(h[4], h[5]);
  lo.w = pack_f16x2(h[6], h[7]);
  hi.x = pack_f16x2(h[8], h[9]);
  hi.y = pack_f16x2(1.f, 0.f);
  hi.z = 0u;
  hi.w = 0u;
  *reinterpret_cast<uint4*>(a_tile + tc::operand_offset(r, 0)) = lo;
  *reinterpret_cast<uint4*>(a_tile + tc::operand_offset(r, 8)) = hi;
}

// exact fp32 minimum of block j of chunk c relative to its base value (rare: blocks whose coarse
// bound reaches the best value seen); the fields come from a direct evaluation of the block base
template <int B1, int B2, int L>
__device__ __noinline__ float tc_exact_block_min(const TableParams& p, unsigned long long c, unsigned int j) {
  constexpr int B = B1 + B2, NF = (L - B) > 0 ? (L - B) : 1;
  const unsigned long long xo = (chunk_prefix(p, c) << L) | ((unsigned long long)(j ^ (j >> 1)) << B);
  long long V;
  float H[B], F[NF];
  base_eval<B, L>(p, xo, B, V, H, F);
  return block_min<B1, B2, 0, NF>(p, H, F);
}

template <int B1, int B2, int L>
__global__ void __launch_bounds__(TC_TPB, TC_CTAS_PER_SM) tc_kernel(const __grid_constant__ TableParams p) {
  constexpr int B = B1 + B2;
  static_assert(B == BMAX, "the tensor-core pass covers 1024-state blocks");
  constexpr int LO = L - B;
  constexpr int NF = LO > 0 ? LO : 1;
  constexpr int NT = (1 << B) / TC_TILE_N;  // MMA tiles per block
  static_assert(NT % 2 == 0, "tiles alternate between the two TMEM buffers");
  extern __shared__ __align__(1024) uint8_t tc_smem[];
  uint8_t* zmat = tc_smem;
  uint8_t* a_tile[2] = {tc_smem + TC_ZBYTES, tc_smem + TC_ZBYTES + TC_ABYTES};
  __shared__ uint64_t bar_a[2], bar_full[2], bar_empty[2];
  __shared__ uint32_t tmem_base;
  __shared__ unsigned long long round_base[2];
  __shared__ int stop_flag[2];

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  // ---- prologue: Z operand (row z: bits of z, Tc(z) + beta) from the fp32 table, TMEM, barriers
  for (int z = tid; z < (1 << B); z += TC_TPB) {
    float h[16];
#pragma unroll
    for (int i = 0; i < B; ++i) h[i] = (float)((z >> i) & 1);
    h[B] = rintf(p.T[z] * p.tc_scale) + (float)p.tc_bias;
#pragma unroll
    for (int i = B + 1; i < 16; ++i) h[i] = 0.f;
    uint4 lo, hi;
    lo.x = pack_f16x2(h[0], h[1]);
    lo.y = pack_f16x2(h[2], h[3]);
    lo.z = pack_f16x2(h[4], h[5]);
    lo.w = pack_f16x2(h[6], h[7]);
    hi.x = pack_f16x2(h[8], h[9]);
    hi.y = pack_f16x2(h[10], h[11]);
    hi.z = pack_f16x2(h[12], h[13]);
    hi.w = pack_f16x2(h[14], h[15]);
    *reinterpret_cast<uint4*>(zmat + tc::operand_offset(z, 0)) = lo;
    *reinterpret_cast<uint4*>(zmat + tc::operand_offset(z, 8)) = hi;
  }
  if (warp == 0) tc::tmem_alloc<2 * TC_TILE_N>(&tmem_base);
  if (tid == 0) {
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      tc::mbar_init(&bar_a[i], TC_WORKERS / 32);
      tc::mbar_init(&bar_full[i], 1);
      tc::mbar_init(&bar_empty[i], TC_WORKERS / 32);
      stop_flag[i] = 0;
    }
  }
  tc::fence_async_smem();
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = tmem_base;

  // MMA issue (thread 0 only).  Tile t of batch g is the (NT g + t)-th tile of this CTA: TMEM buffer
  // t & 1, and its fill / drain is phase (NT/2) g + t/2 of that buffer's barriers.  Tile tt + 2 reuses
  // the buffer of tile tt, so it is issued once every warp has read tile tt back.
  constexpr uint32_t idesc = tc::idesc_f16_f16(TC_WORKERS, TC_TILE_N);
  const uint64_t zdesc = tc::smem_desc(tc::smem_u32(zmat), 128, 256);
  const uint64_t adesc0 = tc::smem_desc(tc::smem_u32(a_tile[0]), 128, 256);
  const uint64_t adesc1 = tc::smem_desc(tc::smem_u32(a_tile[1]), 128, 256);
  auto issue = [&](uint32_t g, int t) {  // tile t of batch g
    const uint64_t ad = (g & 1) ? adesc1 : adesc0;
    // Z rows [N t, N t + N): N/8 8-row groups of 256 B, 32 N t bytes in
    tc::mma_f16(tmem + (t & 1) * TC_TILE_N, ad, zdesc + (uint64_t)(t * (TC_TILE_N * 32 / 16)), idesc, 0u);
    tc::mma_commit(&bar_full[t & 1]);
  };

  Rec best{LLONG_MAX, ~0ull, 0ull, 0u, 0u};
  if (QB_TC_ISSUER_WARP && warp == TC_WORKERS / 32) {
    // dedicated issuer: batch g's tiles once its A rows are published, each into a drained buffer
    if (lane == 0) {
      for (uint32_t g = 0;; ++g) {
        const int s = g & 1;
        tc::mbar_wait(&bar_a[s], (g >> 1) & 1);
        if (*(volatile int*)&stop_flag[s]) break;
        tc::tc_fence_after();
#pragma unroll
        for (int t = 0; t < NT; ++t) {
          if (g > 0 || t >= 2) {
            tc::mbar_wait(&bar_empty[t & 1], ((t >> 1) + 1) & 1);
            tc::tc_fence_after();
          }
          issue(g, t);
        }
      }
    }
    __syncwarp();
  } else {
  const unsigned long long nchunks = p.chunk_end - p.chunk_begin;
  const long long slack = (long long)(B + 1) << p.tc_shift >> 1;
  const bool coarse_exact = p.tc_shift == 0;
  const uint32_t lane_tmem = tmem + ((uint32_t)(warp * 32) << 16);
  int round = 0;
  // the block being prepared (fields) ...
  bool active = false;
  unsigned long long c = 0, ci = 0, key_hi = 0;
  int dir = 0;
  unsigned int j = 0;
  long long V = 0;
  float H[B], F[NF];
  // ... and running per-chunk state of the block being consumed
  long long cmin = LLONG_MAX, skip_min = LLONG_MAX, thr = LLONG_MAX, lim = LLONG_MAX;

  auto fetch_round = [&]() -> bool {  // CTA-wide: the next 128 chunks, one per thread
    if (tid == 0) round_base[round & 1] = atomicAdd(p.work, (unsigned long long)TC_WORKERS);
    named_bar_sync(1, TC_WORKERS);
    const unsigned long long base = round_base[round & 1];
    ++round;
    if (base >= nchunks) return false;
    ci = base + tid;
    active = ci < nchunks;
    j = 0;
    if (active) {
      c = p.chunk_begin + ci;
      const unsigned long long s = chunk_prefix(p, c);
      base_eval<B, L>(p, s << L, L, V, H, F);
      key_hi = chunk_key(p, s, dir);
    } else {
#pragma unroll
      for (int i = 0; i < B; ++i) H[i] = 0.f;
    }
    return true;
  };
  auto publish = [&](int slot) {
    tc_write_row<B>(a_tile[slot], tid, H, p.tc_scale, active);
    tc::fence_async_smem();
    __syncwarp();
    if (lane == 0) tc::mbar_arrive(&bar_a[slot]);
  };
  auto publish_stop = [&](int slot) {  // issuer-warp mode: no batch g, the issuer leaves its loop
    if (QB_TC_ISSUER_WARP) {
      if (tid == 0) stop_flag[slot] = 1;
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&bar_a[slot]);
    }
  };

#ifdef QB_TC_TRACE
  long long tr_prev = 0;
#endif
  bool more = fetch_round();
  if (!more) publish_stop(0);
  if (more) {
    publish(0);
    if (!QB_TC_ISSUER_WARP && tid == 0) {
      tc::mbar_wait(&bar_a[0], 0);
      tc::tc_fence_after();
      issue(0, 0);
      issue(0, 1);
    }
  }
  for (uint32_t g = 0; more; ++g) {
    // the block consumed in this iteration
    const bool cur_active = active;
    const unsigned long long cur_c = c, cur_ci = ci, cur_key_hi = key_hi;
    const int cur_dir = dir;
    const unsigned int cur_j = j;
    const long long Vc = V;
    if (cur_active && cur_j == 0) {  // chunk start: pruning threshold from the device-wide best
      cmin = LLONG_MAX;
      skip_min = LLONG_MAX;
      thr = min(best.val, gbest_dec(__ldcg(p.gbest)));
      lim = thr > LLONG_MAX - slack ? LLONG_MAX : thr + slack;
    }
    // prepare the next block (outer Gray flip, or the next round's chunks) while the tensor core
    // works on this one
    if (j + 1 < (1u << LO)) {
      ++j;
      if (active) {
        const int r = __ffs(j) - 1;
        const float sg = ((j >> (r + 1)) & 1u) ? -1.f : 1.f;
        outer_flip<B, L, B>(p, B + r, sg, V, H, F);
      }
    } else {
      more = fetch_round();
    }
    if (more) publish((g + 1) & 1);
    else publish_stop((g + 1) & 1);

    // fold this block's tiles: four states per VIMNMX3.U16x2
    unsigned m0 = 0xffffffffu, m1 = 0xffffffffu;
#pragma unroll
    for (int t = 0; t < NT; ++t) {
      const int b = t & 1;
#ifdef QB_TC_TRACE
      const long long tr0 = clock64();
#endif
      tc::mbar_wait(&bar_full[b], (t >> 1) & 1);
#ifdef QB_TC_TRACE
      const long long tr1 = clock64();
#endif
      tc::tc_fence_after();
      uint32_t r[TC_TILE_N / 2];
#pragma unroll
      for (int q = 0; q < TC_TILE_N / 64; ++q)
        tc::tmem_ld32_pack16(lane_tmem + b * TC_TILE_N + 64 * q, *reinterpret_cast<uint32_t(*)[32]>(r + 32 * q));
      tc::tmem_wait_ld();
#ifdef QB_TC_TRACE
      const long long tr2 = clock64();
#endif
      tc::tc_fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&bar_empty[b]);
      if (!QB_TC_ISSUER_WARP && tid == 0 && (t + 2 < NT || more)) {  // refill this buffer: tile t + 2 (maybe of batch g + 1)
        tc::mbar_wait(&bar_empty[b], (t >> 1) & 1);
        if (t + 2 >= NT) tc::mbar_wait(&bar_a[(g + 1) & 1], ((g + 1) >> 1) & 1);
        tc::tc_fence_after();
        if (t + 2 < NT) issue(g, t + 2);
        else issue(g + 1, t + 2 - NT);
#ifdef QB_TC_TRACE
        const long long tr3 = clock64();
        if (blockIdx.x == 0 && g >= 40 && g < 42)
          printf("trace g=%u t=%d wait_full %lld ld %lld empty+issue %lld since_prev_tile %lld\n", g, t, tr1 - tr0,
                 tr2 - tr1, tr3 - tr2, tr0 - tr_prev);
        tr_prev = tr0;
#endif
      }
#pragma unroll
      for (int i = 0; i < TC_TILE_N / 2; i += 4) {
        m0 = __vimin3_u16x2(m0, r[i], r[i + 1]);
        m1 = __vimin3_u16x2(m1, r[i + 2], r[i + 3]);
      }
    }
    if (!cur_active) continue;
    const unsigned m = __vminu2(m0, m1);
    const unsigned short m16 = (unsigned short)min(m & 0xffffu, m >> 16);
    const int dmin = (int)__half2float(__ushort_as_half(m16));
    const long long cb = Vc + ((long long)(dmin - p.tc_bias) << p.tc_shift);
    long long val;
    bool evaluated = true;
    if (coarse_exact) {
      val = cb;
    } else if (cb > lim) {  // bound cb - slack > thr: nothing here can beat or tie the best value seen
      skip_min = min(skip_min, cb);
      evaluated = false;
      val = LLONG_MAX;
    } else {
      val = Vc + (long long)tc_exact_block_min<B1, B2, L>(p, cur_c, cur_j);
    }
    if (evaluated) {
      cmin = min(cmin, val);
      if (val <= best.val) {
        const unsigned long long K = block_key(p, cur_key_hi, cur_dir, cur_j, LO);
        if (val < best.val || K < best.K) best = Rec{val, K, cur_c, cur_j, 0u};
        if (val < thr) {
          thr = val;
          lim = val + slack;
          atomicMax(p.gbest, gbest_enc(val));
        }
      }
    }
    if (cur_j + 1 == (1u << LO)) {  // chunk done: its minimum (or lower bound) for the collect pass
      if (skip_min != LLONG_MAX) cmin = min(cmin, skip_min - slack);
      if (p.mode == MODE_SEARCH_RECORD) p.chunk_min[cur_ci] = cmin;
    }
  }
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc<2 * TC_TILE_N>(tmem);
  const Rec r = cta_reduce<TC_TPB>(best);
  if (tid == 0) p.cta_out[blockIdx.x] = r;
}

}  // namespace qb
