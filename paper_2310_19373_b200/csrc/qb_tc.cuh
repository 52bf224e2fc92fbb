// Tensor-core coarse-filter traversal kernel (QB_VARIANT_TC): the coarse block test of
// qb_coarse.cuh with the candidate values of every block formed by tcgen05.mma.
//
// Same chunks, outer Gray walk (Eq. 3 field updates), blocks, certified bound, exact fallback and
// tie keys as the coarse kernel.  What changes is who forms the coarse image
//     C(z) = sum_{i<B} z_i hc_i + Tc(z),   hc_i = rint(H_i 2^-s),  Tc(z) = rint(T(z) 2^-s)
// of the 1024 states of a block and compares it with the block's threshold.  A block of a thread
// whose running best (or the device-wide best) is thr can hold a better or tied state only if some
// C(z) <= Lc = floor((thr + slack - V) 2^-s); with D(z) = C(z) + beta >= 0 and Ld = Lc + beta clamped
// to [-1, 1023], every state's test is one bit of F(z) = D(z) + 1023 - Ld in [0, 2047]:
//     z passes  <=>  D(z) <= Ld  <=>  bit 10 of F(z) is clear.
// One CTA stacks the rows of the 128 blocks its 128 worker threads are on into A [128 x 32] f16 and
// multiplies by the per-instance Z [512 x 32] f16, whose cell row p pairs the states p and p + 512:
//     A row:  hc_0..hc_9, 1, O, 2048, 0 0 0 | hc_0..hc_9, 2048, O, 0 ...          (O = 1023 - Ld)
//     Z row:  bits of p, Tc'(p), 1, 4096, 0 0 0 | 2048 bits of p+512, Tc'(p+512), 2048, 0 ...
//     D[row, p] = 2^23 + F(p) + 2048 F(p + 512)          (Tc' = Tc + beta, fp32 accumulators)
// Every product and partial sum is an integer below 2^24 in magnitude, so the fp32 accumulation is
// exact whatever the tensor core's summation order, and the fixed 2^23 term pins the exponent: the
// low 22 bits of each TMEM cell are F(p) | F(p+512) << 11.  A thread reads its own TMEM lane (512
// cells per block) and ANDs the cells three at a time (LOP3, four states per instruction); the
// block passes iff bit 10 or bit 21 of the AND is clear.  Passing blocks (rare once a good value is
// known) get the exact fp32 table evaluation; a failed block is bounded below by
// V + (Ld - beta + 1) 2^s - slack, which keeps the per-chunk minima of the collect pass valid.  Each
// state's coarse value is still formed (by the tensor core) and compared (by the bit test).
//
// Roles: warps 0-3 are workers (one chunk per thread, CTA-wide rounds of 128 chunks so the rows
// advance in lockstep), warp 4 issues the MMAs from one lane.  Pipelines (mbarriers):
//   bar_a[2]     workers -> issuer: A rows of batch g written (double-buffered by g & 1)
//   bar_full[2]  MMA -> workers: tile in TMEM buffer b done (tcgen05.commit)
//   bar_empty[2] workers -> issuer: TMEM buffer b read back (one arrival per worker warp)
// TMEM: two 128-column tile buffers per CTA, two CTAs per SM (all 512 columns).
#pragma once
#include <cuda_fp16.h>
#include "qb_coarse.cuh"
#include "qb_tc_ptx.cuh"

namespace qb {

namespace tc {
// element (row r, k) of a [rows x 32] f16 K-major SWIZZLE_NONE operand: 8-row x 16-byte core
// matrices, LBO = 128 B (next core matrix along K), SBO = 512 B (next 8-row group)
__host__ __device__ constexpr uint32_t off32(int r, int k) {
  return (uint32_t)((r >> 3) * 512 + (k >> 3) * 128 + (r & 7) * 16 + (k & 7) * 2);
}
constexpr uint32_t kLBO = 128, kSBO = 512, kKStep = 256;  // second K=16 step starts 2 core matrices in
}  // namespace tc

__device__ __forceinline__ void named_bar_sync(int id, int count) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}

__device__ __forceinline__ uint32_t pack_f16x2(float a, float b) {
  const __half2 h = __floats2half2_rn(a, b);
  return *reinterpret_cast<const uint32_t*>(&h);
}

// 32 f16 values (as 8 x uint4) into row r of a K=32 operand tile
__device__ __forceinline__ void tc_store_row(uint8_t* tile, int r, const uint32_t (&w)[16]) {
#pragma unroll
  for (int q = 0; q < 4; ++q)
    *reinterpret_cast<uint4*>(tile + tc::off32(r, 8 * q)) = make_uint4(w[4 * q], w[4 * q + 1], w[4 * q + 2], w[4 * q + 3]);
}

// A row of one block: fields rounded to coarse units and the threshold offset O
template <int B>
__device__ __forceinline__ void tc_write_row(uint8_t* a_tile, int r, const float (&H)[B], float scale, float O,
                                             bool active) {
  static_assert(B == 10, "row layout assumes 10 table bits");
  float h[B];
#pragma unroll
  for (int i = 0; i < B; ++i) h[i] = active ? rintf(H[i] * scale) : 0.f;
  uint32_t w[16];
  w[0] = pack_f16x2(h[0], h[1]);
  w[1] = pack_f16x2(h[2], h[3]);
  w[2] = pack_f16x2(h[4], h[5]);
  w[3] = pack_f16x2(h[6], h[7]);
  w[4] = pack_f16x2(h[8], h[9]);
  w[5] = pack_f16x2(1.f, O);
  w[6] = pack_f16x2(2048.f, 0.f);
  w[7] = 0u;
#pragma unroll
  for (int q = 0; q < 5; ++q) w[8 + q] = w[q];
  w[13] = pack_f16x2(2048.f, O);
  w[14] = 0u;
  w[15] = 0u;
  tc_store_row(a_tile, r, w);
}

// exact fp32 minimum of block j of chunk c relative to its base value (rare: blocks whose coarse
// test passes); the fields come from a direct evaluation of the block base
template <int B1, int B2, int L>
__device__ __noinline__ float tc_exact_block_min(const TableParams& p, unsigned long long c, unsigned int j) {
  constexpr int B = B1 + B2, NF = (L - B) > 0 ? (L - B) : 1;
  const unsigned long long xo = (chunk_prefix(p, c) << L) | ((unsigned long long)(j ^ (j >> 1)) << B);
  long long V;
  float H[B], F[NF];
  base_eval<B, L>(p, xo, B, V, H, F);
  return block_min<B1, B2, 0, NF>(p, H, F);
}

// clamped coarse threshold Ld in [-1, 1023] of a block with base V under pruning limit lim
__device__ __forceinline__ int tc_ld(long long lim, long long V, int shift, int bias) {
  if (lim == LLONG_MAX) return 1023;
  const long long lc = (lim - V) >> shift;  // floor
  return (int)max(-1ll, min(1023ll, lc + bias));
}

template <int B1, int B2, int L>
__global__ void __launch_bounds__(TC_TPB, TC_CTAS_PER_SM) tc_kernel(const __grid_constant__ TableParams p) {
  constexpr int B = B1 + B2;
  static_assert(B == BMAX, "the tensor-core pass covers 1024-state blocks");
  constexpr int LO = L - B;
  constexpr int NF = LO > 0 ? LO : 1;
  constexpr int NT = TC_CELLS / TC_TILE_N;  // MMA tiles per block
  static_assert(NT % 2 == 0, "tiles alternate between the two TMEM buffers");
  extern __shared__ __align__(1024) uint8_t tc_smem[];
  uint8_t* zmat = tc_smem;
  uint8_t* a_tile[2] = {tc_smem + TC_ZBYTES, tc_smem + TC_ZBYTES + TC_ABYTES};
  __shared__ uint64_t bar_a[2], bar_full[2], bar_empty[2];
  __shared__ uint32_t tmem_base;
  __shared__ unsigned long long round_base[2];
  __shared__ int stop_flag[2];

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  // ---- prologue: Z operand from the fp32 table, TMEM, barriers
  for (int pc = tid; pc < TC_CELLS; pc += TC_TPB) {
    const int zh = pc + TC_CELLS;
    float lo[16], hi[16];
#pragma unroll
    for (int i = 0; i < B; ++i) {
      lo[i] = (float)((pc >> i) & 1);
      hi[i] = 2048.f * (float)((zh >> i) & 1);
    }
    lo[B] = rintf(p.T[pc] * p.tc_scale) + (float)p.tc_bias;
    lo[B + 1] = 1.f;
    lo[B + 2] = 4096.f;
    hi[B] = rintf(p.T[zh] * p.tc_scale) + (float)p.tc_bias;
    hi[B + 1] = 2048.f;
    hi[B + 2] = 0.f;
#pragma unroll
    for (int i = B + 3; i < 16; ++i) lo[i] = hi[i] = 0.f;
    uint32_t w[16];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      w[q] = pack_f16x2(lo[2 * q], lo[2 * q + 1]);
      w[8 + q] = pack_f16x2(hi[2 * q], hi[2 * q + 1]);
    }
    tc_store_row(zmat, pc, w);
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

  Rec best{LLONG_MAX, ~0ull, 0ull, 0u, 0u};
  if (warp == TC_WORKERS / 32) {
    // ---------------------------------------------------------------- MMA issuer
    // Tile t of batch g is the (NT g + t)-th tile: TMEM buffer t & 1, and its fill / drain is phase
    // (NT/2) g + t/2 of that buffer's barriers, so every parity is a compile-time constant.
    if (lane == 0) {
      constexpr uint32_t idesc = tc::idesc_f16_f32(TC_WORKERS, TC_TILE_N);
      const uint64_t zdesc = tc::smem_desc(tc::smem_u32(zmat), tc::kLBO, tc::kSBO);
      const uint64_t adesc[2] = {tc::smem_desc(tc::smem_u32(a_tile[0]), tc::kLBO, tc::kSBO),
                                 tc::smem_desc(tc::smem_u32(a_tile[1]), tc::kLBO, tc::kSBO)};
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
          // Z cell rows [128 t, 128 t + 128): 16 8-row groups of 512 B; descriptor addresses in 16 B units
          const uint64_t zd = zdesc + (uint64_t)(t * TC_TILE_N * TC_K * 2 / 16);
          const uint32_t d = tmem + (t & 1) * TC_TILE_N;
          tc::mma_f16(d, adesc[s], zd, idesc, 0u);
          tc::mma_f16(d, adesc[s] + tc::kKStep / 16, zd + tc::kKStep / 16, idesc, 1u);
          tc::mma_commit(&bar_full[t & 1]);
        }
      }
    }
    __syncwarp();
  } else {
    // ---------------------------------------------------------------- workers
    const unsigned long long nchunks = p.chunk_end - p.chunk_begin;
    const long long slack = (long long)(B + 1) << p.tc_shift >> 1;
    const uint32_t lane_tmem = tmem + ((uint32_t)(warp * 32) << 16);
    int round = 0;
    // the block being prepared (fields, threshold) ...
    bool active = false;
    unsigned long long c = 0, ci = 0, key_hi = 0;
    int dir = 0, ld_next = 1023;
    unsigned int j = 0;
    long long V = 0;
    float H[B], F[NF];
    // ... and running per-chunk state of the block being consumed
    long long cmin = LLONG_MAX, skip_min = LLONG_MAX, thr = LLONG_MAX, lim = LLONG_MAX;

    auto fetch_round = [&]() -> bool {  // worker-wide: the next 128 chunks, one per thread
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
        // a new chunk starts from the device-wide best (the thread's own best is in it too)
        thr = min(min(best.val, gbest_dec(__ldcg(p.gbest))), p.seed_val);  // host seed: whole-space searches
        lim = thr > LLONG_MAX - slack ? LLONG_MAX : thr + slack;
      } else {
#pragma unroll
        for (int i = 0; i < B; ++i) H[i] = 0.f;
      }
      return true;
    };
    auto publish = [&](int slot) {
      ld_next = tc_ld(lim, V, p.tc_shift, p.tc_bias);
      tc_write_row<B>(a_tile[slot], tid, H, p.tc_scale, (float)(1023 - ld_next), active);
      tc::fence_async_smem();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&bar_a[slot]);
    };
    auto publish_stop = [&](int slot) {  // no batch g: the issuer leaves its loop
      if (tid == 0) stop_flag[slot] = 1;
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&bar_a[slot]);
    };

    bool more = fetch_round();
    if (more) publish(0);
    else publish_stop(0);
    for (uint32_t g = 0; more; ++g) {
      // the block consumed in this iteration
      const bool cur_active = active;
      const unsigned long long cur_c = c, cur_ci = ci, cur_key_hi = key_hi;
      const int cur_dir = dir, cur_ld = ld_next;
      const unsigned int cur_j = j;
      const long long Vc = V;
      if (cur_active && cur_j == 0) {
        cmin = LLONG_MAX;
        skip_min = LLONG_MAX;
      }

      // AND this block's cells: bit 10 / bit 21 stay set only if every state fails its test
      uint32_t acc[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) acc[k] = 0xffffffffu;
#pragma unroll
      for (int t = 0; t < NT; ++t) {
        const int b = t & 1;
        tc::mbar_wait(&bar_full[b], (t >> 1) & 1);
        tc::tc_fence_after();
        // the whole tile into registers, then hand the buffer back before folding it
        uint32_t r[TC_TILE_N];
#pragma unroll
        for (int q = 0; q < TC_TILE_N / 32; ++q)
          tc::tmem_ld32(lane_tmem + b * TC_TILE_N + 32 * q, *reinterpret_cast<uint32_t(*)[32]>(r + 32 * q));
        tc::tmem_wait_ld();
        tc::tc_fence_before();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(&bar_empty[b]);
#pragma unroll
        for (int i = 0; i < TC_TILE_N; i += 16)
#pragma unroll
          for (int k = 0; k < 8; ++k) acc[k] &= r[i + 2 * k] & r[i + 2 * k + 1];
        if (t == 1) {  // A rows of the next block: needed once tile 2 has drained buffer 0
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
        }
      }
      if (!cur_active) continue;
      const uint32_t all = (acc[0] & acc[1] & acc[2]) & (acc[3] & acc[4] & acc[5]) & (acc[6] & acc[7]);
      const bool pass = (all & 0x200400u) != 0x200400u;
      if (pass) {
        const long long val = Vc + (long long)tc_exact_block_min<B1, B2, L>(p, cur_c, cur_j);
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
      } else {  // every state: C(z) > Ld - beta, so exact >= V + (Ld - beta + 1) 2^s - slack
        skip_min = min(skip_min, Vc + ((long long)(cur_ld - p.tc_bias + 1) << p.tc_shift));
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
