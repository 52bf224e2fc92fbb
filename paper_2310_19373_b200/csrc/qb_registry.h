// Kernel registry shared by the translation units of libqubrute_b200.so.
//
// The kernel templates are instantiated in separate translation units compiled in parallel
// (qb_k_table.cu, qb_k_coarse.cu, qb_k_fieldwalk.cu, qb_k_batch.cu); each exports a table of
// host-side kernel pointers, and qb_api.cu launches through those pointers (cudaLaunchKernel
// resolves the kernel from the host stub address, so no relocatable device code is needed).
#pragma once
#include "qb_common.cuh"
#include "qb_batch_params.h"

#ifndef QB_TPB
#define QB_TPB 128
#endif
#ifndef QB_BIG_B1  // fp32 table split of the 10 large-block bits: u rows x w columns
#define QB_BIG_B1 5
#define QB_BIG_B2 5
#endif
#ifndef QB_COARSE_B1  // coarse pass split of the same bits (measured best 4 x 6)
#define QB_COARSE_B1 4
#define QB_COARSE_B2 6
#endif

namespace qb {

constexpr int TPB = QB_TPB;
constexpr int BIG_B1 = QB_BIG_B1, BIG_B2 = QB_BIG_B2, BIG_BE = BIG_B1 + BIG_B2;

using KFn = void (*)(const TableParams);
using PFn = void (*)(const TableParams, double*, double*, int);
using BatchFn = void (*)(const BatchParams);

// table-kernel family for one block shape (B1, B2) and chunk length L
struct TableFns {
  int B1, B2, L;
  KFn search, mark, blocks, states;
  PFn prefix;
};
// a search kernel over the large-block (BIG_BE) geometry with chunk length L
struct LFn {
  int L;
  KFn fn;
  KFn fin;  // one-CTA record reduction for kernels that do not reduce in their own tail (or null)
};

const TableFns* table_fns(int* count);    // qb_k_table.cu
const LFn* coarse_fns(int* count);        // qb_k_coarse.cu
const LFn* fieldwalk_fns(int* count);     // qb_k_fieldwalk.cu
const LFn* tc_fns(int* count);            // qb_k_tc.cu (tensor-core coarse pass; null fin = finalize_kernel)
const LFn* byte8_fns(int* count);         // qb_k_byte8.cu (table-load byte-packed threshold pass)
const BatchFn* batch_fns(int* count);     // qb_k_batch.cu: index = block bits B (1..BMAX)
BatchFn batch_warp_fn(int* warps, int* nmin, int* nmax);  // qb_k_batch.cu: one warp per instance

}  // namespace qb
