// Batch path parameters (shared by qb_batch.cuh and the host registry).
#pragma once

namespace qb {

constexpr int BATCH_NMAX = 24;
constexpr int BATCH_CAP = 32;
constexpr int BATCH_TPB_MAX = 256;

struct BatchOut {
  unsigned long long x;  // argmin bits
  double value;          // eval_upper(argmin)
  int status;            // 0 ok, 1 candidate overflow (host fallback), 2 no candidate (bug), 3 non-finite input
  int candidates;
};

// Input formats of the batch kernel.  The host folds each instance (QuboInstance convention,
// core.py:66-72) and packs its upper triangle row by row (i <= j), as fp32 when every folded
// coefficient of the piece round-trips through fp32 exactly (config C: 4x fewer H2D bytes than the
// dense fp64 matrix), otherwise as fp64.
enum BatchFmt : int { BATCH_DENSE_F64 = 0, BATCH_UPPER_F32 = 1, BATCH_UPPER_F64 = 2 };

struct BatchParams {
  const void* coeffs;  // [count] instances in format `fmt`
  BatchOut* out;       // [count]
  int n;
  int count;
  int fmt;             // BatchFmt
};

}  // namespace qb
