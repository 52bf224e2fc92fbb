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

struct BatchParams {
  const double* coeffs;  // [count][n][n] fp64; entries below the diagonal are folded in
  BatchOut* out;         // [count]
  int n;
  int count;
};

}  // namespace qb
