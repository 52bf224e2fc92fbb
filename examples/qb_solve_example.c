/* Minimal C consumer of libqubrute_b200.so through include/qubrute_b200.h only (no Python, no
 * torch): builds the reference's worked example and a seeded n=24 instance, solves them with the
 * reference's tie rules and prints the result.  Exit code 0 on success, 2 when no CUDA device
 * is present (the library reports QB_E_NODEV instead of falling back to the CPU).
 *
 *   gcc -O2 -Iinclude examples/qb_solve_example.c -Lpaper_2310_19373_b200 -lqubrute_b200 \
 *       -Wl,-rpath,$PWD/paper_2310_19373_b200 -o build/qb_solve_example
 */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include "qubrute_b200.h"

static uint64_t splitmix64(uint64_t* s) {
  uint64_t z = (*s += 0x9E3779B97F4A7C15ull);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

int main(void) {
  printf("%s\n", qb_version());
  /* host-only: the reference's worked example f(1,1,0) = 2 (test_core.py:88-95) */
  const double q3[9] = {1.0, -2.0, 0.0, 0.0, 3.0, 1.0, 0.0, 0.0, -1.0};
  const double x3[3] = {1.0, 1.0, 0.0};
  printf("eval_upper worked example = %g\n", qb_eval_upper(q3, 3, x3));

  int ndev = 0;
  qb_device_count(&ndev);
  if (ndev == 0 || qb_init(0) != QB_OK) {
    printf("no CUDA device: %s\n", qb_last_error());
    return 2;
  }
  enum { N = 24 };
  static double q[N * N];
  uint64_t seed = 12345;
  for (int i = 0; i < N; ++i)
    for (int j = i; j < N; ++j) q[i * N + j] = (double)((int64_t)(splitmix64(&seed) % 201) - 100);
  qb_result r;
  /* solve_incremental semantics: whole space, ties to the lowest global Gray rank */
  if (qb_solve(q, N, 0, 0, 0, QB_TIE_GRAY, 0, 1, QB_VARIANT_AUTO, &r) != QB_OK) {
    fprintf(stderr, "qb_solve: %s\n", qb_last_error());
    return 1;
  }
  printf("n=%d min %.1f argmin 0x%llx states %llu exact %d kernel %.3f ms\n", N, r.value,
         (unsigned long long)r.argmin_bits, (unsigned long long)r.states, r.exact, r.kernel_ms);
  /* solve_parallel(fixed_bits=3) semantics, split in two shards combined by (value_key, tie_key) */
  qb_result a, b;
  if (qb_solve(q, N, 0, 0, 3, QB_TIE_GRAY, 0, 2, QB_VARIANT_AUTO, &a) != QB_OK ||
      qb_solve(q, N, 0, 0, 3, QB_TIE_GRAY, 1, 2, QB_VARIANT_AUTO, &b) != QB_OK) {
    fprintf(stderr, "qb_solve shard: %s\n", qb_last_error());
    return 1;
  }
  const qb_result* w = (a.value_key < b.value_key || (a.value_key == b.value_key && a.tie_key < b.tie_key)) ? &a : &b;
  printf("2 shards, m=3: min %.1f argmin 0x%llx\n", w->value, (unsigned long long)w->argmin_bits);
  qb_shutdown();
  return 0;
}
