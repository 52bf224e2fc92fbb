/*
 * TEST INFRASTRUCTURE — NOT THE PRODUCT.
 *
 * CPU restatement of the reference's Gray-code QUBO brute force
 * (arxiv 2310.19373, package `qubrute`).  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load this library,
 * and only as the checker or the timed CPU baseline.  The product path
 * (paper_2310_19373_b200) never links or calls it.
 *
 * Pinned against the reference itself: the JSON fixtures under tests/golden were made by
 * importing /root/reference/pkg/src/qubrute (tests/golden/make_golden.py) and
 * tests/test_oracle.py checks every function here against them.
 *
 * Arithmetic follows the reference exactly: fp64, no FMA contraction (build
 * with -ffp-contract=off; numba compiles without fastmath, _kernels.py:4-5),
 * the same summation orders and the same strict-'<' incumbent rule.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* _kernels.py:12-20  eval_upper: f(x) = sum_{i<=j} c[i,j] x_i x_j, row-major order. */
double oc_eval_upper(const double* c, int n, const double* x) {
  double acc = 0.0;
  for (int i = 0; i < n; i++)
    for (int j = i; j < n; j++) acc += c[(size_t)i * n + j] * x[i] * x[j];
  return acc;
}

/* _kernels.py:23-43  naive_scan: ascending integers, one full evaluation per vector,
 * incumbent (0-vector, 0.0), strict '<'.  Returns steps = 2^n - 1. */
uint64_t oc_naive_scan(const double* c, int n, double* x_min, double* v_min) {
  double x[64];
  for (int i = 0; i < n; i++) { x[i] = 0.0; x_min[i] = 0.0; }
  double vm = 0.0;
  uint64_t total = (uint64_t)1 << n;
  for (uint64_t k = 1; k < total; k++) {
    for (int i = 0; i < n; i++) x[i] = (double)((k >> i) & 1);
    double v = oc_eval_upper(c, n, x);
    if (v < vm) {
      memcpy(x_min, x, sizeof(double) * n);
      vm = v;
    }
  }
  *v_min = vm;
  return total - 1;
}

/* core.py:104-111  split: qua = triu(c,1) + its transpose (zero diagonal), lin = diag(c). */
void oc_split(const double* c, int n, double* qua, double* lin) {
  for (int i = 0; i < n; i++) {
    lin[i] = c[(size_t)i * n + i];
    for (int j = 0; j < n; j++) {
      double u = (j > i) ? c[(size_t)i * n + j] : 0.0;   /* triu(c, 1)[i, j] */
      double l = (i > j) ? c[(size_t)j * n + i] : 0.0;   /* triu(c, 1).T[i, j] */
      qua[(size_t)i * n + j] = u + l;
    }
  }
}

/* _kernels.py:46-75  gray_scan: Gray walk over the n_free low bits of x0.
 * Per step: l = ctz(k) by shift loop; flip; row = sum_i qua[l,i] x_i in index
 * order; v += (2x_l - 1)(row + lin[l]); on v < v_min copy x and set v_min to the
 * exact eval_upper of the new incumbent.  Returns steps = 2^n_free - 1. */
uint64_t oc_gray_scan(const double* coeffs, const double* qua, const double* lin, const double* x0,
                      double v0, int n, int n_free, double* x_min, double* v_min) {
  double x[64];
  memcpy(x, x0, sizeof(double) * n);
  memcpy(x_min, x0, sizeof(double) * n);
  double v = v0, vm = v0;
  uint64_t total = (uint64_t)1 << n_free;
  for (uint64_t k = 1; k < total; k++) {
    int l = 0;
    while (((k >> l) & 1) == 0) l++;
    x[l] = 1.0 - x[l];
    double row = 0.0;
    const double* q = qua + (size_t)l * n;
    for (int i = 0; i < n; i++) row += q[i] * x[i];
    v += (2.0 * x[l] - 1.0) * (row + lin[l]);
    if (v < vm) {
      memcpy(x_min, x, sizeof(double) * n);
      vm = oc_eval_upper(coeffs, n, x);
    }
  }
  *v_min = vm;
  return total - 1;
}

/* solver.py:159-170  _scan_subspace for SubspaceSpec(m, suffix): x0 = suffix in bits
 * n-m..n-1 (solver.py:72-79), v0 = eval_upper(x0), gray_scan over n-m free bits,
 * value = exact re-evaluation of the minimiser (core.py:123-130). */
typedef struct {
  uint64_t bits;       /* minimiser, bit i = x_i */
  double value;        /* eval_upper(minimiser) */
  uint64_t steps;
} oc_sub_result;

static oc_sub_result scan_subspace(const double* coeffs, const double* qua, const double* lin, int n,
                                   int m, uint64_t suffix) {
  double x0[64] = {0}, xm[64], vm;
  for (int i = 0; i < n; i++) x0[i] = 0.0;
  for (int t = 0; t < m; t++) x0[n - m + t] = (double)((suffix >> t) & 1);
  double v0 = oc_eval_upper(coeffs, n, x0);
  oc_sub_result r;
  r.steps = oc_gray_scan(coeffs, qua, lin, x0, v0, n, n - m, xm, &vm);
  r.bits = 0;
  for (int i = 0; i < n; i++)
    if (xm[i] != 0.0) r.bits |= (uint64_t)1 << i;
  r.value = oc_eval_upper(coeffs, n, xm);
  return r;
}

typedef struct {
  const double *coeffs, *qua, *lin;
  int n, m;
  uint64_t s_begin, s_end;
  oc_sub_result* out;        /* indexed by suffix - s_begin */
  uint64_t* next;            /* shared work counter (suffix offset) */
  pthread_mutex_t* mu;
} worker_arg;

static void* worker(void* p) {
  worker_arg* a = (worker_arg*)p;
  for (;;) {
    pthread_mutex_lock(a->mu);
    uint64_t s = *a->next;
    if (s < a->s_end - a->s_begin) (*a->next)++;
    pthread_mutex_unlock(a->mu);
    if (s >= a->s_end - a->s_begin) break;
    a->out[s] = scan_subspace(a->coeffs, a->qua, a->lin, a->n, a->m, a->s_begin + s);
  }
  return NULL;
}

/* solver.py:193-229 + 173-185  solve_parallel restricted to suffixes [s_begin, s_end):
 * every subspace scanned (on `threads` pthreads), results combined in ascending
 * suffix order with strict '<' on the exact values (lowest suffix wins ties).
 * evaluations = sum of per-subspace steps.  With s_begin=0, s_end=2^m this is
 * exactly solve_parallel(inst, SolveConfig(threads, fixed_bits=m)); m=0 is
 * solve_incremental; one suffix is solve_subspace. */
int oc_solve_subspaces(const double* coeffs, int n, int m, uint64_t s_begin, uint64_t s_end, int threads,
                       uint64_t* bits, double* value, uint64_t* evaluations) {
  if (n < 1 || n > 62 || m < 0 || m >= n || s_begin >= s_end || s_end > ((uint64_t)1 << m)) return -1;
  double* qua = (double*)malloc(sizeof(double) * n * n);
  double* lin = (double*)malloc(sizeof(double) * n);
  oc_split(coeffs, n, qua, lin);
  uint64_t cnt = s_end - s_begin;
  oc_sub_result* res = (oc_sub_result*)malloc(sizeof(oc_sub_result) * cnt);
  if (threads < 1) threads = 1;
  if ((uint64_t)threads > cnt) threads = (int)cnt;
  uint64_t next = 0;
  pthread_mutex_t mu = PTHREAD_MUTEX_INITIALIZER;
  worker_arg a = {coeffs, qua, lin, n, m, s_begin, s_end, res, &next, &mu};
  if (threads == 1) {
    worker(&a);
  } else {
    pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * threads);
    for (int t = 0; t < threads; t++) pthread_create(&th[t], NULL, worker, &a);
    for (int t = 0; t < threads; t++) pthread_join(th[t], NULL);
    free(th);
  }
  oc_sub_result best = res[0];
  uint64_t ev = res[0].steps;
  for (uint64_t s = 1; s < cnt; s++) {
    ev += res[s].steps;
    if (res[s].value < best.value) best = res[s];
  }
  *bits = best.bits;
  *value = best.value;
  *evaluations = ev;
  free(res); free(qua); free(lin);
  return 0;
}

/* Batch of independent instances (config C): each instance solved like
 * solve_incremental (m = 0), instances spread over `threads` pthreads.  The
 * reference has no batch API; its equivalent is a thread pool over
 * solve_incremental calls. */
typedef struct {
  const double* coeffs; int n; uint64_t count; uint64_t* bits; double* values;
  uint64_t* next; pthread_mutex_t* mu;
} batch_arg;

static void* batch_worker(void* p) {
  batch_arg* a = (batch_arg*)p;
  size_t nn = (size_t)a->n * a->n;
  double* qua = (double*)malloc(sizeof(double) * nn);
  double lin[64];
  for (;;) {
    pthread_mutex_lock(a->mu);
    uint64_t b = *a->next;
    if (b < a->count) (*a->next)++;
    pthread_mutex_unlock(a->mu);
    if (b >= a->count) break;
    const double* c = a->coeffs + b * nn;
    oc_split(c, a->n, qua, lin);
    oc_sub_result r = scan_subspace(c, qua, lin, a->n, 0, 0);
    a->bits[b] = r.bits;
    a->values[b] = r.value;
  }
  free(qua);
  return NULL;
}

int oc_solve_batch(const double* coeffs, int n, uint64_t count, int threads, uint64_t* bits, double* values) {
  if (n < 1 || n > 62) return -1;
  uint64_t next = 0;
  pthread_mutex_t mu = PTHREAD_MUTEX_INITIALIZER;
  batch_arg a = {coeffs, n, count, bits, values, &next, &mu};
  if (threads < 1) threads = 1;
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * threads);
  for (int t = 0; t < threads; t++) pthread_create(&th[t], NULL, batch_worker, &a);
  for (int t = 0; t < threads; t++) pthread_join(th[t], NULL);
  free(th);
  return 0;
}
