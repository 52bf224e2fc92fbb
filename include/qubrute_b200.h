/*
 * qubrute_b200 — B200-native (sm_100a) Gray-code brute-force QUBO solver.
 *
 * C ABI of libqubrute_b200.so.  Plain pointers and sizes only; the caller owns
 * every buffer, the library never retains a caller pointer after returning,
 * device memory / streams are library-owned and persistent per device after
 * qb_init().  Every entry point is safe to call from several host threads
 * (calls on one device are serialised by a per-device mutex); loaded through
 * ctypes.CDLL the GIL is released for the duration of a call.
 *
 * Status codes: QB_OK (0) on success, a negative QB_E_* otherwise; the message
 * is available from qb_last_error() (thread-local).  Argument validation that
 * the reference performs in Python (dimension cap, fixed-bit range, suffix
 * range) is repeated here and reported as QB_E_ARG / QB_E_CAP.
 *
 * The reference ("qubrute", arXiv 2310.19373) has no native interface: its hot
 * path is the numba kernel _kernels.gray_scan reached from solver.py.  The
 * functions below are what a binding of that path needs; each cites the
 * reference interface it replaces.  INTEGRATION.md shows the ctypes binding.
 */
#ifndef QUBRUTE_B200_H
#define QUBRUTE_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define QB_OK 0
#define QB_E_ARG (-1)      /* invalid argument (reference raises ValueError) */
#define QB_E_CAP (-2)      /* n above QB_MAX_DIM (reference raises DimensionCapError) */
#define QB_E_CUDA (-3)     /* CUDA runtime error */
#define QB_E_NODEV (-4)    /* no CUDA device / library not initialised on one */
#define QB_E_INTERNAL (-5) /* invariant violated (reported, never silently ignored) */

#define QB_MAX_DIM 40      /* reference core.py:24 MAX_DIM */

/* Tie rules (which of several exact minimisers is returned). */
#define QB_TIE_GRAY 0      /* lowest (suffix, Gray rank of free bits): solve_incremental (m_tie=0),
                              solve_parallel(fixed_bits=m_tie), solve_subspace -- solver.py:118-229 */
#define QB_TIE_INTEGER 1   /* lowest integer encoding: solve_naive -- solver.py:99-115, _kernels.py:23-43 */

/* Traversal kernel variants. */
#define QB_VARIANT_AUTO 0      /* fastest: coarse-filter kernel for large chunks, table kernel otherwise */
#define QB_VARIANT_TABLE 1     /* blocked Gray walk: outer field updates + inner-block fp32 table */
#define QB_VARIANT_FIELDWALK 2 /* per-step Gray walk with register local fields (Alg. 1 form) */
#define QB_VARIANT_COARSE 3    /* table walk with a packed-int16 block pass + exact re-evaluation */
#define QB_VARIANT_TC 4        /* coarse block pass formed by tcgen05.mma (f16, TMEM) + exact re-evaluation */
#define QB_VARIANT_IMM 5       /* coarse kernel with the instance's coarse table patched into its SASS as
                                  instruction immediates (no table loads), 10-bit blocks */
#define QB_VARIANT_IMM2 6      /* the same with 11-bit coarse super-blocks (two blocks per coarse pass, chunks
                                  of >= 12 free bits) */
#define QB_VARIANT_IMM8 7      /* patched-immediate threshold pass: four states per register as bytes whose top
                                  bit says "above the pruning limit", folded by LOP3 (qb_coarse8.cuh) */
#define QB_VARIANT_IMM8S 8     /* the same over 11-bit super-blocks (chunks of >= 12 free bits) */
#define QB_VARIANT_IMM8A 9     /* row-bound form of IMM8: every row of a block is tested with the least row term
                                  (a certified lower bound of each state), one 2-input add per four states */
#define QB_VARIANT_IMM8AS 10   /* row-bound form of IMM8S; AUTO's first choice where the coarse filter runs (it gives
                                  up and re-runs with IMM8A / IMM8 / IMM when too many blocks fail its test) */
#define QB_VARIANT_IMM8AQ 11   /* row-bound form over 12-bit super-blocks (four blocks per pass, chunks of >= 13
                                  free bits); measured no faster than IMM8AS, kept as an option */
#define QB_VARIANT_BYTE8 12    /* IMM8AS with its table words read from the kernel parameters instead of patched
                                  immediates: no module load (AUTO's first solve of an instance), chunks of >= 12
                                  free bits */

/* Result of one solve (or of one shard of a sharded solve). */
typedef struct qb_result {
  uint64_t argmin_bits;   /* minimiser, bit i = x_i (reference Solution.minimizer, core.py:153-162) */
  double value;           /* eval_upper(minimiser) in the reference's fp64 order (solver.py:169) */
  uint64_t tie_key;       /* position of the minimiser under the tie rule (lower wins) */
  uint64_t value_key;     /* order-preserving 64-bit image of the compared value (lower wins);
                             combine shards by lexicographic min of (value_key, tie_key) */
  uint64_t states;        /* states scanned by this call */
  int32_t exact;          /* 1: values compared exactly (integer-exact path), 0: certified
                             filter + exact re-evaluation of near-minimal candidates */
  int32_t variant;        /* QB_VARIANT_* actually used */
  int32_t scale_exp;      /* e: device values are Q * 2^e rounded to integers */
  int32_t prefix_bits;    /* k: fixed high bits per GPU thread chunk */
  uint64_t candidates;    /* near-minimal states re-evaluated exactly (0 on the exact path) */
  double kernel_ms;       /* device time of all launches of this call (CUDA events on the library stream) */
  double total_ms;        /* wall time inside the call */
  double search_ms;       /* device time of the traversal (search) kernel alone */
  double collect_ms;      /* device time of the candidate-collect kernel (0 on the exact path) */
  int32_t launches;       /* kernels launched by this call */
  int32_t grid;           /* CTAs of the traversal launch */
  uint64_t param_bytes;   /* bytes of kernel parameters copied host->device per launch (Q, T tables) */
  double module_ms;       /* host time patching + loading the patched-immediate kernel (0: cached / not used) */
  int32_t combine;        /* qb_solve_devices: 1 = shards combined by one ncclAllReduce, 0 = on the host */
  int32_t retries;        /* AUTO: optimistic runs of a faster kernel that gave up before this one completed */
  uint64_t exact_blocks;  /* byte-packed threshold kernels: blocks that failed the byte test and were re-evaluated
                             exactly (the rest were certified above the running best), else 0 */
} qb_result;

/* Library / device management. */
const char* qb_version(void);
const char* qb_last_error(void);               /* thread-local message of the last failure */
int qb_device_count(int* count);
int qb_init(int device);                        /* select device for this thread, create stream + workspace */
void qb_shutdown(void);                         /* free all device resources */

/* Direct evaluation, replaces _kernels.eval_upper (_kernels.py:12-20) / core.evaluate
 * (core.py:123-130): same fp64 row-major order, no FMA contraction.  Host only. */
double qb_eval_upper(const double* coeffs, int n, const double* x);

/* Exhaustive solve over the subspace {x : x >> (n - m_fix) == suffix}.
 *   coeffs     n x n fp64 row-major upper-triangular (QuboInstance.coeffs, core.py:35-75)
 *   m_fix      fixed high bits (0: the whole space)                    solver.py:54-79
 *   suffix     value of the fixed high bits
 *   m_tie      tie rule parameter for QB_TIE_GRAY (m_fix <= m_tie < n): 0 = solve_incremental,
 *              m = solve_parallel(fixed_bits=m); for solve_subspace pass m_tie = m_fix
 *   shard, shard_count   scan only shard `shard` of `shard_count` equal slices of the chunk space
 *              (multi-GPU: one shard per rank; combine results by (value_key, tie_key)).  With
 *              shard_count > 1 only the COMBINED result is the solve's answer: every shard prunes against one
 *              host-found attained value of the whole searched space, so a shard that holds neither the minimum
 *              nor a tie may return an empty result (keys ~0, value NaN) or an attained value above its own
 *              minimum; a shard that holds the minimum or a tie always returns it exactly.
 * Replaces solver._scan_subspace + _kernels.gray_scan (solver.py:159-170, _kernels.py:46-75)
 * and the thread-pool fan-out + combine_subspace_minima of solve_parallel (solver.py:193-229). */
int qb_solve(const double* coeffs, int n, int m_fix, uint64_t suffix, int m_tie, int tie_rule,
             uint32_t shard, uint32_t shard_count, int variant, qb_result* out);

/* The same solve sharded over several GPUs from one process (qb_solve with
 * num_gpus): shard i of ndev runs on devices[i] in its own host thread, and the shard results are
 * combined on the host by the lexicographic minimum of (value_key, tie_key), which is the reference's
 * tie rule (combine_subspace_minima, solver.py:173-185).  states / launches / grid / candidates
 * are summed, kernel_ms / search_ms are the maximum over shards.  A device may appear more than
 * once (its shards then run one after another). */
int qb_solve_devices(const double* coeffs, int n, int m_fix, uint64_t suffix, int m_tie, int tie_rule,
                     const int* devices, int ndev, int variant, qb_result* out);

/* Every minimiser of the subspace {x : x >> (n - m_fix) == suffix} (BASELINE config A: "min
 * value + all minimising vectors"; the reference returns one, SPEC.md:273 lists this as a
 * non-goal).  Sorted by the Gray tie rule m_tie, so out[0] is what qb_solve returns.  Writes up
 * to `cap` minimisers; *count receives the total number (which may exceed cap), *value the
 * minimum (eval_upper).  Exact on the integer path; on the float path the candidates within the
 * quantization bound are re-evaluated with eval_upper and those equal to the minimum kept. */
int qb_all_minimisers(const double* coeffs, int n, int m_fix, uint64_t suffix, int m_tie, uint64_t* out,
                      uint64_t cap, uint64_t* count, double* value);

/* Seam 1: the reference operator _kernels.gray_scan(coeffs, qua, lin, x0, v0, n_free)
 * (_kernels.py:46-75) with its exact return contract: x_min (fp64[n], 0/1), v_min
 * (eval_upper(x_min), or v0 when no visited state beats the start), steps = 2^n_free - 1.
 * Requires the free bits of x0 to be zero and v0 == eval_upper(x0), as in every reference call
 * (solver.py:161-166).  qua/lin are accepted for signature parity and cross-checked. */
int qb_gray_scan(const double* coeffs, const double* qua, const double* lin, const double* x0, double v0,
                 int n, int n_free, double* x_min, double* v_min, uint64_t* steps);

/* Batch of independent instances (BASELINE config C): `count` instances of size n (n <= 24),
 * coeffs laid out [count][n][n]; entries below the diagonal are folded into the upper triangle
 * (QuboInstance convention, core.py:66-72).  Instance b is solved like solve_incremental (global
 * Gray-rank tie rule); values[b] = eval_upper(argmin) of the folded matrix.  One CTA per instance, T table in shared memory.  The reference has no batch API:
 * this replaces a loop / thread pool of solve_incremental calls (solver.py:118-136). */
int qb_solve_batch(const double* coeffs, int n, uint64_t count, uint64_t* argmin_bits, double* values,
                   double* kernel_ms);

/* The same for a batch held as float (BASELINE config C stores float32 Q): every coefficient is widened to
 * double exactly, so results are those of qb_solve_batch on the converted array, without the caller first
 * writing that 2x larger array. */
int qb_solve_batch_f32(const float* coeffs, int n, uint64_t count, uint64_t* argmin_bits, double* values,
                       double* kernel_ms);

/* The batch sharded over several GPUs of this process: contiguous slices
 * of the instances, slice i solved by qb_solve_batch on devices[i] from its own host thread, results
 * written in place (the gather is the caller's arrays).  *kernel_ms = the maximum over slices.  A
 * device may appear more than once (its slices then run one after another). */
int qb_solve_batch_devices(const double* coeffs, int n, uint64_t count, const int* devices, int ndev,
                           uint64_t* argmin_bits, double* values, double* kernel_ms);

/* Test hook: chunk-start ("prefix") evaluation used by the traversal kernels, run as a standalone
 * kernel.  For each of `count` chunks c in [c_begin, c_begin+count) of an n-bit problem with
 * k prefix bits, writes the start state's value (fp64, exact on the integer path) and the local
 * fields of the n-k free bits (fields[c][i] = Q_ii + sum_{j != i} Q~_ij x_j).  Mirrors
 * eval_upper / delta (core.py:123-150). */
int qb_prefix_eval(const double* coeffs, int n, int k, uint64_t c_begin, uint64_t count, double* values,
                   double* fields);

/* Test hook (host only): the embedded patched-immediate cubin of `kind` (1: QB_VARIANT_IMM, 512 coarse
 * table words; 2: QB_VARIANT_IMM2, 1024 words; 3 / 5: QB_VARIANT_IMM8 / IMM8A, 256 words; 4 / 6: QB_VARIANT_IMM8S / IMM8AS, 512 words; 7: QB_VARIANT_IMM8AQ, 1024 words) for chunk length L with `words` written into its
 * placeholder immediates -- the image those variants load.
 * *size receives the image size; the image is copied to `out` when cap >= *size. */
int qb_imm_image(int kind, int L, const uint32_t* words, unsigned char* out, uint64_t cap, uint64_t* size);

/* Test hook (host only): the byte image the threshold kernels (kind 3..7 = QB_VARIANT_IMM8, IMM8S, IMM8A, IMM8AS, IMM8AQ)
 * would run `coeffs` with: the packed table words (256 for kinds 3 / 5, 512 for 4 / 6, 1024 for 7), the quantized upper-
 * triangular instance (n * n doubles, integer-valued, coefficient * 2^scale_exp rounded), fl(1 / unit), the range
 * bound Rneg and the certified rounding margin (quantized units).  tests/test_byte_image_cpu.py replays the
 * device's block test on it and checks the range and no-false-negative claims of qb_coarse8.cuh. */
int qb_byte_image(const double* coeffs, int n, int kind, uint32_t* words, double* quantized, float* inv_unit,
                  int32_t* rneg, int64_t* slack, int32_t* scale_exp);

#ifdef __cplusplus
}
#endif
#endif /* QUBRUTE_B200_H */
