/*
 * hafb200.h -- C ABI of the B200 hafnian / loop-hafnian engine (arXiv 1805.12498).
 *
 * This is the drop-in boundary for the reference's kernel-module contract, the
 * object returned by hafnium.kernels.active() (pkg/src/hafnium/kernels/__init__.py:53-56)
 * and called from hafnium.engine._compute (engine.py:163-172) and
 * engine.subset_term (engine.py:210-214).  Each entry point below names the
 * reference function it replaces.
 *
 * Conventions (mirroring the reference contract):
 *   - complex data is interleaved (re, im) doubles: numpy complex128 memory;
 *   - matrices are row-major, C-contiguous; inputs are read-only, outputs are
 *     caller-allocated;
 *   - `atilde` is the PREPARED matrix X.A (rows 2i <-> 2i+1 swapped, diagonal
 *     zeroed for the hafnian), `diag` the loop weights (engine.py:140-150);
 *   - per-term / per-range numeric failures come back as status codes
 *     (0 ok, 1 QR sweep cap hit, 2 non-finite charpoly traces), never as errors;
 *   - the return value is 0 on success, negative on argument / CUDA errors
 *     (message via hafb_last_error(), thread-local); nothing throws across the ABI;
 *   - every call owns its stream and device buffers, so concurrent calls from
 *     different host threads are safe;
 *   - backend: 0 = spectral (Hessenberg + shifted QR), 1 = charpoly;
 *   - arith: 0 = MIRROR (the reference's exact IEEE operation sequence, results
 *     bit-identical to the reference), 1 = FAST (FMA-contracted kernels, results within
 *     the rounding-level bound of paper_1805_12498_b200/accuracy.py) for both backends:
 *     FAST charpoly = Hessenberg + tensor-core charpoly, FAST spectral = the same
 *     Hessenberg + the reference's shifted QR in FMA arithmetic (status 1 on
 *     non-convergence, as the reference); the entry points on a single matrix
 *     (hafb_power_traces, hafb_charpoly_coefficients) run MIRROR.
 *
 * Sizes: n_half = n/2 in [1, 32] (masks are 32-bit on the device; n <= 64).
 */
#ifndef HAFB200_H
#define HAFB200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HAFB_OK 0
#define HAFB_ERR_ARG (-1)
#define HAFB_ERR_CUDA (-2)
#define HAFB_ERR_NODEV (-3)

#define HAFB_BACKEND_SPECTRAL 0
#define HAFB_BACKEND_CHARPOLY 1
#define HAFB_ARITH_MIRROR 0
#define HAFB_ARITH_FAST 1

/* ABI version (bumped on any signature change). */
int hafb_abi_version(void);
/* Last error message of the calling thread ("" if none). */
const char* hafb_last_error(void);
/* Number of visible CUDA devices (0 if none). */
int hafb_device_count(void);

/* Replaces sum_subsets_det (kernels/_numba.py:354-384; numpy twin _numpy.py:182-200):
 * per-range Kahan partial sums over masks 1..2^n_half-1, ranges
 * [1 + r*w, min(1 + (r+1)*w, 2^n_half)), w = ceil((2^n_half - 1)/n_ranges).
 * partials: n_ranges complex; fails: n_ranges statuses (last nonzero per range). */
int hafb_sum_subsets_det(const double* atilde, const double* diag, int n_half, int backend,
                         int include_loops, int n_ranges, int cap_mult, int arith, int device,
                         double* partials, int64_t* fails);

/* Replaces sum_subsets_fast (kernels/_numba.py:387-412; _numpy.py:203-233): worker w
 * Kahan-sums, in one chain, the masks of ranges w, w+W, w+2W, ... (W = workers).
 * wsums: workers complex; wfails: workers statuses. */
int hafb_sum_subsets_fast(const double* atilde, const double* diag, int n_half, int backend,
                          int include_loops, int workers, int n_ranges, int cap_mult, int arith,
                          int device, double* wsums, int64_t* wfails);

/* Generalised range driver (the harness SURVEY.md 8(c) describes for n >= 48):
 * masks [lo, hi) cut into n_chunks chunks of width ceil((hi-lo)/n_chunks), Kahan per
 * chunk in mask order, mask 0 skipped.  hafb_sum_subsets_det == (lo=1, hi=2^D). */
int hafb_sum_mask_range(const double* atilde, const double* diag, int n_half, uint64_t lo,
                        uint64_t hi, int n_chunks, int backend, int include_loops, int cap_mult,
                        int arith, int device, double* partials, int64_t* fails);

/* Replaces subset_term (kernels/_numba.py:297-351), batched over `count` masks
 * (each nonzero and < 2^n_half).  terms: count complex; status: count int32. */
int hafb_terms(const double* atilde, const double* diag, int n_half, const uint64_t* masks,
               int64_t count, int backend, int include_loops, int cap_mult, int arith, int device,
               double* terms, int32_t* status);

/* Batched hafnians (new; the reference loops engine.hafnian): `batch` prepared problems
 * of the same n_half laid out back to back (atilde: batch*n*n complex, diag: batch*n).
 * Each problem runs the deterministic pipeline (n_ranges Kahan ranges + the
 * engine.py:87-97 tree) on the device.  results: batch complex; fails: batch statuses
 * (max over that problem's ranges, as engine._compute takes). */
int hafb_batch(const double* atilde, const double* diag, int batch, int n_half, int backend,
               int include_loops, int n_ranges, int cap_mult, int arith, int device,
               double* results, int64_t* fails);

/* Replaces power_traces_charpoly / power_traces_spectral (kernels/_numba.py:415-433):
 * traces tr(b^k), k = 1..K of one general m x m complex matrix (m <= 64).
 * ok: charpoly -> finite flag; spectral -> converged flag.  sweeps: QR sweeps (spectral). */
int hafb_power_traces(const double* b, int m, int K, int backend, int cap_mult, int arith,
                      int device, double* traces, int64_t* sweeps, int32_t* ok);

/* Replaces charpoly_coefficients (kernels/_numba.py:436-440): monic, ascending, m+1. */
int hafb_charpoly_coefficients(const double* b, int m, int arith, int device, double* coeffs);

/* Device-resident variant of hafb_sum_mask_range for callers that keep inputs in HBM
 * (bench `value`, multi-GPU ranks): all pointers are device pointers, the work is
 * enqueued on `stream` (a cudaStream_t) and the call returns without synchronising.
 * The workspace must be at least hafb_range_workspace_bytes(...) bytes. */
size_t hafb_range_workspace_bytes(int n_half, uint64_t lo, uint64_t hi, int n_chunks);
int hafb_sum_mask_range_async(const double* d_atilde, const double* d_diag, int n_half,
                              uint64_t lo, uint64_t hi, int n_chunks, int backend,
                              int include_loops, int cap_mult, int arith, void* d_workspace,
                              size_t workspace_bytes, double* d_partials, int64_t* d_fails,
                              void* stream);

/* Partial sums for an explicit list of the standard ranges (the partition of
 * hafb_sum_subsets_det with n_ranges ranges): partials[i] is range ranges[i].  This is
 * how the subset space is sharded across GPUs / ranks (LPT over range costs). */
int hafb_sum_range_list(const double* atilde, const double* diag, int n_half, int n_ranges,
                        const int32_t* ranges, int count, int backend, int include_loops,
                        int cap_mult, int arith, int device, double* partials, int64_t* fails);
size_t hafb_range_list_workspace_bytes(int n_half, int n_ranges, int count);
/* Device-resident range-list variant: d_atilde / d_diag / d_partials / d_fails and the
 * workspace are device pointers, `ranges` is a HOST array (the shard plan).  If
 * terms_done_event (a cudaEvent_t) is non-null it is recorded on `stream` between the
 * subset-term kernels and the range reduction (kernel-level timing). */
int hafb_sum_range_list_async(const double* d_atilde, const double* d_diag, int n_half,
                              int n_ranges, const int32_t* ranges, int count, int backend,
                              int include_loops, int cap_mult, int arith, void* d_workspace,
                              size_t workspace_bytes, double* d_partials, int64_t* d_fails,
                              void* stream, void* terms_done_event);

/* hafb_batch on RAW matrices: the input semantics of matrix.py:93-115 (strict
 * symmetry check max|A - A^T| <= symmetry_rtol * max(1, max|A|), upper -> lower
 * mirror) and engine.py:140-150 (zeroed diagonal for the hafnian, loop weights,
 * pair swap) run on the device.  a: batch x n x n complex128 (interleaved).  If a
 * matrix fails the check, *asym_index is its index (first one), *asym_dev / *asym_tol
 * the values, and nothing is computed; otherwise *asym_index = -1. */
int hafb_batch_raw(const double* a, int batch, int n_half, int backend, int include_loops,
                   int n_ranges, int cap_mult, int arith, int device, double symmetry_rtol,
                   double* results, int64_t* fails, int64_t* asym_index, double* asym_dev,
                   double* asym_tol);

/* Exact mode for INTEGER matrices (no reference counterpart:
 * the reference returns a float, inexact beyond 2^53, e.g. cfg3).  The subset sum
 * of engine.py:153-178 evaluated in GF(p) for each prime: per subset the same
 * Hessenberg / charpoly / Newton / exp-coefficient steps as _numba.py:36-351 with
 * field arithmetic (first-nonzero pivot, divisions by k and 2k as inverses mod p).
 * atilde_p: n_primes x n x n residues of the prepared X.A (row-major, the same
 * preparation as `atilde`); diag_p: n_primes x n residues of the loop weights;
 * primes: odd, n < p < 2^31; masks [lo, hi) of the 2^n_half subsets (mask 0 adds 0).
 * residues[i] = (sum of the signed terms) mod primes[i]; the host lifts them to the
 * exact integer by CRT.  device_ms (nullable) = device time of the term kernels. */
int hafb_modp_sums(const uint32_t* atilde_p, const uint32_t* diag_p, const uint32_t* primes,
                   int n_primes, int n_half, uint64_t lo, uint64_t hi, int include_loops,
                   int device, uint64_t* residues, double* device_ms);

/* Calibration: FP64 FMA throughput of `device` measured by a DFMA-saturating probe
 * kernel (the roofline denominator for the subset-term kernels).  tflops = 2 flop/DFMA. */
int hafb_fp64_peak(int device, double* tflops, double* ms);

/* Release the library's cached device memory on `device` (its private stream-ordered
 * pool keeps up to 8 GiB of freed buffers between calls; a large call such as n = 62
 * can leave more until the next synchronisation). */
int hafb_trim_pool(int device);

/* Kernel launches issued by the calling thread since the last reset (the bench's
 * gpu_launches claim). */
int64_t hafb_launch_count(int reset);

#ifdef __cplusplus
}
#endif

#endif /* HAFB200_H */
