/*
 * maternfisher.h — C ABI of the B200 (sm_100a) exact-likelihood engine behind Fisher-BT.
 *
 * This is the drop-in boundary for the reference's hot path (arXiv 2601.11437, package
 * `maternmle`).  Every entry point takes plain pointers and sizes; no torch or CUDA types
 * cross it.  The reference binds the path through Python objects; each function below
 * names the reference interface it replaces (path:line into the reference tree):
 *
 *   mle_ctx_create   <- SpatialDataset(locations, values)           pkg/src/maternmle/matern.py:59-84
 *   mle_loglik       <- log_likelihood(data, theta)                 pkg/src/maternmle/likelihood.py:81-89
 *                       LikelihoodObjective.loglik                  pkg/src/maternmle/optimizer.py:127-134
 *   mle_eval_all     <- grad_and_fisher(data, theta)                pkg/src/maternmle/likelihood.py:107-149
 *                       LikelihoodObjective.eval_all                pkg/src/maternmle/optimizer.py:136-142
 *   mle_build        <- build_cov_matrix / build_dcov_matrix        pkg/src/maternmle/matern.py:186-203
 *   mle_cholesky     <- cholesky_lower(sigma)                       pkg/src/maternmle/likelihood.py:63-78
 *   mle_bessel_k     <- bessel_k(nu, x)                             pkg/src/maternmle/bessel.py:80-100
 *   mle_dnu_xnu_knu  <- dnu_xnu_knu(nu, x)                          pkg/src/maternmle/bessel.py:327-370
 *   mle_dnu_series   <- case2_series / case3_series / case4_series  pkg/src/maternmle/bessel.py:184-318
 *   mle_digamma      <- digamma(nu)                                 pkg/src/maternmle/bessel.py:103-115
 *   mle_matern_elem  <- matern_cov / dcov_dalpha / dcov_dnu / dcov_dsigma2 on distance arrays
 *                                                                    pkg/src/maternmle/matern.py:100-168
 *
 * Return codes (all functions returning int):
 *   MLE_OK (0)            success
 *   MLE_NOT_PD (1)        Cholesky failed; *bad_pivot holds the 0-based failing pivot
 *                         (reference: NotPositiveDefinite(pivot=info-1), likelihood.py:76-77)
 *   MLE_INVALID (2)       invalid argument (reference raises ValueError: matern.py:44-48,
 *                         bessel.py:93-96, 341-345, matern.py:198-201)
 *   MLE_CUDA_ERROR (3)    CUDA runtime failure (message via mle_last_error)
 *
 * Threading: calls on one context are serialised on that context's own CUDA stream;
 * distinct contexts are independent and may be driven from different host threads
 * concurrently (the reference's functions are pure and concurrency-safe).
 */
#ifndef MATERNFISHER_H
#define MATERNFISHER_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MLE_OK 0
#define MLE_NOT_PD 1
#define MLE_INVALID 2
#define MLE_CUDA_ERROR 3

/* Which matrix mle_build writes (reference build_dcov_matrix `which`, matern.py:191-203). */
#define MLE_WHICH_SIGMA 0   /* Sigma(theta)                       build_cov_matrix        */
#define MLE_WHICH_SIGMA2 1  /* dSigma/dsigma2 = C/sigma2, diag 1  build_dcov_matrix sigma2 */
#define MLE_WHICH_ALPHA 2   /* dSigma/dalpha, zero diagonal       build_dcov_matrix alpha  */
#define MLE_WHICH_NU 3      /* dSigma/dnu, zero diagonal          build_dcov_matrix nu     */

/* Phase timers returned by mle_phase_times (milliseconds of device time, last call). */
#define MLE_PHASE_GEN 0
#define MLE_PHASE_POTRF 1
#define MLE_PHASE_SOLVE 2
#define MLE_PHASE_REDUCE 3
#define MLE_PHASE_TOTAL 4
#define MLE_NUM_PHASES 5

typedef struct mle_ctx mle_ctx;

/* Library version string and the last error message of the calling thread. */
const char* mle_version(void);
const char* mle_last_error(void);

/* Number of visible CUDA devices (0 if none); lets a host fail loudly without a GPU. */
int mle_device_count(void);

/*
 * Buffers of destroyed contexts are kept in a per-(device, size) cache and reused by the
 * next context of the same size (no cudaMalloc / cudaFree in the steady state of fitting
 * many datasets).  This returns every idle cached buffer to the driver.  Runtime utility:
 * the reference has no device memory to manage.
 */
int mle_release_cached_memory(void);

/*
 * Kernel profiling of the FP64 trailing-update GEMMs (roofline evidence for bench.py).
 * With profiling enabled, a pass (loglik / eval_all / eval_batch led by this context) runs
 * on one stream and brackets every Ozaki GEMM, slicing and generation launch with CUDA events.
 * mle_kernel_stats then returns, for the last pass, MLE_KSTATS doubles:
 *   [0] GEMM launches  [1] GEMM ms (sum of launch durations)  [2] FP64-equivalent tile
 *   flops  [3] int8 tensor-core ops (28 slice products per FP64 MAC)  [4] slicing launches  [5] slicing
 *   ms  [6] slicing algorithmic bytes  [7] host time to enqueue the last pass (ms; also
 *   maintained when profiling is off)  [8] main-stream idle time between the previous pass on
 *   this device and the host's first enqueue of this one (ms)  [9] time this pass then waited
 *   for pending speculation and its parameter upload (ms)  [10] generation launches (Sigma
 *   and derivative matrices)  [11] generation ms  [12] generation algorithmic bytes (8 B per
 *   lower-triangle element per matrix written).
 * Diagnostic only: no reference counterpart.
 */
#define MLE_KSTATS 13
/* (max L_jj / min L_jj)^2 of the context's last successful factorization (0 before any): a
 * cheap lower bound of cond(Sigma), reported for diagnostics. */
int mle_ctx_cond_estimate(const mle_ctx* ctx, double* out);
/* 1 when the context evaluates eval_all in sequential-derivative mode: the derivative blocks
 * do not fit on the device beside the factor (BASELINE config 5, n = 100,000, on one B200),
 * so they are generated, reduced (B_i = L^-1 S_i L^-T) and summed one at a time in one work
 * matrix, finished blocks parked in the unused upper triangles of the two resident arrays.
 * Chosen at mle_ctx_create from n, the nugget and the device's memory (MLE_SEQ_DERIVS=0|1
 * overrides).  Results agree with the batched path to the rounding of the final sums; the
 * log-likelihood is bit-identical.  No reference counterpart (likelihood.py:107-149 holds
 * every matrix at once). */
int mle_ctx_seq_derivs(const mle_ctx* ctx);
int mle_kernel_profile(mle_ctx* ctx, int enable);
int mle_kernel_stats(const mle_ctx* ctx, double* out);

/*
 * Create a context owning device-resident copies of the n locations (n x 2, row-major
 * x,y pairs) and the n observed values z.  `device` selects the GPU.  `nugget` >= 0 adds
 * tau^2 to the diagonal of Sigma (0 reproduces the reference, which has no nugget).  With a
 * nugget, eval_all treats dSigma/dsigma^2 = (Sigma - tau^2 I)/sigma^2 as a third derivative
 * block (config 5; oracle/maternmle_cpu.py eval_all_nugget -- not in the reference).
 * All O(n^2) matrices are allocated lazily on first use.
 */
int mle_ctx_create(const double* locs_xy, const double* z, int64_t n, int device,
                   double nugget, mle_ctx** out);
void mle_ctx_destroy(mle_ctx* ctx);
int64_t mle_ctx_n(const mle_ctx* ctx);

/* Replace the observed values z (same n); used to refit a new field on the same locations. */
int mle_ctx_set_values(mle_ctx* ctx, const double* z);

/* Exact log-likelihood at theta = [sigma2, alpha, nu]. */
int mle_loglik(mle_ctx* ctx, const double theta[3], double* loglik, int64_t* bad_pivot);

/* Log-likelihood, score (3) and Fisher information (3x3 row-major, exactly symmetric). */
int mle_eval_all(mle_ctx* ctx, const double theta[3], double* loglik, double grad[3],
                 double fisher[9], int64_t* bad_pivot);

/*
 * Batched evaluation: `count` requests, one per distinct context, run as ONE pass (every
 * kernel launch covers all requests of the same device and padded size).  modes[i]:
 * 0 skip, 1 loglik, 2 eval_all.  thetas: count x 3.  results: count x 13 doubles
 * [loglik, grad[3], fisher[9] row-major] (grad/fisher only for mode 2).  rcs[i] / pivots[i]
 * carry each request's own MLE_OK / MLE_NOT_PD / MLE_INVALID and failing pivot.  Returns
 * MLE_OK when the batch ran (individual requests may still have failed), otherwise the
 * error that stopped it.  Replaces running the reference's LikelihoodObjective once per
 * replicate / L9 start sequentially (optimizer.py:188-197; "the nine L9
 * evaluations may run concurrently").
 */
int mle_eval_batch(mle_ctx* const* ctxs, int count, const double* thetas, const int* modes,
                   double* results, int64_t* pivots, int* rcs);

/*
 * One exact draw z = L w from N(0, Sigma(theta)) on the context's locations, with w the
 * caller's n standard normals: the device factorization followed by a device L w
 * (replaces simulate_grf, pkg/src/maternmle/simulate.py:100-106, whose `lower @ normals`
 * cannot run on a host at n >= 65,536).  The factor stays cached for theta.
 */
int mle_simulate(mle_ctx* ctx, const double theta[3], const double* w, double* z_out,
                 int64_t* bad_pivot);

/* Write one full n x n matrix (row-major == column-major, symmetric) to host memory. */
int mle_build(mle_ctx* ctx, const double theta[3], int which, double* out_host);

/* Device-time breakdown of the last mle_loglik / mle_eval_all call (MLE_NUM_PHASES doubles)
 * followed by: standard-count FP64 flops of the factor/solve phase, algorithmic bytes
 * written by generation, and the number of kernels the call launched
 * (MLE_NUM_PHASES + 3 doubles in total). */
int mle_phase_times(const mle_ctx* ctx, double* out);

/* Kernels this library has launched since it was loaded, all contexts and devices
 * (diagnostics: the bench reads it around its timed region). */
int64_t mle_launch_count(void);

/* Dense lower Cholesky of a host n x n symmetric matrix (row-major; only the lower triangle
 * is read).  l_out receives L with a zeroed strict upper triangle (LAPACK clean=1). */
int mle_cholesky(const double* a, int64_t n, int device, double* l_out, int64_t* bad_pivot);

/* Elementwise special functions on the GPU, m points, host in/out. */
int mle_bessel_k(double nu, const double* x, int64_t m, int device, double* out);
int mle_dnu_xnu_knu(double nu, const double* x, int64_t m, int device, double* out);

/* One order-derivative series on its own domain (drop-in for case2_series / case3_series /
 * case4_series, bessel.py:184-318): which_case 2 (0 < x < 8.5, nu off integers), 3
 * (8.5 <= x < 30), 4 (x >= 30); nu > 0.  Domain violations return MLE_INVALID. */
int mle_dnu_series(int which_case, double nu, const double* x, int64_t m, int device,
                   double* out);

/* digamma psi(x) (drop-in for bessel.digamma, bessel.py:103-115; host arithmetic, the per-theta
 * prologue's own routine).  Poles (non-positive integers) return MLE_INVALID. */
int mle_digamma(const double* x, int64_t m, double* out);

/* Elementwise Matern covariance / derivatives at distances h (h >= 0) for theta:
 * which = MLE_WHICH_* selects C, dC/dsigma2, dC/dalpha or dC/dnu; h = 0 gives the
 * zero-lag limit (sigma2, 1, 0, 0). */
int mle_matern_elem(const double theta[3], int which, const double* h, int64_t m, int device,
                    double* out);


/* ---- Distributed engine (configs 4-5 over several GPUs) ----------------------
 * One context per rank.  Outer blocks of 512 columns are owned cyclically (block b by rank
 * b % world); a rank holds the full-height column panels of Sigma -> L and of the derivative
 * blocks for its blocks.  The host driver (paper_2601_11437_b200/distributed.py) runs, per
 * evaluation:
 *   begin(theta) on every rank;
 *   for b: factor(b) on its owner -> broadcast P_b -> update(b) on every rank;
 *   (eval_all) for b: wblock(b) on the owner -> broadcast W_b -> forward(b) everywhere;
 *   (eval_all) for b: owner re-sends W_b, right_operand(b) -> broadcast X_b -> right(b);
 *   partials() on every rank -> all-reduce(sum).
 * Exchange buffers are device memory owned by the caller (NCCL sends them); sizes from
 * mle_dctx_layout.  Every call returns after this rank's stream drained (unless
 * mle_dctx_set_async).  Replaces the
 * reference's single-process likelihood.py:107-149 for n beyond one GPU's memory.
 */
typedef struct mle_dctx mle_dctx;
int mle_dctx_create(const double* locs_xy, const double* z, int64_t n, int device,
                    double nugget, int rank, int world, mle_dctx** out);
void mle_dctx_destroy(mle_dctx* d);
/* out[0] N, [1] blocks, [2] P-exchange bytes, [3] W-exchange bytes, [4] X-exchange bytes,
 * [5] derivative blocks (2, or 3 with a nugget), [6] blocks owned by this rank */
int mle_dctx_layout(const mle_dctx* d, int64_t* out);
int mle_dctx_begin(mle_dctx* d, const double theta[3], int derivs);
int mle_dctx_factor(mle_dctx* d, int b, void* exch_p);
int mle_dctx_update(mle_dctx* d, int b, const void* exch_p);
int mle_dctx_wblock(mle_dctx* d, int b, void* exch_w);
int mle_dctx_forward(mle_dctx* d, int b, const void* exch_w);
int mle_dctx_right_operand(mle_dctx* d, int b, void* exch_x);
int mle_dctx_right(mle_dctx* d, int b, const void* exch_w, const void* exch_x);
/* Look-ahead variants: only the panels of blocks j with lo <= j < hi.  right_range with
 * exch_w == NULL takes W_b from the rank's W cache (mle_dctx_wcache). */
int mle_dctx_update_range(mle_dctx* d, int b, const void* exch_p, int lo, int hi);
int mle_dctx_right_range(mle_dctx* d, int b, const void* exch_w, const void* exch_x, int lo,
                         int hi);
/* on = 1: the step calls above return as soon as their work is queued on the rank's stream
 * (mle_dctx_stream) instead of draining it; the caller orders its collectives against that
 * stream (CUDA events; NCCL on a communication stream).  begin / partials stay synchronous. */
int mle_dctx_set_async(mle_dctx* d, int on);
/* Two-sided reduction on the panels (the single-context engine's path from N >= 16,384):
 * per block b: wblock(b) and 2s_owner(b) on the owner (steps 1-3, S21 slices into exch_x),
 * panel_slices(b) (P_b into exch_p), broadcast both, 2s_update_range(b) on every rank
 * (step 4, the syr2k of its panels j > b), 2s_finish(b) on the owner (step 5); then the
 * deferred sweep: for b >= 1, W_b broadcast and forward_range(b, W, 0, b) on every rank. */
int mle_dctx_2s_owner(mle_dctx* d, int b, void* exch_x);
int mle_dctx_2s_finish(mle_dctx* d, int b);
int mle_dctx_2s_update_range(mle_dctx* d, int b, const void* exch_x, const void* exch_p, int lo,
                             int hi);
int mle_dctx_panel_slices(mle_dctx* d, int b, void* exch_p);
int mle_dctx_forward_range(mle_dctx* d, int b, const void* exch_w, int lo, int hi);
int mle_dctx_stream(const mle_dctx* d, void** stream);
/* Keep every block's W_b on this rank (~3.5 N^2 bytes) so that the right sweep reuses the
 * forward sweep's W_b instead of a second broadcast; MLE_CUDA_ERROR if it does not fit. */
int mle_dctx_wcache(mle_dctx* d, int on);
/* out: MLE_DCTX_SUMS partial sums [logdet, quad, trA, trN, <A,A>, <A,N>, <N,N>, trM, <A,M>,
 * <N,M>, <M,M>, yBy_A, yBy_N, yBy_M], then the failure flag and the 0-based pivot */
#define MLE_DCTX_SUMS 14
int mle_dctx_partials(mle_dctx* d, double* out);
/* The same sums per owned panel (ascending blocks; out[q * MLE_DCTX_SUMS + k]), then the
 * failure flag and pivot: adding panels in block order makes results independent of world. */
int mle_dctx_panel_partials(mle_dctx* d, double* out);

#ifdef __cplusplus
}
#endif

#endif /* MATERNFISHER_H */
