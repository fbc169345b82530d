/*
 * utv_steps.h -- step-level entry points of libutv.so: each exposes one row of the hot
 * path so that it can be checked against the oracle in isolation.
 * Conventions as in utv.h (FP64, column-major, device pointers, the handle's stream,
 * status returns, no host synchronisation unless stated).
 */
#ifndef UTV_STEPS_H_
#define UTV_STEPS_H_

#include "utv.h"

#ifdef __cplusplus
extern "C" {
#endif

/* a1 -- Gaussian sketch (reading R6).  G (mrows x b, ldg >= mrows):
 * entry (i, c) = Box-Muller of Philox4x32-10 with key (lo32 seed, hi32 seed) and counter
 * (lo32 g, hi32 g, c/2, step), g = row0 + i. */
utv_status utv_sketch(utv_handle handle, uint64_t seed, int64_t step, int64_t row0, int64_t mrows,
                      int64_t b, double* G, int64_t ldg);

/* a1 (integer part) -- raw Philox4x32-10: out[4i..4i+3] = philox(ctr[4i..4i+3], key[2i..2i+1])
 * for i < n (device arrays of uint32).  Bit-exact. */
utv_status utv_philox(utv_handle handle, int64_t n, const uint32_t* ctr, const uint32_t* key,
                      uint32_t* out);

/* a3 / a5 -- Householder QR of P (m x w, m >= w, in place; R8):
 * out P = R in the upper triangle, zeros strictly below; W (m x w, ldw >= m) the explicit
 * unit-lower Householder vectors; tau (w); T (w x w, ldt >= w) upper triangular with
 * H_0 ... H_{w-1} = I - W T W^T (LAPACK dlarfg/dlarft conventions). */
utv_status utv_hqr(utv_handle handle, int64_t m, int64_t w, double* P, int64_t ldp, double* W,
                   int64_t ldw, double* tau, double* T, int64_t ldt);

/* a7 -- SVD of a b x b upper-triangular block (readings R9, R9b): one-sided
 * Jacobi on R^T.  Out: U_s, V_s (b x b), sigma (b, non-negative, non-increasing) with
 * R ~= U_s diag(sigma) V_s^T.  *sweeps (if non-NULL) gets the sweep count (synchronises).
 * Requires 1 <= b <= 256.  UTV_ERR_NUMERICAL if Jacobi needed more than 30 sweeps. */
utv_status utv_svd_small(utv_handle handle, int64_t b, const double* R, int64_t ldr, double* Us,
                         int64_t ldu, double* sigma, double* Vs, int64_t ldv, int32_t* sweeps);

/* a7 in place -- "[A11, U_SVD, V_SVD] := SVD(A11)": the b x b upper-triangular block
 * A11 (lda) is replaced by diag(sigma); U_s, V_s, sigma as utv_svd_small.  Asynchronous: a
 * Jacobi failure is recorded in the handle and reported by utv_svd_status. */
utv_status utv_svd_block(utv_handle handle, int64_t b, double* A11, int64_t lda, double* Us,
                         int64_t ldu, double* sigma, double* Vs, int64_t ldv);

/* Read (and clear) the Jacobi status accumulated by utv_svd_block calls: *failed != 0 if any
 * block exceeded 30 sweeps; *max_sweeps the largest sweep count (synchronises). */
utv_status utv_svd_status(utv_handle handle, int32_t* failed, int32_t* max_sweeps);

/* a9 -- Z (n x k, ldz) := T(0:n, 0:n)^{-1} Z for upper-triangular T (ldt) (back substitution of
 * eq:simplesoln P:894-901 in 256-row blocks: block solve + DMMA GEMM updates). */
utv_status utv_trsm_upper(utv_handle handle, int64_t n, const double* T, int64_t ldt, double* Z,
                          int64_t ldz, int64_t k);

/* a2 / a4 / a6 primitive -- FP64 DMMA GEMM: C = alpha op(A) op(B) + beta C, op = transpose
 * when ta / tb != 0 (C is not read when beta == 0). */
utv_status utv_gemm(utv_handle handle, int ta, int tb, int64_t M, int64_t N, int64_t K, double alpha,
                    const double* A, int64_t lda, const double* B, int64_t ldb, double beta,
                    double* C, int64_t ldc);

/* a8 -- Compute_rank (R10) of T's diagonal (n entries); synchronises. */
utv_status utv_rank(utv_handle handle, int64_t n, const double* T, int64_t ldt, double tau,
                    int64_t* rank);

/* a8 on a vector: the same rule for the n diagonal entries d[0..n-1] gathered contiguously
 * (multi-GPU path, where diag(T) is spread over the column owners); synchronises. */
utv_status utv_rank_diag(utv_handle handle, int64_t n, const double* d, double tau, int64_t* rank);

/* ---- test / tuning knobs ---------------------------------------------------------------
 * Process-wide switches that force one implementation choice, so that parity tests can reach
 * on small inputs the code paths that only full-size problems take (and benchmarks can sweep
 * them).  They change how a result is computed, never what is computed.  value < 0 (or 0 where
 * stated) restores the automatic choice.  Not synchronised: set them while no call is running.
 *   UTV_TUNE_GEMM_CFG     DMMA GEMM tile configuration 0..5 (csrc/gemm.cu Shape<> table)
 *   UTV_TUNE_GEMM_SPLITS  split-K factor >= 1 (0 = cost model), clamped to the workspace
 *   UTV_TUNE_GEMM_PATH    1 = the cp.async kernel instead of the TMA kernel (0 = automatic)
 *   UTV_TUNE_QR_GLOBAL    1 = the global-memory sub-panel kernel of a3/a5 at any panel height
 *   UTV_TUNE_QR_CTAS      cap on the cooperative CTAs of a sub-panel launch (0 = automatic)
 *   UTV_TUNE_DIST_CHUNKS  multi-GPU handles: column chunks (1..4) of the sketch / power-iteration
 *                         and X = A W_V products, each chunk's AllReduce overlapping the next
 *                         chunk's GEMM on the communication stream (0 = automatic: 2)
 *   UTV_TUNE_SVD_LAG      multi-GPU handles: steps (1..8) by which the application of a diagonal
 *                         block's SVD may trail its panel QR (0 = automatic: 1 at P = 1, else 8)
 *   UTV_TUNE_QR_CHOLQR    a3/a5 panel algorithm: 0 = automatic (CholeskyQR2 + Householder
 *                         reconstruction on 64-column sub-panels of >= 2048 rows -- a last
 *                         sub-panel narrower than 48 columns excepted --, the Householder sub-panel
 *                         kernels where it declines, chosen on the device; reading R22),
 *                         1 = Householder kernels only, 2 = CholeskyQR2 attempted on every
 *                         sub-panel at any height and width
 * Returns UTV_ERR_ARG for an unknown key; *old (if non-NULL) gets the previous value. */
enum {
  UTV_TUNE_GEMM_CFG = 1,
  UTV_TUNE_GEMM_SPLITS = 2,
  UTV_TUNE_GEMM_PATH = 3,
  UTV_TUNE_QR_GLOBAL = 4,
  UTV_TUNE_QR_CTAS = 5,
  UTV_TUNE_DIST_CHUNKS = 6,
  UTV_TUNE_SVD_LAG = 7,
  UTV_TUNE_QR_CHOLQR = 8
};
utv_status utv_tune(int key, int64_t value, int64_t* old);

/* ---- instrumentation (bench.py) -----------------------------------------------------
 * When enabled, every kernel launch of the library on this handle is bracketed by CUDA events
 * on the handle's stream and tagged with a family; flops / bytes are the ALGORITHMIC counts of
 * the launch (GEMM: 2MNK flops, 8(MK + KN + MN[+MN if beta != 0]) bytes). */
enum {
  UTV_PROF_GEMM = 0,    /* FP64 DMMA GEMM (+ its split-K reduce) */
  UTV_PROF_PANEL = 1,   /* cooperative Householder sub-panel kernel */
  UTV_PROF_SVD = 2,     /* Jacobi SVD kernels */
  UTV_PROF_SKETCH = 3,  /* Philox sketch */
  UTV_PROF_SOLVE = 4,   /* rank + block triangular solve */
  UTV_PROF_MISC = 5,    /* copies, zeroing, identity, finiteness guard */
  UTV_PROF_FAMILIES = 6
};
typedef struct {
  int64_t launches;     /* kernel launches */
  int64_t calls;        /* event-bracketed launch groups */
  double ms;            /* sum of event-measured durations */
  double flops;         /* algorithmic flops */
  double bytes;         /* algorithmic bytes */
} utv_prof_entry;

/* enable != 0: start recording (clears previous records); 0: stop. */
utv_status utv_profile(utv_handle handle, int enable);
/* Fill out[0 .. UTV_PROF_FAMILIES-1] from the records so far (synchronises the stream). */
utv_status utv_profile_read(utv_handle handle, utv_prof_entry* out);
/* Write every record so far as CSV (family, launches, ms, flops, M, N, K, tag) to `path`
 * (diagnostics; synchronises). */
utv_status utv_profile_dump(utv_handle handle, const char* path);

#ifdef __cplusplus
}
#endif

#endif /* UTV_STEPS_H_ */
