// gemm.cuh -- FP64 DMMA GEMM (column-major, BLAS-like semantics).
#pragma once
#include "common.cuh"
#include <algorithm>

namespace utv {

// C(M x N) = alpha * op(A) * op(B) + beta * C; op(X) = X^T when the flag is set.
// beta == 0 does not read C.  Split-K (deterministic) is used for small-output /
// long-K products when `work` has room; it needs dgemm_workspace_doubles().
void dgemm(cudaStream_t st, bool ta, bool tb, int64_t M, int64_t N, int64_t K, double alpha, const double* A,
           int64_t lda, const double* B, int64_t ldb, double beta, double* C, int64_t ldc, double* work,
           size_t work_doubles, int num_sms);

// utv_tune knobs: cfg 0..5 (else automatic), splits >= 1 (else automatic), path 1 = cp.async kernel
void dgemm_force(int cfg, int splits, int path);
int dgemm_split_count(int64_t M, int64_t N, int64_t K, int num_sms);
size_t dgemm_workspace_doubles(int64_t M, int64_t N, int64_t K, int num_sms);

}  // namespace utv
