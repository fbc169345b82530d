// kernels.cuh -- launchers of the sm_100a randUTV kernels (internal to libutv.so).
#pragma once
#include "common.cuh"
#include "gemm.cuh"

namespace utv {

// ---- a1: Philox4x32-10 Gaussian sketch (sketch.cu) --------------------------------------
void launch_sketch(cudaStream_t st, uint64_t seed, int64_t step, int64_t row0, int64_t mrows, int64_t b, double* G,
                   int64_t ldg, int num_sms);
void launch_philox_words(cudaStream_t st, const uint32_t* ctr, const uint32_t* key, int64_t n, uint32_t* out);

// ---- a3/a5: Householder panel QR (panel_qr.cu) -------------------------------------------
struct PanelWork {
  double* part;          // >= 2 * num_sms * 64 doubles (double-buffered per-CTA partials)
  double* z1;            // >= 32 * w doubles
  double* z2;            // >= 32 * w doubles
  double* gram;          // >= w * w doubles
  double* x;             // >= w * 32 doubles
  double* gemm_work;     // split-K workspace
  size_t gemm_work_doubles;
  unsigned* bar;         // 2 unsigned, bar[0] == 0 between launches
  int num_sms;
  // CholeskyQR2 + reconstruction path (cholqr.cu); cq == nullptr disables it (side stream)
  double* cq = nullptr;  // >= rows * 64 doubles (Q_1 of a sub-panel)
  double* csm = nullptr; // >= cholqr_small_doubles()
  int* dflag = nullptr;  // device accept / reject flag (selects the algorithm on the device)
};
// In place: P (rows x w) -> R (upper triangle), zeros strictly below; W (rows x w) the explicit
// unit-lower Householder vectors; tau (w); T (w x w, upper, zeros below) with
// Q = H_0 ... H_{w-1} = I - W T W^T.  Requires rows >= w.
// utv_tune knobs: force the global-memory sub-panel kernel; cap the cooperative CTAs (0 = auto)
void panel_force(int global_variant, int ctas, int cholqr = 0);
// CholeskyQR2 + Householder reconstruction of columns [jb, jb + nb) (cholqr.cu, reading R22),
// enqueued; *pw.dflag on the device ends 0 (accepted) or nonzero (declined, nothing written).
int cholqr_max_width();
size_t cholqr_small_doubles();
void cholqr_subpanel(cudaStream_t st, int64_t rows, int64_t jb, int nb, double* P, int64_t ldp, double* W,
                     int64_t ldw, double* tau, double* T, int64_t ldt, const PanelWork& pw);
void panel_qr(cudaStream_t st, int64_t rows, int64_t w, double* P, int64_t ldp, double* W, int64_t ldw, double* tau,
              double* T, int64_t ldt, const PanelWork& pw);

// ---- a7: small SVD (jacobi.cu) -----------------------------------------------------------
struct SvdWork {
  double* W;      // bw * bw
  double* J;      // bw * bw
  double* Ws;     // bw * bw
  double* Wh;     // bw * bw
  double* Tq;     // bw * bw
  double* X;      // bw * bw
  double* Q;      // bw * bw
  double* tau;    // bw
  int* rot;       // kMaxSweeps ints
  int* info;      // 2 ints: sweeps, status
  PanelWork pw;
};
constexpr int kMaxSweeps = 30;
// R (bw x bw upper triangular, ldr) -> U_s, sigma, V_s with R ~= U_s diag(sigma) V_s^T.
// Asynchronous; info[1] != 0 flags non-convergence (checked by the caller).
void svd_small(cudaStream_t st, int64_t bw, const double* R, int64_t ldr, double* Us, int64_t ldu, double* sigma,
               double* Vs, int64_t ldv, const SvdWork& sw);

// ---- a8/a9: rank and solve (solve.cu) ----------------------------------------------------
void launch_rank(cudaStream_t st, int64_t n, const double* T, int64_t ldt, double tau, int64_t* r_dev);
// In place z := T(j0:j1, j0:j1)^{-1} z for the rows j0..j1-1 of Z (ldz), k columns.
void launch_trsv_block(cudaStream_t st, int64_t j0, int64_t j1, const double* T, int64_t ldt, double* Z, int64_t ldz,
                       int64_t k);
// In place z := T11^{-1} z (r x k, ldz) for a T11 whose b x b diagonal blocks are DIAGONAL (randUTV
// without Nullify: A11 := Sigma): one GEMV launch per block + one scaling pass (b <= 256).
void launch_diag_block_solve(cudaStream_t st, int64_t r, int64_t b, const double* T, int64_t ldt, double* Z,
                             int64_t ldz, int64_t k);

// ---- misc (misc.cu) ----------------------------------------------------------------------
void launch_set_identity(cudaStream_t st, int64_t rows, int64_t cols, double* A, int64_t lda);
void launch_set_zero(cudaStream_t st, int64_t rows, int64_t cols, double* A, int64_t lda);
void launch_set_diag(cudaStream_t st, int64_t bw, const double* sigma, double* A, int64_t lda);
void launch_copy(cudaStream_t st, int64_t rows, int64_t cols, const double* src, int64_t lds, double* dst, int64_t ldd);
void launch_zero_strict_lower(cudaStream_t st, int64_t rows, int64_t cols, double* A, int64_t lda);
void launch_axpy(cudaStream_t st, int64_t n, double alpha, const double* x, double* y);   // y += alpha x (contiguous)
// multi-GPU block-cyclic helpers (misc.cu): see the kernels' comments
void launch_assemble_y(cudaStream_t st, int64_t np, int64_t cols, int64_t b, int64_t i, int P, int64_t Lmax,
                       const double* recv, double* Y, int64_t ldy);
void launch_gather_local(cudaStream_t st, int64_t nloc, int64_t cols, int64_t b, int64_t i, int P, int p,
                         const double* W, int64_t ldw, double* D, int64_t ldd);
// flag[0] |= any non-finite entry in A (rows x cols)
void launch_check_finite(cudaStream_t st, int64_t rows, int64_t cols, const double* A, int64_t lda, int* flag);

// ---- Nullify_top_right_part_of_T helpers (misc.cu) -----------------------------------------
void launch_rz_build(cudaStream_t st, int64_t bw, int64_t nz, const double* T, int64_t ldt, int64_t i0, int64_t r,
                     double* M, int64_t ldm);
void launch_rz_writeback(cudaStream_t st, int64_t bw, int64_t nz, const double* M, int64_t ldm, double* T,
                         int64_t ldt, int64_t i0, int64_t r);
void launch_reverse_rows(cudaStream_t st, int64_t bw, const double* src, int64_t lds, double* dst, int64_t ldd);
// Wide least squares (R21): dst (cols x rows) = src^T; permutations (mode 0 rows reversed, 1 columns
// reversed, 2 J src^T J upper triangle of a square upper-triangular src).
void launch_transpose(cudaStream_t st, int64_t rows, int64_t cols, const double* src, int64_t lds, double* dst,
                      int64_t ldd);
void launch_permute(cudaStream_t st, int mode, int64_t rows, int64_t cols, const double* src, int64_t lds, double* dst,
                    int64_t ldd);

}  // namespace utv
