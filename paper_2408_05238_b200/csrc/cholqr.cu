// cholqr.cu -- a3 / a5 fast path: the Householder factorization of a tall sub-panel (P:795-796
// "unpivoted_QR(Y)", "unpivoted_QR([A11; A21])"; compact WY P:663-666) computed as
// CholeskyQR2 followed by Householder reconstruction (reading R22 in DESIGN.md).
//
// For a full-rank sub-panel P (R x nb, nb <= 64) the QR factorization with a prescribed sign on
// diag(R) is unique, so the W, T, R that LAPACK's dlarfg/dlarft convention (reading R8) produces
// can be recovered from ANY orthonormal basis Q of P with P = Q R (diag R > 0):
//   Q - [S; 0] = W U'   (LU without pivoting of the top nb x nb block, s_j = -sign of the j-th
//                        Schur-complement pivot, so |pivot| >= 1: no growth),
//   W = [L; Q_2 U'^{-1}],   T = -U' S L^{-T},   R_householder = S R,   tau = diag(T).
// Q and R come from CholeskyQR2 (R_1 = chol(P^T P), Q_1 = P R_1^{-1}, R_2 = chol(Q_1^T Q_1),
// R = R_2 R_1), and W_2 = Q_2 U'^{-1} = P_2 (U' R)^{-1}.  Per sub-panel: two skinny DMMA Gram GEMMs
// over the R rows (P^T P, Q_1^T Q_1), two row-parallel triangular solves over the R rows
// (cqr_trsm_kernel: P R_1^{-1}, P_2 (U' R)^{-1}, substitution in registers), two single-CTA
// nb x nb kernels (Cholesky / LU with one CTA barrier per column, row solves, products) -- no
// per-column grid barrier, no explicit triangular inverse, no host wait.  CholeskyQR2 is accurate
// only while kappa(P) is moderate: a non-positive Cholesky pivot, or a first pass with
// ||Q_1^T Q_1 - I||_F > 1e-4 (kappa(P) beyond ~1e6), declines the sub-panel -- a device flag, which
// makes the rest of this sequence return at entry and the Householder kernels the caller enqueued
// behind it (panel_qr.cu, under PredScope) run instead.  Rank-deficient panels (the
// exact-rank transition of randUTV, zero columns) always take the Householder path, which keeps the
// paper's tau = 0 convention for zero columns; so do sub-panels with a column whose part below the
// diagonal vanishes (an LU pivot of magnitude 1), where dlarfg does not reflect.
#include "kernels.cuh"
#include "prof.cuh"

namespace utv {
namespace {

constexpr int CQ_NB = 64;               // widest sub-panel
constexpr int CQ_LD = CQ_NB + 1;        // padded shared-memory row
constexpr int CQ_MAT = CQ_NB * CQ_LD;   // doubles per nb x nb shared-memory matrix
constexpr int CQ_THREADS = 256;

// diagnostics: %globaltimer at the phase boundaries of cqr_recon_kernel (build with -DUTV_CQR_TRACE)
__device__ long long g_cqr_trace[16];
// diagnostics: sub-panels attempted / accepted by the CholeskyQR2 path on this device (tests read them
// through utv_debug_cqr_stats to see which sub-panels declined to the Householder kernels)
__device__ unsigned long long g_cqr_stats[2];
#ifdef UTV_CQR_TRACE
#define CQ_TRACE(k) do { __syncthreads(); if (threadIdx.x == 0) { long long t_; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_)); g_cqr_trace[k] = t_; } } while (0)
#else
#define CQ_TRACE(k) do { } while (0)
#endif

// 1 / d to within an ulp without the IEEE division sequence (whose ~220-cycle latency would sit on
// the per-column critical path of the factorizations): MUFU reciprocal seed + two Newton steps.
__device__ __forceinline__ double rcp(double d) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(d));
  double e = fma(-d, r, 1.0);
  r = fma(r, e, r);
  e = fma(-d, r, 1.0);
  return fma(r, e, r);
}

// nb x nb matrices in shared memory are row-major: a[r * CQ_LD + c].  Every routine below is called
// by all CQ_THREADS threads of the CTA and ends with a CTA barrier.
__device__ void load_cm(const double* __restrict__ g, int64_t ld, int nb, double* a) {
  for (int e = threadIdx.x; e < nb * nb; e += CQ_THREADS) {
    const int r = e % nb, c = e / nb;
    a[r * CQ_LD + c] = g[(size_t)c * ld + r];
  }
  __syncthreads();
}

// c = alpha a b (nb x nb, no aliasing): thread (ty, tx) of a 16 x 16 grid owns the 4 x 4 outputs
// (ty + 16 i, tx + 16 j) in registers -- 8 shared-memory loads per 16 FMAs, conflict-free.
__device__ void mm(double* __restrict__ c, const double* __restrict__ a, const double* __restrict__ b, int nb,
                   double alpha) {
  const int ty = threadIdx.x >> 4, tx = threadIdx.x & 15;
  double acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;
  for (int k = 0; k < nb; ++k) {
    double av[4], bv[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) av[i] = a[(ty + 16 * i) * CQ_LD + k];
#pragma unroll
    for (int j = 0; j < 4; ++j) bv[j] = b[k * CQ_LD + tx + 16 * j];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j] += av[i] * bv[j];
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j)
      if (ty + 16 * i < nb && tx + 16 * j < nb) c[(ty + 16 * i) * CQ_LD + tx + 16 * j] = alpha * acc[i][j];
  __syncthreads();
}

// In-place LU without pivoting, right-looking with ONE CTA barrier per column: thread (ty, tx) of
// a 16 x 16 grid updates rows j+1+ty+16p x columns j+1+tx+16q of the Schur complement, forming its
// rows' multipliers l_i = a_ij / pivot itself; the multipliers are stored (by tx == 0) and the
// pivots written back one step later, when no thread reads them any more.  The strict lower part
// of a becomes L (unit diagonal implied), the rest U.  SIGN: column j's pivot d is first shifted by
// s_j = -sign(d) (sign(0) = +; s_j -> sg[j]): the LU of Q_top - S of the reconstruction.
// Returns (uniformly -- every thread sees the same pivots) bit 0 = a zero / non-positive (!SIGN,
// Cholesky use) or non-finite pivot, bit 1 (SIGN) = |d| within 1e-8 of 1.
template <bool SIGN>
__device__ int lu_fast(double* a, int nb, double* sg, double* pv) {
  const int tid = threadIdx.x, ty = tid >> 4, tx = tid & 15;
  int st = 0;
  double lprev[4] = {0.0, 0.0, 0.0, 0.0};
  for (int j = 0; j < nb; ++j) {
    if (tx == 0 && j > 0) {                            // multipliers of column j - 1
#pragma unroll
      for (int p = 0; p < 4; ++p) {
        const int i = j + ty + 16 * p;
        if (i < nb) a[i * CQ_LD + j - 1] = lprev[p];
      }
    }
    // every load of the step before any store (the compiler cannot reorder them across the
    // possibly-aliasing stores itself)
    const double d = a[j * CQ_LD + j];
    double rj[4], ai[4], v[4][4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int l = j + 1 + tx + 16 * q;
      rj[q] = l < nb ? a[j * CQ_LD + l] : 0.0;
    }
#pragma unroll
    for (int p = 0; p < 4; ++p) {
      const int i = j + 1 + ty + 16 * p;
      ai[p] = i < nb ? a[i * CQ_LD + j] : 0.0;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int l = j + 1 + tx + 16 * q;
        v[p][q] = (i < nb && l < nb) ? a[i * CQ_LD + l] : 0.0;
      }
    }
    double piv = d;
    if constexpr (SIGN) {
      const double sj = d >= 0.0 ? -1.0 : 1.0;
      piv = d - sj;
      if (!(fabs(d) < 1.0 - 1.0e-8)) st |= 2;
      if (!isfinite(piv)) st |= 1;
      if (tid == 0) sg[j] = sj;
    } else {
      if (!(d > 0.0) || !isfinite(d)) st |= 1;
    }
    if (tid == 0) pv[j] = piv;
    const double pinv = rcp(piv);
#pragma unroll
    for (int p = 0; p < 4; ++p) {
      const int i = j + 1 + ty + 16 * p;
      const double li = ai[p] * pinv;
      lprev[p] = li;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int l = j + 1 + tx + 16 * q;
        if (i < nb && l < nb) a[i * CQ_LD + l] = v[p][q] - li * rj[q];
      }
    }
    __syncthreads();
  }
  for (int j = tid; j < nb; j += CQ_THREADS) a[j * CQ_LD + j] = pv[j];
  __syncthreads();
  return st;
}

// Row substitution in registers, two threads per row (lanes 2q and 2q+1 of a warp; h = lane & 1 owns
// columns 32h .. 32h+31 in x[0..31]): on entry x = this thread's half of a right-hand-side row, on
// exit the half of the solution of x M = rhs for the upper triangular CQ_NB x CQ_NB M in shared
// memory (minv[k] = 1 / M_kk; UNIT: unit diagonal).  Right-looking: x_k is formed by its owner,
// passed to the partner by a shuffle and folded into every later partial sum (32 independent
// accumulators per thread).  M must be padded with zeros beyond nb (minv = 1); every lane of the
// warp must take part (the shuffles), rows beyond the problem compute on zeros.
template <bool UNIT>
__device__ __forceinline__ void solve_row_upper2(double (&x)[32], const double* M, const double* minv) {
  const int lane = threadIdx.x & 31, h = lane & 1, pair = lane & ~1;
#pragma unroll
  for (int k = 0; k < CQ_NB; ++k) {
    const int own = k >> 5, kk = k & 31;
    double xk = 0.0;
    if (h == own) {
      xk = UNIT ? x[kk] : x[kk] * minv[k];
      x[kk] = xk;
    }
    xk = __shfl_sync(0xffffffffu, xk, pair | own);
    const double* Mk = M + k * CQ_LD + 32 * h;
#pragma unroll
    for (int c = 0; c < 32; ++c)
      if (32 * h + c > k) x[c] -= xk * Mk[c];
  }
}

// After lu_fast<false> of an SPD matrix (U = D L^T): R = D^{-1/2} U (upper, zeros below).
__device__ void lu_to_chol(double* a, int nb) {
  for (int e = threadIdx.x; e < nb * nb; e += CQ_THREADS) {
    const int r = e / nb, c = e % nb;
    if (c > r) a[r * CQ_LD + c] /= sqrt(a[r * CQ_LD + r]);
    else if (c < r) a[r * CQ_LD + c] = 0.0;
  }
  __syncthreads();
  for (int r = threadIdx.x; r < nb; r += CQ_THREADS) a[r * CQ_LD + r] = sqrt(a[r * CQ_LD + r]);
  __syncthreads();
}

// Kernel 1: R_1 = chol(G_1) (column-major, zeros below); flag = 0 (accepted) or 1 (a non-positive
// or non-finite pivot: the Householder path).
__global__ void __launch_bounds__(CQ_THREADS, 1)
cqr_chol_kernel(int nb, const double* __restrict__ G, int64_t ldg, double* __restrict__ R1, int* __restrict__ flag) {
  extern __shared__ double sm[];
  double* a = sm;
  __shared__ double pv[CQ_NB];
  load_cm(G, ldg, nb, a);
  const bool ok = lu_fast<false>(a, nb, nullptr, pv) == 0;
  if (threadIdx.x == 0) {
    *flag = ok ? 0 : 1;
    atomicAdd(&g_cqr_stats[0], 1ull);
  }
  if (!ok) return;
  lu_to_chol(a, nb);
  for (int e = threadIdx.x; e < nb * nb; e += CQ_THREADS) {
    const int r = e % nb, c = e / nb;
    R1[e] = a[r * CQ_LD + c];
  }
}

// X = P M^{-1} (rows x nb; M upper triangular nb x nb, column-major ld nb): two threads per row,
// the substitution in registers (solve_row_upper2).  Skipped when the flag is set.  In place
// allowed (X == P): each thread reads its half row before the pair writes.
constexpr int TRSM_THREADS = 128;
template <bool WITH_T>
__global__ void __launch_bounds__(TRSM_THREADS)
cqr_trsm_kernel(int64_t rows, int nb, const double* P, int64_t ldp, const double* __restrict__ M, int ldm,
                double* X, int64_t ldx, const int* __restrict__ flag, const double* __restrict__ LU,
                const double* __restrict__ sg, double* __restrict__ T, int64_t ldt, double* __restrict__ tau) {
  if (*(volatile const int*)flag != 0) return;
  __shared__ double Ms[CQ_NB * CQ_LD];
  __shared__ double minv[CQ_NB];
  if (WITH_T && blockIdx.x == gridDim.x - 1) {
    // side job of the last CTA (overlaps the row passes of the others): T = -U' S L^{-T} of the
    // reconstruction by row solves t_r L^T = -(U' S)_r, from the LU (col-major, ld CQ_NB) and signs
    for (int e = threadIdx.x; e < CQ_NB * CQ_NB; e += TRSM_THREADS) {   // Ms = L^T (unit, padded)
      const int r = e / CQ_NB, c = e % CQ_NB;
      Ms[r * CQ_LD + c] = (r < nb && c < nb && c > r) ? LU[(size_t)r * CQ_NB + c] : 0.0;
    }
    for (int k = threadIdx.x; k < CQ_NB; k += TRSM_THREADS) minv[k] = 1.0;
    __syncthreads();
    const int r = threadIdx.x >> 1, h = threadIdx.x & 1;
    double x[32];
#pragma unroll
    for (int c = 0; c < 32; ++c) {
      const int col = 32 * h + c;
      x[c] = (r < nb && col < nb && col >= r) ? -LU[(size_t)col * CQ_NB + r] * sg[col] : 0.0;
    }
    solve_row_upper2<true>(x, Ms, minv);
#pragma unroll
    for (int c = 0; c < 32; ++c) {
      const int col = 32 * h + c;
      if (r < nb && col < nb) T[(size_t)col * ldt + r] = col >= r ? x[c] : 0.0;
      if (r < nb && col == r) tau[r] = x[c];
    }
    return;
  }
  const unsigned nrow_ctas = WITH_T ? gridDim.x - 1 : gridDim.x;
  for (int e = threadIdx.x; e < CQ_NB * CQ_NB; e += TRSM_THREADS) {
    const int r = e % CQ_NB, c = e / CQ_NB;
    Ms[r * CQ_LD + c] = (r < nb && c < nb && r <= c) ? M[(size_t)c * ldm + r] : 0.0;
  }
  __syncthreads();
  for (int k = threadIdx.x; k < CQ_NB; k += TRSM_THREADS) minv[k] = k < nb ? 1.0 / Ms[k * CQ_LD + k] : 1.0;
  __syncthreads();
  const int h = threadIdx.x & 1;
  constexpr int RPB = TRSM_THREADS / 2;                 // rows per CTA pass
  const int64_t npass = (rows + RPB - 1) / RPB;
  for (int64_t ps = blockIdx.x; ps < npass; ps += nrow_ctas) {   // uniform per CTA (shuffles)
    const int64_t i = ps * RPB + (threadIdx.x >> 1);
    const bool live = i < rows;
    double x[32];
#pragma unroll
    for (int c = 0; c < 32; ++c) {
      const int col = 32 * h + c;
      x[c] = (live && col < nb) ? P[(size_t)col * ldp + i] : 0.0;
    }
    solve_row_upper2<false>(x, Ms, minv);
#pragma unroll
    for (int c = 0; c < 32; ++c) {
      const int col = 32 * h + c;
      if (live && col < nb) X[(size_t)col * ldx + i] = x[c];
    }
  }
}

// Kernel 2 (skipped when kernel 1 flagged): ||G_2 - I||_F <= 1e-4 (else flag 4: CholeskyQR2 needs a
// nearly orthonormal first pass, i.e. kappa(P) below ~1e6), R_2 = chol(G_2), R = R_2 R_1,
// Q_top = Q_1top R_2^{-1}, the LU of Q_top - S with the dlarfg signs, then the outputs of the
// sub-panel's top nb rows:  P top block := S R (upper, zeros below), W top block := L (unit lower),
// rows above the sub-panel of W := 0, M := U' R (column-major, for W_2 = P_2 M^{-1}), and the LU
// (column-major, ld CQ_NB) + signs from which the W_2 launch's extra CTA forms T = -U' S L^{-T} and
// tau = diag(T) (row solves T L^T = -U' S) while the other CTAs solve the rows.
__global__ void __launch_bounds__(CQ_THREADS, 1)
cqr_recon_kernel(int nb, const double* __restrict__ G2, int64_t ldg, const double* __restrict__ Q1, int64_t ldq,
                 const double* __restrict__ R1, int* __restrict__ flag, double* __restrict__ P, int64_t ldp,
                 double* __restrict__ W, int64_t ldw, int64_t wtop, double* __restrict__ Mout,
                 double* __restrict__ LUout, double* __restrict__ Sout) {
  if (*(volatile int*)flag != 0) return;
  extern __shared__ double sm[];
  double* a = sm;
  double* b = sm + CQ_MAT;
  double* m = sm + 2 * CQ_MAT;
  double* y = sm + 3 * CQ_MAT;
  __shared__ double s[CQ_NB], pv[CQ_NB], minv[CQ_NB];
  __shared__ double red[CQ_THREADS / 32];
  const int tid = threadIdx.x;
  CQ_TRACE(0);
  load_cm(G2, ldg, nb, a);
  double e2 = 0.0;
  for (int e = tid; e < nb * nb; e += CQ_THREADS) {
    const int r = e / nb, c = e % nb;
    const double d = a[r * CQ_LD + c] - (r == c ? 1.0 : 0.0);
    e2 += d * d;
  }
  for (int o = 16; o > 0; o >>= 1) e2 += __shfl_xor_sync(0xffffffffu, e2, o);
  if ((tid & 31) == 0) red[tid >> 5] = e2;
  __syncthreads();
  e2 = 0.0;
  for (int w = 0; w < CQ_THREADS / 32; ++w) e2 += red[w];
  if (!(e2 <= 1.0e-8)) {                              // uniform
    if (tid == 0) *flag = 4;
    return;
  }
  CQ_TRACE(5);
  if (lu_fast<false>(a, nb, nullptr, pv) != 0) {       // R_2 = chol(G_2) -> a
    if (tid == 0) *flag = 2;
    return;
  }
  lu_to_chol(a, nb);
  CQ_TRACE(1);
  load_cm(R1, nb, nb, b);
  mm(y, a, b, nb, 1.0);                               // y = R = R_2 R_1
  CQ_TRACE(6);
  for (int e = tid; e < CQ_NB * CQ_NB; e += CQ_THREADS) {   // b = R_2 padded for the row solves
    const int r = e / CQ_NB, c = e % CQ_NB;
    b[r * CQ_LD + c] = (r < nb && c < nb) ? a[r * CQ_LD + c] : 0.0;
  }
  for (int k = tid; k < CQ_NB; k += CQ_THREADS) minv[k] = k < nb ? 1.0 / a[k * CQ_LD + k] : 1.0;
  __syncthreads();
  if (tid < 2 * CQ_NB) {                             // m row r = Q_1top row r R_2^{-1} (2 threads / row)
    const int r = tid >> 1, h = tid & 1;
    double x[32];
#pragma unroll
    for (int c = 0; c < 32; ++c) x[c] = (r < nb && 32 * h + c < nb) ? Q1[(size_t)(32 * h + c) * ldq + r] : 0.0;
    solve_row_upper2<false>(x, b, minv);
#pragma unroll
    for (int c = 0; c < 32; ++c)
      if (r < nb && 32 * h + c < nb) m[r * CQ_LD + 32 * h + c] = x[c];
  }
  __syncthreads();
  CQ_TRACE(2);
  // |d| = 1 exactly when column j's part below the diagonal is zero after the previous reflectors,
  // where dlarfg takes tau = 0 (no reflection, R_jj keeps alpha's sign) -- a discontinuity the
  // reconstruction cannot resolve through rounding, so such sub-panels decline (flag 3): e.g. the
  // last column of a square panel, or a panel whose rows below the top block are zero.
  const int st = lu_fast<true>(m, nb, s, pv);          // m = L \ U', s = signs
  if (st != 0) {
    if (tid == 0) *flag = 3;
    return;
  }
  CQ_TRACE(3);
  for (int e = tid; e < nb * nb; e += CQ_THREADS) {
    const int r = e % nb, c = e / nb;
    P[(size_t)c * ldp + r] = r <= c ? s[r] * y[r * CQ_LD + c] : 0.0;          // S R
    W[(size_t)c * ldw + r] = r < c ? 0.0 : (r == c ? 1.0 : m[r * CQ_LD + c]);  // L
  }
  for (int64_t e = tid; e < wtop * nb; e += CQ_THREADS) {   // rows above the sub-panel
    const int64_t i = e % wtop, c = e / wtop;
    W[c * ldw + (i - wtop)] = 0.0;
  }
  for (int e = tid; e < CQ_NB * CQ_NB; e += CQ_THREADS) {   // a = U' (zeros below); the LU and the
    const int r = e / CQ_NB, c = e % CQ_NB;                  // signs for the T side job (trsm kernel)
    const bool in = r < nb && c < nb;
    a[r * CQ_LD + c] = (in && c >= r) ? m[r * CQ_LD + c] : 0.0;
    LUout[(size_t)c * CQ_NB + r] = in ? m[r * CQ_LD + c] : 0.0;
  }
  for (int k = tid; k < CQ_NB; k += CQ_THREADS) Sout[k] = k < nb ? s[k] : 1.0;
  __syncthreads();
  CQ_TRACE(7);
  CQ_TRACE(8);
  mm(m, a, y, nb, 1.0);                               // m = M = U' R
  for (int e = tid; e < nb * nb; e += CQ_THREADS) {
    const int r = e % nb, c = e / nb;
    Mout[e] = m[r * CQ_LD + c];
  }
  if (tid == 0) atomicAdd(&g_cqr_stats[1], 1ull);
  CQ_TRACE(4);
}

}  // namespace

int cholqr_max_width() { return CQ_NB; }

size_t cholqr_small_doubles() { return 4 * (size_t)CQ_NB * CQ_NB + CQ_NB; }

// Enqueue the CholeskyQR2 + reconstruction of columns [jb, jb + nb) of the panel (rows jb:rows).
// On the device, pw.dflag ends 0 (accepted: P, W, T, tau written) or nonzero (declined: nothing of
// P, W, T, tau written); the caller enqueues the Householder kernels under PredScope(pw.dflag, 1),
// so no host wait is needed.
void cholqr_subpanel(cudaStream_t st, int64_t rows, int64_t jb, int nb, double* P, int64_t ldp, double* W,
                     int64_t ldw, double* tau, double* T, int64_t ldt, const PanelWork& pw) {
  const int64_t R = rows - jb;
  double* Pb = P + cm(jb, jb, ldp);
  double* Wb = W + cm(jb, jb, ldw);
  double* G = pw.csm;
  double* R1 = G + CQ_NB * CQ_NB;
  double* M = R1 + CQ_NB * CQ_NB;
  double* LU = M + CQ_NB * CQ_NB;              // the signed LU of Q_top - S and the signs (T side job)
  double* Sg = LU + CQ_NB * CQ_NB;
  const size_t smem1 = (size_t)CQ_MAT * sizeof(double), smem2 = 4 * (size_t)CQ_MAT * sizeof(double);
  static std::atomic<unsigned long long> attr1{0}, attr2{0};
  ensure_smem_attr(cqr_chol_kernel, (int)smem1, attr1);
  ensure_smem_attr(cqr_recon_kernel, (int)smem2, attr2);
  dgemm(st, true, false, nb, nb, R, 1.0, Pb, ldp, Pb, ldp, 0.0, G, nb, pw.gemm_work, pw.gemm_work_doubles,
        pw.num_sms);                                                              // G_1 = P^T P
  {
    ProfScope prof(st, kProfPanel, 1, (double)nb * nb * nb / 3.0, 16.0 * nb * nb);
    prof.shape(nb, nb, 1, 10);
    cqr_chol_kernel<<<1, CQ_THREADS, smem1, st>>>(nb, G, nb, R1, pw.dflag);
    UTV_CUDA(cudaGetLastError());
  }
  {
    ProfScope prof(st, kProfPanel, 1, (double)R * nb * nb, 16.0 * (double)R * nb);
    prof.shape(R, nb, 1, 12);
    const int64_t blocks = std::min<int64_t>((R + TRSM_THREADS / 2 - 1) / (TRSM_THREADS / 2), 8 * (int64_t)pw.num_sms);
    cqr_trsm_kernel<false><<<(unsigned)blocks, TRSM_THREADS, 0, st>>>(R, nb, Pb, ldp, R1, nb, pw.cq, R, pw.dflag,
                                                                      nullptr, nullptr, nullptr, 0, nullptr);
    UTV_CUDA(cudaGetLastError());                                               // Q_1 = P R_1^{-1}
  }
  dgemm(st, true, false, nb, nb, R, 1.0, pw.cq, R, pw.cq, R, 0.0, G, nb, pw.gemm_work, pw.gemm_work_doubles,
        pw.num_sms);                                                              // G_2 = Q_1^T Q_1
  {
    ProfScope prof(st, kProfPanel, 1, 3.0 * nb * nb * nb, 40.0 * nb * nb);
    prof.shape(nb, nb, 1, 11);
    cqr_recon_kernel<<<1, CQ_THREADS, smem2, st>>>(nb, G, nb, pw.cq, R, R1, pw.dflag, Pb, ldp, Wb, ldw, jb, M, LU,
                                                   Sg);
    UTV_CUDA(cudaGetLastError());
  }
  {
    // W_2 = P_2 (U' R)^{-1}, and on one extra CTA T = -U' S L^{-T}, tau (overlapping the row passes)
    ProfScope prof(st, kProfPanel, 1, (double)(R - nb) * nb * nb, 16.0 * (double)(R - nb) * nb);
    prof.shape(R - nb, nb, 1, 12);
    const int64_t blocks =
        std::min<int64_t>((R - nb + TRSM_THREADS / 2 - 1) / (TRSM_THREADS / 2), 8 * (int64_t)pw.num_sms) + 1;
    cqr_trsm_kernel<true><<<(unsigned)blocks, TRSM_THREADS, 0, st>>>(R - nb, nb, Pb + nb, ldp, M, nb, Wb + nb, ldw,
                                                                     pw.dflag, LU, Sg, T + cm(jb, jb, ldt), ldt,
                                                                     tau + jb);
    UTV_CUDA(cudaGetLastError());
  }
  if (R > nb) {
    PredScope accepted(pw.dflag, 0);
    launch_set_zero(st, R - nb, nb, Pb + nb, ldp);
  }
}

}  // namespace utv

extern "C" int utv_debug_cqr_trace(long long* out) {   // diagnostics only (not part of utv.h)
  return (int)cudaMemcpyFromSymbol(out, utv::g_cqr_trace, sizeof(long long) * 16);
}

// diagnostics only (not part of utv.h): out[0] = sub-panels attempted, out[1] = accepted by the
// CholeskyQR2 path on the current device since the last reset (synchronises the device)
extern "C" int utv_debug_cqr_stats(unsigned long long* out, int reset) {
  int e = (int)cudaDeviceSynchronize();
  if (!e && out) e = (int)cudaMemcpyFromSymbol(out, utv::g_cqr_stats, sizeof(unsigned long long) * 2);
  if (!e && reset) {
    const unsigned long long z[2] = {0, 0};
    e = (int)cudaMemcpyToSymbol(utv::g_cqr_stats, z, sizeof(z));
  }
  return e;
}
