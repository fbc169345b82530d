// panel_qr.cu -- a3 / a5: Householder QR of a tall-skinny panel ("unpivoted_QR(Y)",
// P:809-811 "unpivoted_QR([A11; A21])"), compact-WY output ("W unit lower
// trapezoidal"), sign and T-factor conventions of LAPACK dlarfg/dlarft (reading R8).
//
// B200 design.  A b-wide panel has m' rows (50 000 .. 200 000), so one column step is a
// global reduction over the whole chip.  The panel is factored in 32-column sub-panels:
//  * qr2_kernel: one cooperative launch per sub-panel (<= 148 CTAs, each owning a contiguous
//    row range; data stays in L2).  Per column ONE grid barrier: a single fused pass per CTA
//    applies reflector j to its rows and accumulates, for column j+1, the squared norm, the
//    inner products with the remaining columns (-> w = v^T P) and with the previous
//    Householder vectors (-> the dlarft column of T).  Partials are reduced redundantly by
//    every CTA in a fixed order (deterministic, no atomics on data).
//  * between sub-panels: the block reflector is applied to the rest of the panel with three
//    DMMA GEMMs (W^T P, T^T ., P -= W .), and the off-diagonal blocks of T are assembled from
//    the needed blocks of the Gram matrix W^T W:  T_12 = -T_11 (W_1^T W_2) T_22.
// Tall panels (>= 2048 rows) first try CholeskyQR2 + Householder reconstruction on 64-column
// sub-panels (cholqr.cu, reading R22): both algorithms are enqueued and a device flag selects
// one, so the host never waits (the kernels of the other return at entry).
#include "kernels.cuh"
#include "prof.cuh"
#include <cstdlib>

namespace utv {

__device__ long long g_qr_trace[64 * 8];   // diagnostics: per column phase timestamps (CTA 0)
__device__ long long g_qr_arrive[2 * 256];  // diagnostics: globaltimer at barrier arrival / departure, column 5
__device__ __forceinline__ long long gtimer() { long long t; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t)); return t; }
namespace {
constexpr int NBMAX = 32;
constexpr int QR_THREADS = 256;
constexpr int SROW = NBMAX + 1;            // padded shared-memory row (conflict-free per column)
constexpr int SMEM_ROWS_MAX = 768;         // CTA rows cached in shared memory (<= 198 KiB)

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return __shfl_sync(0xffffffffu, v, 0);
}

// Transpose-reduce 32 per-lane values over the warp with 31 shuffles (instead of 32 x 5): after
// the 5 halving levels lane l holds the warp total of value index l.  Fixed order (deterministic).
__device__ __forceinline__ double warp_transpose_reduce(double (&a)[NBMAX]) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int lvl = 0; lvl < 5; ++lvl) {
    const int o = 16 >> lvl;               // exchange partner distance == half the live width
    const bool upper = lane & o;
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      if (i < o) {
        const double send = upper ? a[i] : a[i + o];
        const double keep = upper ? a[i + o] : a[i];
        a[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
      }
    }
  }
  return a[0];
}

// Block-reduce acc[0..nb) (rows i > j of this CTA) and store this CTA's partials.
template <bool GLOBAL>
__device__ __forceinline__ void block_reduce_store(double (&acc)[NBMAX], int nb, double* red_w, double* part_out,
                                                   int stride) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const double s = warp_transpose_reduce(acc);
  red_w[warp * NBMAX + lane] = s;
  __syncthreads();
  if (threadIdx.x < nb) {
    double t = 0.0;
    for (int w = 0; w < QR_THREADS / 32; ++w) t += red_w[w * NBMAX + threadIdx.x];
    if constexpr (GLOBAL) __stcg(part_out + (size_t)threadIdx.x * stride, t);
    else part_out[threadIdx.x] = t;
  }
}

// Unblocked Householder QR of the R x nb sub-panel P (rows 0..R-1 from its diagonal),
// LAPACK storage during the kernel (R on/above the diagonal, v strictly below), explicit W and
// zeros below R written at the end.  CTA c owns rows [c L, (c+1) L); SMEM: those rows live in
// shared memory for the whole kernel, else each row is re-read from global (L2) per column with
// all its loads in flight.  One grid barrier per column.
template <bool SMEM, bool HYB = false, int SR = SROW>
__global__ void __launch_bounds__(QR_THREADS, 1)
qr2_kernel(int64_t R, int nb, double* __restrict__ P, int64_t ldp, double* __restrict__ W, int64_t ldw, int64_t wtop,
           double* __restrict__ tau, double* __restrict__ T, int64_t ldt, double* __restrict__ part,
           unsigned* __restrict__ bar, int64_t Ls, Pred pr) {
  if (pred_skip(pr)) return;                 // uniform: every CTA returns before the grid barrier state
  // SMEM: the first Ls rows of each CTA's range live in shared memory for the whole kernel, the
  // rest (tall panels: hybrid) are re-read from global memory / L2 per column; !SMEM: Ls = 0.
  extern __shared__ double sp[];             // [Ls][SR] (SMEM only)
  __shared__ double red_w[(QR_THREADS / 32) * NBMAX];
  __shared__ double red[NBMAX];
  __shared__ double piv[NBMAX];              // row j: W values (< j) and P values (>= j)
  __shared__ double sw[NBMAX];               // w_l = v^T P[:, l]
  __shared__ double swz[NBMAX];              // sw, zero for l <= j and l >= nb (SMEM row update)
  __shared__ double ssg[NBMAX];              // s_p = W[:, p]^T v
  __shared__ double sT[NBMAX * NBMAX];
  __shared__ unsigned s_gen;

  const unsigned G = gridDim.x;
  const int tid = threadIdx.x;
  const int64_t L = (R + G - 1) / G;
  const int64_t r0 = (int64_t)blockIdx.x * L;
  const int64_t r1 = min(R, r0 + L);
  const int64_t rs = SMEM ? (HYB ? min(r1, r0 + Ls) : r1) : r0;   // rows [r0, rs) in shared memory
  auto in_smem = [&](int64_t i) { return SMEM && i < rs; };
  if (tid == 0) s_gen = ld_acquire_gpu(bar);
  if (blockIdx.x == 0) {
    for (int64_t e = tid; e < wtop * nb; e += QR_THREADS) {   // rows above the sub-panel in W
      const int64_t i = e % wtop, c = e / wtop;
      W[c * ldw + (i - wtop)] = 0.0;
    }
    for (int e = tid; e < NBMAX * NBMAX; e += QR_THREADS) sT[e] = 0.0;
  }
  if constexpr (SMEM) {
    for (int64_t e = tid; e < (rs - r0) * nb; e += QR_THREADS) {
      const int64_t il = e % (rs - r0), c = e / (rs - r0);
      sp[il * SR + c] = P[cm(r0 + il, c, ldp)];
    }
  }
  __syncthreads();
  unsigned gen = s_gen;

  double acc[NBMAX];
  double scal_prev = 0.0;                    // SMEM path: scal of the previous column
#pragma unroll
  for (int v = 0; v < NBMAX; ++v) acc[v] = 0.0;
  for (int64_t i = r0 + tid; i < r1; i += QR_THREADS) {        // column 0: rows i > 0
    if (i < 1) continue;
    const bool sm = in_smem(i);
    const double x0 = sm ? sp[(i - r0) * SR] : P[cm(i, 0, ldp)];
#pragma unroll
    for (int p = 0; p < NBMAX; ++p)
      if (p < nb) acc[p] += x0 * (sm ? sp[(i - r0) * SR + p] : P[cm(i, p, ldp)]);
  }

  // part: double-buffered by column parity; slot (buf, c) = CTA c's partial sums at [0, nb) and,
  // for the CTA owning pivot row j, that row at [NBMAX, NBMAX + nb).  A CTA runs at most one column
  // ahead of the slowest, so writes for column j+1 never touch the buffer read for column j, and
  // the owner updates row j in place while the others use the published copy.
  // value-major: element (buf, v, c) at part[(buf * 2 NBMAX + v) * G + c], so the 32 lanes of a warp
  // reading CTAs c..c+31 of one value touch one 256-byte segment (coalesced)
  auto pelem = [&](int buf, int v, unsigned c) { return part + ((size_t)buf * 2 * NBMAX + v) * G + c; };
  auto tr = [&](int j, int ph) {            // phase timestamps (build with -DUTV_QR_TRACE)
#ifdef UTV_QR_TRACE
    if (blockIdx.x == 0 && tid == 0 && j < 64) g_qr_trace[j * 8 + ph] = clock64();
#else
    (void)j; (void)ph;
#endif
  };
  // dlarft column j of T (T[0:j, j] = -tau_j T[0:j, 0:j] s_j, T[j, j] = tau_j; s_j = ssg) is
  // assembled by CTA 0 one column LATE, between publishing its arrival at column j+1's grid barrier
  // and polling for the others -- off the per-column critical path (thread l < j owns row l of T;
  // ssg keeps column j's values until column j+1's dlarfg, after the barrier).
  double tj_prev = 0.0;
  auto t_column = [&](int jc, double tjc) {
    if (blockIdx.x != 0 || jc < 0) return;
    if (tid < jc) {
      double s = 0.0;
      for (int l = tid; l < jc; ++l) s += sT[tid * NBMAX + l] * ssg[l];
      sT[tid * NBMAX + jc] = -tjc * s;
    }
    if (tid == 0) { sT[jc * NBMAX + jc] = tjc; tau[jc] = tjc; }
  };
  for (int j = 0; j < nb; ++j) {
    tr(j, 0);
    const int buf = j & 1;
    const unsigned owner = (unsigned)(j / L);
    if (G == 1) {
      block_reduce_store<false>(acc, nb, red_w, red, 1);
      if (tid < nb) piv[tid] = in_smem(j) ? sp[(j - r0) * SR + tid] : P[cm(j, tid, ldp)];
      t_column(j - 1, tj_prev);
      __syncthreads();
    } else {
      block_reduce_store<true>(acc, nb, red_w, pelem(buf, 0, blockIdx.x), (int)G);
      if (blockIdx.x == owner && tid < nb)
        __stcg(pelem(buf, NBMAX + tid, owner), in_smem(j) ? sp[(j - r0) * SR + tid] : P[cm(j, tid, ldp)]);
      tr(j, 3);
#ifdef UTV_QR_TRACE
      if (j == 5 && tid == 0 && blockIdx.x < 256) g_qr_arrive[blockIdx.x] = gtimer();
#endif
      grid_arrive(bar, gen);
      t_column(j - 1, tj_prev);
      grid_wait(bar, G, gen);
#ifdef UTV_QR_TRACE
      if (j == 5 && tid == 0 && blockIdx.x < 256) g_qr_arrive[256 + blockIdx.x] = gtimer();
#endif
      tr(j, 4);
      // fixed-order reduction of the G partials (identical in every CTA): warp w owns values
      // v = w + 8u; lane l sums CTAs c = l + 32q with all loads in flight, then a fixed butterfly
      const int warp = tid >> 5, lane = tid & 31;
      constexpr int QMAX = 5;                // G <= 160
      double vals[NBMAX / 8][QMAX];
#pragma unroll
      for (int u = 0; u < NBMAX / 8; ++u)
#pragma unroll
        for (int q = 0; q < QMAX; ++q) {
          const unsigned c = lane + 32u * q;
          const int v = warp + 8 * u;
          vals[u][q] = (c < G && v < nb) ? __ldcg(pelem(buf, v, c)) : 0.0;
        }
#pragma unroll
      for (int u = 0; u < NBMAX / 8; ++u) {
        double s = vals[u][0];
#pragma unroll
        for (int q = 1; q < QMAX; ++q) s += vals[u][q];
        s = warp_sum(s);
        if (lane == 0 && warp + 8 * u < nb) red[warp + 8 * u] = s;
      }
      if (tid < nb) piv[tid] = __ldcg(pelem(buf, NBMAX + tid, owner));
      __syncthreads();
    }
    tr(j, 1);
    // dlarfg on x = P[j:, j], evaluated redundantly by every thread (identical inputs and
    // operations, so identical results) instead of by thread 0 plus a broadcast barrier
    double tj, beta, scal;
    {
      const double alpha = piv[j];
      const double xi = sqrt(red[j]);
      if (xi == 0.0) {
        tj = 0.0; beta = alpha; scal = 0.0;
      } else {
        beta = -copysign(hypot(alpha, xi), alpha);
        tj = (beta - alpha) / beta;
        scal = 1.0 / (alpha - beta);
      }
    }
    if (tid < nb) {
      // SMEM path: the previous column's running sums used its pre-scaling values x (the stored
      // Householder entries are x * scal_prev), so that one partial sum is rescaled here
      const double rv = (SMEM && tid == j - 1) ? red[tid] * scal_prev : red[tid];
      if (tid > j) sw[tid] = piv[tid] + rv * scal;            // v^T P[:, l], v_j = 1
      else if (tid < j) ssg[tid] = piv[tid] + rv * scal;      // W[:, p]^T v
    }
    if (SMEM && tid < NBMAX) swz[tid] = (tid > j && tid < nb) ? piv[tid] + red[tid] * scal : 0.0;
    __syncthreads();
    tj_prev = tj;
#pragma unroll
    for (int v = 0; v < NBMAX; ++v) acc[v] = 0.0;
    tr(j, 2);
    const bool next = (j + 1 < nb);
    if constexpr (SMEM) {
      // Rows in shared memory: the pivot columns are read and written with a runtime index, and
      // the reflector is applied to every column with the zero-padded swz (no per-column selects);
      // column j keeps its pre-scaling value in registers, so acc[j] is rescaled next column.
      for (int64_t i = r0 + tid; i < rs; i += QR_THREADS) {
        if (i < j) continue;
        double* srow = sp + (i - r0) * SR;
        double row[NBMAX];
#pragma unroll
        for (int c = 0; c < NBMAX; ++c) row[c] = (c < nb) ? srow[c] : 0.0;
        const double xj = srow[j];
        const double xj1 = next ? srow[j + 1] : 0.0;
        const double swj1 = next ? swz[j + 1] : 0.0;
        const double v = (i == j) ? 1.0 : xj * scal;
        const double newj = (i == j) ? beta : v;
        const double tv = tj * v;
        const bool acc_next = next && i > j + 1;
        const double xn = xj1 - tv * swj1;
#pragma unroll
        for (int c = 0; c < NBMAX; ++c) row[c] -= tv * swz[c];
#pragma unroll
        for (int c = 0; c < NBMAX; ++c)
          if (c < nb) srow[c] = row[c];
        srow[j] = newj;
        if (acc_next) {
#pragma unroll
          for (int c = 0; c < NBMAX; ++c) acc[c] += xn * row[c];
        }
      }
      scal_prev = scal;
      if constexpr (!HYB) {
        __syncthreads();
        continue;
      }
    }
    // rows in global memory (all of them, or the hybrid variant's tail); with SMEM the running sum
    // of column j uses the pre-scaling x_j like the shared-memory rows (rescaled next column)
    for (int64_t i = rs + tid; i < r1; i += QR_THREADS) {
      if (i < j) continue;                   // rows above the pivot: untouched
      // load the whole row first (all loads in flight; no shared-memory store in between that the
      // compiler would have to order them against), then compute, store and accumulate.  j is
      // runtime, so every index is static and selected with unrolled compares.
      double row[NBMAX];
#pragma unroll
      for (int c = 0; c < NBMAX; ++c) row[c] = (c < nb) ? P[cm(i, c, ldp)] : 0.0;
      double xj = 0.0, xj1 = 0.0, swj1 = 0.0;
#pragma unroll
      for (int c = 0; c < NBMAX; ++c) {
        if (c == j) xj = row[c];
        if (c == j + 1) { xj1 = row[c]; swj1 = (c < nb) ? sw[c] : 0.0; }
      }
      const double v = (i == j) ? 1.0 : xj * scal;
      const double newj = (i == j) ? beta : v;   // v stored below the diagonal (LAPACK)
      const double tv = tj * v;
      const bool acc_next = next && i > j + 1; // column j+1: norm, v^T-products, Gram column
      const double xn = xj1 - tv * swj1;
#pragma unroll
      for (int c = 0; c < NBMAX; ++c) {
        if (c == j) row[c] = newj;
        else if (c > j && c < nb) row[c] -= tv * sw[c];
      }
#pragma unroll
      for (int c = 0; c < NBMAX; ++c)
        if (c >= j && c < nb) P[cm(i, c, ldp)] = row[c];
      if (acc_next) {
#pragma unroll
        for (int c = 0; c < NBMAX; ++c) acc[c] += xn * ((SMEM && c == j) ? xj : row[c]);
      }
    }
    if (SMEM) scal_prev = scal;
    __syncthreads();
  }
  t_column(nb - 1, tj_prev);                 // the last column of T
  __syncthreads();
  // write back: P = R (upper) / 0 (below); W = explicit unit-lower Householder vectors
  for (int64_t e = tid; e < (r1 - r0) * nb; e += QR_THREADS) {
    const int64_t il = e % (r1 - r0), c = e / (r1 - r0), i = r0 + il;
    const double x = in_smem(i) ? sp[il * SR + c] : P[cm(i, c, ldp)];
    P[cm(i, c, ldp)] = i <= c ? x : 0.0;
    W[cm(i, c, ldw)] = i < c ? 0.0 : (i == c ? 1.0 : x);
  }
  if (blockIdx.x == 0) {
    for (int e = tid; e < nb * nb; e += QR_THREADS) {
      const int r = e % nb, c = e / nb;
      T[cm(r, c, ldt)] = sT[r * NBMAX + c];
    }
  }
  if (G > 1) grid_sync_finish(bar, gen);
}

}  // namespace

namespace {
int g_qr_force_global = 0;   // utv_tune(UTV_TUNE_QR_GLOBAL): the global-memory qr2 variant at any size
int g_qr_ctas = 0;           // utv_tune(UTV_TUNE_QR_CTAS): cap on the cooperative CTAs (0 = automatic)
int g_qr_cholqr = 0;         // utv_tune(UTV_TUNE_QR_CHOLQR): 0 auto, 1 Householder only, 2 CholeskyQR2 forced
}  // namespace

void panel_force(int global_variant, int ctas, int cholqr) {
  g_qr_force_global = global_variant ? 1 : 0;
  g_qr_ctas = ctas > 0 ? ctas : 0;
  g_qr_cholqr = (cholqr >= 0 && cholqr <= 2) ? cholqr : 0;
}

namespace {
// Shared-memory rows per CTA of the 16-column sub-panel kernel (row stride 17 doubles) within the
// 227 KB opt-in limit (dynamic + the kernel's ~11 KB static shared memory).
constexpr int SROW16 = 17;
constexpr int SMEM_ROWS_MAX16 = 1600;

// One cooperative launch of the sub-panel kernel on columns [j0, j0 + nb) of the panel (rows j0:rows).
void qr2_launch(cudaStream_t st, int64_t rows, int64_t j0, int nb, double* P, int64_t ldp, double* W, int64_t ldw,
                double* tau, double* T, int64_t ldt, const PanelWork& pw, bool narrow) {
  const int64_t R = rows - j0;
  // one CTA (no grid barrier) up to 768 rows; else ~256+ rows per CTA, at most one per SM
  static const int env_max = [] { const char* e = std::getenv("UTV_QR_MAXCTAS"); return e ? std::atoi(e) : 0; }();
  const int cap = g_qr_ctas > 0 ? g_qr_ctas : env_max;
  const int gmax = cap > 0 ? std::min(cap, pw.num_sms) : std::min(pw.num_sms, 160);
  const int G = R <= 768 ? 1 : (int)std::max<int64_t>(1, std::min<int64_t>(gmax, (R + 255) / 256));
  const int64_t Lr = (R + G - 1) / G;
  // shared-memory rows: all of a CTA's rows (32 columns up to 768 rows per CTA; the 16-column
  // sub-panels of tall panels up to 1600), or the first SMEM_ROWS_MAX with the rest re-read from
  // L2 per column (hybrid); the global-memory variant only when forced (UTV_TUNE_QR_GLOBAL)
  const bool smem = !g_qr_force_global;
  int64_t Ls = smem ? std::min<int64_t>(Lr, narrow ? SMEM_ROWS_MAX16 : SMEM_ROWS_MAX) : 0;
  int64_t Rv = R; int nbv = nb; double* Pb = P + cm(j0, j0, ldp); double* Wb = W + cm(j0, j0, ldw);
  int64_t wtop = j0; double* taub = tau + j0; double* Tb = T + cm(j0, j0, ldt);
  Pred pr = launch_pred();
  void* args[] = {&Rv, &nbv, &Pb, (void*)&ldp, &Wb, (void*)&ldw, &wtop, &taub, &Tb, (void*)&ldt,
                  (void*)&pw.part, (void*)&pw.bar, &Ls, &pr};
  ProfScope prof(st, kProfPanel, 1, 2.0 * (double)R * nb * nb, 16.0 * (double)R * nb);
  // tag: 0 = global-memory variant, 1 = shared-memory variant, 3 = hybrid, 6 = 16-column shared-memory
  prof.shape(R, nb, G, !smem ? 0 : (narrow ? 6 : (Ls < Lr ? 3 : 1)));
  static std::atomic<unsigned long long> attr{0}, attr_h{0}, attr_n{0};
  ensure_smem_attr(qr2_kernel<true>, (int)(SMEM_ROWS_MAX * SROW * sizeof(double)), attr);
  ensure_smem_attr(qr2_kernel<true, true>, (int)(SMEM_ROWS_MAX * SROW * sizeof(double)), attr_h);
  ensure_smem_attr(qr2_kernel<true, false, SROW16>, (int)(SMEM_ROWS_MAX16 * SROW16 * sizeof(double)), attr_n);
  const size_t smem_bytes = smem ? (size_t)Ls * (narrow ? SROW16 : SROW) * sizeof(double) : 0;
  void* kern = !smem ? (void*)qr2_kernel<false>
                     : (narrow ? (void*)qr2_kernel<true, false, SROW16>
                               : (Ls < Lr ? (void*)qr2_kernel<true, true> : (void*)qr2_kernel<true>));
  UTV_CUDA(cudaLaunchCooperativeKernel(kern, dim3(G), dim3(QR_THREADS), args, smem_bytes, st));
}

// Rows per CTA of a sub-panel with R rows (the grid qr2_launch chooses).
int64_t qr2_rows_per_cta(int64_t R, const PanelWork& pw) {
  static const int env_max = [] { const char* e = std::getenv("UTV_QR_MAXCTAS"); return e ? std::atoi(e) : 0; }();
  const int cap = g_qr_ctas > 0 ? g_qr_ctas : env_max;
  const int gmax = cap > 0 ? std::min(cap, pw.num_sms) : std::min(pw.num_sms, 160);
  const int G = R <= 768 ? 1 : (int)std::max<int64_t>(1, std::min<int64_t>(gmax, (R + 255) / 256));
  return (R + G - 1) / G;
}
}  // namespace

namespace {
// Q_b^T applied from the left to the panel columns right of sub-panel [jb, jb + nb) (rows jb:rows),
// transposed so the skinny dimension nb is the GEMMs' N: Z1^T = P_r^T W_b ; Z2^T = Z1^T T_b ;
// P_r -= W_b (Z2^T)^T
void apply_subpanel(cudaStream_t st, int64_t rows, int64_t jb, int64_t nb, int64_t wr, double* P, int64_t ldp,
                    const double* W, int64_t ldw, const double* T, int64_t ldt, const PanelWork& pw) {
  if (wr <= 0) return;
  const int64_t R = rows - jb;
  double* Pr = P + cm(jb, jb + nb, ldp);
  const double* Wb = W + cm(jb, jb, ldw);
  const double* Tb = T + cm(jb, jb, ldt);
  dgemm(st, true, false, wr, nb, R, 1.0, Pr, ldp, Wb, ldw, 0.0, pw.z1, wr, pw.gemm_work, pw.gemm_work_doubles,
        pw.num_sms);
  dgemm(st, false, false, wr, nb, nb, 1.0, pw.z1, wr, Tb, ldt, 0.0, pw.z2, wr, pw.gemm_work, pw.gemm_work_doubles,
        pw.num_sms);
  dgemm(st, false, true, R, wr, nb, -1.0, Wb, ldw, pw.z2, wr, 1.0, Pr, ldp, pw.gemm_work, pw.gemm_work_doubles,
        pw.num_sms);
}

// dlarft's off-diagonal blocks of T[c0:c1, c0:c1] from the sub-panel blocks of width bw on its
// diagonal: Gram S = W^T W (rows c0:rows; W is zero above each column's diagonal), then
// T[0:jb, blk] = -T[0:jb, 0:jb] (S[0:jb, blk] T_bb) (indices relative to c0).
void assemble_t(cudaStream_t st, int64_t rows, int64_t c0, int64_t c1, int64_t bw, const double* W, int64_t ldw,
                double* T, int64_t ldt, const PanelWork& pw) {
  const int64_t cw = c1 - c0;
  if (cw <= bw) return;
  const double* Wc = W + cm(c0, c0, ldw);
  double* Tc = T + cm(c0, c0, ldt);
  // only the blocks W_i^T W_j with i < j are needed: S' = W(:, 0:jl)^T W(:, bw:cw) (jl = the last
  // block's first column), element (p, q) = W_p^T W_(q + bw) (44% fewer flops than the full Gram
  // at 4 sub-panels)
  const int64_t jl = ((cw - 1) / bw) * bw;
  dgemm(st, true, false, jl, cw - bw, rows - c0, 1.0, Wc, ldw, Wc + cm(0, bw, ldw), ldw, 0.0, pw.gram, jl,
        pw.gemm_work, pw.gemm_work_doubles, pw.num_sms);
  for (int64_t jb = bw; jb < cw; jb += bw) {
    const int64_t nb = std::min<int64_t>(bw, cw - jb);
    dgemm(st, false, false, jb, nb, nb, 1.0, pw.gram + cm(0, jb - bw, jl), jl, Tc + cm(jb, jb, ldt), ldt, 0.0, pw.x,
          jb, pw.gemm_work, pw.gemm_work_doubles, pw.num_sms);
    dgemm(st, false, false, jb, nb, jb, -1.0, Tc, ldt, pw.x, jb, 0.0, Tc + cm(0, jb, ldt), ldt, pw.gemm_work,
          pw.gemm_work_doubles, pw.num_sms);
  }
}

// Householder QR (qr2 sub-panel kernels) of columns [c0, c1) of the panel, rows c0:rows; rows
// above c0 of W are zeroed by the kernels (wtop), T[c0:c1, c0:c1] assembled.
void panel_hqr(cudaStream_t st, int64_t rows, int64_t c0, int64_t c1, double* P, int64_t ldp, double* W,
               int64_t ldw, double* tau, double* T, int64_t ldt, const PanelWork& pw) {
  for (int64_t jb = c0; jb < c1; jb += NBMAX) {
    const int nb = (int)std::min<int64_t>(NBMAX, c1 - jb);
    const int64_t R = rows - jb;
    double* Wb = W + cm(jb, jb, ldw);
    double* Tb = T + cm(jb, jb, ldt);
    const int64_t Lr = qr2_rows_per_cta(R, pw);
    if (!g_qr_force_global && Lr > SMEM_ROWS_MAX && Lr <= SMEM_ROWS_MAX16 && nb > 16) {
      // Tall panel: rows per CTA exceed what 32 columns fit in shared memory but 16 columns fit.
      // The 32-column sub-panel is factored as two 16-column halves (each entirely in shared memory)
      // with Q_a^T applied to the second half in between; T_bb = [T_a, -T_a (W_a^T W_b) T_b; 0, T_b].
      const int na = 16, nc = nb - 16;
      qr2_launch(st, rows, jb, na, P, ldp, W, ldw, tau, T, ldt, pw, true);
      apply_subpanel(st, rows, jb, na, nc, P, ldp, W, ldw, T, ldt, pw);
      qr2_launch(st, rows, jb + na, nc, P, ldp, W, ldw, tau, T, ldt, pw, true);
      double* Wc = W + cm(jb, jb + na, ldw);                                    // rows jb.. (zero above jb + na)
      dgemm(st, true, false, na, nc, R, 1.0, Wb, ldw, Wc, ldw, 0.0, pw.x, na, pw.gemm_work, pw.gemm_work_doubles,
            pw.num_sms);                                                         // S_ac = W_a^T W_c
      dgemm(st, false, false, na, nc, nc, 1.0, pw.x, na, T + cm(jb + na, jb + na, ldt), ldt, 0.0, pw.z1, na,
            pw.gemm_work, pw.gemm_work_doubles, pw.num_sms);                     // S_ac T_c
      dgemm(st, false, false, na, nc, na, -1.0, Tb, ldt, pw.z1, na, 0.0, T + cm(jb, jb + na, ldt), ldt,
            pw.gemm_work, pw.gemm_work_doubles, pw.num_sms);                     // -T_a (S_ac T_c)
    } else {
      qr2_launch(st, rows, jb, nb, P, ldp, W, ldw, tau, T, ldt, pw, false);
    }
    apply_subpanel(st, rows, jb, nb, c1 - jb - nb, P, ldp, W, ldw, T, ldt, pw);
  }
  assemble_t(st, rows, c0, c1, NBMAX, W, ldw, T, ldt, pw);
}

// CholeskyQR2 sub-panels from this many rows on (below, the one-CTA / few-CTA Householder kernel
// is as fast); UTV_CQR_MIN_ROWS overrides (diagnostics)
int64_t cholqr_min_rows() {
  static const int64_t v = [] { const char* e = std::getenv("UTV_CQR_MIN_ROWS"); return e ? std::atoll(e) : 2048; }();
  return v;
}
}  // namespace

void panel_qr(cudaStream_t st, int64_t rows, int64_t w, double* P, int64_t ldp, double* W, int64_t ldw, double* tau,
              double* T, int64_t ldt, const PanelWork& pw) {
  if (w <= 0) return;
  launch_set_zero(st, w, w, T, ldt);
  // g_qr_cholqr: 0 = automatic (tall sub-panels), 1 = Householder kernels only, 2 = CholeskyQR2 at any height
  const bool force = g_qr_cholqr == 2;
  const bool cq = pw.cq && g_qr_cholqr != 1 && !g_qr_force_global && (force || rows >= cholqr_min_rows());
  if (!cq) {
    panel_hqr(st, rows, 0, w, P, ldp, W, ldw, tau, T, ldt, pw);
    return;
  }
  const int64_t bw = cholqr_max_width();
  for (int64_t jb = 0; jb < w; jb += bw) {
    const int nb = (int)std::min<int64_t>(bw, w - jb);
    // narrow last sub-panels (< 48 columns) are cheaper on the Householder kernels (~6 us per column
    // against a ~270 us fixed cost of the CholeskyQR2 sequence at 50000 rows)
    const bool tall = force || (rows - jb >= cholqr_min_rows() && nb >= 48);
    if (tall) {
      // both algorithms enqueued, the device flag picks one: no host wait (the Householder kernels
      // of a sub-panel CholeskyQR2 accepted return at entry, ~3 us per launch)
      cholqr_subpanel(st, rows, jb, nb, P, ldp, W, ldw, tau, T, ldt, pw);
      PredScope declined(pw.dflag, 1);
      panel_hqr(st, rows, jb, jb + nb, P, ldp, W, ldw, tau, T, ldt, pw);
    } else {
      panel_hqr(st, rows, jb, jb + nb, P, ldp, W, ldw, tau, T, ldt, pw);
    }
    apply_subpanel(st, rows, jb, nb, w - jb - nb, P, ldp, W, ldw, T, ldt, pw);
  }
  assemble_t(st, rows, 0, w, bw, W, ldw, T, ldt, pw);
}

}  // namespace utv

extern "C" int utv_debug_qr_trace(long long* out) {   // diagnostics only (not part of utv.h)
  int e = (int)cudaMemcpyFromSymbol(out, utv::g_qr_trace, sizeof(long long) * 64 * 8);
  return e ? e : (int)cudaMemcpyFromSymbol(out + 512, utv::g_qr_arrive, sizeof(long long) * 512);
}
