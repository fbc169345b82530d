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
//    the Gram matrix W^T W:  T_12 = -T_11 (W_1^T W_2) T_22.
#include "kernels.cuh"
#include "prof.cuh"

namespace utv {

namespace {
constexpr int NBMAX = 32;
constexpr int QR_THREADS = 256;

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return __shfl_sync(0xffffffffu, v, 0);
}

// acc[v], v < nb: p < j -> sum x_i W[i,p]; v == j -> sum x_i^2; v > j -> sum x_i P[i,v]
// (rows i > j of the CTA range).  Block-reduce and store this CTA's partials.
__device__ __forceinline__ void block_reduce_store(double (&acc)[NBMAX], int nb, double* red_w, double* part_out) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
  for (int v = 0; v < NBMAX; ++v) {
    if (v < nb) {
      double s = warp_sum(acc[v]);
      if (lane == 0) red_w[warp * NBMAX + v] = s;
    }
  }
  __syncthreads();
  if (threadIdx.x < nb) {
    double s = 0.0;
    for (int w = 0; w < QR_THREADS / 32; ++w) s += red_w[w * NBMAX + threadIdx.x];
    __stcg(part_out + threadIdx.x, s);
  }
}

__global__ void __launch_bounds__(QR_THREADS, 1)
qr2_kernel(int64_t R, int nb, double* __restrict__ P, int64_t ldp, double* __restrict__ W, int64_t ldw, int64_t wtop,
           double* __restrict__ tau, double* __restrict__ T, int64_t ldt, double* __restrict__ part,
           unsigned* __restrict__ bar) {
  __shared__ double red_w[(QR_THREADS / 32) * NBMAX];
  __shared__ double red[NBMAX];
  __shared__ double piv[NBMAX];      // pivot row j (published by its owner)
  __shared__ double sw[NBMAX];       // w_l = v^T P[:, l]
  __shared__ double ssg[NBMAX];      // s_p = W[:, p]^T v
  __shared__ double sT[NBMAX * NBMAX];
  __shared__ double s_tau, s_beta, s_scal;
  __shared__ unsigned s_gen;

  const unsigned G = gridDim.x;
  const int tid = threadIdx.x;
  const int64_t L = (R + G - 1) / G;
  const int64_t r0 = (int64_t)blockIdx.x * L;
  const int64_t r1 = min(R, r0 + L);
  unsigned gen = 0;
  if (tid == 0) { s_gen = *((volatile unsigned*)bar + 1); }
  __syncthreads();
  gen = s_gen;

  // zero the rows above the sub-panel in W (columns 0..nb-1)
  if (blockIdx.x == 0) {
    for (int64_t e = tid; e < wtop * nb; e += QR_THREADS) {
      const int64_t i = e % wtop, c = e / wtop;
      W[c * ldw + (i - wtop)] = 0.0;
    }
    for (int e = tid; e < NBMAX * NBMAX; e += QR_THREADS) sT[e] = 0.0;
  }

  double acc[NBMAX];
#pragma unroll
  for (int v = 0; v < NBMAX; ++v) acc[v] = 0.0;
  // reduction for column 0
  for (int64_t i = r0 + tid; i < r1; i += QR_THREADS) {
    if (i < 1) continue;
    const double x = P[cm(i, 0, ldp)];
    acc[0] += x * x;
#pragma unroll
    for (int l = 1; l < NBMAX; ++l)
      if (l < nb) acc[l] += x * P[cm(i, l, ldp)];
  }

  // part is double-buffered by column parity: slot (buf, c) holds CTA c's partial sums
  // [0, nb) and, for the CTA owning the pivot row j, that row's values P[j, l] at [NBMAX + l].
  // A CTA can run at most one column ahead of the slowest (it blocks in the next barrier), so
  // the writes for column j+1 never touch the buffer still being read for column j, and the
  // owner may update row j in place while the others use the published copy.
  auto slot = [&](int buf, unsigned c) { return part + ((size_t)buf * G + c) * (2 * NBMAX); };
  for (int j = 0; j < nb; ++j) {
    const int buf = j & 1;
    const unsigned owner = (unsigned)(j / L);
    block_reduce_store(acc, nb, red_w, slot(buf, blockIdx.x));
    if (blockIdx.x == owner && tid >= j && tid < nb) __stcg(slot(buf, owner) + NBMAX + tid, P[cm(j, tid, ldp)]);
    grid_sync(bar, G, gen);
    {
      // fixed-order reduction of the G partials (identical in every CTA): warp w owns the
      // values v = w, w+8, ...; lane l sums CTAs c = l, l+32, ...; then a fixed butterfly.
      const int warp = tid >> 5, lane = tid & 31;
      for (int v = warp; v < nb; v += QR_THREADS / 32) {
        double s = 0.0;
        for (unsigned c = lane; c < G; c += 32) s += __ldcg(slot(buf, c) + v);
        s = warp_sum(s);
        if (lane == 0) red[v] = s;
      }
      if (tid >= j && tid < nb) piv[tid] = __ldcg(slot(buf, owner) + NBMAX + tid);
    }
    __syncthreads();
    if (tid == 0) {
      const double alpha = piv[j];
      const double xi = sqrt(red[j]);
      double t, beta, scal;
      if (xi == 0.0) {
        t = 0.0; beta = alpha; scal = 0.0;
      } else {
        beta = -copysign(hypot(alpha, xi), alpha);
        t = (beta - alpha) / beta;
        scal = 1.0 / (alpha - beta);
      }
      s_tau = t; s_beta = beta; s_scal = scal;
    }
    __syncthreads();
    const double tj = s_tau, scal = s_scal;
    if (tid < nb) {
      if (tid > j) sw[tid] = piv[tid] + red[tid] * scal;
      else if (tid < j) ssg[tid] = __ldcg(W + cm(j, tid, ldw)) + red[tid] * scal;
    }
    __syncthreads();
    if (blockIdx.x == 0) {
      // dlarft: T[0:j, j] = -tau_j T[0:j, 0:j] s ; T[j, j] = tau_j
      if (tid < j) {
        double s = 0.0;
        for (int l = tid; l < j; ++l) s += sT[tid * NBMAX + l] * ssg[l];
        sT[tid * NBMAX + j] = -tj * s;
      }
      if (tid == 0) { sT[j * NBMAX + j] = tj; tau[j] = tj; }
    }
#pragma unroll
    for (int v = 0; v < NBMAX; ++v) acc[v] = 0.0;
    const bool next = (j + 1 < nb);
    for (int64_t i = r0 + tid; i < r1; i += QR_THREADS) {
      if (i < j) { W[cm(i, j, ldw)] = 0.0; continue; }
      double v;
      if (i == j) { v = 1.0; P[cm(j, j, ldp)] = s_beta; }
      else { v = P[cm(i, j, ldp)] * scal; P[cm(i, j, ldp)] = 0.0; }
      W[cm(i, j, ldw)] = v;
      const double tv = tj * v;
      const bool acc_next = next && (i > j + 1);
      double xn = 0.0;
#pragma unroll
      for (int l = 1; l < NBMAX; ++l) {
        if (l > j && l < nb) {
          double pl = P[cm(i, l, ldp)];
          if (tj != 0.0) { pl -= tv * sw[l]; P[cm(i, l, ldp)] = pl; }
          if (l == j + 1) xn = pl;
          else if (acc_next) acc[l] += xn * pl;
        }
      }
      if (acc_next) {
#pragma unroll
        for (int p = 0; p < NBMAX; ++p) {
          if (p <= j) acc[p] += xn * (p == j ? v : W[cm(i, p, ldw)]);
          else if (p == j + 1) acc[p] += xn * xn;
        }
      }
    }
    __syncthreads();
  }
  if (blockIdx.x == 0) {
    for (int e = tid; e < nb * nb; e += QR_THREADS) {
      const int r = e % nb, c = e / nb;
      T[cm(r, c, ldt)] = sT[r * NBMAX + c];
    }
  }
}

}  // namespace

void panel_qr(cudaStream_t st, int64_t rows, int64_t w, double* P, int64_t ldp, double* W, int64_t ldw, double* tau,
              double* T, int64_t ldt, const PanelWork& pw) {
  if (w <= 0) return;
  launch_set_zero(st, w, w, T, ldt);
  for (int64_t jb = 0; jb < w; jb += NBMAX) {
    const int nb = (int)std::min<int64_t>(NBMAX, w - jb);
    const int64_t R = rows - jb;
    const int G = (int)std::max<int64_t>(1, std::min<int64_t>(pw.num_sms, (R + 127) / 128));
    int64_t Rv = R; int nbv = nb; double* Pb = P + cm(jb, jb, ldp); double* Wb = W + cm(jb, jb, ldw);
    int64_t wtop = jb; double* taub = tau + jb; double* Tb = T + cm(jb, jb, ldt);
    void* args[] = {&Rv, &nbv, &Pb, (void*)&ldp, &Wb, (void*)&ldw, &wtop, &taub, &Tb, (void*)&ldt,
                    (void*)&pw.part, (void*)&pw.bar};
    {
      ProfScope prof(st, kProfPanel, 1, 2.0 * (double)R * nb * nb, 16.0 * (double)R * nb);
      UTV_CUDA(cudaLaunchCooperativeKernel((void*)qr2_kernel, dim3(G), dim3(QR_THREADS), args, 0, st));
    }
    const int64_t wr = w - jb - nb;
    if (wr > 0) {
      double* Pr = P + cm(jb, jb + nb, ldp);
      // Z1 = W_b^T P_r ; Z2 = T_b^T Z1 ; P_r -= W_b Z2      (apply Q_b^T from the left)
      dgemm(st, true, false, nb, wr, R, 1.0, Wb, ldw, Pr, ldp, 0.0, pw.z1, nb, pw.gemm_work, pw.gemm_work_doubles,
            pw.num_sms);
      dgemm(st, true, false, nb, wr, nb, 1.0, Tb, ldt, pw.z1, nb, 0.0, pw.z2, nb, pw.gemm_work,
            pw.gemm_work_doubles, pw.num_sms);
      dgemm(st, false, false, R, wr, nb, -1.0, Wb, ldw, pw.z2, nb, 1.0, Pr, ldp, pw.gemm_work,
            pw.gemm_work_doubles, pw.num_sms);
    }
  }
  if (w > NBMAX) {
    // Gram S = W^T W (upper part used), then T[0:jb, blk] = -T[0:jb,0:jb] (S[0:jb, blk] T_bb)
    dgemm(st, true, false, w, w, rows, 1.0, W, ldw, W, ldw, 0.0, pw.gram, w, pw.gemm_work, pw.gemm_work_doubles,
          pw.num_sms);
    for (int64_t jb = NBMAX; jb < w; jb += NBMAX) {
      const int64_t nb = std::min<int64_t>(NBMAX, w - jb);
      dgemm(st, false, false, jb, nb, nb, 1.0, pw.gram + cm(0, jb, w), w, T + cm(jb, jb, ldt), ldt, 0.0, pw.x, jb,
            pw.gemm_work, pw.gemm_work_doubles, pw.num_sms);
      dgemm(st, false, false, jb, nb, jb, -1.0, T, ldt, pw.x, jb, 0.0, T + cm(0, jb, ldt), ldt, pw.gemm_work,
            pw.gemm_work_doubles, pw.num_sms);
    }
  }
}

}  // namespace utv
