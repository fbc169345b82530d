// jacobi.cu -- a7: the small SVD of the b x b block R ("[A11, U_SVD, V_SVD] :=
// SVD(A11)").  The paper leaves the method open; reading R9: one-sided Hestenes
// Jacobi on W := R^T with rotations accumulated into U_s, pair skip tolerance sqrt(b) eps
// (relative), numerically-zero columns (||w||^2 <= eps^2 ||R||_F^2, reading R9b) never rotated,
// columns stably sorted by norm, then (V_s, R') := Householder QR of the sorted W with an
// explicit Q, column signs flipped so R'_jj >= 0, sigma_j := R'_jj.
//
// B200 design: block one-sided Jacobi.  The b columns are split into 2P blocks of 16; a
// thread-block cluster of P CTAs (P = ceil(b/32), 8 at b = 256) runs a round-robin tournament over
// the blocks (2P-1 rounds per sweep, one hardware cluster barrier per round).  In each round a CTA stages
// its two blocks (32 columns of W and of J, 128 KiB at b = 256) in shared memory and runs a
// full inner cyclic sweep over the 496 column pairs, 16 disjoint pairs at a time (one warp per
// pair, 8 rows per lane, fixed-order warp reductions broadcast from lane 0).  The pair order
// differs from the oracle's cyclic-by-rows order, so sigma agrees to rounding and U_s / V_s
// agree up to rotations inside clusters of equal singular values (x is invariant).
#include "kernels.cuh"
#include "prof.cuh"

namespace utv {

__device__ long long g_jac_trace[32 * 8];   // diagnostics (-DUTV_JAC_TRACE): CTA 0 phase clocks
// diagnostics: %globaltimer at the start and end of CTA 0 of every jacobi_kernel launch (ring of
// kJacRing), the in-situ execution time of the side-stream SVD (its stream events also count the
// wait for a free 8-SM cluster slot)
constexpr int kJacRing = 4096;
__device__ unsigned long long g_jac_ns[2 * kJacRing];
__device__ unsigned g_jac_cnt;
__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
namespace {
constexpr int JBLK = 16;
constexpr int JT = 512;

__device__ __forceinline__ void cluster_barrier() {
  // hardware cluster barrier (~0.2 us): release / acquire order the global-memory column
  // exchange between the CTAs of the cluster
  asm volatile("barrier.cluster.arrive.release.aligned;\n"
               "barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}

__device__ __forceinline__ void dmma16884(double (&d)[4], double a0, double a1, double b0) {
  asm volatile(
      "mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
      : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3])
      : "d"(a0), "d"(a1), "d"(b0));
}

__device__ __forceinline__ double warp_sum_bcast(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return __shfl_sync(0xffffffffu, v, 0);
}

__global__ void __launch_bounds__(JT, 1)
jacobi_kernel(int bw, double* __restrict__ W, double* __restrict__ J, const double* __restrict__ fro2, double tol,
              int max_sweeps, int* __restrict__ rot, int* __restrict__ info, unsigned* __restrict__ bar) {
  extern __shared__ __align__(16) double jsm[];
  double* sW = jsm;
  double* sJ = jsm + 2 * JBLK * bw;
  __shared__ double sQ[2 * JBLK * (2 * JBLK + 1)];   // this round's rotations, column c at sQ + c*33
  __shared__ int s_gcol[2 * JBLK];
  __shared__ int s_rot;
  __shared__ double s_nrm[2 * JBLK];
  __shared__ int s_done;
  __shared__ unsigned s_slot;
  const int P = gridDim.x, nblk = 2 * P, c = blockIdx.x;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  (void)bar;
  const double eps = 0x1.0p-52;
  const double small2 = eps * eps * fro2[0];   // R9b: numerically-zero column floor
  if (c == 0 && tid == 0) {
    s_slot = atomicAdd(&g_jac_cnt, 1u) % kJacRing;
    g_jac_ns[2 * s_slot] = globaltimer_ns();
  }

  int sweep = 0;
  bool converged = false;
  for (sweep = 0; sweep < max_sweeps; ++sweep) {
    for (int r = 0; r < nblk - 1; ++r) {
#ifdef UTV_JAC_TRACE
      const int trk = sweep * 15 + r;
      if (c == 0 && tid == 0 && trk < 32) g_jac_trace[trk * 8 + 0] = clock64();
#endif
      const int bp = (c == 0) ? 0 : 1 + (c - 1 + r) % (nblk - 1);
      const int kq = nblk - 1 - c;
      const int bq = (kq == 0) ? 0 : 1 + (kq - 1 + r) % (nblk - 1);
      if (tid < 2 * JBLK) s_gcol[tid] = tid < JBLK ? bp * JBLK + tid : bq * JBLK + (tid - JBLK);
      if (tid == 0) s_rot = 0;
      __syncthreads();
      // stage the 32 columns: all global loads of a thread in flight, then the shared stores
      constexpr int PER = 2 * JBLK * 256 / JT;
      {
        double lw[PER], lj[PER];
#pragma unroll
        for (int it = 0; it < PER; ++it) {
          const int e = tid + it * JT;
          const bool valid = e < 2 * JBLK * bw;
          const int col = valid ? e / bw : 0, row = valid ? e % bw : 0, gc = s_gcol[col];
          const bool ok = valid && gc < bw;
          lw[it] = ok ? __ldcg(W + (size_t)gc * bw + row) : 0.0;
          lj[it] = ok ? __ldcg(J + (size_t)gc * bw + row) : 0.0;
        }
#pragma unroll
        for (int it = 0; it < PER; ++it) {
          const int e = tid + it * JT;
          if (e < 2 * JBLK * bw) { sW[e] = lw[it]; sJ[e] = lj[it]; }
        }
      }
      // the round's rotations are accumulated in the 32 x 32 sQ (= I here) and applied to the
      // staged J columns once, at the end of the round (J_blk := J_blk sQ), instead of rotating the
      // b-row J columns at every step: half the shared-memory traffic of the inner sweep
      for (int e = tid; e < 2 * JBLK * 2 * JBLK; e += JT) {
        const int c = e / (2 * JBLK), r = e % (2 * JBLK);
        sQ[c * (2 * JBLK + 1) + r] = r == c ? 1.0 : 0.0;
      }
      __syncthreads();
      // squared column norms, recomputed from the data once per round and then updated exactly
      // per rotation (alpha' = alpha - t gamma, beta' = beta + t gamma): one inner product per pair
      for (int col = warp; col < 2 * JBLK; col += JT / 32) {
        double s2 = 0.0;
        for (int row = lane; row < bw; row += 32) s2 += sW[col * bw + row] * sW[col * bw + row];
        s2 = warp_sum_bcast(s2);
        if (lane == 0) s_nrm[col] = s2;
      }
      __syncthreads();
#ifdef UTV_JAC_TRACE
      if (c == 0 && tid == 0 && trk < 32) g_jac_trace[trk * 8 + 1] = clock64();
#endif
      constexpr int RPL = 256 / 32;                    // rows per lane (bw <= 256)
      for (int ir = 0; ir < 2 * JBLK - 1; ++ir) {
        if (warp < JBLK) {
          int a = (warp == 0) ? 0 : 1 + (warp - 1 + ir) % (2 * JBLK - 1);
          const int kb = 2 * JBLK - 1 - warp;
          int b = (kb == 0) ? 0 : 1 + (kb - 1 + ir) % (2 * JBLK - 1);
          int ga = s_gcol[a], gb = s_gcol[b];
          if (ga > gb) { int t0 = a; a = b; b = t0; t0 = ga; ga = gb; gb = t0; }
          if (gb < bw) {
            double* wi = sW + a * bw;
            double* wj = sW + b * bw;
            double x[RPL], y[RPL];
#pragma unroll
            for (int k = 0; k < RPL; ++k) {
              const int row = lane + 32 * k;
              x[k] = row < bw ? wi[row] : 0.0;
              y[k] = row < bw ? wj[row] : 0.0;
            }
            double gm = 0.0;
#pragma unroll
            for (int k = 0; k < RPL; ++k) gm += x[k] * y[k];
            gm = warp_sum_bcast(gm);
            const double al = s_nrm[a], be = s_nrm[b];
            const bool skip = (gm == 0.0) || al <= small2 || be <= small2 || fabs(gm) <= tol * sqrt(al * be);
            if (!skip) {
              // t = sign(zeta) / (|zeta| + sqrt(1 + zeta^2)), zeta = (be - al) / (2 gm), rewritten
              // as t = 2 gm sign(be - al) / (|be - al| + sqrt((be - al)^2 + 4 gm^2)) (one division)
              const double d = be - al;
              const double t = (d >= 0.0 ? 2.0 * gm : -2.0 * gm) / (fabs(d) + sqrt(d * d + 4.0 * gm * gm));
              const double cs = rsqrt(1.0 + t * t);
              const double sn = cs * t;
              double* qi = sQ + a * (2 * JBLK + 1);
              double* qj = sQ + b * (2 * JBLK + 1);
              const double u = qi[lane], v = qj[lane];     // 2 JBLK == 32 rows: one per lane
#pragma unroll
              for (int k = 0; k < RPL; ++k) {
                const int row = lane + 32 * k;
                if (row < bw) {
                  wi[row] = cs * x[k] - sn * y[k];
                  wj[row] = sn * x[k] + cs * y[k];
                }
              }
              qi[lane] = cs * u - sn * v;
              qj[lane] = sn * u + cs * v;
              __syncwarp();                                  // every lane has read s_nrm[a], s_nrm[b]
              if (lane == 0) {
                s_nrm[a] = fmax(al - t * gm, 0.0);
                s_nrm[b] = be + t * gm;
                atomicAdd(&s_rot, 1);
              }
            }
          }
        }
        __syncthreads();
      }
#ifdef UTV_JAC_TRACE
      if (c == 0 && tid == 0 && trk < 32) g_jac_trace[trk * 8 + 2] = clock64();
#endif
      {
        // J_blk := J_blk sQ (bw x 32 x 32) on the FP64 tensor cores: warp w owns rows 16w..16w+15,
        // all four 8-column tiles; the result goes straight to global memory
        const int g = lane >> 2, t4 = lane & 3;
        if (16 * warp < bw) {
          double d[4][4] = {};
#pragma unroll
          for (int ks = 0; ks < 2 * JBLK / 4; ++ks) {
            const int k0 = 4 * ks + t4;
            const int ra = 16 * warp + g, rb = ra + 8;
            const double a0 = ra < bw ? sJ[k0 * bw + ra] : 0.0;
            const double a1 = rb < bw ? sJ[k0 * bw + rb] : 0.0;
#pragma unroll
            for (int nt = 0; nt < 4; ++nt) dmma16884(d[nt], a0, a1, sQ[(8 * nt + g) * (2 * JBLK + 1) + k0]);
          }
#pragma unroll
          for (int nt = 0; nt < 4; ++nt)
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const int row = 16 * warp + g + ((q & 2) ? 8 : 0), col = 8 * nt + 2 * t4 + (q & 1);
              const int gc = s_gcol[col];
              if (row < bw && gc < bw) __stcg(J + (size_t)gc * bw + row, d[nt][q]);
            }
        }
        double lw[PER];
#pragma unroll
        for (int it = 0; it < PER; ++it) {
          const int e = tid + it * JT;
          lw[it] = e < 2 * JBLK * bw ? sW[e] : 0.0;
        }
#pragma unroll
        for (int it = 0; it < PER; ++it) {
          const int e = tid + it * JT;
          if (e < 2 * JBLK * bw) {
            const int col = e / bw, row = e % bw, gc = s_gcol[col];
            if (gc < bw) __stcg(W + (size_t)gc * bw + row, lw[it]);
          }
        }
      }
#ifdef UTV_JAC_TRACE
      if (c == 0 && tid == 0 && trk < 32) g_jac_trace[trk * 8 + 3] = clock64();
#endif
      if (tid == 0 && s_rot) atomicAdd(rot + sweep, s_rot);
      cluster_barrier();
#ifdef UTV_JAC_TRACE
      if (c == 0 && tid == 0 && trk < 32) g_jac_trace[trk * 8 + 4] = clock64();
#endif
    }
    if (tid == 0) s_done = (atomicAdd(rot + sweep, 0) == 0);
    __syncthreads();
    if (s_done) { converged = true; break; }
  }
  if (c == 0 && tid == 0) {   // accumulated over the steps of one factorization
    g_jac_ns[2 * s_slot + 1] = globaltimer_ns();
    atomicMax(info, converged ? sweep + 1 : sweep);
    if (!converged) atomicOr(info + 1, 1);
  }
}

// ||R||_F^2 of W (= R^T), fixed-order; one CTA.
__global__ void fro2_kernel(int bw, const double* __restrict__ W, double* __restrict__ out) {
  __shared__ double red[32];
  double s = 0.0;
  for (int e = threadIdx.x; e < bw * bw; e += blockDim.x) s += W[e] * W[e];
  s = warp_sum_bcast(s);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)blockDim.x / 32; ++w) t += red[w];
    out[0] = t;
  }
}

// W := R^T, J := I
__global__ void jacobi_init_kernel(int bw, const double* __restrict__ R, int64_t ldr, double* __restrict__ W,
                                   double* __restrict__ J) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < bw * bw; e += gridDim.x * blockDim.x) {
    const int i = e % bw, j = e / bw;
    W[e] = R[cm(j, i, ldr)];
    J[e] = i == j ? 1.0 : 0.0;
  }
}

// stable sort of the columns by norm (descending): Ws = W P, Us = J P
__global__ void jacobi_sort_kernel(int bw, const double* __restrict__ W, const double* __restrict__ J,
                                   double* __restrict__ Ws, double* __restrict__ Us, int64_t ldu) {
  __shared__ double nrm[256];
  __shared__ int pos[256];
  for (int j = threadIdx.x; j < bw; j += blockDim.x) {
    double s = 0.0;
    for (int r = 0; r < bw; ++r) s += W[(size_t)j * bw + r] * W[(size_t)j * bw + r];
    nrm[j] = sqrt(s);
  }
  __syncthreads();
  for (int j = threadIdx.x; j < bw; j += blockDim.x) {
    int p = 0;
    for (int l = 0; l < bw; ++l) p += (nrm[l] > nrm[j]) || (nrm[l] == nrm[j] && l < j);
    pos[j] = p;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < bw * bw; e += blockDim.x) {
    const int r = e % bw, j = e / bw, p = pos[j];
    Ws[(size_t)p * bw + r] = W[e];
    Us[cm(r, p, ldu)] = J[e];
  }
}

// V_s[:, j] = sgn_j (e_j - Q[:, j]), sigma_j = |R'_jj|
__global__ void jacobi_vs_kernel(int bw, const double* __restrict__ Q, const double* __restrict__ Rp,
                                 double* __restrict__ Vs, int64_t ldv, double* __restrict__ sigma) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < bw * bw; e += gridDim.x * blockDim.x) {
    const int r = e % bw, j = e / bw;
    const double d = Rp[(size_t)j * bw + j];
    const double v = (r == j ? 1.0 : 0.0) - Q[e];
    Vs[cm(r, j, ldv)] = d < 0.0 ? -v : v;
    if (r == 0) sigma[j] = fabs(d);
  }
}
}  // namespace

void svd_small(cudaStream_t st, int64_t bw64, const double* R, int64_t ldr, double* Us, int64_t ldu, double* sigma,
               double* Vs, int64_t ldv, const SvdWork& sw) {
  const int bw = (int)bw64;
  if (bw <= 0) return;
  {
  ProfScope prof_a(st, kProfSvd, 4, 0.0, 0.0);
  jacobi_init_kernel<<<std::max(1, std::min(bw * bw / 256, 256)), 256, 0, st>>>(bw, R, ldr, sw.W, sw.J);
  UTV_CUDA(cudaGetLastError());
  fro2_kernel<<<1, 1024, 0, st>>>(bw, sw.W, sw.X);   // X[0] = ||R||_F^2 (scratch)
  UTV_CUDA(cudaGetLastError());
  UTV_CUDA(cudaMemsetAsync(sw.rot, 0, sizeof(int) * kMaxSweeps, st));
  static std::atomic<unsigned long long> attr{0};
  ensure_smem_attr(jacobi_kernel, 4 * JBLK * 256 * (int)sizeof(double), attr);
  int P = (bw + 2 * JBLK - 1) / (2 * JBLK);
  size_t smem = (size_t)4 * JBLK * bw * sizeof(double);
  int bwv = bw;
  const double* fro2 = sw.X;
  double tol = sqrt((double)bw) * 0x1.0p-52;
  int maxs = kMaxSweeps;
  void* args[] = {&bwv, (void*)&sw.W, (void*)&sw.J, &fro2, &tol, &maxs, (void*)&sw.rot, (void*)&sw.info,
                  (void*)&sw.pw.bar};
  {
    // one thread-block cluster of P <= 8 CTAs (portable size): cluster barriers between rounds
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(P);
    cfg.blockDim = dim3(JT);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = P;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    UTV_CUDA(cudaLaunchKernelExC(&cfg, (const void*)jacobi_kernel, args));
  }
  jacobi_sort_kernel<<<1, 256, 0, st>>>(bw, sw.W, sw.J, sw.Ws, Us, ldu);
  UTV_CUDA(cudaGetLastError());
  }
  panel_qr(st, bw, bw, sw.Ws, bw, sw.Wh, bw, sw.tau, sw.Tq, bw, sw.pw);
  dgemm(st, false, true, bw, bw, bw, 1.0, sw.Tq, bw, sw.Wh, bw, 0.0, sw.X, bw, sw.pw.gemm_work,
        sw.pw.gemm_work_doubles, sw.pw.num_sms);
  dgemm(st, false, false, bw, bw, bw, 1.0, sw.Wh, bw, sw.X, bw, 0.0, sw.Q, bw, sw.pw.gemm_work,
        sw.pw.gemm_work_doubles, sw.pw.num_sms);
  ProfScope prof_b(st, kProfSvd, 1, 0.0, 0.0);
  jacobi_vs_kernel<<<std::max(1, std::min(bw * bw / 256, 256)), 256, 0, st>>>(bw, sw.Q, sw.Ws, Vs, ldv, sigma);
  UTV_CUDA(cudaGetLastError());
}

}  // namespace utv

// diagnostics only (not part of utv.h): copies min(count, max) (start, end) globaltimer pairs of
// the most recent jacobi_kernel launches to out (2 * max entries) and returns the launch count
// since the last reset (reset != 0 zeroes it after the copy); -1 on a CUDA error
extern "C" int utv_debug_jac_times(unsigned long long* out, int max, int reset) {
  unsigned cnt = 0;
  if (cudaMemcpyFromSymbol(&cnt, utv::g_jac_cnt, sizeof(unsigned)) != cudaSuccess) return -1;
  const int n = (int)std::min<unsigned>(cnt, (unsigned)std::min(max, utv::kJacRing));
  if (n > 0 && cudaMemcpyFromSymbol(out, utv::g_jac_ns, sizeof(unsigned long long) * 2 * n) != cudaSuccess) return -1;
  if (reset) {
    const unsigned z = 0;
    if (cudaMemcpyToSymbol(utv::g_jac_cnt, &z, sizeof(unsigned)) != cudaSuccess) return -1;
  }
  return (int)cnt;
}

extern "C" int utv_debug_jac_trace(long long* out) {   // diagnostics only (not part of utv.h)
  return (int)cudaMemcpyFromSymbol(out, utv::g_jac_trace, sizeof(long long) * 32 * 8);
}
