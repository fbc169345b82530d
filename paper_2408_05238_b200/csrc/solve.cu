// solve.cu -- a8 Compute_rank (reading R10: relative to max_l T_ll,
// prefix rule) and the block triangular solve of a9, x_simple = V(:,1:r) T11^{-1} U_1^T b
// (eq:simplesoln P:894-901).  The large parts of a9 (the updates above each diagonal block and
// X = V(:, 0:r) z) are DMMA GEMMs; these kernels are the latency-bound pieces.
#include "kernels.cuh"
#include "prof.cuh"

namespace utv {

namespace {
__global__ void rank_kernel(int64_t n, const double* __restrict__ T, int64_t ldt, double tau, int64_t* r_out) {
  __shared__ double smax[32];
  __shared__ long long sidx[32];
  __shared__ double s_dmax;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  double m = 0.0;
  for (int64_t j = threadIdx.x; j < n; j += blockDim.x) m = fmax(m, T[cm(j, j, ldt)]);
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if (lane == 0) smax[warp] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    double d = 0.0;
    for (int w = 0; w < nw; ++w) d = fmax(d, smax[w]);
    s_dmax = d;
  }
  __syncthreads();
  const double dmax = s_dmax;
  long long first = (long long)n;
  for (int64_t j = threadIdx.x; j < n; j += blockDim.x)
    if (T[cm(j, j, ldt)] <= tau * dmax) { first = (long long)j; break; }
  for (int o = 16; o > 0; o >>= 1) {
    long long other = __shfl_xor_sync(0xffffffffu, first, o);
    first = other < first ? other : first;
  }
  if (lane == 0) sidx[warp] = first;
  __syncthreads();
  if (threadIdx.x == 0) {
    long long f = (long long)n;
    for (int w = 0; w < nw; ++w) f = sidx[w] < f ? sidx[w] : f;
    *r_out = (dmax == 0.0) ? 0 : (int64_t)f;
  }
}

// Back substitution on one diagonal block (<= 256 rows), k RHS in chunks of 16, in sub-blocks of 32
// from the bottom: warp 0 solves the 32 x 32 diagonal triangle with lane l owning row l (the pivot
// broadcast by shuffles, no block barrier per column), then every thread p above the sub-block
// subtracts its 32 terms T(p, i) z(i).  Per element the operations and their order (i descending,
// divide when all later columns are in) are those of plain column back substitution.
constexpr int TS_ROWS = 256, TS_K = 16, TS_SB = 32;
__global__ void __launch_bounds__(TS_ROWS) trsv_block_kernel(int64_t j0, int64_t j1, const double* __restrict__ T,
                                                             int64_t ldt, double* __restrict__ Z, int64_t ldz,
                                                             int64_t k) {
  __shared__ double z[TS_K][TS_ROWS];
  const int bs = (int)(j1 - j0);
  const int p = threadIdx.x, lane = p & 31;
  for (int64_t c0 = 0; c0 < k; c0 += TS_K) {
    const int kc = (int)((k - c0) < TS_K ? (k - c0) : TS_K);
    for (int e = threadIdx.x; e < bs * kc; e += blockDim.x) {
      const int q = e % bs, c = e / bs;
      z[c][q] = Z[cm(j0 + q, c0 + c, ldz)];
    }
    __syncthreads();
    for (int sb = ((bs - 1) / TS_SB) * TS_SB; sb >= 0; sb -= TS_SB) {
      const int w = (bs - sb) < TS_SB ? (bs - sb) : TS_SB;
      if (p < 32) {                                                    // diagonal 32 x 32 triangle
        double t[TS_SB];
#pragma unroll
        for (int u = 0; u < TS_SB; ++u)
          t[u] = (u < w && lane < w && lane <= u) ? T[cm(j0 + sb + lane, j0 + sb + u, ldt)] : 1.0;
        for (int c = 0; c < kc; ++c) {
          double zl = lane < w ? z[c][sb + lane] : 0.0;
#pragma unroll
          for (int u = TS_SB - 1; u >= 0; --u) {
            if (u >= w) continue;                                      // uniform
            if (lane == u) zl /= t[u];
            const double zi = __shfl_sync(0xffffffffu, zl, u);
            if (lane < u) zl -= t[u] * zi;
          }
          if (lane < w) z[c][sb + lane] = zl;
        }
      }
      __syncthreads();
      if (p < sb) {                                                    // rows above: 32 terms each
        double t[TS_SB];
#pragma unroll
        for (int u = 0; u < TS_SB; ++u) t[u] = u < w ? T[cm(j0 + p, j0 + sb + u, ldt)] : 0.0;
        for (int c = 0; c < kc; ++c) {
          double acc = z[c][p];
#pragma unroll
          for (int u = TS_SB - 1; u >= 0; --u)
            if (u < w) acc -= t[u] * z[c][sb + u];
          z[c][p] = acc;
        }
      }
      __syncthreads();
    }
    for (int e = threadIdx.x; e < bs * kc; e += blockDim.x) {
      const int q = e % bs, c = e / bs;
      Z[cm(j0 + q, c0 + c, ldz)] = z[c][q];
    }
    __syncthreads();
  }
}

// a9 when T11's b x b diagonal blocks are diagonal (randUTV sets A11 := Sigma, so
// without Nullify T11 = blockdiag(Sigma_i) + strictly-upper blocks): bottom-up over the blocks,
// block q (rows j0:j1) contributes acc(0:j0) -= T(0:j0, j0:j1) (acc(j0:j1) ./ diag(T)(j0:j1)).
// acc(j0:j1) is final once the blocks below are in and no later launch writes it, so one pass
// z = acc ./ diag(T) at the end gives z = T11^{-1} C.  One HBM-bound GEMV launch per block, z_q
// (scaled redundantly per CTA) in shared memory.
constexpr int DS_THREADS = 256, DS_K = 8, DS_B = 256, DS_ROWS = 32, DS_WARPS = DS_THREADS / 32;
// CTA = 32 rows (lane = row, each warp column load is one coalesced 256-byte segment) x the block's
// columns split over the 8 warps, then a fixed-order reduction of the 8 partial sums.
__global__ void __launch_bounds__(DS_THREADS) diag_block_gemv_kernel(int64_t j0, int64_t j1,
                                                                     const double* __restrict__ T, int64_t ldt,
                                                                     double* __restrict__ Z, int64_t ldz, int64_t k) {
  __shared__ double zq[DS_K][DS_B];
  __shared__ double red[DS_WARPS][DS_K][DS_ROWS];
  const int bs = (int)(j1 - j0);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t i = (int64_t)blockIdx.x * DS_ROWS + lane;
  for (int64_t c0 = 0; c0 < k; c0 += DS_K) {
    const int kc = (int)((k - c0) < DS_K ? (k - c0) : DS_K);
    for (int e = threadIdx.x; e < bs * kc; e += DS_THREADS) {
      const int q = e % bs, c = e / bs;
      zq[c][q] = Z[cm(j0 + q, c0 + c, ldz)] / T[cm(j0 + q, j0 + q, ldt)];
    }
    __syncthreads();
    double acc[DS_K];
#pragma unroll
    for (int c = 0; c < DS_K; ++c) acc[c] = 0.0;
    if (i < j0) {
      const double* Ti = T + cm(i, j0, ldt);
#pragma unroll 4
      for (int q = warp; q < bs; q += DS_WARPS) {
        const double t = __ldg(Ti + (size_t)q * ldt);
#pragma unroll
        for (int c = 0; c < DS_K; ++c)
          if (c < kc) acc[c] += t * zq[c][q];
      }
    }
#pragma unroll
    for (int c = 0; c < DS_K; ++c)
      if (c < kc) red[warp][c][lane] = acc[c];
    __syncthreads();
    if (warp == 0 && i < j0) {
      for (int c = 0; c < kc; ++c) {
        double sum = 0.0;
#pragma unroll
        for (int w = 0; w < DS_WARPS; ++w) sum += red[w][c][lane];
        Z[cm(i, c0 + c, ldz)] -= sum;
      }
    }
    __syncthreads();
  }
}

__global__ void diag_scale_kernel(int64_t r, int64_t k, const double* __restrict__ T, int64_t ldt, double* Z,
                                  int64_t ldz) {
  const int64_t total = r * k;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e % r, c = e / r;
    Z[cm(i, c, ldz)] /= T[cm(i, i, ldt)];
  }
}
}  // namespace

void launch_diag_block_solve(cudaStream_t st, int64_t r, int64_t b, const double* T, int64_t ldt, double* Z,
                             int64_t ldz, int64_t k) {
  if (r <= 0 || k <= 0) return;
  if (b > DS_B) throw CudaError{cudaErrorInvalidValue, "launch_diag_block_solve: b > 256", __LINE__};
  for (int64_t j0 = ((r - 1) / b) * b; j0 > 0; j0 -= b) {
    const int64_t j1 = std::min(r, j0 + b);
    ProfScope prof(st, kProfSolve, 1, 2.0 * (double)j0 * (j1 - j0) * k, 8.0 * (double)j0 * (j1 - j0) + 16.0 * j0 * k);
    diag_block_gemv_kernel<<<(unsigned)((j0 + DS_ROWS - 1) / DS_ROWS), DS_THREADS, 0, st>>>(j0, j1, T, ldt, Z, ldz,
                                                                                            k);
    UTV_CUDA(cudaGetLastError());
  }
  ProfScope prof(st, kProfSolve, 1, (double)r * k, 16.0 * (double)r * k + 8.0 * r);
  diag_scale_kernel<<<(unsigned)std::min<int64_t>((r * k + 255) / 256, 1024), 256, 0, st>>>(r, k, T, ldt, Z, ldz);
  UTV_CUDA(cudaGetLastError());
}

void launch_rank(cudaStream_t st, int64_t n, const double* T, int64_t ldt, double tau, int64_t* r_dev) {
  ProfScope prof(st, kProfSolve, 1, 0.0, 8.0 * (double)n);
  rank_kernel<<<1, 1024, 0, st>>>(n, T, ldt, tau, r_dev);
  UTV_CUDA(cudaGetLastError());
}

void launch_trsv_block(cudaStream_t st, int64_t j0, int64_t j1, const double* T, int64_t ldt, double* Z, int64_t ldz,
                       int64_t k) {
  if (j1 <= j0 || k <= 0) return;
  ProfScope prof(st, kProfSolve, 1, (double)(j1 - j0) * (j1 - j0) * k,
                 8.0 * (j1 - j0) * (j1 - j0) / 2 + 16.0 * (j1 - j0) * k);
  trsv_block_kernel<<<1, TS_ROWS, 0, st>>>(j0, j1, T, ldt, Z, ldz, k);
  UTV_CUDA(cudaGetLastError());
}

}  // namespace utv
