// misc.cu -- elementwise helpers (identity init, zeroing, copies, finiteness guard).
// All HBM-bound grid-stride kernels over column-major matrices.
#include "kernels.cuh"
#include "prof.cuh"

namespace utv {

namespace {
thread_local Pred t_pred{nullptr, 0};
}  // namespace
Pred launch_pred() { return t_pred; }
PredScope::PredScope(const int* flag, int want) : old(t_pred) { t_pred = Pred{flag, want}; }
PredScope::~PredScope() { t_pred = old; }

namespace {
__global__ void set_identity_kernel(int64_t rows, int64_t cols, double* A, int64_t lda) {
  const int64_t total = rows * cols;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e % rows, j = e / rows;
    A[cm(i, j, lda)] = i == j ? 1.0 : 0.0;
  }
}
__global__ void set_zero_kernel(int64_t rows, int64_t cols, double* A, int64_t lda, Pred pr) {
  if (pred_skip(pr)) return;
  const int64_t total = rows * cols;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e % rows, j = e / rows;
    A[cm(i, j, lda)] = 0.0;
  }
}
__global__ void set_diag_kernel(int64_t bw, const double* sigma, double* A, int64_t lda) {
  const int64_t total = bw * bw;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e % bw, j = e / bw;
    A[cm(i, j, lda)] = i == j ? sigma[i] : 0.0;
  }
}
__global__ void copy_kernel(int64_t rows, int64_t cols, const double* __restrict__ S, int64_t lds, double* __restrict__ D,
                            int64_t ldd) {
  const int64_t total = rows * cols;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e % rows, j = e / rows;
    D[cm(i, j, ldd)] = S[cm(i, j, lds)];
  }
}
__global__ void zero_strict_lower_kernel(int64_t rows, int64_t cols, double* A, int64_t lda) {
  const int64_t total = rows * cols;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e % rows, j = e / rows;
    if (i > j) A[cm(i, j, lda)] = 0.0;
  }
}
__global__ void check_finite_kernel(int64_t rows, int64_t cols, const double* __restrict__ A, int64_t lda, int* flag) {
  const int64_t total = rows * cols;
  int bad = 0;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e % rows, j = e / rows;
    bad |= !isfinite(A[cm(i, j, lda)]);
  }
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(flag, 1);
}
int grid_for(int64_t total) { return (int)std::max<int64_t>(1, std::min<int64_t>((total + 255) / 256, 148 * 16)); }
}  // namespace

void launch_set_identity(cudaStream_t st, int64_t rows, int64_t cols, double* A, int64_t lda) {
  if (rows * cols <= 0) return;
  ProfScope prof(st, kProfMisc, 1, 0.0, 8.0 * (double)(rows * cols));
  set_identity_kernel<<<grid_for(rows * cols), 256, 0, st>>>(rows, cols, A, lda);
  UTV_CUDA(cudaGetLastError());
}
void launch_set_zero(cudaStream_t st, int64_t rows, int64_t cols, double* A, int64_t lda) {
  if (rows * cols <= 0) return;
  ProfScope prof(st, kProfMisc, 1, 0.0, 8.0 * (double)(rows * cols));
  set_zero_kernel<<<grid_for(rows * cols), 256, 0, st>>>(rows, cols, A, lda, launch_pred());
  UTV_CUDA(cudaGetLastError());
}
void launch_set_diag(cudaStream_t st, int64_t bw, const double* sigma, double* A, int64_t lda) {
  if (bw <= 0) return;
  ProfScope prof(st, kProfMisc, 1, 0.0, 8.0 * (double)(bw * bw));
  set_diag_kernel<<<grid_for(bw * bw), 256, 0, st>>>(bw, sigma, A, lda);
  UTV_CUDA(cudaGetLastError());
}
__global__ void axpy_kernel(int64_t n, double alpha, const double* __restrict__ x, double* __restrict__ y) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x)
    y[e] += alpha * x[e];
}
// Multi-GPU layout helpers (block-cyclic columns, block b, owner(blk) = blk mod P).
// assemble_y: Y (np x cols, ldy) in global block order from the all-gathered per-rank row blocks
// (rank o's trailing blocks, packed, at recv + o*Lmax*cols with ld Lmax): global block u = blk - i
// comes from rank (i+u) mod P, where it is trailing block number u / P.
__global__ void assemble_y_kernel(int64_t np, int64_t cols, int64_t b, int64_t i, int P, int64_t Lmax,
                                  const double* __restrict__ recv, double* __restrict__ Y, int64_t ldy) {
  const int64_t total = np * cols;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = e % np, c = e / np;
    const int64_t u = row / b, rr = row % b;
    const int64_t o = (i + u) % P, t = u / P;
    Y[cm(row, c, ldy)] = recv[o * Lmax * cols + cm(t * b + rr, c, Lmax)];
  }
}
// gather_local: the rows of W (np x cols, global trailing order from block i) that belong to rank p's
// trailing blocks, packed: local trailing block t is global block u = ((p - i) mod P) + t P.
__global__ void gather_local_kernel(int64_t nloc, int64_t cols, int64_t b, int64_t i, int P, int p,
                                    const double* __restrict__ W, int64_t ldw, double* __restrict__ D, int64_t ldd) {
  const int64_t total = nloc * cols;
  const int64_t u0 = (((int64_t)p - i) % P + P) % P;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = e % nloc, c = e / nloc;
    const int64_t t = row / b, rr = row % b;
    D[cm(row, c, ldd)] = W[cm((u0 + t * P) * b + rr, c, ldw)];
  }
}

void launch_axpy(cudaStream_t st, int64_t n, double alpha, const double* x, double* y) {
  if (n <= 0) return;
  ProfScope prof(st, kProfMisc, 1, 2.0 * (double)n, 24.0 * (double)n);
  axpy_kernel<<<grid_for(n), 256, 0, st>>>(n, alpha, x, y);
  UTV_CUDA(cudaGetLastError());
}
void launch_assemble_y(cudaStream_t st, int64_t np, int64_t cols, int64_t b, int64_t i, int P, int64_t Lmax,
                       const double* recv, double* Y, int64_t ldy) {
  if (np * cols <= 0) return;
  ProfScope prof(st, kProfMisc, 1, 0.0, 16.0 * (double)(np * cols));
  assemble_y_kernel<<<grid_for(np * cols), 256, 0, st>>>(np, cols, b, i, P, Lmax, recv, Y, ldy);
  UTV_CUDA(cudaGetLastError());
}
void launch_gather_local(cudaStream_t st, int64_t nloc, int64_t cols, int64_t b, int64_t i, int P, int p,
                         const double* W, int64_t ldw, double* D, int64_t ldd) {
  if (nloc * cols <= 0) return;
  ProfScope prof(st, kProfMisc, 1, 0.0, 16.0 * (double)(nloc * cols));
  gather_local_kernel<<<grid_for(nloc * cols), 256, 0, st>>>(nloc, cols, b, i, P, p, W, ldw, D, ldd);
  UTV_CUDA(cudaGetLastError());
}

void launch_copy(cudaStream_t st, int64_t rows, int64_t cols, const double* src, int64_t lds, double* dst, int64_t ldd) {
  if (rows * cols <= 0) return;
  ProfScope prof(st, kProfMisc, 1, 0.0, 8.0 * (double)(rows * cols));
  copy_kernel<<<grid_for(rows * cols), 256, 0, st>>>(rows, cols, src, lds, dst, ldd);
  UTV_CUDA(cudaGetLastError());
}
void launch_zero_strict_lower(cudaStream_t st, int64_t rows, int64_t cols, double* A, int64_t lda) {
  if (rows * cols <= 0) return;
  ProfScope prof(st, kProfMisc, 1, 0.0, 8.0 * (double)(rows * cols));
  zero_strict_lower_kernel<<<grid_for(rows * cols), 256, 0, st>>>(rows, cols, A, lda);
  UTV_CUDA(cudaGetLastError());
}
void launch_check_finite(cudaStream_t st, int64_t rows, int64_t cols, const double* A, int64_t lda, int* flag) {
  if (rows * cols <= 0) return;
  ProfScope prof(st, kProfMisc, 1, 0.0, 8.0 * (double)(rows * cols));
  check_finite_kernel<<<grid_for(rows * cols), 256, 0, st>>>(rows, cols, A, lda, flag);
  UTV_CUDA(cudaGetLastError());
}

}  // namespace utv

// ---- Nullify_top_right_part_of_T helpers ----------------------------------
// The RZ factorization of a row slab S = [L | D] (L = T(i0:i0+bw, i0:i0+bw) upper triangular,
// D = T(i0:i0+bw, r:n)) from the right is a Householder QR of
//   M = diag(J, I) S^T J     (J = exchange matrix),
// whose top bw x bw block is upper triangular, so each reflector touches exactly one top row and
// the D rows: the RZ structure.  S C = [J R^T J, 0] with C = I - W' T W'^T, W' = diag(J, I) W.
namespace utv {
namespace {
__global__ void rz_build_kernel(int64_t bw, int64_t nz, const double* __restrict__ T, int64_t ldt, int64_t i0,
                                int64_t r, double* __restrict__ M, int64_t ldm) {
  const int64_t rows = bw + nz, total = rows * bw;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = e % rows, q = e / rows;
    const int64_t srow = i0 + bw - 1 - q;
    M[cm(p, q, ldm)] = p < bw ? T[cm(srow, i0 + bw - 1 - p, ldt)] : T[cm(srow, r + (p - bw), ldt)];
  }
}
// T(i0:i0+bw, i0:i0+bw) = J R^T J (R = upper bw x bw of M), T(i0:i0+bw, r:n) = 0
__global__ void rz_writeback_kernel(int64_t bw, int64_t nz, const double* __restrict__ M, int64_t ldm,
                                    double* __restrict__ T, int64_t ldt, int64_t i0, int64_t r) {
  const int64_t total = bw * (bw + nz);
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t a = e % bw, c = e / bw;
    if (c < bw) {
      const int64_t pr = bw - 1 - c, pc = bw - 1 - a;      // R(pr, pc), upper: pr <= pc  <=>  a <= c
      T[cm(i0 + a, i0 + c, ldt)] = pr <= pc ? M[cm(pr, pc, ldm)] : 0.0;
    } else {
      T[cm(i0 + a, r + (c - bw), ldt)] = 0.0;
    }
  }
}
// dst (bw x bw) = J * src(0:bw, 0:bw)  (row reversal of the top block of W)
__global__ void reverse_rows_kernel(int64_t bw, const double* __restrict__ src, int64_t lds, double* __restrict__ dst,
                                    int64_t ldd) {
  const int64_t total = bw * bw;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = e % bw, q = e / bw;
    dst[cm(p, q, ldd)] = src[cm(bw - 1 - p, q, lds)];
  }
}
int grid_for2(int64_t total) { return (int)std::max<int64_t>(1, std::min<int64_t>((total + 255) / 256, 148 * 16)); }
}  // namespace

void launch_rz_build(cudaStream_t st, int64_t bw, int64_t nz, const double* T, int64_t ldt, int64_t i0, int64_t r,
                     double* M, int64_t ldm) {
  ProfScope prof(st, kProfMisc, 1, 0.0, 16.0 * (double)bw * (bw + nz));
  rz_build_kernel<<<grid_for2(bw * (bw + nz)), 256, 0, st>>>(bw, nz, T, ldt, i0, r, M, ldm);
  UTV_CUDA(cudaGetLastError());
}
void launch_rz_writeback(cudaStream_t st, int64_t bw, int64_t nz, const double* M, int64_t ldm, double* T,
                         int64_t ldt, int64_t i0, int64_t r) {
  ProfScope prof(st, kProfMisc, 1, 0.0, 16.0 * (double)bw * (bw + nz));
  rz_writeback_kernel<<<grid_for2(bw * (bw + nz)), 256, 0, st>>>(bw, nz, M, ldm, T, ldt, i0, r);
  UTV_CUDA(cudaGetLastError());
}
void launch_reverse_rows(cudaStream_t st, int64_t bw, const double* src, int64_t lds, double* dst, int64_t ldd) {
  ProfScope prof(st, kProfMisc, 1, 0.0, 16.0 * (double)bw * bw);
  reverse_rows_kernel<<<grid_for2(bw * bw), 256, 0, st>>>(bw, src, lds, dst, ldd);
  UTV_CUDA(cudaGetLastError());
}
}  // namespace utv

// ---- Wide least squares (m < n, reading R21) ------------------------------
// A^T through a 32 x 33 shared-memory tile: coalesced column reads of A and column writes of A^T.
namespace utv {
namespace {
constexpr int kTr = 32;
__global__ void transpose_kernel(int64_t rows, int64_t cols, const double* __restrict__ src, int64_t lds,
                                 double* __restrict__ dst, int64_t ldd) {
  __shared__ double tile[kTr][kTr + 1];
  const int64_t r0 = (int64_t)blockIdx.x * kTr, c0 = (int64_t)blockIdx.y * kTr;
  for (int j = threadIdx.y; j < kTr; j += blockDim.y) {               // src column c0 + j
    const int64_t r = r0 + threadIdx.x, c = c0 + j;
    if (r < rows && c < cols) tile[j][threadIdx.x] = src[cm(r, c, lds)];
  }
  __syncthreads();
  for (int j = threadIdx.y; j < kTr; j += blockDim.y) {               // dst column r0 + j = src row r0 + j
    const int64_t dr = c0 + threadIdx.x, dc = r0 + j;
    if (dr < cols && dc < rows) dst[cm(dr, dc, ldd)] = tile[threadIdx.x][j];
  }
}
// mode 0: dst = J src (rows reversed); mode 1: dst = src J (columns reversed);
// mode 2 (square, rows == cols): dst = J src^T J restricted to its upper triangle (0 below), i.e.
// the upper-triangular form of the lower-triangular src^T when src is upper triangular.
__global__ void permute_kernel(int mode, int64_t rows, int64_t cols, const double* __restrict__ src, int64_t lds,
                               double* __restrict__ dst, int64_t ldd) {
  const int64_t total = rows * cols;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e % rows, j = e / rows;
    double v;
    if (mode == 0) v = src[cm(rows - 1 - i, j, lds)];
    else if (mode == 1) v = src[cm(i, cols - 1 - j, lds)];
    else v = i <= j ? src[cm(rows - 1 - j, rows - 1 - i, lds)] : 0.0;
    dst[cm(i, j, ldd)] = v;
  }
}
}  // namespace

void launch_transpose(cudaStream_t st, int64_t rows, int64_t cols, const double* src, int64_t lds, double* dst,
                      int64_t ldd) {
  if (rows * cols <= 0) return;
  ProfScope prof(st, kProfMisc, 1, 0.0, 16.0 * (double)(rows * cols));
  const dim3 grid((unsigned)((rows + kTr - 1) / kTr), (unsigned)((cols + kTr - 1) / kTr));
  transpose_kernel<<<grid, dim3(kTr, 8), 0, st>>>(rows, cols, src, lds, dst, ldd);
  UTV_CUDA(cudaGetLastError());
}
void launch_permute(cudaStream_t st, int mode, int64_t rows, int64_t cols, const double* src, int64_t lds, double* dst,
                    int64_t ldd) {
  if (rows * cols <= 0) return;
  ProfScope prof(st, kProfMisc, 1, 0.0, 16.0 * (double)(rows * cols));
  permute_kernel<<<grid_for2(rows * cols), 256, 0, st>>>(mode, rows, cols, src, lds, dst, ldd);
  UTV_CUDA(cudaGetLastError());
}
}  // namespace utv
