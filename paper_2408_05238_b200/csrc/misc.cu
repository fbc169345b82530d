// misc.cu -- elementwise helpers (identity init, zeroing, copies, finiteness guard).
// All HBM-bound grid-stride kernels over column-major matrices.
#include "kernels.cuh"
#include "prof.cuh"

namespace utv {

namespace {
__global__ void set_identity_kernel(int64_t rows, int64_t cols, double* A, int64_t lda) {
  const int64_t total = rows * cols;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e % rows, j = e / rows;
    A[cm(i, j, lda)] = i == j ? 1.0 : 0.0;
  }
}
__global__ void set_zero_kernel(int64_t rows, int64_t cols, double* A, int64_t lda) {
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
  set_zero_kernel<<<grid_for(rows * cols), 256, 0, st>>>(rows, cols, A, lda);
  UTV_CUDA(cudaGetLastError());
}
void launch_set_diag(cudaStream_t st, int64_t bw, const double* sigma, double* A, int64_t lda) {
  if (bw <= 0) return;
  ProfScope prof(st, kProfMisc, 1, 0.0, 8.0 * (double)(bw * bw));
  set_diag_kernel<<<grid_for(bw * bw), 256, 0, st>>>(bw, sigma, A, lda);
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
