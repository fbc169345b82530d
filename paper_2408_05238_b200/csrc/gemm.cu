// gemm.cu -- FP64 tensor-core (DMMA) GEMM for sm_100a: C = alpha * op(A) op(B) + beta * C.
//
// This single kernel carries ~99% of randUTV's flops (SURVEY 8(a) a2, a4, a6 and the a7
// slab updates).  B200 has no FP64 kind of tcgen05.mma, so the FP64 tensor
// path is the warp-level `mma.sync.aligned.m16n8k4.row.col.f64` (SASS DMMA.8x8x4),
// measured at 37.2 TFLOP/s per GPU (profiles/r01_fp64_peaks.json).
//
// Design (B200-first):
//  * 128x128x16 CTA tile, 8 warps as 2 (M) x 4 (N), warp tile 64x32 = 4x4 m16n8 fragments,
//    64 FP64 accumulators per thread; 1 CTA / SM (register bound).
//  * Operands staged global->shared with 128-bit `cp.async.cg` (zero-fill for ragged edges)
//    in a 4-stage ring; the layout in shared memory follows the operand's contiguous
//    dimension (no transpose in flight): MN-major [BK][BMN+8], K-major [BMN][BK+4]; both
//    paddings make every fragment load exactly 2 wavefronts (conflict-free for LDS.64).
//  * Deterministic split-K for skinny outputs with long K (panel Gram/projection products):
//    partials to a workspace, reduced in a fixed order by dgemm_splitk_reduce.
#include "gemm.cuh"
#include "prof.cuh"

namespace utv {

namespace {

constexpr int BM = 128, BN = 128, BK = 16, STAGES = 4, THREADS = 256;
constexpr int LD_MN = BM + 8;          // MN-major tile: [BK][BM + 8]
constexpr int LD_K = BK + 4;           // K-major tile:  [BM][BK + 4]
constexpr int TILE_DBL = (BK * LD_MN > BM * LD_K) ? BK * LD_MN : BM * LD_K;  // 2560
constexpr int STAGE_DBL = 2 * TILE_DBL;
constexpr size_t SMEM_BYTES = (size_t)STAGES * STAGE_DBL * sizeof(double);  // 160 KiB

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}

template <int VEC>
__device__ __forceinline__ void cp_async(unsigned dst, const double* src, int src_bytes) {
  if constexpr (VEC == 2) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src), "r"(src_bytes));
  } else {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(dst), "l"(src), "r"(src_bytes));
  }
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

__device__ __forceinline__ void dmma_16x8x4(double (&d)[4], double a0, double a1, double b0) {
  asm volatile(
      "mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
      : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3])
      : "d"(a0), "d"(a1), "d"(b0));
}

// Load one 128 x 16 operand tile (rows along MN, columns along K) into shared memory.
// MN_MAJOR: element (mn, k) at ptr[mn + k*ld]; otherwise at ptr[k + mn*ld].
template <bool MN_MAJOR, int VEC>
__device__ __forceinline__ void load_tile(double* s, const double* __restrict__ g, int64_t ld, int64_t mn0,
                                          int64_t MN, int64_t k0, int64_t kend) {
  const int tid = threadIdx.x;
  if constexpr (MN_MAJOR) {
    constexpr int CPR = BM / VEC;               // chunks per k-row
    constexpr int NCH = BK * CPR;
#pragma unroll
    for (int c = tid; c < NCH; c += THREADS) {
      const int kk = c / CPR, mm = (c % CPR) * VEC;
      const int64_t gk = k0 + kk, gm = mn0 + mm;
      int64_t rem = MN - gm; int valid = (gk < kend && rem > 0) ? (int)(rem < VEC ? rem : VEC) : 0;
      const double* src = valid ? g + gm + gk * ld : g;
      cp_async<VEC>(smem_u32(s + kk * LD_MN + mm), src, valid * 8);
    }
  } else {
    constexpr int CPR = BK / VEC;
    constexpr int NCH = BM * CPR;
#pragma unroll
    for (int c = tid; c < NCH; c += THREADS) {
      const int mm = c / CPR, kk = (c % CPR) * VEC;
      const int64_t gk = k0 + kk, gm = mn0 + mm;
      int64_t rem = kend - gk; int valid = (gm < MN && rem > 0) ? (int)(rem < VEC ? rem : VEC) : 0;
      const double* src = valid ? g + gk + gm * ld : g;
      cp_async<VEC>(smem_u32(s + mm * LD_K + kk), src, valid * 8);
    }
  }
}

template <bool MN_MAJOR>
__device__ __forceinline__ double frag(const double* s, int mn, int k) {
  return MN_MAJOR ? s[k * LD_MN + mn] : s[mn * LD_K + k];
}

// A operand (m, k): TA=false -> A[m + k lda] (MN-major); TA=true -> A[k + m lda] (K-major).
// B operand (k, n): TB=false -> B[k + n ldb] (K-major);  TB=true -> B[n + k ldb] (MN-major).
template <bool TA, bool TB, int VEC>
__global__ void __launch_bounds__(THREADS, 1)
dgemm_dmma_kernel(int64_t M, int64_t N, int64_t K, double alpha, const double* __restrict__ A, int64_t lda,
                  const double* __restrict__ B, int64_t ldb, double beta, double* __restrict__ C, int64_t ldc,
                  int64_t k_chunk, double* __restrict__ partial) {
  extern __shared__ __align__(128) double smem[];
  constexpr bool A_MN = !TA;
  constexpr bool B_MN = TB;

  const int64_t n0 = (int64_t)blockIdx.x * BN;
  const int64_t m0 = (int64_t)blockIdx.y * BM;
  const int64_t kbeg = (int64_t)blockIdx.z * k_chunk;
  const int64_t kend = min(K, kbeg + k_chunk);
  const int nkt = (int)((kend - kbeg + BK - 1) / BK);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wm = warp >> 2, wn = warp & 3;       // 2 x 4 warps
  const int g = lane >> 2, t = lane & 3;

  double acc[4][4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int r = 0; r < 4; ++r) acc[i][j][r] = 0.0;

  auto stage_a = [&](int s) { return smem + s * STAGE_DBL; };
  auto stage_b = [&](int s) { return smem + s * STAGE_DBL + TILE_DBL; };

#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < nkt) {
      const int64_t k0 = kbeg + (int64_t)s * BK;
      load_tile<A_MN, VEC>(stage_a(s), A, lda, m0, M, k0, kend);
      load_tile<B_MN, VEC>(stage_b(s), B, ldb, n0, N, k0, kend);
    }
    cp_async_commit();
  }

  for (int kt = 0; kt < nkt; ++kt) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    {
      const int pf = kt + STAGES - 1;
      if (pf < nkt) {
        const int s = pf % STAGES;
        const int64_t k0 = kbeg + (int64_t)pf * BK;
        load_tile<A_MN, VEC>(stage_a(s), A, lda, m0, M, k0, kend);
        load_tile<B_MN, VEC>(stage_b(s), B, ldb, n0, N, k0, kend);
      }
      cp_async_commit();
    }
    const double* sa = stage_a(kt % STAGES);
    const double* sb = stage_b(kt % STAGES);
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      double af[4][2], bf[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int mr = wm * 64 + i * 16 + g;
        af[i][0] = frag<A_MN>(sa, mr, kk + t);
        af[i][1] = frag<A_MN>(sa, mr + 8, kk + t);
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) bf[j] = frag<B_MN>(sb, wn * 32 + j * 8 + g, kk + t);
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma_16x8x4(acc[i][j], af[i][0], af[i][1], bf[j]);
    }
  }
  cp_async_wait<0>();

  // Epilogue: fragment (i, j): rows m0+wm*64+i*16+g (+8), cols n0+wn*32+j*8+2t (+1).
  if (partial) {
    double* P = partial + (size_t)blockIdx.z * (size_t)M * (size_t)N;
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          const int64_t m = m0 + wm * 64 + i * 16 + g + (r >> 1) * 8;
          const int64_t n = n0 + wn * 32 + j * 8 + 2 * t + (r & 1);
          if (m < M && n < N) P[cm(m, n, M)] = acc[i][j][r];
        }
  } else {
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          const int64_t m = m0 + wm * 64 + i * 16 + g + (r >> 1) * 8;
          const int64_t n = n0 + wn * 32 + j * 8 + 2 * t + (r & 1);
          if (m < M && n < N) {
            double v = alpha * acc[i][j][r];
            if (beta != 0.0) v += beta * C[cm(m, n, ldc)];
            C[cm(m, n, ldc)] = v;
          }
        }
  }
}

// C = alpha * sum_{z=0}^{S-1} partial[z] + beta * C, summed in order z = 0..S-1.
__global__ void dgemm_splitk_reduce(int64_t M, int64_t N, int S, double alpha, const double* __restrict__ partial,
                                    double beta, double* __restrict__ C, int64_t ldc) {
  const int64_t total = M * N;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int z = 0; z < S; ++z) s += partial[(size_t)z * total + e];
    const int64_t m = e % M, n = e / M;
    double v = alpha * s;
    if (beta != 0.0) v += beta * C[cm(m, n, ldc)];
    C[cm(m, n, ldc)] = v;
  }
}

template <bool TA, bool TB, int VEC>
void launch_t(cudaStream_t st, int64_t M, int64_t N, int64_t K, double alpha, const double* A, int64_t lda,
              const double* B, int64_t ldb, double beta, double* C, int64_t ldc, int splits, int64_t kc,
              double* partial) {
  static bool attr_set = false;
  auto kern = dgemm_dmma_kernel<TA, TB, VEC>;
  if (!attr_set) {
    UTV_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM_BYTES));
    attr_set = true;
  }
  dim3 grid((unsigned)((N + BN - 1) / BN), (unsigned)((M + BM - 1) / BM), (unsigned)splits);
  kern<<<grid, THREADS, SMEM_BYTES, st>>>(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, kc, partial);
  UTV_CUDA(cudaGetLastError());
}

template <int VEC>
void dispatch(cudaStream_t st, bool ta, bool tb, int64_t M, int64_t N, int64_t K, double alpha, const double* A,
              int64_t lda, const double* B, int64_t ldb, double beta, double* C, int64_t ldc, int splits,
              int64_t kc, double* partial) {
  if (!ta && !tb) launch_t<false, false, VEC>(st, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, splits, kc, partial);
  else if (ta && !tb) launch_t<true, false, VEC>(st, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, splits, kc, partial);
  else if (!ta && tb) launch_t<false, true, VEC>(st, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, splits, kc, partial);
  else launch_t<true, true, VEC>(st, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, splits, kc, partial);
}

}  // namespace

int dgemm_split_count(int64_t M, int64_t N, int64_t K, int num_sms) {
  const int64_t tiles = ((M + BM - 1) / BM) * ((N + BN - 1) / BN);
  if (tiles >= num_sms || K < 4 * 256) return 1;
  int64_t s = (2 * (int64_t)num_sms + tiles - 1) / tiles;
  s = std::min<int64_t>(s, K / 256);                 // >= 256 deep per split
  s = std::min<int64_t>(s, 128);
  return (int)std::max<int64_t>(s, 1);
}

size_t dgemm_workspace_doubles(int64_t M, int64_t N, int64_t K, int num_sms) {
  int s = dgemm_split_count(M, N, K, num_sms);
  return s > 1 ? (size_t)s * (size_t)M * (size_t)N : 0;
}

void dgemm(cudaStream_t st, bool ta, bool tb, int64_t M, int64_t N, int64_t K, double alpha, const double* A,
           int64_t lda, const double* B, int64_t ldb, double beta, double* C, int64_t ldc, double* work,
           size_t work_doubles, int num_sms) {
  if (M <= 0 || N <= 0) return;
  if (K <= 0 || alpha == 0.0) {
    // C = beta * C (K == 0): reuse the reduce kernel with S = 0
    ProfScope prof(st, kProfMisc, 1, 0.0, 16.0 * (double)M * N);
    dgemm_splitk_reduce<<<std::max<int64_t>(1, std::min<int64_t>((M * N + 255) / 256, 4096)), 256, 0, st>>>(
        M, N, 0, 0.0, nullptr, beta, C, ldc);
    UTV_CUDA(cudaGetLastError());
    return;
  }
  const bool aligned = ((reinterpret_cast<uintptr_t>(A) | reinterpret_cast<uintptr_t>(B)) % 16 == 0) &&
                       (lda % 2 == 0) && (ldb % 2 == 0);
  int splits = dgemm_split_count(M, N, K, num_sms);
  if (splits > 1 && (size_t)splits * (size_t)M * (size_t)N > work_doubles) {
    splits = (int)std::max<size_t>(1, work_doubles / ((size_t)M * (size_t)N));
  }
  int64_t kc = K;
  if (splits > 1) {
    kc = ((K + splits - 1) / splits + BK - 1) / BK * BK;
    splits = (int)((K + kc - 1) / kc);
  }
  double* partial = splits > 1 ? work : nullptr;
  ProfScope prof(st, kProfGemm, splits > 1 ? 2 : 1, 2.0 * (double)M * (double)N * (double)K,
                 8.0 * ((double)M * K + (double)K * N + (double)M * N * (beta != 0.0 ? 2.0 : 1.0)));
  if (aligned)
    dispatch<2>(st, ta, tb, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, splits, kc, partial);
  else
    dispatch<1>(st, ta, tb, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, splits, kc, partial);
  if (splits > 1) {
    const int64_t total = M * N;
    int blocks = (int)std::min<int64_t>((total + 255) / 256, 8 * (int64_t)num_sms);
    dgemm_splitk_reduce<<<blocks, 256, 0, st>>>(M, N, splits, alpha, partial, beta, C, ldc);
    UTV_CUDA(cudaGetLastError());
  }
}

}  // namespace utv
