// gemm.cu -- FP64 tensor-core (DMMA) GEMM for sm_100a: C = alpha * op(A) op(B) + beta * C.
//
// This single kernel carries ~97% of randUTV's executed flops (SURVEY 8(a) a2, a4, a6 and the a7
// slab updates).  B200 has no FP64 kind of tcgen05.mma, so the FP64 tensor
// path is the warp-level `mma.sync.aligned.m16n8k4.row.col.f64` (SASS DMMA.8x8x4),
// measured at 37.2 TFLOP/s per GPU (profiles/r01_fp64_peaks.json).
//
// Design (B200-first):
//  * CTA tile BM x BN x 16 (Shape<> table: 128x128 / 1 CTA per SM for long K, 128x64 / 2 per SM
//    for short K), warp tile (16 MI) x (8 NJ) m16n8 fragments, 64 FP64 accumulators per thread.
//  * Default path (dgemm_tma_kernel): operand tiles staged by TMA (cp.async.bulk.tensor, one
//    elected thread, completion on a per-stage mbarrier) into a 6-stage (4 at 2 CTAs/SM) ring;
//    K-major tiles use the 128-byte swizzle, MN-major tiles a rank-3 map whose box lands as
//    [mn/8][k][8] -- both make every fragment LDS.64 exactly 2 wavefronts.  Slots are released
//    per warp on "empty" mbarriers (no CTA-wide barrier in the main loop).
//  * Fallback (dgemm_dmma_kernel, 8-byte aligned operands / odd leading dimensions): the same
//    tiles staged with cp.async (zero-fill for ragged edges), padded layouts MN-major
//    [BK][BMN+8] and K-major [BMN][BK+4].
//  * Deterministic split-K for skinny outputs with long K (panel Gram/projection products):
//    partials to a workspace, reduced in a fixed order by dgemm_splitk_reduce.
#include "gemm.cuh"
#include "prof.cuh"
#include <cuda.h>            // CUtensorMap (type only; the encoder is fetched from the driver at run time)
#include <cmath>
#include <cstdlib>
#include <mutex>

namespace utv {

namespace {

constexpr int BK = 16;
constexpr int LD_K = BK + 4;           // K-major tile row: [BMN][BK + 4]

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

// Shared-memory footprint (doubles) of one BMN x BK operand tile.
template <int BMN, bool MN_MAJOR>
constexpr int tile_doubles() { return MN_MAJOR ? BK * (BMN + 8) : BMN * LD_K; }

// Tile configurations: CTA tile BM x BN, WM x WN warps, warp tile (16 MI) x (8 NJ), MI*NJ*4 = 64
// FP64 accumulators per thread.
//   0: 128 x 128, 2 x 4 warps of 64 x 32, 256 threads, 1 CTA / SM   (long K)
//   1: 128 x  64, 2 x 2 warps of 64 x 32, 128 threads, 2 CTAs / SM  (short K: one CTA's epilogue
//      overlaps the other's main loop)
//   2: 128 x 128, 4 x 2 warps of 32 x 64, 256 threads, 1 CTA / SM
//   3:  64 x 128, 2 x 2 warps of 32 x 64, 128 threads, 2 CTAs / SM
//   4: 128 x  32, 4 x 1 warps of 32 x 32, 128 threads, 3 CTAs / SM  (N <= 32: the panel's
//      P_r^T W products and the few-RHS updates, which would waste most of a 64/128-wide tile)
//   5:  64 x  64, 2 x 2 warps of 32 x 32, 128 threads, 3 CTAs / SM  (short K, the default: with 12
//      warps per SM two CTAs keep the DMMA pipe busy through the third one's epilogue; K = 512
//      update 34.1 -> 34.6 TF/s, K = 256 32.8 -> 33.8 vs config 1; 4 CTAs / SM was worse)
template <int ID> struct Shape;
template <> struct Shape<0> { static constexpr int BM = 128, WM = 2, WN = 4, MI = 4, NJ = 4, CTAS = 1; };
template <> struct Shape<1> { static constexpr int BM = 128, WM = 2, WN = 2, MI = 4, NJ = 4, CTAS = 2; };
template <> struct Shape<2> { static constexpr int BM = 128, WM = 4, WN = 2, MI = 2, NJ = 8, CTAS = 1; };
template <> struct Shape<3> { static constexpr int BM = 64, WM = 2, WN = 2, MI = 2, NJ = 8, CTAS = 2; };
template <> struct Shape<4> { static constexpr int BM = 128, WM = 4, WN = 1, MI = 2, NJ = 4, CTAS = 3; };
template <> struct Shape<5> { static constexpr int BM = 64, WM = 2, WN = 2, MI = 2, NJ = 4, CTAS = 3; };
constexpr int kNumShapes = 6;
constexpr int kNarrowCfg = 4;
__host__ __device__ constexpr int shape_bm(int id) { return (id == 3 || id == 5) ? 64 : 128; }
__host__ __device__ constexpr int shape_bn(int id) { return (id == 1 || id == 5) ? 64 : (id == 4 ? 32 : 128); }
__host__ __device__ constexpr int shape_ctas(int id) { return (id == 4 || id == 5) ? 3 : ((id == 1 || id == 3) ? 2 : 1); }
__host__ __device__ constexpr int smem_budget_kb(int ctas) { return ctas == 1 ? 200 : (ctas == 2 ? 108 : 72); }

template <bool TA, bool TB, int ID>
struct Cfg {
  static constexpr int BM = Shape<ID>::BM, WM = Shape<ID>::WM, WN = Shape<ID>::WN;
  static constexpr int MI = Shape<ID>::MI, NJ = Shape<ID>::NJ;
  static_assert(16 * MI * WM == BM, "warp tiles must cover BM");
  static constexpr int BN = 8 * NJ * WN;
  static_assert(BM == shape_bm(ID) && BN == shape_bn(ID), "shape table out of sync");
  static constexpr int THREADS = 32 * WM * WN;
  static constexpr bool A_MN = !TA, B_MN = TB;
  static constexpr int A_DBL = tile_doubles<BM, A_MN>();
  static constexpr int B_DBL = tile_doubles<BN, B_MN>();
  static constexpr int STAGE_DBL = A_DBL + B_DBL;
  static constexpr int CTAS_PER_SM = Shape<ID>::CTAS;
  static constexpr int SMEM_BUDGET = smem_budget_kb(CTAS_PER_SM) * 1024;
  static constexpr int STAGES_FIT = SMEM_BUDGET / (STAGE_DBL * 8);
  static constexpr int STAGES = STAGES_FIT > 4 ? 4 : STAGES_FIT;
  static constexpr size_t SMEM = (size_t)STAGES * STAGE_DBL * sizeof(double);
  static_assert(STAGES >= 3, "not enough shared memory for a 3-stage pipeline");
};

// Load one BMN x 16 operand tile (rows along MN, columns along K) into shared memory.
// MN_MAJOR: element (mn, k) at ptr[mn + k*ld]; otherwise at ptr[k + mn*ld].
template <int BMN, bool MN_MAJOR, int VEC, int THREADS>
__device__ __forceinline__ void load_tile(double* s, const double* __restrict__ g, int64_t ld, int64_t mn0,
                                          int64_t MN, int64_t k0, int64_t kend) {
  const int tid = threadIdx.x;
  if constexpr (MN_MAJOR) {
    constexpr int CPR = BMN / VEC;              // chunks per k-row
    constexpr int NCH = BK * CPR;
#pragma unroll
    for (int c = tid; c < NCH; c += THREADS) {
      const int kk = c / CPR, mm = (c % CPR) * VEC;
      const int64_t gk = k0 + kk, gm = mn0 + mm;
      int64_t rem = MN - gm; int valid = (gk < kend && rem > 0) ? (int)(rem < VEC ? rem : VEC) : 0;
      const double* src = valid ? g + gm + gk * ld : g;
      cp_async<VEC>(smem_u32(s + kk * (BMN + 8) + mm), src, valid * 8);
    }
  } else {
    constexpr int CPR = BK / VEC;
    constexpr int NCH = BMN * CPR;
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

template <int BMN, bool MN_MAJOR>
__device__ __forceinline__ double frag(const double* s, int mn, int k) {
  return MN_MAJOR ? s[k * (BMN + 8) + mn] : s[mn * LD_K + k];
}

// A operand (m, k): TA=false -> A[m + k lda] (MN-major); TA=true -> A[k + m lda] (K-major).
// B operand (k, n): TB=false -> B[k + n ldb] (K-major);  TB=true -> B[n + k ldb] (MN-major).
template <bool TA, bool TB, int VEC, int ID>
__global__ void __launch_bounds__(Cfg<TA, TB, ID>::THREADS, Cfg<TA, TB, ID>::CTAS_PER_SM)
dgemm_dmma_kernel(int64_t M, int64_t N, int64_t K, double alpha, const double* __restrict__ A, int64_t lda,
                  const double* __restrict__ B, int64_t ldb, double beta, double* __restrict__ C, int64_t ldc,
                  int64_t k_chunk, double* __restrict__ partial, Pred pr) {
  if (pred_skip(pr)) return;
  using CF = Cfg<TA, TB, ID>;
  constexpr int BM = CF::BM, BN = CF::BN, THREADS = CF::THREADS, STAGES = CF::STAGES;
  constexpr int WN = CF::WN, MI = CF::MI, NJ = CF::NJ, WTM = 16 * MI, WTN = 8 * NJ;
  constexpr bool A_MN = CF::A_MN, B_MN = CF::B_MN;
  extern __shared__ __align__(128) double smem[];

  // Grouped rasterisation: consecutive CTAs walk GROUP_M tile-rows x all tile-columns in
  // column order, so the CTAs resident at one time share a few MB of A and B rows in L2
  // (a plain row-major order re-streams the whole B operand from HBM for every tile-row).
  const int64_t tiles_m = (M + BM - 1) / BM, tiles_n = (N + BN - 1) / BN;
  constexpr int64_t GROUP_M = 16;
  const int64_t pid = blockIdx.x;
  const int64_t per_group = GROUP_M * tiles_n;
  const int64_t first_m = (pid / per_group) * GROUP_M;
  const int64_t gsz = min(tiles_m - first_m, GROUP_M);
  const int64_t m0 = (first_m + (pid % per_group) % gsz) * BM;
  const int64_t n0 = ((pid % per_group) / gsz) * BN;
  const int64_t kbeg = (int64_t)blockIdx.z * k_chunk;
  const int64_t kend = min(K, kbeg + k_chunk);
  const int nkt = (int)((kend - kbeg + BK - 1) / BK);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wm = warp / WN, wn = warp % WN;      // WM x WN warps
  const int g = lane >> 2, t = lane & 3;

  double acc[MI][NJ][4];
#pragma unroll
  for (int i = 0; i < MI; ++i)
#pragma unroll
    for (int j = 0; j < NJ; ++j)
#pragma unroll
      for (int r = 0; r < 4; ++r) acc[i][j][r] = 0.0;

  auto stage_a = [&](int s) { return smem + s * CF::STAGE_DBL; };
  auto stage_b = [&](int s) { return smem + s * CF::STAGE_DBL + CF::A_DBL; };

#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < nkt) {
      const int64_t k0 = kbeg + (int64_t)s * BK;
      load_tile<BM, A_MN, VEC, THREADS>(stage_a(s), A, lda, m0, M, k0, kend);
      load_tile<BN, B_MN, VEC, THREADS>(stage_b(s), B, ldb, n0, N, k0, kend);
    }
    cp_async_commit();
  }

  // Software pipeline: the fragments of k-step s+1 are loaded (LDS) while the DMMAs of step s
  // run (register double buffer), and the barrier that publishes the next stage is taken
  // before the last k-step of the current one, so its latency overlaps 16 DMMAs.
  double af[2][MI][2], bf[2][NJ];
  auto load_frags = [&](int buf, const double* sa, const double* sb, int kk) {
#pragma unroll
    for (int i = 0; i < MI; ++i) {
      const int mr = wm * WTM + i * 16 + g;
      af[buf][i][0] = frag<BM, A_MN>(sa, mr, kk + t);
      af[buf][i][1] = frag<BM, A_MN>(sa, mr + 8, kk + t);
    }
#pragma unroll
    for (int j = 0; j < NJ; ++j) bf[buf][j] = frag<BN, B_MN>(sb, wn * WTN + j * 8 + g, kk + t);
  };

  cp_async_wait<STAGES - 2>();
  __syncthreads();
  if (nkt > 0) load_frags(0, stage_a(0), stage_b(0), 0);

  for (int kt = 0; kt < nkt; ++kt) {
    const double* sa = stage_a(kt % STAGES);
    const double* sb = stage_b(kt % STAGES);
#pragma unroll
    for (int ks = 0; ks < BK / 4; ++ks) {
      const int cur = ks & 1;
      if (ks == BK / 4 - 1) {
        // stage kt+1 must be visible to every warp; stage kt-1 has been fully read
        cp_async_wait<STAGES - 3 >= 0 ? STAGES - 3 : 0>();
        __syncthreads();
        const int pf = kt + STAGES - 1;
        if (pf < nkt) {
          const int s = pf % STAGES;
          const int64_t k0 = kbeg + (int64_t)pf * BK;
          load_tile<BM, A_MN, VEC, THREADS>(stage_a(s), A, lda, m0, M, k0, kend);
          load_tile<BN, B_MN, VEC, THREADS>(stage_b(s), B, ldb, n0, N, k0, kend);
        }
        cp_async_commit();
        if (kt + 1 < nkt) load_frags(cur ^ 1, stage_a((kt + 1) % STAGES), stage_b((kt + 1) % STAGES), 0);
      } else {
        load_frags(cur ^ 1, sa, sb, (ks + 1) * 4);
      }
#pragma unroll
      for (int i = 0; i < MI; ++i)
#pragma unroll
        for (int j = 0; j < NJ; ++j) dmma_16x8x4(acc[i][j], af[cur][i][0], af[cur][i][1], bf[cur][j]);
    }
  }
  cp_async_wait<0>();

  // Epilogue: fragment (i, j): rows m0+wm*WTM+i*16+g (+8), cols n0+wn*32+j*8+2t (+1).
  if (partial) {
    double* P = partial + (size_t)blockIdx.z * (size_t)M * (size_t)N;
#pragma unroll
    for (int i = 0; i < MI; ++i)
#pragma unroll
      for (int j = 0; j < NJ; ++j)
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          const int64_t m = m0 + wm * WTM + i * 16 + g + (r >> 1) * 8;
          const int64_t n = n0 + wn * WTN + j * 8 + 2 * t + (r & 1);
          if (m < M && n < N) P[cm(m, n, M)] = acc[i][j][r];
        }
  } else {
    if (beta != 0.0) {
      // batch the C loads first (memory-level parallelism), then combine and store
#pragma unroll
      for (int i = 0; i < MI; ++i)
#pragma unroll
        for (int j = 0; j < NJ; ++j)
#pragma unroll
          for (int r = 0; r < 4; ++r) {
            const int64_t m = m0 + wm * WTM + i * 16 + g + (r >> 1) * 8;
            const int64_t n = n0 + wn * WTN + j * 8 + 2 * t + (r & 1);
            const double c = (m < M && n < N) ? __ldg(C + cm(m, n, ldc)) : 0.0;
            acc[i][j][r] = alpha * acc[i][j][r] + beta * c;
          }
    } else {
#pragma unroll
      for (int i = 0; i < MI; ++i)
#pragma unroll
        for (int j = 0; j < NJ; ++j)
#pragma unroll
          for (int r = 0; r < 4; ++r) acc[i][j][r] *= alpha;
    }
#pragma unroll
    for (int i = 0; i < MI; ++i)
#pragma unroll
      for (int j = 0; j < NJ; ++j)
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          const int64_t m = m0 + wm * WTM + i * 16 + g + (r >> 1) * 8;
          const int64_t n = n0 + wn * WTN + j * 8 + 2 * t + (r & 1);
          if (m < M && n < N) C[cm(m, n, ldc)] = acc[i][j][r];
        }
  }
}

// ------------------------------------------------------------------------------------------
// TMA-fed variant (the default for 16-byte aligned operands with even leading dimensions).
// One elected thread issues the bulk-tensor copies of a whole k-tile (cp.async.bulk.tensor,
// completion counted on a per-stage mbarrier), so the warps spend their issue slots on LDS +
// DMMA only (the cp.async path spends ~60 integer instructions per 16-byte chunk on addresses).
// Shared-memory layouts, chosen so every fragment LDS.64 is exactly 2 wavefronts:
//  * K-major operand: one box {16 k, BMN rows} with SWIZZLE_128B: element (mn, k) at byte
//    mn*128 + (((k>>1) ^ (mn&7)) << 4) + (k&1)*8.  A fragment reads 8 rows (g) x 4 k (t): the
//    swizzle spreads the 8 rows over all 8 16-byte chunks.
//  * MN-major operand: BMN/8 boxes {8 mn, 16 k} (no swizzle): element (mn, k) at byte
//    (mn>>3)*1024 + k*64 + (mn&7)*8.  A fragment reads 4 k rows (t) x 8 mn (g) of 64 B.
// At the CTA barrier of k-tile kt the slot of k-tile kt-1 is refilled with k-tile kt+STAGES-1
// (STAGES-1 tiles in flight).  TMA zero-fills out-of-bounds boxes (ragged M/N/K).
// ------------------------------------------------------------------------------------------
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];\n"
      ::"r"(smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}

__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1,
                                            int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];\n"
      ::"r"(smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}

// mn_3d: the MN-major operand has a rank-3 map {8 mn_lo, K, MN/8 mn_hi} (MN % 8 == 0) and the
// whole tile is one box {8, 16, BMN/8}; otherwise BMN/8 rank-2 boxes {8, 16}.  Same smem layout.
template <int BMN, bool MN_MAJOR>
__device__ __forceinline__ void tma_tile(char* s, const CUtensorMap* map, uint64_t* bar, int mn0, int k0,
                                         bool mn_3d) {
  if constexpr (MN_MAJOR) {
    if (mn_3d) {
      tma_load_3d(s, map, bar, 0, k0, mn0 >> 3);
    } else {
#pragma unroll
      for (int j = 0; j < BMN / 8; ++j) tma_load_2d(s + j * 1024, map, bar, mn0 + 8 * j, k0);
    }
  } else {
    tma_load_2d(s, map, bar, k0, mn0);
  }
}

template <bool TA, bool TB, int ID>
struct TmaCfg {
  static constexpr int BM = Shape<ID>::BM, WM = Shape<ID>::WM, WN = Shape<ID>::WN;
  static constexpr int MI = Shape<ID>::MI, NJ = Shape<ID>::NJ;
  static constexpr int BN = 8 * NJ * WN;
  static constexpr int THREADS = 32 * WM * WN;
  static constexpr bool A_MN = !TA, B_MN = TB;
  static constexpr int A_BYTES = BM * BK * 8, B_BYTES = BN * BK * 8;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int CTAS_PER_SM = Shape<ID>::CTAS;
  static constexpr int SMEM_BUDGET = (CTAS_PER_SM == 1 ? 210 : smem_budget_kb(CTAS_PER_SM)) * 1024;
  static constexpr int STAGES_FIT = SMEM_BUDGET / STAGE_BYTES;
  static constexpr int STAGES = STAGES_FIT > 6 ? 6 : STAGES_FIT;
  static constexpr size_t SMEM = (size_t)STAGES * STAGE_BYTES + 1024;   // + alignment slack
  static_assert(STAGES >= 3, "not enough shared memory for a 3-stage pipeline");
};

template <int BMN, bool MN_MAJOR>
__device__ __forceinline__ double tma_frag(const char* s, int mn, int k) {
  if constexpr (MN_MAJOR) {
    return *reinterpret_cast<const double*>(s + (mn >> 3) * 1024 + k * 64 + (mn & 7) * 8);
  } else {
    return *reinterpret_cast<const double*>(s + mn * 128 + ((((k >> 1) ^ (mn & 7))) << 4) + (k & 1) * 8);
  }
}

template <bool TA, bool TB, int ID>
__global__ void __launch_bounds__(TmaCfg<TA, TB, ID>::THREADS, TmaCfg<TA, TB, ID>::CTAS_PER_SM)
dgemm_tma_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, int64_t M,
                 int64_t N, int64_t K, double alpha, double beta, double* __restrict__ C, int64_t ldc,
                 int64_t k_chunk, double* __restrict__ partial, int mn_3d, Pred pr) {
  if (pred_skip(pr)) return;
  using CF = TmaCfg<TA, TB, ID>;
  constexpr int BM = CF::BM, BN = CF::BN, STAGES = CF::STAGES;
  constexpr int WN = CF::WN, MI = CF::MI, NJ = CF::NJ, WTM = 16 * MI, WTN = 8 * NJ;
  constexpr bool A_MN = CF::A_MN, B_MN = CF::B_MN;
  constexpr int NWARPS = CF::THREADS / 32;
  extern __shared__ __align__(1024) char smem_raw[];
  __shared__ uint64_t full[STAGES], empty[STAGES];
  // 1024-byte aligned (SWIZZLE_128B); offsetting the __shared__ array keeps LDS addressing
  char* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);

  const int64_t tiles_m = (M + BM - 1) / BM, tiles_n = (N + BN - 1) / BN;
  const int64_t GROUP_M = (mn_3d >> 8) ? (mn_3d >> 8) : 16;    // raster group height (tile rows)
  const int64_t pid = blockIdx.x;
  const int64_t per_group = GROUP_M * tiles_n;
  const int64_t first_m = (pid / per_group) * GROUP_M;
  const int64_t gsz = min(tiles_m - first_m, GROUP_M);
  const int m0 = (int)((first_m + (pid % per_group) % gsz) * BM);
  const int n0 = (int)(((pid % per_group) / gsz) * BN);
  const int64_t kbeg = (int64_t)blockIdx.z * k_chunk;
  const int64_t kend = min(K, kbeg + k_chunk);
  const int nkt = (int)((kend - kbeg + BK - 1) / BK);

  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int wm = warp / WN, wn = warp % WN;
  const int g = lane >> 2, t = lane & 3;

  auto stage_a = [&](int s) { return smem + s * CF::STAGE_BYTES; };
  auto stage_b = [&](int s) { return smem + s * CF::STAGE_BYTES + CF::A_BYTES; };
  auto issue = [&](int kt) {
    const int s = kt % STAGES;
    const int k0 = (int)(kbeg + (int64_t)kt * BK);
    mbar_expect_tx(&full[s], CF::STAGE_BYTES);
    tma_tile<BM, A_MN>(stage_a(s), &tmA, &full[s], m0, k0, mn_3d & 1);
    tma_tile<BN, B_MN>(stage_b(s), &tmB, &full[s], n0, k0, mn_3d & 2);
  };

  if (tid == 0) {
#pragma unroll
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NWARPS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  }
  __syncthreads();
  if (tid == 0) {
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
    for (int s = 0; s < STAGES - 1 && s < nkt; ++s) issue(s);
  }

  double acc[MI][NJ][4];
#pragma unroll
  for (int i = 0; i < MI; ++i)
#pragma unroll
    for (int j = 0; j < NJ; ++j)
#pragma unroll
      for (int r = 0; r < 4; ++r) acc[i][j][r] = 0.0;

  double af[2][MI][2], bf[2][NJ];
  auto load_frags = [&](int buf, const char* sa, const char* sb, int kk) {
#pragma unroll
    for (int i = 0; i < MI; ++i) {
      const int mr = wm * WTM + i * 16 + g;
      af[buf][i][0] = tma_frag<BM, A_MN>(sa, mr, kk + t);
      af[buf][i][1] = tma_frag<BM, A_MN>(sa, mr + 8, kk + t);
    }
#pragma unroll
    for (int j = 0; j < NJ; ++j) bf[buf][j] = tma_frag<BN, B_MN>(sb, wn * WTN + j * 8 + g, kk + t);
  };

  if (nkt > 0) {
    mbar_wait(&full[0], 0);
    load_frags(0, stage_a(0), stage_b(0), 0);
  }
  for (int kt = 0; kt < nkt; ++kt) {
    const int slot = kt % STAGES;
    const char* sa = stage_a(slot);
    const char* sb = stage_b(slot);
#pragma unroll
    for (int ks = 0; ks < BK / 4; ++ks) {
      const int cur = ks & 1;
      if (ks == 0 && kt > 0) {
        // This warp's DMMAs of k-tile kt-1 have consumed their fragment registers, so all of its
        // LDS from that slot have returned: release the slot (one arrival per warp).
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[(kt - 1) % STAGES]);
      }
      if (ks == BK / 4 - 1) {
        // Refill the slot of k-tile kt-1 once every warp has released it (no CTA-wide barrier:
        // only the issuing warp can wait, and only on a warp that is a whole k-tile behind).
        // Slot kt itself is not safe here: its last LDS may still be in flight, and the TMA
        // write is not ordered after them (observed as rare corrupted tiles).
        if (tid == 0 && kt + STAGES - 1 < nkt) {
          if (kt > 0) mbar_wait(&empty[(kt - 1) % STAGES], (unsigned)(((kt - 1) / STAGES) & 1));
          issue(kt + STAGES - 1);
        }
        if (kt + 1 < nkt) {
          const int s1 = (kt + 1) % STAGES;
          mbar_wait(&full[s1], (unsigned)(((kt + 1) / STAGES) & 1));
          load_frags(cur ^ 1, stage_a(s1), stage_b(s1), 0);
        }
      } else {
        load_frags(cur ^ 1, sa, sb, (ks + 1) * 4);
      }
#pragma unroll
      for (int i = 0; i < MI; ++i)
#pragma unroll
        for (int j = 0; j < NJ; ++j) dmma_16x8x4(acc[i][j], af[cur][i][0], af[cur][i][1], bf[cur][j]);
    }
  }

  if (partial) {
    double* P = partial + (size_t)blockIdx.z * (size_t)M * (size_t)N;
#pragma unroll
    for (int i = 0; i < MI; ++i)
#pragma unroll
      for (int j = 0; j < NJ; ++j)
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          const int64_t m = m0 + wm * WTM + i * 16 + g + (r >> 1) * 8;
          const int64_t n = n0 + wn * WTN + j * 8 + 2 * t + (r & 1);
          if (m < M && n < N) P[cm(m, n, M)] = acc[i][j][r];
        }
  } else {
    if (beta != 0.0) {
#pragma unroll
      for (int i = 0; i < MI; ++i)
#pragma unroll
        for (int j = 0; j < NJ; ++j)
#pragma unroll
          for (int r = 0; r < 4; ++r) {
            const int64_t m = m0 + wm * WTM + i * 16 + g + (r >> 1) * 8;
            const int64_t n = n0 + wn * WTN + j * 8 + 2 * t + (r & 1);
            const double c = (m < M && n < N) ? __ldg(C + cm(m, n, ldc)) : 0.0;
            acc[i][j][r] = alpha * acc[i][j][r] + beta * c;
          }
    } else {
#pragma unroll
      for (int i = 0; i < MI; ++i)
#pragma unroll
        for (int j = 0; j < NJ; ++j)
#pragma unroll
          for (int r = 0; r < 4; ++r) acc[i][j][r] *= alpha;
    }
#pragma unroll
    for (int i = 0; i < MI; ++i)
#pragma unroll
      for (int j = 0; j < NJ; ++j)
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          const int64_t m = m0 + wm * WTM + i * 16 + g + (r >> 1) * 8;
          const int64_t n = n0 + wn * WTN + j * 8 + 2 * t + (r & 1);
          if (m < M && n < N) C[cm(m, n, ldc)] = acc[i][j][r];
        }
  }
}

// C = alpha * sum_{z=0}^{S-1} partial[z] + beta * C, summed in order z = 0..S-1.
__global__ void dgemm_splitk_reduce(int64_t M, int64_t N, int S, double alpha, const double* __restrict__ partial,
                                    double beta, double* __restrict__ C, int64_t ldc, Pred pr) {
  if (pred_skip(pr)) return;
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

template <bool TA, bool TB, int VEC, int ID>
void launch_t(cudaStream_t st, int64_t M, int64_t N, int64_t K, double alpha, const double* A, int64_t lda,
              const double* B, int64_t ldb, double beta, double* C, int64_t ldc, int splits, int64_t kc,
              double* partial) {
  using CF = Cfg<TA, TB, ID>;
  static std::atomic<unsigned long long> attr_set{0};
  auto kern = dgemm_dmma_kernel<TA, TB, VEC, ID>;
  ensure_smem_attr(kern, (int)CF::SMEM, attr_set);
  dim3 grid((unsigned)(((N + CF::BN - 1) / CF::BN) * ((M + CF::BM - 1) / CF::BM)), 1u, (unsigned)splits);
  kern<<<grid, CF::THREADS, CF::SMEM, st>>>(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, kc, partial, launch_pred());
  UTV_CUDA(cudaGetLastError());
}

// cuTensorMapEncodeTiled from the driver (no link-time dependency on libcuda).
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  return fn;
}

// Tensor map of a column-major operand: dim0 = the contiguous extent (rows0), dim1 = cols.
// MN-major tiles use boxes {8, 16}; K-major tiles one box {16, BMN} with the 128-byte swizzle.
bool make_tmap(CUtensorMap* map, const double* ptr, int64_t rows0, int64_t cols, int64_t ld, bool mn_major,
               int bmn, bool* rank3 = nullptr) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return false;
  if (rank3) *rank3 = false;
  if (mn_major && rank3 && rows0 % 8 == 0) {
    // {8 mn_lo, cols, rows0/8 mn_hi}, strides {ld, 8} doubles: one box {8, 16, bmn/8} per tile
    const cuuint64_t dims3[3] = {8, (cuuint64_t)cols, (cuuint64_t)(rows0 / 8)};
    const cuuint64_t strides3[2] = {(cuuint64_t)ld * 8, 64};
    const cuuint32_t box3[3] = {8, (cuuint32_t)BK, (cuuint32_t)(bmn / 8)};
    const cuuint32_t estr3[3] = {1, 1, 1};
    if (fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(ptr), dims3, strides3, box3, estr3,
           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS) {
      *rank3 = true;
      return true;
    }
  }
  const cuuint64_t dims[2] = {(cuuint64_t)rows0, (cuuint64_t)cols};
  const cuuint64_t strides[1] = {(cuuint64_t)ld * 8};
  const cuuint32_t box[2] = {mn_major ? 8u : (cuuint32_t)BK, mn_major ? (cuuint32_t)BK : (cuuint32_t)bmn};
  const cuuint32_t estr[2] = {1, 1};
  return fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(ptr), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, mn_major ? CU_TENSOR_MAP_SWIZZLE_NONE : CU_TENSOR_MAP_SWIZZLE_128B,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <bool TA, bool TB, int ID>
bool launch_tma_t(cudaStream_t st, int64_t M, int64_t N, int64_t K, double alpha, const double* A, int64_t lda,
                  const double* B, int64_t ldb, double beta, double* C, int64_t ldc, int splits, int64_t kc,
                  double* partial) {
  using CF = TmaCfg<TA, TB, ID>;
  CUtensorMap ta_map, tb_map;
  // A operand (M x K): !TA -> column-major M x K (MN-major); TA -> stored K x M (K-major)
  bool a3 = false, b3 = false;
  if (!make_tmap(&ta_map, A, TA ? K : M, TA ? M : K, lda, !TA, CF::BM, &a3)) return false;
  // B operand (K x N): !TB -> stored K x N (K-major); TB -> stored N x K (MN-major)
  if (!make_tmap(&tb_map, B, TB ? N : K, TB ? K : N, ldb, TB, CF::BN, &b3)) return false;
  static const int group_m = [] { const char* e = std::getenv("UTV_GEMM_GROUP_M"); return e ? std::atoi(e) : 0; }();
  const int mn_3d = (a3 ? 1 : 0) | (b3 ? 2 : 0) | (group_m << 8);
  static std::atomic<unsigned long long> attr_set{0};
  auto kern = dgemm_tma_kernel<TA, TB, ID>;
  ensure_smem_attr(kern, (int)CF::SMEM, attr_set);
  dim3 grid((unsigned)(((N + CF::BN - 1) / CF::BN) * ((M + CF::BM - 1) / CF::BM)), 1u, (unsigned)splits);
  kern<<<grid, CF::THREADS, CF::SMEM, st>>>(ta_map, tb_map, M, N, K, alpha, beta, C, ldc, kc, partial, mn_3d,
                                            launch_pred());
  UTV_CUDA(cudaGetLastError());
  return true;
}

template <int ID>
bool dispatch_tma(cudaStream_t st, bool ta, bool tb, int64_t M, int64_t N, int64_t K, double alpha, const double* A,
                  int64_t lda, const double* B, int64_t ldb, double beta, double* C, int64_t ldc, int splits,
                  int64_t kc, double* partial) {
  if (!ta && !tb) return launch_tma_t<false, false, ID>(st, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, splits, kc, partial);
  if (ta && !tb) return launch_tma_t<true, false, ID>(st, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, splits, kc, partial);
  if (!ta && tb) return launch_tma_t<false, true, ID>(st, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, splits, kc, partial);
  return launch_tma_t<true, true, ID>(st, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, splits, kc, partial);
}

template <int VEC, int ID>
void dispatch(cudaStream_t st, bool ta, bool tb, int64_t M, int64_t N, int64_t K, double alpha, const double* A,
              int64_t lda, const double* B, int64_t ldb, double beta, double* C, int64_t ldc, int splits,
              int64_t kc, double* partial) {
  if (!ta && !tb) launch_t<false, false, VEC, ID>(st, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, splits, kc, partial);
  else if (ta && !tb) launch_t<true, false, VEC, ID>(st, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, splits, kc, partial);
  else if (!ta && tb) launch_t<false, true, VEC, ID>(st, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, splits, kc, partial);
  else launch_t<true, true, VEC, ID>(st, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, splits, kc, partial);
}

// Test / tuning knobs (utv_tune, include/utv_steps.h): -1 / 0 = automatic.
int g_force_cfg = -1;      // tile configuration 0..5
int g_force_splits = 0;    // split-K factor >= 1 (clamped to the workspace)
int g_force_path = 0;      // 1 = the cp.async fallback kernel instead of TMA

}  // namespace

void dgemm_force(int cfg, int splits, int path) {
  g_force_cfg = cfg >= 0 && cfg < kNumShapes ? cfg : -1;
  g_force_splits = splits > 0 ? splits : 0;
  g_force_path = path;
}

// Launch plan: tile configuration and split-K factor from a small cost model (waves of CTAs x
// per-tile time + the split-K reduce traffic).  Fixes wave quantisation: e.g. 782 tiles on 148
// SMs is 5.28 waves -> 6 (88%); split 3 gives 2346 tiles = 15.85 -> 16 waves (99%).
struct Plan { int cfg; int splits; int64_t kc; };

int g_cfg_long = 0, g_cfg_short = 5;     // defaults (overridable: UTV_GEMM_CFG_LONG / _SHORT)

static Plan plan_for(int cfg, int64_t M, int64_t N, int64_t K, int num_sms, size_t work_doubles, double* t_out) {
  const int bm = shape_bm(cfg), bn = shape_bn(cfg), ctas = shape_ctas(cfg);
  Plan best{cfg, 1, K};
  double best_t = 1e300;
  const double slots = (double)num_sms * ctas;
  const double tiles = (double)((M + bm - 1) / bm) * (double)((N + bn - 1) / bn);
  const double rate = 37.2e12 * 0.85 / slots;              // flop/s per CTA slot
  for (int s = 1; s <= 128; ++s) {
    if (s > 1 && (K / s < 256 || (size_t)s * (size_t)M * (size_t)N > work_doubles)) break;
    const int64_t kc = s == 1 ? K : ((K + s - 1) / s + BK - 1) / BK * BK;
    const int sp = (int)((K + kc - 1) / kc);
    const double waves = std::ceil(tiles * sp / slots);
    double t = waves * (2.0 * bm * bn * (double)kc / rate + 2.5e-6);
    if (sp > 1) t += 8.0 * (double)M * (double)N * (sp + 1) / 5.0e12 + 4e-6;
    // measured (profiles/r01_timeline): unsplit long-K launches run 1-6% below the split ones
    // of the same size even when their wave count is whole (one CTA streaming all of K)
    if (sp == 1 && K > 2048) t *= 1.05;
    if (t < best_t * 0.995) { best_t = t; best = Plan{cfg, sp, kc}; }
  }
  *t_out = best_t;
  return best;
}

static Plan make_plan(int64_t M, int64_t N, int64_t K, int num_sms, size_t work_doubles) {
  static const bool env_read = [] {
    if (const char* e = std::getenv("UTV_GEMM_CFG_LONG")) g_cfg_long = std::atoi(e) % kNumShapes;
    if (const char* e = std::getenv("UTV_GEMM_CFG_SHORT")) g_cfg_short = std::atoi(e) % kNumShapes;
    return true;
  }();
  (void)env_read;
  const bool forced = g_force_cfg >= 0;
  const int cfg = forced ? g_force_cfg : (N <= 32 ? kNarrowCfg : (K <= 1024 ? g_cfg_short : g_cfg_long));
  if (g_force_splits > 0) {
    // forced split-K: as many splits as requested that the workspace holds (>= 1 k-tile each)
    int64_t s = std::min<int64_t>(g_force_splits, (K + BK - 1) / BK);
    while (s > 1 && (size_t)s * (size_t)M * (size_t)N > work_doubles) --s;
    const int64_t kc = s <= 1 ? K : ((K + s - 1) / s + BK - 1) / BK * BK;
    return Plan{cfg, (int)((K + kc - 1) / kc), kc};
  }
  double t0 = 0.0;
  Plan p0 = plan_for(cfg, M, N, K, num_sms, work_doubles, &t0);
  if (!forced && cfg == 0 && K > 1024) {
    // long K: the 64 x 64 / 3-CTA tile balances small and mid-size outputs better; it runs ~2%
    // below the 128 x 128 tile when both fill the machine
    double t5 = 0.0;
    Plan p5 = plan_for(5, M, N, K, num_sms, work_doubles, &t5);
    if (t5 * 1.02 < t0) return p5;
  }
  return p0;
}

int dgemm_split_count(int64_t M, int64_t N, int64_t K, int num_sms) {
  return make_plan(M, N, K, num_sms, (size_t)-1).splits;
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
        M, N, 0, 0.0, nullptr, beta, C, ldc, launch_pred());
    UTV_CUDA(cudaGetLastError());
    return;
  }
  const bool aligned = ((reinterpret_cast<uintptr_t>(A) | reinterpret_cast<uintptr_t>(B)) % 16 == 0) &&
                       (lda % 2 == 0) && (ldb % 2 == 0);
  const Plan plan = make_plan(M, N, K, num_sms, work ? work_doubles : 0);
  const int splits = plan.splits;
  const int64_t kc = plan.kc;
  double* partial = splits > 1 ? work : nullptr;
  ProfScope prof(st, kProfGemm, splits > 1 ? 2 : 1, 2.0 * (double)M * (double)N * (double)K,
                 8.0 * ((double)M * K + (double)K * N + (double)M * N * (beta != 0.0 ? 2.0 : 1.0)));
  prof.shape(M, N, K, (ta ? 1 : 0) | (tb ? 2 : 0) | (plan.cfg << 2) | (splits << 8));
  static const bool use_tma = [] {
    const char* e = std::getenv("UTV_GEMM_TMA");
    return !(e && e[0] == '0');
  }();
  const bool tma_ok = use_tma && g_force_path != 1 && aligned && M < (1ll << 31) && N < (1ll << 31) && K < (1ll << 31);
  bool done = false;
  if (tma_ok) {
    switch (plan.cfg) {
      case 0: done = dispatch_tma<0>(st, ta, tb, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, splits, kc, partial); break;
      case 1: done = dispatch_tma<1>(st, ta, tb, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, splits, kc, partial); break;
      case 2: done = dispatch_tma<2>(st, ta, tb, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, splits, kc, partial); break;
      case 3: done = dispatch_tma<3>(st, ta, tb, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, splits, kc, partial); break;
      case 4: done = dispatch_tma<4>(st, ta, tb, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, splits, kc, partial); break;
      default: done = dispatch_tma<5>(st, ta, tb, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, splits, kc, partial); break;
    }
  }
  if (!done) {                     // cp.async fallback: the narrow tile runs as 128 x 64 there
    if (aligned) {
      switch (plan.cfg) {
        case 0: dispatch<2, 0>(st, ta, tb, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, splits, kc, partial); break;
        case 1: dispatch<2, 1>(st, ta, tb, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, splits, kc, partial); break;
        case 2: dispatch<2, 2>(st, ta, tb, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, splits, kc, partial); break;
        case 3: dispatch<2, 3>(st, ta, tb, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, splits, kc, partial); break;
        default: dispatch<2, 1>(st, ta, tb, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, splits, kc, partial); break;
      }
    } else {
      switch (plan.cfg) {
        case 0: dispatch<1, 0>(st, ta, tb, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, splits, kc, partial); break;
        case 1: dispatch<1, 1>(st, ta, tb, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, splits, kc, partial); break;
        case 2: dispatch<1, 2>(st, ta, tb, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, splits, kc, partial); break;
        case 3: dispatch<1, 3>(st, ta, tb, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, splits, kc, partial); break;
        default: dispatch<1, 1>(st, ta, tb, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, splits, kc, partial); break;
      }
    }
  }
  if (splits > 1) {
    const int64_t total = M * N;
    int blocks = (int)std::min<int64_t>((total + 255) / 256, 8 * (int64_t)num_sms);
    dgemm_splitk_reduce<<<blocks, 256, 0, st>>>(M, N, splits, alpha, partial, beta, C, ldc, launch_pred());
    UTV_CUDA(cudaGetLastError());
  }
}

}  // namespace utv
