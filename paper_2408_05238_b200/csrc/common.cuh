// common.cuh -- shared definitions for the sm_100a randUTV kernels (libutv.so).
// Product code: nothing here is shared with oracle/ (the CPU checker).
#pragma once
#include <cuda_runtime.h>
#include <atomic>
#include <cstdint>
#include <cstdio>
#include <string>

namespace utv {

constexpr int kNumSMsDefault = 148;

// Status codes mirror include/utv.h.
enum Status : int {
  kOk = 0, kErrArg = -1, kErrShape = -2, kErrAlloc = -3, kErrCuda = -4,
  kErrNccl = -5, kErrNumerical = -6, kErrUnsupported = -7
};

struct CudaError {
  cudaError_t err;
  const char* what;
  int line;
};

#define UTV_CUDA(x)                                                         \
  do {                                                                      \
    cudaError_t e_ = (x);                                                   \
    if (e_ != cudaSuccess) throw ::utv::CudaError{e_, #x, __LINE__};        \
  } while (0)

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per device: function attributes live in
// each device's context, so a process-wide "done" flag would leave a second device unset (handles
// of an in-process group on several GPUs).  Racing threads may both set it, which is harmless.
template <typename K>
inline void ensure_smem_attr(K kern, int bytes, std::atomic<unsigned long long>& done) {
  int dev = 0;
  UTV_CUDA(cudaGetDevice(&dev));
  const unsigned long long bit = 1ull << (dev & 63);
  if (done.load(std::memory_order_acquire) & bit) return;
  UTV_CUDA(cudaFuncSetAttribute(reinterpret_cast<const void*>(kern), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                bytes));
  done.fetch_or(bit, std::memory_order_release);
}

// Device-side launch predicate.  The panel factorization enqueues both of its algorithms for a
// sub-panel (CholeskyQR2 and the Householder kernels) and lets a device flag written by the
// CholeskyQR2 check choose, so the host never waits for it: a kernel launched while a PredScope is
// active on the launching thread runs only if (*flag != 0) == want, otherwise every CTA returns at
// entry (before touching shared state such as a grid barrier).  flag == nullptr: always runs.
struct Pred {
  const int* flag;
  int want;
};
Pred launch_pred();                           // the calling thread's current predicate
struct PredScope {
  Pred old;
  PredScope(const int* flag, int want);
  ~PredScope();
};
__device__ __forceinline__ bool pred_skip(Pred p) {
  return p.flag && ((*(volatile const int*)p.flag != 0) != (p.want != 0));
}

// Column-major element access.
__host__ __device__ __forceinline__ size_t cm(int64_t i, int64_t j, int64_t ld) {
  return (size_t)i + (size_t)j * (size_t)ld;
}

// Grid barrier for cooperative launches (all CTAs co-resident).  bar[0] = release generation
// (written by CTA 0 only), bar[32 + c * kFlagStride] = arrival flag of CTA c (written by CTA c
// only; one 128-byte line per flag, so the G x G polls of a barrier spread over G L2 lines
// instead of hammering the 5 lines of packed flags -- measured 6.6 us -> see DESIGN): no
// contended atomics -- each CTA publishes its arrival with a release store, CTA 0 polls the
// flags in parallel (one thread per CTA) and publishes the release; everyone else polls bar[0].
// `gen` must start as bar[0] read at kernel entry; every CTA calls it the same number of times.
// Requires >= (32 + gridDim.x * kFlagStride) unsigned of zero-initialised (or monotone) storage.
constexpr int kFlagStride = 32;               // unsigned per arrival flag (128 bytes)

__device__ __forceinline__ unsigned ld_acquire_gpu(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned ld_relaxed_gpu(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_gpu(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ void grid_sync(unsigned* bar, unsigned nblocks, unsigned& gen) {
  const unsigned next = gen + 1;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    st_release_gpu(bar + 32 + blockIdx.x * kFlagStride, next);
  }
  if (blockIdx.x == 0) {
    for (unsigned c = threadIdx.x; c < nblocks; c += blockDim.x)
      while ((int)(ld_acquire_gpu(bar + 32 + c * kFlagStride) - next) < 0) { }
    __syncthreads();
    if (threadIdx.x == 0) st_release_gpu(bar, next);
  } else if (threadIdx.x == 0) {
    while ((int)(ld_acquire_gpu(bar) - next) < 0) { }
  }
  gen = next;
  __syncthreads();
}

// Single-hop variant: no master -- every CTA polls all arrival flags (one thread per CTA), so
// the release costs one L2 round trip after the last arrival instead of two.  Same storage and
// monotone generations as grid_sync; the caller stores the final generation to bar[0] at the end
// of the kernel (grid_sync_finish) so the next launch starts from it.
__device__ __forceinline__ void grid_sync_all(unsigned* bar, unsigned nblocks, unsigned& gen) {
  const unsigned next = gen + 1;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    st_release_gpu(bar + 32 + blockIdx.x * kFlagStride, next);
  }
  // poll with relaxed loads (an acquire load invalidates L1 on every iteration), then ONE acquire
  // load of the observed flag (synchronises-with CTA c's release; bar.sync below extends it to the
  // whole CTA) instead of a full fence
  for (unsigned c = threadIdx.x; c < nblocks; c += blockDim.x) {
    while ((int)(ld_relaxed_gpu(bar + 32 + c * kFlagStride) - next) < 0) { }
    (void)ld_acquire_gpu(bar + 32 + c * kFlagStride);
  }
  gen = next;
  __syncthreads();
}
// grid_sync_all split in two so that a CTA can do independent work between publishing its arrival
// and polling for the others' (the qr2 kernel assembles the previous dlarft column of T there).
// The arrival is ONE release store: bar.sync orders the CTA's earlier writes (the partial sums,
// the pivot row) before thread 0's st.release.gpu (PTX memory model: causality order is
// transitive through the CTA-scope barrier and the GPU-scope release/acquire pair), so no
// separate __threadfence (MEMBAR.SC.GPU + L1 invalidate in SASS) precedes it.
__device__ __forceinline__ void grid_arrive(unsigned* bar, unsigned gen) {
  __syncthreads();
  if (threadIdx.x == 0) st_release_gpu(bar + 32 + blockIdx.x * kFlagStride, gen + 1);
}
__device__ __forceinline__ void grid_wait(unsigned* bar, unsigned nblocks, unsigned& gen) {
  const unsigned next = gen + 1;
  for (unsigned c = threadIdx.x; c < nblocks; c += blockDim.x) {
    while ((int)(ld_relaxed_gpu(bar + 32 + c * kFlagStride) - next) < 0) { }
    (void)ld_acquire_gpu(bar + 32 + c * kFlagStride);
  }
  gen = next;
  __syncthreads();
}
__device__ __forceinline__ void grid_sync_finish(unsigned* bar, unsigned gen) {
  if (blockIdx.x == 0 && threadIdx.x == 0) st_release_gpu(bar, gen);
}

constexpr size_t kGridBarrierBytes = 32768;   // >= (32 + max CTAs * kFlagStride) * 4

}  // namespace utv
