// common.cuh -- shared definitions for the sm_100a randUTV kernels (libutv.so).
// Product code: nothing here is shared with oracle/ (the CPU checker).
#pragma once
#include <cuda_runtime.h>
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

// Column-major element access.
__host__ __device__ __forceinline__ size_t cm(int64_t i, int64_t j, int64_t ld) {
  return (size_t)i + (size_t)j * (size_t)ld;
}

// Deterministic grid barrier for cooperative launches (all CTAs co-resident).
// bar[0] = arrival counter, bar[1] = generation.  Every CTA must call it the
// same number of times.
__device__ __forceinline__ void grid_sync(unsigned* bar, unsigned nblocks, unsigned& gen) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    unsigned arrived = atomicAdd(&bar[0], 1u);
    if (arrived == nblocks - 1) {
      atomicExch(&bar[0], 0u);
      __threadfence();
      atomicAdd(&bar[1], 1u);
    } else {
      volatile unsigned* vgen = bar + 1;
      while (*vgen == gen) { __nanosleep(32); }
    }
    __threadfence();
  }
  ++gen;
  __syncthreads();
}

}  // namespace utv
