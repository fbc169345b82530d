// prof.cuh -- optional launch instrumentation (bench.py's roofline / gpu_launches evidence).
// When a handle enables profiling, every kernel launch of the library is bracketed by CUDA
// events on its stream and tagged with a family; flops / bytes are the ALGORITHMIC counts.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include <vector>

namespace utv {

enum ProfFamily : int { kProfGemm = 0, kProfPanel = 1, kProfSvd = 2, kProfSketch = 3, kProfSolve = 4,
                        kProfMisc = 5, kProfN = 6 };

struct ProfRec {
  int family;
  int launches;
  double flops, bytes;
  cudaEvent_t e0, e1;
  int64_t M = 0, N = 0, K = 0;   // GEMM shape (diagnostics)
  int tag = 0;                   // GEMM: ta | tb << 1 | cfg << 2 | splits << 8
  cudaStream_t stream = nullptr;  // timeline diagnostics (prof_dump)
};

struct Profiler {
  bool on = false;
  std::vector<ProfRec> recs;
  std::vector<cudaEvent_t> pool;
  size_t pool_used = 0;
  cudaEvent_t get();
  void reset();
  ~Profiler();
};

// The profiler of the handle currently executing an API call on this thread (or null).
extern thread_local Profiler* g_prof;

struct ProfScope {
  ProfRec* rec = nullptr;
  size_t idx = 0;
  cudaStream_t st;
  ProfScope(cudaStream_t s, int family, int launches, double flops = 0.0, double bytes = 0.0);
  ~ProfScope();
  void shape(int64_t M, int64_t N, int64_t K, int tag);
};


// Write every record (family, launches, ms, flops, M, N, K, tag) as CSV; returns records written.
long prof_dump(Profiler& p, const char* path);

}  // namespace utv
