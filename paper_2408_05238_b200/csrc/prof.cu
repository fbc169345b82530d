// prof.cu -- see prof.cuh.
#include "prof.cuh"
#include <cstdio>

namespace utv {

thread_local Profiler* g_prof = nullptr;

cudaEvent_t Profiler::get() {
  if (pool_used == pool.size()) {
    cudaEvent_t e;
    if (cudaEventCreate(&e) != cudaSuccess) { cudaGetLastError(); return nullptr; }
    pool.push_back(e);
  }
  return pool[pool_used++];
}

void Profiler::reset() {
  recs.clear();
  pool_used = 0;
}

Profiler::~Profiler() {
  for (auto e : pool) cudaEventDestroy(e);
}

ProfScope::ProfScope(cudaStream_t s, int family, int launches, double flops, double bytes) : st(s) {
  Profiler* p = g_prof;
  if (!p || !p->on) return;
  ProfRec r{family, launches, flops, bytes, p->get(), nullptr};
  r.stream = s;
  if (r.e0) cudaEventRecord(r.e0, s);
  p->recs.push_back(r);
  idx = p->recs.size() - 1;
  rec = &p->recs[idx];
}

ProfScope::~ProfScope() {
  Profiler* p = g_prof;
  if (!rec || !p) return;
  ProfRec& r = p->recs[idx];
  r.e1 = p->get();
  if (r.e1) cudaEventRecord(r.e1, st);
}

void ProfScope::shape(int64_t M, int64_t N, int64_t K, int tag) {
  Profiler* p = g_prof;
  if (!rec || !p) return;
  ProfRec& r = p->recs[idx];
  r.M = M; r.N = N; r.K = K; r.tag = tag;
}

long prof_dump(Profiler& p, const char* path) {
  FILE* f = std::fopen(path, "w");
  if (!f) return -1;
  std::fprintf(f, "family,launches,ms,flops,M,N,K,tag,start_ms,stream\n");
  long n = 0;
  const cudaEvent_t origin = p.recs.empty() ? nullptr : p.recs.front().e0;
  for (const ProfRec& r : p.recs) {
    float ms = 0.f, t0 = 0.f;
    if (r.e0 && r.e1 && cudaEventElapsedTime(&ms, r.e0, r.e1) != cudaSuccess) { cudaGetLastError(); ms = -1.f; }
    if (origin && r.e0 && cudaEventElapsedTime(&t0, origin, r.e0) != cudaSuccess) { cudaGetLastError(); t0 = -1.f; }
    std::fprintf(f, "%d,%d,%.6f,%.6e,%lld,%lld,%lld,%d,%.6f,%llx\n", r.family, r.launches, ms, r.flops, (long long)r.M,
                 (long long)r.N, (long long)r.K, r.tag, t0, (unsigned long long)(uintptr_t)r.stream);
    ++n;
  }
  std::fclose(f);
  return n;
}

}  // namespace utv
