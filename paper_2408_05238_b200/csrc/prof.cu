// prof.cu -- see prof.cuh.
#include "prof.cuh"

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

}  // namespace utv
