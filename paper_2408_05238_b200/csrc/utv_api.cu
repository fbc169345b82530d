// utv_api.cu -- the C ABI of libutv.so (include/utv.h, include/utv_steps.h) and the host
// orchestration of randUTV on one B200: the per-step launch sequence of fig:alg_utv
// over the sm_100a kernels, the handle's workspace arena and error mapping.
#include <dlfcn.h>
#include <nccl.h>             // types and constants only; the functions are resolved with dlsym

#include <chrono>
#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <new>
#include <string>
#include <thread>
#include <vector>

#include "../../include/utv.h"
#include "../../include/utv_steps.h"
#include "kernels.cuh"
#include "prof.cuh"

using namespace utv;

// ------------------------------------------------------------------------------------------
// Communicators of the multi-GPU path: NCCL (one process per GPU, utv_create_dist)
// or an in-process group of ranks driven by host threads (utv_create_local_group).  In-place
// sum-AllReduce, Broadcast and AllGather of FP64 device buffers, enqueued on the caller's stream.
// ------------------------------------------------------------------------------------------
struct Comm {
  int nranks = 1, rank = 0;
  virtual ~Comm() {}
  virtual void abort() {}          // a failing rank releases its peers
  // Wait for the stream (replaces cudaStreamSynchronize on the multi-GPU path): NCCL polls the
  // communicator's asynchronous error state and gives up after a timeout, so that a rank whose
  // peer died does not wait forever (the caller's error path then aborts the communicator).
  virtual void wait(cudaStream_t st) { UTV_CUDA(cudaStreamSynchronize(st)); }
  virtual void allreduce(double* buf, size_t n, cudaStream_t st) = 0;
  virtual void bcast(double* buf, size_t n, int root, cudaStream_t st) = 0;
  virtual void allgather(const double* send, double* recv, size_t n, cudaStream_t st) = 0;
};

struct CommError {
  std::string msg;
};

// NCCL, resolved at run time (libnccl.so.2 -- the one torch already loaded, if any), so that
// libutv.so has no link-time NCCL dependency.
struct NcclApi {
  void* lib = nullptr;
  ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*allReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*allGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*errorString)(ncclResult_t) = nullptr;
  ncclResult_t (*commAbort)(ncclComm_t) = nullptr;
  ncclResult_t (*commGetAsyncError)(ncclComm_t, ncclResult_t*) = nullptr;
};

const NcclApi* nccl_api() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* l = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!l) l = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!l) return;
    NcclApi a;
    a.lib = l;
    a.getUniqueId = reinterpret_cast<decltype(a.getUniqueId)>(dlsym(l, "ncclGetUniqueId"));
    a.commInitRank = reinterpret_cast<decltype(a.commInitRank)>(dlsym(l, "ncclCommInitRank"));
    a.commDestroy = reinterpret_cast<decltype(a.commDestroy)>(dlsym(l, "ncclCommDestroy"));
    a.allReduce = reinterpret_cast<decltype(a.allReduce)>(dlsym(l, "ncclAllReduce"));
    a.broadcast = reinterpret_cast<decltype(a.broadcast)>(dlsym(l, "ncclBroadcast"));
    a.allGather = reinterpret_cast<decltype(a.allGather)>(dlsym(l, "ncclAllGather"));
    a.errorString = reinterpret_cast<decltype(a.errorString)>(dlsym(l, "ncclGetErrorString"));
    a.commAbort = reinterpret_cast<decltype(a.commAbort)>(dlsym(l, "ncclCommAbort"));
    a.commGetAsyncError = reinterpret_cast<decltype(a.commGetAsyncError)>(dlsym(l, "ncclCommGetAsyncError"));
    if (a.getUniqueId && a.commInitRank && a.commDestroy && a.allReduce && a.broadcast && a.allGather && a.errorString &&
        a.commAbort && a.commGetAsyncError)
      api = a;
  });
  return api.lib ? &api : nullptr;
}

struct NcclComm : Comm {
  const NcclApi* api = nullptr;
  ncclComm_t comm = nullptr;
  bool aborted = false;
  void check(ncclResult_t r, const char* what) {
    if (r != ncclSuccess) throw CommError{std::string(what) + ": " + api->errorString(r)};
  }
  void live() {
    if (aborted) throw CommError{"the NCCL communicator was aborted by an earlier failure; destroy the handle"};
  }
  // ncclCommAbort: ends this rank's in-flight NCCL kernels and connections (a peer blocked in a
  // collective with this rank then sees an error or its own timeout instead of hanging).
  void abort() override {
    if (comm && !aborted) {
      api->commAbort(comm);
      comm = nullptr;
      aborted = true;
    }
  }
  void wait(cudaStream_t st) override {
    live();
    static const double limit = [] {
      const char* e = std::getenv("UTV_COMM_TIMEOUT_S");
      return e ? std::atof(e) : 3600.0;
    }();
    const auto t0 = std::chrono::steady_clock::now();
    for (int it = 0;; ++it) {
      const cudaError_t e = cudaStreamQuery(st);
      if (e == cudaSuccess) return;
      if (e != cudaErrorNotReady) throw CudaError{e, "cudaStreamQuery (multi-GPU wait)", __LINE__};
      ncclResult_t ae = ncclSuccess;
      if (api->commGetAsyncError(comm, &ae) == ncclSuccess && ae != ncclSuccess && ae != ncclInProgress)
        throw CommError{std::string("NCCL asynchronous error: ") + api->errorString(ae)};
      if (std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() > limit)
        throw CommError{"timed out waiting for the peer ranks (UTV_COMM_TIMEOUT_S)"};
      if (it > 64) std::this_thread::sleep_for(std::chrono::microseconds(50));
    }
  }
  void allreduce(double* buf, size_t n, cudaStream_t st) override {
    live();
    if (n) check(api->allReduce(buf, buf, n, ncclFloat64, ncclSum, comm, st), "ncclAllReduce");
  }
  void bcast(double* buf, size_t n, int root, cudaStream_t st) override {
    live();
    if (n) check(api->broadcast(buf, buf, n, ncclFloat64, root, comm, st), "ncclBroadcast");
  }
  void allgather(const double* send, double* recv, size_t n, cudaStream_t st) override {
    live();
    if (n) check(api->allGather(send, recv, n, ncclFloat64, comm, st), "ncclAllGather");
  }
  ~NcclComm() override {
    if (comm && api) api->commDestroy(comm);
  }
};

// In-process group: every rank is a host thread with its own handle and stream.  Collectives
// rendezvous on the host (each rank first drains its stream), then every rank combines the peers'
// device buffers in rank order (deterministic, identical on all ranks) with peer copies / adds.
struct LocalGroup {
  int n = 0;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  uint64_t gen = 0;
  bool aborted = false;            // set by a rank whose call failed: every barrier then throws
  std::vector<const double*> ptr;
  explicit LocalGroup(int n_) : n(n_), ptr(n_, nullptr) {}
  void barrier() {
    std::unique_lock<std::mutex> lk(mu);
    if (aborted) throw CommError{"a peer rank of the in-process group failed"};
    const uint64_t g = gen;
    if (++arrived == n) {
      arrived = 0;
      ++gen;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return gen != g || aborted; });
      if (gen == g) throw CommError{"a peer rank of the in-process group failed"};
    }
  }
  void abort() {
    std::lock_guard<std::mutex> lk(mu);
    aborted = true;
    cv.notify_all();
  }
};

struct LocalComm : Comm {
  std::shared_ptr<LocalGroup> g;
  int device = 0;
  double* tmp = nullptr;
  double* stage = nullptr;        // a peer's buffer copied to this device (ranks on other GPUs)
  size_t tmp_n = 0;
  void ensure_tmp(size_t n) {
    if (tmp_n >= n) return;
    if (tmp) cudaFree(tmp);
    if (stage) cudaFree(stage);
    tmp = stage = nullptr; tmp_n = 0;
    UTV_CUDA(cudaMalloc((void**)&tmp, n * sizeof(double)));
    UTV_CUDA(cudaMalloc((void**)&stage, n * sizeof(double)));
    tmp_n = n;
  }
  bool local(const void* p) const {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) { cudaGetLastError(); return false; }
    return a.type == cudaMemoryTypeDevice && a.device == device;
  }
  void allreduce(double* buf, size_t n, cudaStream_t st) override {
    if (!n) return;
    ensure_tmp(n);
    UTV_CUDA(cudaStreamSynchronize(st));
    g->ptr[rank] = buf;
    g->barrier();
    UTV_CUDA(cudaMemcpyAsync(tmp, g->ptr[0], n * sizeof(double), cudaMemcpyDefault, st));
    for (int r = 1; r < nranks; ++r) {
      const double* src = g->ptr[r];
      if (!local(src)) {                      // kernels read only this device's memory
        UTV_CUDA(cudaMemcpyAsync(stage, src, n * sizeof(double), cudaMemcpyDefault, st));
        src = stage;
      }
      launch_axpy(st, (int64_t)n, 1.0, src, tmp);
    }
    UTV_CUDA(cudaStreamSynchronize(st));
    g->barrier();                                            // every rank has read every buffer
    UTV_CUDA(cudaMemcpyAsync(buf, tmp, n * sizeof(double), cudaMemcpyDefault, st));
  }
  void bcast(double* buf, size_t n, int root, cudaStream_t st) override {
    if (!n) return;
    UTV_CUDA(cudaStreamSynchronize(st));
    g->ptr[rank] = buf;
    g->barrier();
    if (rank != root) {
      UTV_CUDA(cudaMemcpyAsync(buf, g->ptr[root], n * sizeof(double), cudaMemcpyDefault, st));
      UTV_CUDA(cudaStreamSynchronize(st));
    }
    g->barrier();
  }
  void allgather(const double* send, double* recv, size_t n, cudaStream_t st) override {
    if (!n) return;
    UTV_CUDA(cudaStreamSynchronize(st));
    g->ptr[rank] = send;
    g->barrier();
    for (int r = 0; r < nranks; ++r)
      UTV_CUDA(cudaMemcpyAsync(recv + (size_t)r * n, g->ptr[r], n * sizeof(double), cudaMemcpyDefault, st));
    UTV_CUDA(cudaStreamSynchronize(st));
    g->barrier();
  }
  void abort() override { g->abort(); }
  ~LocalComm() override {
    if (tmp) cudaFree(tmp);
    if (stage) cudaFree(stage);
  }
};

// Caller-supplied communicator (utv_create_with_comm): the collectives are forwarded to host
// callbacks in program order; a non-zero return fails the call.
struct CallbackComm : Comm {
  utv_comm_ops ops{};
  void check(int rc, const char* what) {
    if (rc != 0) throw CommError{std::string("user communicator: ") + what + " returned " + std::to_string(rc)};
  }
  void abort() override { if (ops.abort) ops.abort(ops.ctx); }
  void allreduce(double* buf, size_t n, cudaStream_t st) override {
    if (n) check(ops.allreduce_sum(ops.ctx, buf, (int64_t)n, st), "allreduce_sum");
  }
  void bcast(double* buf, size_t n, int root, cudaStream_t st) override {
    if (n) check(ops.broadcast(ops.ctx, buf, (int64_t)n, root, st), "broadcast");
  }
  void allgather(const double* send, double* recv, size_t n, cudaStream_t st) override {
    if (n) check(ops.allgather(ops.ctx, send, recv, (int64_t)n, st), "allgather");
  }
};

// Factored V: instead of accumulating V explicitly (2 n^3 flops at square
// shapes, 23% of the work at q = 2), keep every step's block reflector (W_V, T_V) and V_s:
//   V = Q_1 Q_2 ... Q_s D_1 ... D_s   (D_i = V_s on block i commutes with Q_j, j > i: H5),
// and apply it to [z; 0] in the solve.  Used by utv_lstsq (V is not an output there).
struct FactoredV {
  double* W;       // sum_i n'_i b doubles: W_V of step i at woff[i] (ld n'_i)
  double* T;       // nsteps b^2: T_V of step i (ld b)
  double* Vs;      // nsteps b^2: V_s of step i (ld b)
  std::vector<size_t> woff;
  std::vector<int64_t> j0, np;
  std::vector<char> has_q;
};

// Kept factorization (UTV_KEEP_FACTORS, the reuse that v23t cannot offer,
// P:1726-1728): the last factorization's U and V in factored form, so that utv_solve_rhs can
// solve for a new right-hand side with the T left in the caller's A.
//   U = Q_U,1 ... Q_U,s  blockdiag(U_s,i)     (U_s,i on block i commutes with Q_U,j, j > i)
//   V = Q_V,1 ... Q_V,s  blockdiag(V_s,i)     (FactoredV)
struct Kept {
  bool valid = false;
  bool dist = false;       // multi-GPU handle: T is block-cyclically sharded
  int64_t m = 0, n = 0, b = 0, r = 0;
  double* buf = nullptr; size_t buf_doubles = 0;
  FactoredV fv;
  double* Wu = nullptr;    // sum_i m'_i bw_i doubles: W_U of step i at uoff[i] (ld m'_i = m - j0_i)
  double* Tu = nullptr;    // nsteps b^2: T_U of step i (ld b)
  double* Us = nullptr;    // nsteps b^2: U_s of step i (ld b)
  std::vector<size_t> uoff;
};

struct utv_handle_s {
  int device = 0;
  cudaStream_t stream = nullptr;
  int num_sms = kNumSMsDefault;
  std::string last_error;
  // workspace arena (device)
  double* ws = nullptr;
  size_t ws_doubles = 0;
  unsigned* bar = nullptr;       // grid-barrier state: [0] count, [1] generation (main stream)
  unsigned* bar2 = nullptr;      // grid-barrier state of the SVD side stream
  cudaStream_t side = nullptr;   // a7 (small SVD + its 4 updates) overlaps the next step's sketch
  cudaEvent_t ev_panel = nullptr, ev_svd = nullptr, ev_us = nullptr;
  cudaEvent_t ev_r = nullptr;     // this step's R is in A11 (a5 done): the side-stream SVD may start
  // multi-GPU overlap: collectives of column chunks run on a communication stream (high priority)
  // while the main stream computes the next chunk; the owner's SVDs may lag up to kLagMax steps
  static constexpr int kChunks = 4, kLagMax = 8;
  cudaStream_t cst = nullptr;
  cudaEvent_t ev_cq[kChunks] = {}, ev_cd[kChunks] = {};
  cudaEvent_t ev_svdq[kLagMax + 1] = {};
  int* info = nullptr;           // Jacobi sweeps / failure flag
  int* flag = nullptr;           // finiteness flag
  int64_t* d_rank = nullptr;
  int64_t* h_rank = nullptr;     // pinned
  int* h_info = nullptr;         // pinned (info[0..1], flag)
  // lstsq buffers
  double* vbuf = nullptr; size_t vbuf_doubles = 0;
  double* stage = nullptr; size_t stage_doubles = 0;   // host-pointer staging (A, B, X)
  double* nbuf = nullptr; size_t nbuf_doubles = 0;     // factored Nullify blocks (C_1..C_p)
  // out-of-core streaming (UTV_HOST_STREAMED)
  double* ooc = nullptr; size_t ooc_doubles = 0;       // resident column blocks + staging + panel
  int64_t dev_budget = 0;                              // bytes; 0 = free HBM at call time - 1 GiB
  int64_t ooc_h2d = 0, ooc_d2h = 0, ooc_resident_cols = 0;
  cudaStream_t h2d = nullptr, d2h = nullptr;
  static constexpr int kStg = 3;
  cudaEvent_t ev_loaded[kStg] = {}, ev_free[kStg] = {}, ev_done = nullptr, ev_wb = nullptr;
  // multi-GPU (utv_create_dist / utv_create_local_group)
  Comm* comm = nullptr;
  double* agree = nullptr;       // device scratch of the multi-GPU argument agreement (2 doubles)
  bool agreed_failure = false;   // the failing call was agreed on by every rank: no abort needed
  bool collective_phase = false; // this call has entered the ranks' collectives (abort on failure)
  int coop_share = 1;            // ranks of an in-process group sharing this device (cooperative-CTA cap)
  double* dbuf = nullptr; size_t dbuf_doubles = 0;
  Kept kept;                     // UTV_KEEP_FACTORS
  int64_t dist_block = 0;        // multi-GPU: block size of the last utv_factor / utv_lstsq (T's layout)
  Profiler prof;
};

namespace {

int g_dist_chunks = 0;   // utv_tune(UTV_TUNE_DIST_CHUNKS): 0 = automatic
int g_svd_lag = 0;       // utv_tune(UTV_TUNE_SVD_LAG): 0 = automatic

struct ApiError {
  utv_status st;
  std::string msg;
};

void fail(utv_status st, const std::string& m) { throw ApiError{st, m}; }

template <typename F>
utv_status guarded(utv_handle h, F&& f) {
  if (!h) return UTV_ERR_ARG;
  try {
    int cur = -1;
    cudaGetDevice(&cur);
    if (cur != h->device) UTV_CUDA(cudaSetDevice(h->device));
    struct ProfBind {
      explicit ProfBind(Profiler* p) { g_prof = p; }
      ~ProfBind() { g_prof = nullptr; }
    } bind(h->prof.on ? &h->prof : nullptr);
    h->agreed_failure = false;
    h->collective_phase = false;
    try {
      f();
    } catch (...) {
      // abort only once the ranks are inside the call's collectives (a failure before that is
      // rank-local: no peer is waiting for this rank yet, or the ranks agreed on the failure)
      if (h->comm && h->collective_phase && !h->agreed_failure) h->comm->abort();
      throw;
    }
    h->last_error.clear();
    return UTV_OK;
  } catch (const ApiError& e) {
    h->last_error = e.msg;
    return e.st;
  } catch (const CudaError& e) {
    h->last_error = std::string("CUDA error '") + cudaGetErrorString(e.err) + "' in " + e.what + " (utv_api/kernels line " +
                    std::to_string(e.line) + ")";
    cudaGetLastError();
    return e.err == cudaErrorMemoryAllocation ? UTV_ERR_ALLOC : UTV_ERR_CUDA;
  } catch (const CommError& e) {
    h->last_error = e.msg;
    return UTV_ERR_NCCL;
  } catch (const std::bad_alloc&) {
    h->last_error = "host allocation failed";
    return UTV_ERR_ALLOC;
  }
}

void ensure_buf(double** p, size_t* have, size_t need) {
  if (*have >= need) return;
  if (*p) { UTV_CUDA(cudaFree(*p)); *p = nullptr; *have = 0; }
  cudaError_t e = cudaMalloc((void**)p, need * sizeof(double));
  if (e != cudaSuccess) {
    cudaGetLastError();
    *p = nullptr;
    fail(UTV_ERR_ALLOC, "device allocation of " + std::to_string(need * sizeof(double)) + " bytes failed");
  }
  *have = need;
}

// Workspace layout for one factorization (offsets in doubles).
struct Layout {
  size_t G, Y, Z, Wv, Tv, tauv, X, X2, Wu, S, Tu, tauu, Z1, Z2, tmp, R, Us, Us2, Vs, sig, sig2;
  size_t sW, sJ, sWs, sWh, sTq, sX, sQ, stau, part, pz1, pz2, gram, px, gemm, zsolve, cq, csm;
  size_t part2, pz1b, pz2b, gram2, px2, gemm2, tmp2;
  size_t nM, nW, ntau, nT, nWt, nY, nY2;
  size_t gemm_doubles, gemm2_doubles;
  size_t total;
};

Layout plan(int64_t m, int64_t n, int64_t k, int64_t b, int num_sms) {
  Layout L{};
  size_t off = 0;
  auto take = [&](size_t cnt) { size_t o = off; off += (cnt + 31) / 32 * 32; return o; };
  const size_t mx = (size_t)std::max(m, n);
  const size_t nk = (size_t)std::max<int64_t>(n, std::max<int64_t>(k, 1));
  L.G = take((size_t)m * b);
  L.Y = take((size_t)n * b);
  L.Z = take((size_t)m * b);
  L.Wv = take((size_t)n * 2 * b);          // WVZ = [W_V | P'^T]
  L.Tv = take((size_t)b * b);
  L.tauv = take(b);
  L.X = take(mx * b);
  L.X2 = take(mx * b);
  L.Wu = take((size_t)m * 2 * b);          // LU = [X2 | W_U]
  L.S = take((size_t)b * b);
  L.Tu = take((size_t)b * b);
  L.tauu = take(b);
  L.Z1 = take((size_t)b * nk);
  L.Z2 = take((size_t)b * nk);
  L.tmp = take(std::max<size_t>(mx * b, (size_t)b * nk));
  L.R = take((size_t)b * b);
  L.Us = take((size_t)b * b);
  L.Us2 = take((size_t)b * b);
  L.Vs = take((size_t)b * b);
  L.sig = take(b);
  L.sig2 = take(b);
  L.sW = take((size_t)b * b);
  L.sJ = take((size_t)b * b);
  L.sWs = take((size_t)b * b);
  L.sWh = take((size_t)b * b);
  L.sTq = take((size_t)b * b);
  L.sX = take((size_t)b * b);
  L.sQ = take((size_t)b * b);
  L.stau = take(b);
  L.part = take((size_t)num_sms * 128);   // 2 buffers x G x (32 sums + 32 pivot values)
  L.pz1 = take((size_t)64 * b);          // 64-column sub-panels (CholeskyQR2 path)
  L.pz2 = take((size_t)64 * b);
  L.gram = take((size_t)b * b);
  L.px = take((size_t)b * 64);
  L.cq = take((size_t)std::max<int64_t>(mx, n + b) * cholqr_max_width());   // Q_1 of a sub-panel
  L.csm = take(cholqr_small_doubles());
  L.zsolve = take((size_t)n * std::max<int64_t>(k, 1));
  // split-K partials: the b x b Gram products (<= 128 b^2) and up to 4 splits of the long-K
  // max(m,n) x b sketch products (wave-quantisation fix, see gemm.cu make_plan)
  L.gemm_doubles = std::max<size_t>({(size_t)128 * b * std::max<int64_t>(b, 32), (size_t)1 << 22, 4 * mx * b});
  L.gemm = take(L.gemm_doubles);
  // side-stream (SVD) copies of the panel workspace
  L.part2 = take((size_t)num_sms * 128);
  L.pz1b = take((size_t)32 * b);
  L.pz2b = take((size_t)32 * b);
  L.gram2 = take((size_t)b * b);
  L.px2 = take((size_t)b * 32);
  L.gemm2_doubles = std::max<size_t>((size_t)128 * b * std::max<int64_t>(b, 32), (size_t)1 << 20);
  L.gemm2 = take(L.gemm2_doubles);
  L.tmp2 = take(std::max<size_t>(mx * b, (size_t)b * nk));
  // Nullify_top_right_part_of_T (only touched when UTV_NULLIFY_T12 is set)
  L.nM = take((size_t)(b + n) * b);
  L.nW = take((size_t)(b + n) * b);
  L.ntau = take(b);
  L.nT = take((size_t)b * b);
  L.nWt = take((size_t)b * b);
  L.nY = take(std::max<size_t>(mx * b, (size_t)n * std::max<int64_t>(k, 1)));
  L.nY2 = take(mx * b);
  L.total = off;
  return L;
}

struct Ctx {
  utv_handle h;
  cudaStream_t st;
  Layout L;
  double* w;
  cudaStream_t side;
  PanelWork pw, pw2;
  SvdWork sw;                    // uses pw2: runs on the side stream
  double* at(size_t off) const { return w + off; }
  void gemm(bool ta, bool tb, int64_t M, int64_t N, int64_t K, double alpha, const double* A, int64_t lda,
            const double* B, int64_t ldb, double beta, double* C, int64_t ldc) const {
    dgemm(st, ta, tb, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, at(L.gemm), L.gemm_doubles, h->num_sms);
  }
  void gemm_side(bool ta, bool tb, int64_t M, int64_t N, int64_t K, double alpha, const double* A, int64_t lda,
                 const double* B, int64_t ldb, double beta, double* C, int64_t ldc) const {
    dgemm(side, ta, tb, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, at(L.gemm2), L.gemm2_doubles, h->num_sms);
  }
};

Ctx make_ctx(utv_handle h, int64_t m, int64_t n, int64_t k, int64_t b) {
  Ctx c;
  c.h = h;
  c.st = h->stream;
  c.L = plan(m, n, k, b, h->num_sms);
  ensure_buf(&h->ws, &h->ws_doubles, c.L.total);
  c.w = h->ws;
  const Layout& L = c.L;
  c.side = h->side;
  static const bool svd_inline = [] { const char* e = std::getenv("UTV_SVD_INLINE"); return e && e[0] == '1'; }();
  if (svd_inline) c.side = h->stream;               // diagnostics: no side-stream overlap
  // the main-stream panel kernels leave 16 SMs free for the concurrent side-stream Jacobi
  // Cooperative (grid-barrier) panel kernels: ranks of an in-process group that share a device split
  // its SMs, so that all their grids stay co-resident even when launched at the same time.
  c.pw = PanelWork{c.at(L.part), c.at(L.pz1), c.at(L.pz2), c.at(L.gram), c.at(L.px), c.at(L.gemm), L.gemm_doubles,
                   h->bar, std::max(1, (h->num_sms - 16) / h->coop_share)};
  c.pw.cq = c.at(L.cq);
  c.pw.csm = c.at(L.csm);
  // info[0..1]: Jacobi sweeps / status, info[2 .. 2 + kMaxSweeps): its per-sweep rotation counts
  // (side stream); the CholeskyQR2 accept flag of the main-stream panels lives past them
  static_assert(2 + kMaxSweeps <= 48, "info layout");
  c.pw.dflag = h->info + 48;
  c.pw2 = PanelWork{c.at(L.part2), c.at(L.pz1b), c.at(L.pz2b), c.at(L.gram2), c.at(L.px2), c.at(L.gemm2),
                    L.gemm2_doubles, h->bar2, std::max(1, h->num_sms / h->coop_share)};
  c.sw = SvdWork{c.at(L.sW), c.at(L.sJ), c.at(L.sWs), c.at(L.sWh), c.at(L.sTq), c.at(L.sX), c.at(L.sQ), c.at(L.stau),
                 h->info + 2, h->info, c.pw2};
  return c;
}

void check_opts(const utv_opts* o) {
  if (!o) fail(UTV_ERR_ARG, "opts is NULL");
  if (o->block < 1) fail(UTV_ERR_ARG, "opts->block < 1");
  if (o->block > 256) fail(UTV_ERR_UNSUPPORTED, "opts->block > 256 is not supported by this build");
  if (o->power_iters < 0) fail(UTV_ERR_ARG, "opts->power_iters < 0");
  if (!(o->tau >= 0.0 && o->tau < 1.0)) fail(UTV_ERR_ARG, "opts->tau not in [0, 1)");
}

void check_ld(const char* name, int64_t ld, int64_t rows) {
  if (ld < std::max<int64_t>(1, rows)) fail(UTV_ERR_ARG, std::string(name) + " < max(1, rows)");
}

// Copy a (rows x cols) column-major matrix between (possibly host) buffers on the stream.
void copy2d(cudaStream_t st, void* dst, int64_t ldd, const void* src, int64_t lds, int64_t rows, int64_t cols,
            cudaMemcpyKind kind) {
  if (rows <= 0 || cols <= 0) return;
  UTV_CUDA(cudaMemcpy2DAsync(dst, (size_t)ldd * 8, src, (size_t)lds * 8, (size_t)rows * 8, (size_t)cols, kind, st));
}

size_t factored_w_doubles(int64_t n, int64_t b) {
  size_t tot = 0;
  for (int64_t j0 = 0; j0 < n; j0 += b)
    if (n - j0 > b) tot += (size_t)(n - j0) * b;
  return tot;
}

size_t kept_u_doubles(int64_t m, int64_t n, int64_t b) {
  size_t tot = 0;
  for (int64_t j0 = 0; j0 < n; j0 += b) tot += (size_t)(m - j0) * (size_t)std::min(b, n - j0);
  return tot;
}

// Allocate the kept-factor store (UTV_KEEP_FACTORS) for an m x n factorization with block b.
Kept& kept_prepare(utv_handle h, int64_t m, int64_t n, int64_t b, bool dist) {
  Kept& kp = h->kept;
  kp.valid = false;
  const int64_t nsteps = (n + b - 1) / b;
  const size_t wdbl = factored_w_doubles(n, b), tdbl = (size_t)nsteps * b * b, udbl = kept_u_doubles(m, n, b);
  ensure_buf(&kp.buf, &kp.buf_doubles, wdbl + 4 * tdbl + udbl + 64);
  kp.fv = FactoredV{};
  kp.fv.W = kp.buf; kp.fv.T = kp.buf + wdbl; kp.fv.Vs = kp.fv.T + tdbl;
  kp.Tu = kp.fv.Vs + tdbl; kp.Us = kp.Tu + tdbl; kp.Wu = kp.Us + tdbl;
  kp.uoff.clear();
  kp.m = m; kp.n = n; kp.b = b; kp.r = 0; kp.dist = dist;
  return kp;
}

// Record step `step`'s W_U (mp x bw at Wu, ld ldwu) and T_U (ld b) in the kept store.
void kept_push_u(cudaStream_t st, Kept& kp, int64_t step, int64_t mp, int64_t bw, const double* Wu, int64_t ldwu,
                 const double* Tu) {
  const size_t off = kp.uoff.empty() ? 0 : kp.uoff.back() + (size_t)(kp.m - (step - 1) * kp.b) * kp.b;
  kp.uoff.push_back(off);
  launch_copy(st, mp, bw, Wu, ldwu, kp.Wu + off, mp);
  launch_copy(st, bw, bw, Tu, kp.b, kp.Tu + (size_t)step * kp.b * kp.b, kp.b);
}

// C := U^T C with the kept factors, step by step as in the factorization: Q_U,i^T on rows j0:m,
// then U_s,i^T on rows j0:j0+bw (C m x k, device, ldc).
void kept_apply_ut(const Ctx& c, const Kept& kp, double* Cm, int64_t ldc, int64_t k) {
  double *Z1 = c.at(c.L.Z1), *Z2 = c.at(c.L.Z2);
  const int64_t m = kp.m, n = kp.n, b = kp.b;
  for (int64_t j0 = 0, i = 0; j0 < n; j0 += b, ++i) {
    const int64_t bw = std::min(b, n - j0), mp = m - j0;
    const double* W = kp.Wu + kp.uoff[i];
    double* Cr = Cm + j0;
    c.gemm(true, false, bw, k, mp, 1.0, W, mp, Cr, ldc, 0.0, Z1, bw);
    c.gemm(true, false, bw, k, bw, 1.0, kp.Tu + (size_t)i * b * b, b, Z1, bw, 0.0, Z2, bw);
    c.gemm(false, false, mp, k, bw, -1.0, W, mp, Z2, bw, 1.0, Cr, ldc);
    c.gemm(true, false, bw, k, bw, 1.0, kp.Us + (size_t)i * b * b, b, Cr, ldc, 0.0, Z1, bw);
    launch_copy(c.st, bw, k, Z1, bw, Cr, ldc);
  }
}

// The randUTV factorization on device buffers (fig:alg_utv).
void factor_impl(const Ctx& c, int64_t m, int64_t n, double* A, int64_t lda, double* V, int64_t ldv, double* U,
                 int64_t ldu, double* B, int64_t ldb, int64_t k, const utv_opts& o, FactoredV* fv = nullptr,
                 Kept* kp = nullptr) {
  cudaStream_t st = c.st;
  const Layout& L = c.L;
  const int64_t b = o.block;
  const int ns = c.h->num_sms;
  UTV_CUDA(cudaMemsetAsync(c.h->info, 0, 4 * sizeof(int), st));
  UTV_CUDA(cudaMemsetAsync(c.h->flag, 0, sizeof(int), st));
  launch_check_finite(st, m, n, A, lda, c.h->flag);
  if (B && k > 0) launch_check_finite(st, m, k, B, ldb, c.h->flag);
  if (V) launch_set_identity(st, n, n, V, ldv);
  if (U) launch_set_identity(st, m, m, U, ldu);
  double *G = c.at(L.G), *Y = c.at(L.Y), *Z = c.at(L.Z), *WVZ = c.at(L.Wv), *Tv = c.at(L.Tv), *tauv = c.at(L.tauv);
  double *X = c.at(L.X), *Xv2 = c.at(L.X2), *LU = c.at(L.Wu), *Tu = c.at(L.Tu), *tauu = c.at(L.tauu);
  double* S = c.at(L.S);
  double *Z1 = c.at(L.Z1), *Z2 = c.at(L.Z2), *tmp = c.at(L.tmp2), *Us = c.at(L.Us), *Vs = c.at(L.Vs),
         *sig = c.at(L.sig);
  cudaStream_t sd = c.side;
  bool svd_pending = false;
  bool us_pending = false, us_applied = false;      // deferred A12 := U_s^T A12 (see below)
  int64_t us_j0 = 0, us_bw = 0;
  const double* us_ptr = nullptr;                   // U_s of the pending A12 update
  // the side stream must not start before the work enqueued on the main stream so far
  UTV_CUDA(cudaEventRecord(c.h->ev_panel, st));
  UTV_CUDA(cudaStreamWaitEvent(sd, c.h->ev_panel, 0));

  for (int64_t j0 = 0, step = 0; j0 < n; j0 += b, ++step) {
    const int64_t bw = std::min(b, n - j0), mp = m - j0, np = n - j0, nr = np - bw;
    double* Ap = A + cm(j0, j0, lda);
    // ---- apply transformations from the right ----
    // Fused two-sided update (SURVEY 8(a) a4+a6, K5): the trailing block A_r = A[j0:m, j0+b:n]
    // gets the right update and the left update in ONE pass with K = 2b,
    //   A_r -= [X2_r | W_U] [W_r^T ; P'],  P' = T_U^T (W_U^T A_r - (W_U^T X2_r) W_r^T),
    // exact algebra of  Q_U^T (A_r - X2_r W_r^T)  with X2 = A W_V T_V (R1: all rows) and W_r =
    // W_V[b:n'].  Only the top rows 0:j0 and the panel block column get a separate K = b update.
    // LU = [X2 | W_U] (ld m), WVZ = [W_V | P'^T] (ld n').
    double* X2 = LU;
    double* Wu = LU + cm(j0, b, m);
    const bool right = np > b;                        // R5: no sketch for the last block
    if (right) {
      launch_sketch(st, o.seed, step, j0, mp, b, G, mp, ns);                          // a1
      c.gemm(true, false, np, b, mp, 1.0, Ap, lda, G, mp, 0.0, Y, np);                // Y = A'^T G
      for (int32_t it = 0; it < o.power_iters; ++it) {                                // a2 (R7)
        c.gemm(false, false, mp, b, np, 1.0, Ap, lda, Y, np, 0.0, Z, mp);             // Z = A' Y
        c.gemm(true, false, np, b, mp, 1.0, Ap, lda, Z, mp, 0.0, Y, np);              // Y = A'^T Z
      }
      double* Tvs = fv ? fv->T + (size_t)step * b * b : Tv;                            // T_V (kept if factored)
      panel_qr(st, np, b, Y, np, WVZ, np, tauv, Tvs, b, c.pw);                        // a3: W_V
      if (fv) {
        fv->woff.push_back(fv->woff.empty() ? 0 : fv->woff.back() + (size_t)fv->np.back() * b);
        fv->j0.push_back(j0); fv->np.push_back(np); fv->has_q.push_back(1);
        launch_copy(st, np, b, WVZ, np, fv->W + fv->woff.back(), np);
      }
      double* Ac = A + cm(0, j0, lda);                                                 // a4, R1: all rows
      c.gemm(false, false, m, b, np, 1.0, Ac, lda, WVZ, np, 0.0, X, m);               // X = A W_V
      c.gemm(false, false, m, b, b, 1.0, X, m, Tvs, b, 0.0, X2, m);                   // X2 = X T_V
      if (j0 > 0)                                                                      // top rows
        c.gemm(false, true, j0, np, b, -1.0, X2, m, WVZ, np, 1.0, Ac, lda);
      c.gemm(false, true, mp, bw, b, -1.0, X2 + j0, m, WVZ, np, 1.0, Ap, lda);       // panel block column
      if (V) {
        double* Vc = V + cm(0, j0, ldv);
        c.gemm(false, false, n, b, np, 1.0, Vc, ldv, WVZ, np, 0.0, X, n);
        c.gemm(false, false, n, b, b, 1.0, X, n, Tvs, b, 0.0, Xv2, n);
        c.gemm(false, true, n, np, b, -1.0, Xv2, n, WVZ, np, 1.0, Vc, ldv);
      }
    }
    // ---- apply transformations from the left ----
    panel_qr(st, mp, bw, Ap, lda, Wu, m, tauu, Tu, b, c.pw);                            // a5 (+R13)
    // a7's SVD reads only R = A11 and writes only A11 (:= Sigma) and side-stream buffers, which
    // nothing on the main stream touches before the next step's right update (that waits for
    // ev_svd): start it now, so that it overlaps this step's left update -- whose short-lived
    // CTAs free an 8-SM cluster slot quickly -- rather than the next step's long-K sketch GEMMs
    UTV_CUDA(cudaEventRecord(c.h->ev_r, st));
    UTV_CUDA(cudaStreamWaitEvent(sd, c.h->ev_r, 0));
    double* Vsi = fv ? fv->Vs + (size_t)step * b * b : Vs;                             // V_s (kept if factored)
    double* Usi = kp ? kp->Us + (size_t)step * b * b                                   // kept until applied
                     : ((step & 1) ? c.at(L.Us2) : Us);
    svd_small(sd, bw, Ap, lda, Usi, b, sig, Vsi, b, c.sw);                             // a7
    launch_set_diag(sd, bw, sig, Ap, lda);
    if (kp) kept_push_u(st, *kp, step, mp, bw, Wu, m, Tu);                              // keep W_U, T_U
    if (nr > 0) {                                                                       // a6, R3
      double* Ar = A + cm(j0, j0 + bw, lda);
      c.gemm(true, false, bw, nr, mp, 1.0, Wu, m, Ar, lda, 0.0, Z1, bw);              // W_U^T A_r
      if (right) {
        c.gemm(true, false, bw, b, mp, 1.0, Wu, m, X2 + j0, m, 0.0, S, bw);            // W_U^T X2_r
        c.gemm(false, true, bw, nr, b, -1.0, S, bw, WVZ + bw, np, 1.0, Z1, bw);      // - S W_r^T
        // P'^T = Z1^T T_U  into WVZ[bw:n', b:2b]
        c.gemm(true, false, nr, bw, bw, 1.0, Z1, bw, Tu, b, 0.0, WVZ + cm(bw, b, np), np);
        c.gemm(false, true, mp, nr, 2 * b, -1.0, X2 + j0, m, WVZ + bw, np, 1.0, Ar, lda);  // fused, K = 2b
      } else {
        c.gemm(true, false, bw, nr, bw, 1.0, Tu, b, Z1, bw, 0.0, Z2, bw);
        c.gemm(false, false, mp, nr, bw, -1.0, Wu, m, Z2, bw, 1.0, Ar, lda);
      }
    }
    if (B && k > 0) {                                                                   // C := Q_U^T C (v23t)
      double* Cr = B + cm(j0, 0, ldb);
      c.gemm(true, false, bw, k, mp, 1.0, Wu, m, Cr, ldb, 0.0, Z1, bw);
      c.gemm(true, false, bw, k, bw, 1.0, Tu, b, Z1, bw, 0.0, Z2, bw);
      c.gemm(false, false, mp, k, bw, -1.0, Wu, m, Z2, bw, 1.0, Cr, ldb);
    }
    if (U) {
      double* Uc = U + cm(0, j0, ldu);
      c.gemm(false, false, m, bw, mp, 1.0, Uc, ldu, Wu, m, 0.0, X, m);
      c.gemm(false, false, m, bw, bw, 1.0, X, m, Tu, b, 0.0, Xv2, m);
      c.gemm(false, true, m, mp, bw, -1.0, Xv2, m, Wu, m, 1.0, Uc, ldu);
    }
    // ---- deferred A12 := U_s^T A12 of the PREVIOUS step (main stream) ----
    // Rows j0':j0'+b of the trailing columns (step i-1's A12) are only right-multiplied after step
    // i-1 (right updates of the top rows; nothing else reads them), and a left multiplication
    // commutes with those, so U_s^T is applied here -- one step late -- instead of making the X
    // GEMM of this step wait for the side-stream SVD (the SVD now has a whole step to finish).
    if (us_pending) {
      UTV_CUDA(cudaStreamWaitEvent(st, c.h->ev_svd, 0));
      double* A12p = A + cm(us_j0, us_j0 + us_bw, lda);
      c.gemm(true, false, us_bw, n - us_j0 - us_bw, us_bw, 1.0, us_ptr, b, A12p, lda, 0.0, c.at(L.tmp), us_bw);
      launch_copy(st, us_bw, n - us_j0 - us_bw, c.at(L.tmp), us_bw, A12p, lda);
      UTV_CUDA(cudaEventRecord(c.h->ev_us, st));
      us_pending = false;
      us_applied = true;
    }
    // ---- the four updates of the small SVD ----
    // a7 on the side stream (the SVD itself was launched after a5): the updates touch A01, A12,
    // V(:, block), C(block, :), U(:, block), so they wait for this step's main-stream work on
    // those (C and U left updates, the deferred A12 of step i-1).  The next step's sketch, power
    // iterations and QR(Y) read only the trailing matrix, so they overlap it; the next right
    // update (which writes A12's rows) waits for ev_svd (reading H5: the updates commute, they
    // must not race).
    UTV_CUDA(cudaEventRecord(c.h->ev_panel, st));
    UTV_CUDA(cudaStreamWaitEvent(sd, c.h->ev_panel, 0));
    if (j0 > 0) {                                                                       // A01 := A01 V_s
      // A01's last b rows were just rotated by the deferred U_s^T of step i-1 (main stream)
      if (us_applied) UTV_CUDA(cudaStreamWaitEvent(sd, c.h->ev_us, 0));
      double* A01 = A + cm(0, j0, lda);
      c.gemm_side(false, false, j0, bw, bw, 1.0, A01, lda, Vsi, b, 0.0, tmp, j0);
      launch_copy(sd, j0, bw, tmp, j0, A01, lda);
    }
    if (nr > 0) {                                                                       // A12 := U_s^T A12
      us_pending = true;                                                                // next step, main
      us_j0 = j0; us_bw = bw; us_ptr = Usi;
    }
    if (V) {                                                                            // V1 := V1 V_s
      double* V1 = V + cm(0, j0, ldv);
      c.gemm_side(false, false, n, bw, bw, 1.0, V1, ldv, Vsi, b, 0.0, tmp, n);
      launch_copy(sd, n, bw, tmp, n, V1, ldv);
    }
    if (B && k > 0) {                                                                   // C1 := U_s^T C1
      double* C1 = B + cm(j0, 0, ldb);
      c.gemm_side(true, false, bw, k, bw, 1.0, Usi, b, C1, ldb, 0.0, tmp, bw);
      launch_copy(sd, bw, k, tmp, bw, C1, ldb);
    }
    if (U) {                                                                            // U1 := U1 U_s
      double* U1 = U + cm(0, j0, ldu);
      c.gemm_side(false, false, m, bw, bw, 1.0, U1, ldu, Usi, b, 0.0, tmp, m);
      launch_copy(sd, m, bw, tmp, m, U1, ldu);
    }
    UTV_CUDA(cudaEventRecord(c.h->ev_svd, sd));
    svd_pending = true;
  }
  if (svd_pending) UTV_CUDA(cudaStreamWaitEvent(st, c.h->ev_svd, 0));
  if (us_pending) {                                                                     // the last A12
    double* A12p = A + cm(us_j0, us_j0 + us_bw, lda);
    c.gemm(true, false, us_bw, n - us_j0 - us_bw, us_bw, 1.0, us_ptr, b, A12p, lda, 0.0, c.at(L.tmp), us_bw);
    launch_copy(st, us_bw, n - us_j0 - us_bw, c.at(L.tmp), us_bw, A12p, lda);
  }
  if (m > n) launch_set_zero(st, m - n, n, A + n, lda);   // rows below T (already 0 by R13; kept explicit)
}

// Reads back the Jacobi / finiteness flags and the rank (one synchronisation).
int64_t finish_factor(const Ctx& c, int64_t n, const double* T, int64_t ldt, double tau, bool want_rank) {
  cudaStream_t st = c.st;
  if (want_rank) {
    launch_rank(st, n, T, ldt, tau, c.h->d_rank);
    UTV_CUDA(cudaMemcpyAsync(c.h->h_rank, c.h->d_rank, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  }
  UTV_CUDA(cudaMemcpyAsync(c.h->h_info, c.h->info, 2 * sizeof(int), cudaMemcpyDeviceToHost, st));
  UTV_CUDA(cudaMemcpyAsync(c.h->h_info + 2, c.h->flag, sizeof(int), cudaMemcpyDeviceToHost, st));
  if (c.h->comm) c.h->comm->wait(st);
  else UTV_CUDA(cudaStreamSynchronize(st));
  if (c.h->h_info[2]) fail(UTV_ERR_NUMERICAL, "NaN or Inf in A or B");
  if (c.h->h_info[1]) fail(UTV_ERR_NUMERICAL, "Jacobi SVD of a diagonal block did not converge in 30 sweeps");
  return want_rank ? *c.h->h_rank : -1;
}

// X = V(:, 0:r) T(0:r,0:r)^{-1} C(0:r, :) on device buffers.
void solve_impl(const Ctx& c, int64_t n, int64_t r, const double* T, int64_t ldt, const double* V, int64_t ldv,
                const double* Cm, int64_t ldc, int64_t k, double* X, int64_t ldx) {
  cudaStream_t st = c.st;
  if (k <= 0) return;
  if (r <= 0) { launch_set_zero(st, n, k, X, ldx); return; }
  double* Zb = c.at(c.L.zsolve);
  launch_copy(st, r, k, Cm, ldc, Zb, r);
  constexpr int64_t SB = 256;
  for (int64_t j0 = ((r - 1) / SB) * SB; j0 >= 0; j0 -= SB) {
    const int64_t j1 = std::min(r, j0 + SB);
    launch_trsv_block(st, j0, j1, T, ldt, Zb, r, k);
    if (j0 > 0) c.gemm(false, false, j0, k, j1 - j0, -1.0, T + cm(0, j0, ldt), ldt, Zb + j0, r, 1.0, Zb, r);
  }
  c.gemm(false, false, n, k, r, 1.0, V, ldv, Zb, r, 0.0, X, ldx);
}

// Nullify_top_right_part_of_T (fig:alg_nullify_t12), blocked bottom-up
// in row blocks of b: for rows i0:i1 the RZ factorization of the slab [T(i0:i1, i0:i1) | T(i0:i1, r:n)]
// is the Householder QR of M = diag(J, I) S^T J (panel_qr, same dlarfg conventions as the oracle's
// row-by-row sweep), giving S C = [J R^T J, 0] with C = I - W' T_z W'^T, W' = diag(J, I) W; C is
// applied to the rows above ("Update(C11, D1, C01, D0)") and to V ("Update(C11, D1, E1, F)") as
// DMMA GEMMs over the two column ranges (i0:i1) and (r:n).  With V factored, C is kept (ns).
struct NullStore {
  double* Wtop = nullptr;   // per block q: b x b (ld b)      W'_top = J W_top
  double* Wbot = nullptr;   // per block q: nz x b (ld nz)    W'_bot
  double* Tz = nullptr;     // per block q: b x b (ld b)
  std::vector<int64_t> i0, bw;
  int64_t nz = 0;
};

void nullify_impl(const Ctx& c, int64_t n, int64_t r, double* T, int64_t ldt, double* V, int64_t ldv, int64_t b,
                  NullStore* ns) {
  const int64_t nz = n - r;
  if (nz <= 0 || r <= 0) return;
  cudaStream_t st = c.st;
  const int64_t ldm = b + nz;
  double *M = c.at(c.L.nM), *W = c.at(c.L.nW), *tz = c.at(c.L.ntau), *Tz = c.at(c.L.nT), *Wt = c.at(c.L.nWt);
  double *Y = c.at(c.L.nY), *Y2 = c.at(c.L.nY2);
  if (ns) ns->nz = nz;
  for (int64_t i1 = r, q = 0; i1 > 0; ++q) {
    const int64_t i0 = std::max<int64_t>(0, i1 - b), bw = i1 - i0;
    launch_rz_build(st, bw, nz, T, ldt, i0, r, M, ldm);
    panel_qr(st, bw + nz, bw, M, ldm, W, ldm, tz, Tz, b, c.pw);
    launch_rz_writeback(st, bw, nz, M, ldm, T, ldt, i0, r);
    launch_reverse_rows(st, bw, W, ldm, Wt, b);
    const double* Wb = W + bw;                                           // W'_bot (ld ldm)
    auto apply_rows = [&](double* X, int64_t ldx, int64_t rows) {        // X(:, cols) <- X(:, cols) C
      double* Xl = X + cm(0, i0, ldx);
      double* Xr = X + cm(0, r, ldx);
      c.gemm(false, false, rows, bw, bw, 1.0, Xl, ldx, Wt, b, 0.0, Y, rows);
      c.gemm(false, false, rows, bw, nz, 1.0, Xr, ldx, Wb, ldm, 1.0, Y, rows);
      c.gemm(false, false, rows, bw, bw, 1.0, Y, rows, Tz, b, 0.0, Y2, rows);
      c.gemm(false, true, rows, bw, bw, -1.0, Y2, rows, Wt, b, 1.0, Xl, ldx);
      c.gemm(false, true, rows, nz, bw, -1.0, Y2, rows, Wb, ldm, 1.0, Xr, ldx);
    };
    if (i0 > 0) apply_rows(T, ldt, i0);                                  // rows above
    if (V) apply_rows(V, ldv, n);
    if (ns) {
      launch_copy(st, bw, bw, Wt, b, ns->Wtop + (size_t)q * b * b, b);
      launch_copy(st, nz, bw, Wb, ldm, ns->Wbot + (size_t)q * nz * b, nz);
      launch_copy(st, bw, bw, Tz, b, ns->Tz + (size_t)q * b * b, b);
      ns->i0.push_back(i0);
      ns->bw.push_back(bw);
    }
    i1 = i0;
  }
}

size_t null_store_doubles(int64_t n, int64_t r, int64_t b) {
  if (r <= 0 || n - r <= 0) return 0;
  const size_t nblk = (size_t)((r + b - 1) / b);
  return nblk * ((size_t)(n - r) * b + 2 * (size_t)b * b);
}

// X = V(:, 0:r) z with V in factored form: X = Q_1 ... Q_s D [C_1 ... C_p] [z; 0]  (X is n x k).
// z_ready: z = T11^{-1} C(0:r) is already in the zsolve buffer (ld r; the streamed path solves it
// block by block as T's columns arrive) -- T and Cm are then not read.
void solve_factored(const Ctx& c, int64_t n, int64_t r, const double* T, int64_t ldt, const double* Cm, int64_t ldc,
                    int64_t k, double* X, int64_t ldx, const FactoredV& fv, int64_t b,
                    const NullStore* ns = nullptr, bool z_ready = false) {
  cudaStream_t st = c.st;
  if (k <= 0) return;
  launch_set_zero(st, n, k, X, ldx);
  if (r <= 0) return;
  double* Zb = c.at(c.L.zsolve);
  if (!z_ready) {
    launch_copy(st, r, k, Cm, ldc, Zb, r);
    static const bool force_trsv = [] { const char* e = std::getenv("UTV_SOLVE_TRSV"); return e && e[0] == '1'; }();
    if ((!ns || ns->i0.empty()) && b <= 256 && !force_trsv) {
      // without Nullify T11's b x b diagonal blocks are Sigma_i (diagonal): GEMVs + one scaling
      launch_diag_block_solve(st, r, b, T, ldt, Zb, r, k);
    } else {
      constexpr int64_t SB = 256;
      for (int64_t j0 = ((r - 1) / SB) * SB; j0 >= 0; j0 -= SB) {             // z = T11^{-1} C(0:r)
        const int64_t j1 = std::min(r, j0 + SB);
        launch_trsv_block(st, j0, j1, T, ldt, Zb, r, k);
        if (j0 > 0) c.gemm(false, false, j0, k, j1 - j0, -1.0, T + cm(0, j0, ldt), ldt, Zb + j0, r, 1.0, Zb, r);
      }
    }
  }
  double* tmp = c.at(c.L.Z1);
  double* tmp2 = c.at(c.L.Z2);
  const bool nul = ns && !ns->i0.empty();
  if (!nul) {
    for (int64_t j0 = 0, step = 0; j0 < r; j0 += b, ++step) {                // D: X(blk) = V_s,i z(blk)
      const int64_t bw = std::min(b, n - j0), zr = std::min(bw, r - j0);
      c.gemm(false, false, bw, k, zr, 1.0, fv.Vs + (size_t)step * b * b, b, Zb + j0, r, 0.0, X + j0, ldx);
    }
  } else {
    // y = C_1 ... C_p [z; 0] (the last-processed nullify block first), then D on every block
    double* Yv = c.at(c.L.nY);                                            // n x k
    launch_set_zero(st, n, k, Yv, n);
    launch_copy(st, r, k, Zb, r, Yv, n);
    const int64_t nz = ns->nz;
    for (int64_t q = (int64_t)ns->i0.size() - 1; q >= 0; --q) {
      const int64_t i0 = ns->i0[q], bw = ns->bw[q];
      const double* Wt = ns->Wtop + (size_t)q * b * b;
      const double* Wb = ns->Wbot + (size_t)q * nz * b;
      c.gemm(true, false, bw, k, bw, 1.0, Wt, b, Yv + i0, n, 0.0, tmp, b);
      c.gemm(true, false, bw, k, nz, 1.0, Wb, nz, Yv + r, n, 1.0, tmp, b);
      c.gemm(false, false, bw, k, bw, 1.0, ns->Tz + (size_t)q * b * b, b, tmp, b, 0.0, tmp2, b);
      c.gemm(false, false, bw, k, bw, -1.0, Wt, b, tmp2, b, 1.0, Yv + i0, n);
      c.gemm(false, false, nz, k, bw, -1.0, Wb, nz, tmp2, b, 1.0, Yv + r, n);
    }
    for (int64_t j0 = 0, step = 0; j0 < n; j0 += b, ++step) {                // D on all blocks
      const int64_t bw = std::min(b, n - j0);
      c.gemm(false, false, bw, k, bw, 1.0, fv.Vs + (size_t)step * b * b, b, Yv + j0, n, 0.0, X + j0, ldx);
    }
  }
  for (int64_t i = (int64_t)fv.woff.size() - 1; i >= 0; --i) {                // X = Q_i X, i = s..1
    const int64_t j0 = fv.j0[i], np = fv.np[i];
    const double* W = fv.W + fv.woff[i];
    c.gemm(true, false, b, k, np, 1.0, W, np, X + j0, ldx, 0.0, tmp, b);
    c.gemm(false, false, b, k, b, 1.0, fv.T + (size_t)(j0 / b) * b * b, b, tmp, b, 0.0, tmp2, b);
    c.gemm(false, false, np, k, b, -1.0, W, np, tmp2, b, 1.0, X + j0, ldx);
  }
}

// ------------------------------------------------------------------------------------------
// Out-of-core randUTV (UTV_HOST_STREAMED, the paper's out-of-core regime
// P:1580-1675).  A stays in (pinned) host memory and is overwritten by T there.
// HBM holds the workspace, the factored V, a staging ring of kStg chunks (cw columns, all rows)
// and as many trailing column blocks as the device budget allows: columns [c_res, n) are loaded
// once and stay resident (the last blocks are the ones every step touches); columns < c_res are
// streamed H2D on one copy stream and D2H on another, overlapped with the DMMA GEMMs of the
// previous / next chunk (the column-block decomposition of every product is exact).  Per step:
//   passes over the trailing columns, rows j0:m:  Z = A'Y (accumulated), Y = A'^T Z   (q times)
//   QR(Y) -> W_V, T_V;  pass, all rows:  X = A W_V (accumulated);  X2 = X T_V
//   block i (loaded): right update, panel QR, SVD, written back
//   one read+write pass over the columns > i:  right update (all rows), Q_U^T (rows j0:m),
//   U_s^T (rows j0:j0+b), and the NEXT step's sketch product Y' = A''^T G' (rows j0+b:m,
//   which the U_s^T update does not touch) -- so each step streams 2q+2 reads + 1 write.
// ------------------------------------------------------------------------------------------
struct Ooc {
  utv_handle h = nullptr;
  int64_t m = 0, n = 0, b = 0;
  double* hA = nullptr;
  int64_t lda = 0;
  int64_t c_res = 0;      // first resident column (multiple of b)
  double* res = nullptr;  // device, m x (n - c_res), ld m
  int64_t cw = 0;         // staging chunk width (columns, multiple of b)
  double* stg[utv_handle_s::kStg] = {};
  double* pb[2] = {};     // device m x b: a step's own block column when it is streamed (by step parity)
  int next = 0;
};

// h2d waits for every write-back enqueued so far (host data consistency).
void ooc_sync_wb(Ooc& o) {
  UTV_CUDA(cudaEventRecord(o.h->ev_wb, o.h->d2h));
  UTV_CUDA(cudaStreamWaitEvent(o.h->h2d, o.h->ev_wb, 0));
}

// Enqueue a host -> device copy on h2d and make the main stream wait for it.
void ooc_load(Ooc& o, const Ctx& c, double* dst, int64_t ldd, int64_t row0, int64_t rows, int64_t col, int64_t w,
              cudaEvent_t done) {
  utv_handle h = o.h;
  copy2d(h->h2d, dst, ldd, o.hA + cm(row0, col, o.lda), o.lda, rows, w, cudaMemcpyHostToDevice);
  h->ooc_h2d += rows * w * 8;
  UTV_CUDA(cudaEventRecord(done, h->h2d));
  UTV_CUDA(cudaStreamWaitEvent(c.st, done, 0));
}

void ooc_store(Ooc& o, const Ctx& c, const double* src, int64_t lds, int64_t row0, int64_t rows, int64_t col,
               int64_t w, cudaEvent_t done) {
  utv_handle h = o.h;
  UTV_CUDA(cudaEventRecord(h->ev_done, c.st));
  UTV_CUDA(cudaStreamWaitEvent(h->d2h, h->ev_done, 0));
  copy2d(h->d2h, o.hA + cm(row0, col, o.lda), o.lda, src, lds, rows, w, cudaMemcpyDeviceToHost);
  h->ooc_d2h += rows * w * 8;
  if (done) UTV_CUDA(cudaEventRecord(done, h->d2h));
}

// One pass over columns [c0, n), rows row0:m: fn(dev, ld, col, w) on the main stream with dev at
// (row0, col).  Resident columns first (one call), then the streamed chunks through the ring.
template <typename F>
void ooc_pass(Ooc& o, const Ctx& c, int64_t c0, int64_t row0, bool write_back, F&& fn) {
  utv_handle h = o.h;
  const int64_t rows = o.m - row0;
  const int64_t r0 = std::max(c0, o.c_res);
  if (r0 < o.n) fn(o.res + cm(row0, r0 - o.c_res, o.m), o.m, r0, o.n - r0);
  // chunks of one pass are disjoint, so only earlier passes' write-backs must land first
  if (c0 < std::min(o.n, o.c_res)) ooc_sync_wb(o);
  for (int64_t col = c0; col < std::min(o.n, o.c_res); col += o.cw) {
    const int64_t w = std::min(o.cw, o.c_res - col);
    const int s = o.next;
    o.next = (o.next + 1) % utv_handle_s::kStg;
    double* d = o.stg[s];
    UTV_CUDA(cudaStreamWaitEvent(h->h2d, h->ev_free[s], 0));          // slot's previous chunk done
    ooc_load(o, c, d, o.m, row0, rows, col, w, h->ev_loaded[s]);
    fn(d, o.m, col, w);
    if (write_back) {
      ooc_store(o, c, d, o.m, row0, rows, col, w, h->ev_free[s]);
    } else {
      UTV_CUDA(cudaEventRecord(h->ev_free[s], c.st));
    }
  }
}

// Device pointer (row 0, ld *ld) of the column block [j0, j0 + w), rows 0:rows loaded if streamed.
double* ooc_block(Ooc& o, const Ctx& c, int64_t j0, int64_t w, int64_t rows, int64_t* ld, int buf = 0) {
  *ld = o.m;
  if (j0 >= o.c_res) return o.res + cm(0, j0 - o.c_res, o.m);
  UTV_CUDA(cudaEventRecord(o.h->ev_done, c.st));                      // the buffer's previous readers
  UTV_CUDA(cudaStreamWaitEvent(o.h->h2d, o.h->ev_done, 0));
  ooc_sync_wb(o);
  ooc_load(o, c, o.pb[buf], o.m, 0, rows, j0, w, o.h->ev_loaded[0]);
  return o.pb[buf];
}

void ooc_block_store(Ooc& o, const Ctx& c, int64_t j0, int64_t w, int buf) {
  if (j0 >= o.c_res) return;
  ooc_store(o, c, o.pb[buf], o.m, 0, o.m, j0, w, nullptr);
}

// diag(T) is gathered into dg (n) as each block's sigma is set; C (device, ldc) becomes U^T B.
void factor_ooc(const Ctx& c, Ooc& o, double* Cd, int64_t ldc, int64_t k, const utv_opts& opt, FactoredV* fv,
                double* dg) {
  cudaStream_t st = c.st;
  const Layout& L = c.L;
  const int64_t b = opt.block, m = o.m, n = o.n;
  const int ns = c.h->num_sms;
  UTV_CUDA(cudaMemsetAsync(c.h->info, 0, 4 * sizeof(int), st));
  UTV_CUDA(cudaMemsetAsync(c.h->flag, 0, sizeof(int), st));
  if (Cd && k > 0) launch_check_finite(st, m, k, Cd, ldc, c.h->flag);
  double *G = c.at(L.G), *Y = c.at(L.Y), *Z = c.at(L.Z), *WV = c.at(L.Wv), *tauv = c.at(L.tauv);
  double *X = c.at(L.X), *X2 = c.at(L.X2), *Wu = c.at(L.Wu), *Tu = c.at(L.Tu), *tauu = c.at(L.tauu);
  double *Z1 = c.at(L.Z1), *Z2 = c.at(L.Z2), *tmp = c.at(L.tmp2), *Us = c.at(L.Us), *sig = c.at(L.sig);
  // resident columns: loaded once
  if (o.c_res < n) {
    UTV_CUDA(cudaEventRecord(o.h->ev_done, st));
    UTV_CUDA(cudaStreamWaitEvent(o.h->h2d, o.h->ev_done, 0));
    ooc_load(o, c, o.res, m, 0, m, o.c_res, n - o.c_res, o.h->ev_loaded[0]);
    launch_check_finite(st, m, n - o.c_res, o.res, m, c.h->flag);
  }
  bool y_ready = false;
  bool fin_pending = false, us_pend = false;        // the previous step's SVD results (see below)
  int64_t fin_step = 0, fin_j0 = 0, fin_bw = 0;
  for (int64_t j0 = 0, step = 0; j0 < n; j0 += b, ++step) {
    const int64_t bw = std::min(b, n - j0), mp = m - j0, np = n - j0, nr = np - bw;
    const bool right = np > b;                                                     // R5
    double* Tvs = fv->T + (size_t)step * b * b;
    if (right) {
      if (!y_ready) {                                                              // a1 + Y = A'^T G
        launch_sketch(st, opt.seed, step, j0, mp, b, G, mp, ns);
        ooc_pass(o, c, j0, j0, false, [&](double* d, int64_t ld, int64_t col, int64_t w) {
          if (step == 0 && col < o.c_res) launch_check_finite(st, mp, w, d, ld, c.h->flag);
          c.gemm(true, false, w, b, mp, 1.0, d, ld, G, mp, 0.0, Y + (col - j0), np);
        });
      }
      for (int32_t it = 0; it < opt.power_iters; ++it) {                          // a2 (R7)
        launch_set_zero(st, mp, b, Z, mp);
        ooc_pass(o, c, j0, j0, false, [&](double* d, int64_t ld, int64_t col, int64_t w) {
          c.gemm(false, false, mp, b, w, 1.0, d, ld, Y + (col - j0), np, 1.0, Z, mp);
        });
        ooc_pass(o, c, j0, j0, false, [&](double* d, int64_t ld, int64_t col, int64_t w) {
          c.gemm(true, false, w, b, mp, 1.0, d, ld, Z, mp, 0.0, Y + (col - j0), np);
        });
      }
      panel_qr(st, np, b, Y, np, WV, np, tauv, Tvs, b, c.pw);                     // a3
      fv->woff.push_back(fv->woff.empty() ? 0 : fv->woff.back() + (size_t)fv->np.back() * b);
      fv->j0.push_back(j0); fv->np.push_back(np); fv->has_q.push_back(1);
      launch_copy(st, np, b, WV, np, fv->W + fv->woff.back(), np);
      launch_set_zero(st, m, b, X, m);                                             // a4, R1: all rows
      ooc_pass(o, c, j0, 0, false, [&](double* d, int64_t ld, int64_t col, int64_t w) {
        c.gemm(false, false, m, b, w, 1.0, d, ld, WV + (col - j0), np, 1.0, X, m);
      });
      c.gemm(false, false, m, b, b, 1.0, X, m, Tvs, b, 0.0, X2, m);
    }
    // ---- block i: right update, the previous step's deferred SVD results, panel QR (a5),
    // C := Q_U^T C, and this step's SVD launched on the side stream (a7).  The SVD results are
    // applied one step later (as on the in-core path): A12 := U_s^T A12 commutes with the next
    // step's right updates, and block i itself is finalised (Sigma, A01 V_s) and written back at
    // the next step, so the Jacobi overlaps the next step's link-bound passes.
    const int buf = (int)(step & 1);
    int64_t lda_i = m;
    double* Ai = ooc_block(o, c, j0, bw, m, &lda_i, buf);
    // n <= b: no sketch pass ran, so a streamed block 0 has not been checked for NaN / Inf yet
    if (step == 0 && !right && j0 < o.c_res) launch_check_finite(st, m, bw, Ai, lda_i, c.h->flag);
    if (right) c.gemm(false, true, m, bw, b, -1.0, X2, m, WV, np, 1.0, Ai, lda_i);
    if (fin_pending) {
      UTV_CUDA(cudaStreamWaitEvent(st, c.h->ev_svd, 0));
      const double* Usp = (fin_step & 1) ? c.at(L.Us2) : Us;
      const double* sgp = (fin_step & 1) ? c.at(L.sig2) : sig;
      const double* Vsp = fv->Vs + (size_t)fin_step * b * b;
      // block i's part of A12(i-1): rows fin_j0:fin_j0+fin_bw
      c.gemm(true, false, fin_bw, bw, fin_bw, 1.0, Usp, b, Ai + fin_j0, lda_i, 0.0, Z1, fin_bw);
      launch_copy(st, fin_bw, bw, Z1, fin_bw, Ai + fin_j0, lda_i);
      // finalise block i-1: A11 := Sigma, A01 := A01 V_s, C1 := U_s^T C1, diag(T), write back
      int64_t ldf = m;
      double* Af = fin_j0 >= o.c_res ? o.res + cm(0, fin_j0 - o.c_res, m) : o.pb[fin_step & 1];
      launch_set_diag(st, fin_bw, sgp, Af + fin_j0, ldf);
      launch_copy(st, fin_bw, 1, sgp, fin_bw, dg + fin_j0, n);
      if (fin_j0 > 0) {
        c.gemm(false, false, fin_j0, fin_bw, fin_bw, 1.0, Af, ldf, Vsp, b, 0.0, tmp, fin_j0);
        launch_copy(st, fin_j0, fin_bw, tmp, fin_j0, Af, ldf);
      }
      if (Cd && k > 0) {
        c.gemm(true, false, fin_bw, k, fin_bw, 1.0, Usp, b, Cd + fin_j0, ldc, 0.0, Z1, fin_bw);
        launch_copy(st, fin_bw, k, Z1, fin_bw, Cd + fin_j0, ldc);
      }
      ooc_block_store(o, c, fin_j0, fin_bw, (int)(fin_step & 1));
      fin_pending = false;
      us_pend = nr > 0;                  // rows fin_j0:+fin_bw of the columns > block i: in the U pass
    }
    panel_qr(st, mp, bw, Ai + j0, lda_i, Wu, m, tauu, Tu, b, c.pw);
    if (Cd && k > 0) {
      double* Cr = Cd + j0;
      c.gemm(true, false, bw, k, mp, 1.0, Wu, m, Cr, ldc, 0.0, Z1, bw);
      c.gemm(true, false, bw, k, bw, 1.0, Tu, b, Z1, bw, 0.0, Z2, bw);
      c.gemm(false, false, mp, k, bw, -1.0, Wu, m, Z2, bw, 1.0, Cr, ldc);
    }
    {
      double* Vsi = fv->Vs + (size_t)step * b * b;
      double* Usi = buf ? c.at(L.Us2) : Us;
      double* sgi = buf ? c.at(L.sig2) : sig;
      UTV_CUDA(cudaEventRecord(c.h->ev_panel, st));
      UTV_CUDA(cudaStreamWaitEvent(c.side, c.h->ev_panel, 0));
      svd_small(c.side, bw, Ai + j0, lda_i, Usi, b, sgi, Vsi, b, c.sw);
      UTV_CUDA(cudaEventRecord(c.h->ev_svd, c.side));
    }
    // ---- one read+write pass over the trailing columns (+ the next step's sketch product)
    if (nr > 0) {
      const bool next_sketch = nr > b;
      if (next_sketch) launch_sketch(st, opt.seed, step + 1, j0 + b, mp - b, b, G, mp - b, ns);
      const bool upd_prev = us_pend;
      const double* Usp = ((step - 1) & 1) ? c.at(L.Us2) : Us;
      const int64_t pj0 = j0 - b;
      ooc_pass(o, c, j0 + bw, 0, true, [&](double* d, int64_t ld, int64_t col, int64_t w) {
        if (right) c.gemm(false, true, m, w, b, -1.0, X2, m, WV + (col - j0), np, 1.0, d, ld);
        if (upd_prev) {                                                            // A12(i-1) := U_s^T A12
          c.gemm(true, false, b, w, b, 1.0, Usp, b, d + pj0, ld, 0.0, Z1, b);
          launch_copy(st, b, w, Z1, b, d + pj0, ld);
        }
        double* dr = d + j0;                                                       // a6, R3
        c.gemm(true, false, bw, w, mp, 1.0, Wu, m, dr, ld, 0.0, Z1, bw);
        c.gemm(true, false, bw, w, bw, 1.0, Tu, b, Z1, bw, 0.0, Z2, bw);
        c.gemm(false, false, mp, w, bw, -1.0, Wu, m, Z2, bw, 1.0, dr, ld);
        if (next_sketch)
          c.gemm(true, false, w, b, mp - b, 1.0, d + j0 + b, ld, G, mp - b, 0.0, Y + (col - j0 - b), np - b);
      });
      y_ready = next_sketch;
    }
    us_pend = false;
    fin_pending = true;
    fin_step = step; fin_j0 = j0; fin_bw = bw;
  }
  // the last block: its SVD results
  if (fin_pending) {
    UTV_CUDA(cudaStreamWaitEvent(st, c.h->ev_svd, 0));
    const double* Usp = (fin_step & 1) ? c.at(L.Us2) : Us;
    const double* sgp = (fin_step & 1) ? c.at(L.sig2) : sig;
    const double* Vsp = fv->Vs + (size_t)fin_step * b * b;
    int64_t ldf = m;
    double* Af = fin_j0 >= o.c_res ? o.res + cm(0, fin_j0 - o.c_res, m) : o.pb[fin_step & 1];
    launch_set_diag(st, fin_bw, sgp, Af + fin_j0, ldf);
    launch_copy(st, fin_bw, 1, sgp, fin_bw, dg + fin_j0, n);
    if (fin_j0 > 0) {
      c.gemm(false, false, fin_j0, fin_bw, fin_bw, 1.0, Af, ldf, Vsp, b, 0.0, tmp, fin_j0);
      launch_copy(st, fin_j0, fin_bw, tmp, fin_j0, Af, ldf);
    }
    if (Cd && k > 0) {
      c.gemm(true, false, fin_bw, k, fin_bw, 1.0, Usp, b, Cd + fin_j0, ldc, 0.0, Z1, fin_bw);
      launch_copy(st, fin_bw, k, Z1, fin_bw, Cd + fin_j0, ldc);
    }
    ooc_block_store(o, c, fin_j0, fin_bw, (int)(fin_step & 1));
  }
}

// z = T11^{-1} C(0:r) into the zsolve buffer, T's column blocks fetched bottom-up (rows 0:j1).
void solve_z_ooc(const Ctx& c, Ooc& o, int64_t r, const double* Cd, int64_t ldc, int64_t k) {
  cudaStream_t st = c.st;
  if (r <= 0 || k <= 0) return;
  double* Zb = c.at(c.L.zsolve);
  double* D = c.at(c.L.R);
  launch_copy(st, r, k, Cd, ldc, Zb, r);
  const int64_t b = o.b;
  for (int64_t j0 = ((r - 1) / b) * b; j0 >= 0; j0 -= b) {
    const int64_t j1 = std::min(r, j0 + b), w = j1 - j0;
    int64_t ldt = o.m;
    const double* Tb = ooc_block(o, c, j0, w, j1, &ldt);
    launch_copy(st, w, w, Tb + j0, ldt, D, b);
    launch_trsv_block(st, 0, w, D, b, Zb + j0, r, k);
    if (j0 > 0) c.gemm(false, false, j0, k, w, -1.0, Tb, ldt, Zb + j0, r, 1.0, Zb, r);
  }
}

bool is_device_ptr(const void* p) {
  if (!p) return true;
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) { cudaGetLastError(); return false; }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

bool is_pinned_host_ptr(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) { cudaGetLastError(); return false; }
  return a.type == cudaMemoryTypeHost;
}

// Pins a host matrix for the DMA engines if the caller did not (unpinned when the object dies).
struct HostPin {
  void* p = nullptr;
  void pin(double* A, int64_t m, int64_t n, int64_t lda) {
    if (n <= 0 || is_pinned_host_ptr(A)) return;
    UTV_CUDA(cudaHostRegister(A, ((size_t)(n - 1) * lda + m) * sizeof(double), cudaHostRegisterDefault));
    p = A;
  }
  ~HostPin() { if (p) { cudaHostUnregister(p); cudaGetLastError(); } }
};

// The copy streams and events of the out-of-core mode (created once per handle).
void ooc_streams(utv_handle h) {
  if (h->h2d) return;
  UTV_CUDA(cudaStreamCreateWithFlags(&h->h2d, cudaStreamNonBlocking));
  UTV_CUDA(cudaStreamCreateWithFlags(&h->d2h, cudaStreamNonBlocking));
  for (int s = 0; s < utv_handle_s::kStg; ++s) {
    UTV_CUDA(cudaEventCreateWithFlags(&h->ev_loaded[s], cudaEventDisableTiming));
    UTV_CUDA(cudaEventCreateWithFlags(&h->ev_free[s], cudaEventDisableTiming));
  }
  UTV_CUDA(cudaEventCreateWithFlags(&h->ev_done, cudaEventDisableTiming));
  UTV_CUDA(cudaEventCreateWithFlags(&h->ev_wb, cudaEventDisableTiming));
}

// utv_lstsq with UTV_HOST_STREAMED: A (host, overwritten by T), B / X host or device.
int64_t lstsq_streamed(utv_handle h, int64_t m, int64_t n, int64_t k, double* A, int64_t lda, double* B, int64_t ldb,
                       double* X, int64_t ldx, const utv_opts& opt) {
  if (is_device_ptr(A)) fail(UTV_ERR_ARG, "UTV_HOST_STREAMED needs A in host memory");
  if (opt.flags & (UTV_NULLIFY_T12 | UTV_EXPLICIT_V))
    fail(UTV_ERR_UNSUPPORTED, "UTV_HOST_STREAMED is implemented for the fast option with factored V only");
  cudaStream_t st = h->stream;
  const int64_t b = opt.block;
  HostPin pin;
  pin.pin(A, m, n, lda);
  ooc_streams(h);
  h->ooc_h2d = h->ooc_d2h = 0;
  // fixed device memory: workspace, factored V, then the OOC arena (C, X, diag, panel, staging)
  Ctx c = make_ctx(h, m, n, k, b);
  const int64_t nsteps = (n + b - 1) / b;
  const size_t wdbl = factored_w_doubles(n, b), tdbl = (size_t)nsteps * b * b;
  ensure_buf(&h->vbuf, &h->vbuf_doubles, wdbl + 2 * tdbl + 64);
  FactoredV fv;
  fv.W = h->vbuf; fv.T = h->vbuf + wdbl; fv.Vs = fv.T + tdbl;
  static const int64_t chunk_blocks = [] {
    const char* e = std::getenv("UTV_OOC_CHUNK_BLOCKS");
    return e ? std::max<int64_t>(1, std::atoll(e)) : (int64_t)4;
  }();
  const int64_t cw = std::min<int64_t>(chunk_blocks * b, (n + b - 1) / b * b);
  const size_t kk = (size_t)std::max<int64_t>(k, 1);
  const size_t fixed = (size_t)m * kk + (size_t)n * kk + (size_t)n + 64 + 2 * (size_t)m * b +
                       (size_t)utv_handle_s::kStg * m * cw;
  size_t free_b = 0, total_b = 0;
  UTV_CUDA(cudaMemGetInfo(&free_b, &total_b));
  const size_t used_b = (h->ws_doubles + h->vbuf_doubles + h->ooc_doubles) * sizeof(double);
  size_t avail = free_b + h->ooc_doubles * sizeof(double);                 // the OOC arena is reused
  avail = avail > ((size_t)1 << 30) ? avail - ((size_t)1 << 30) : 0;       // 1 GiB head room
  if (h->dev_budget > 0) {
    const size_t cap = (size_t)h->dev_budget > used_b - h->ooc_doubles * sizeof(double)
                           ? (size_t)h->dev_budget - (used_b - h->ooc_doubles * sizeof(double)) : 0;
    avail = std::min(avail, cap);
  }
  if (avail < fixed * sizeof(double))
    fail(UTV_ERR_ALLOC, "device budget too small for the streamed working set (" +
                            std::to_string(fixed * sizeof(double) + used_b) + " bytes needed)");
  int64_t res_cols = (int64_t)((avail / sizeof(double) - fixed) / (size_t)m);
  if (const char* e = std::getenv("UTV_OOC_MAX_RESIDENT_COLS"))              // tests / benchmarks
    res_cols = std::min<int64_t>(res_cols, std::max<int64_t>(0, std::atoll(e)));
  Ooc o;
  o.h = h; o.m = m; o.n = n; o.b = b; o.hA = A; o.lda = lda; o.cw = cw;
  o.c_res = res_cols >= n ? 0 : std::min<int64_t>(n, (n - res_cols + b - 1) / b * b);
  const size_t total = fixed + (size_t)m * (n - o.c_res);
  if (h->ooc_doubles < total) {
    if (h->ooc) { UTV_CUDA(cudaFree(h->ooc)); h->ooc = nullptr; h->ooc_doubles = 0; }
    ensure_buf(&h->ooc, &h->ooc_doubles, total);
  }
  double* p = h->ooc;
  double* Cd = p; p += (size_t)m * kk;
  double* Xd = p; p += (size_t)n * kk;
  double* dg = p; p += (size_t)n + 64;
  o.pb[0] = p; p += (size_t)m * b;
  o.pb[1] = p; p += (size_t)m * b;
  for (int s = 0; s < utv_handle_s::kStg; ++s) { o.stg[s] = p; p += (size_t)m * cw; }
  o.res = p;
  h->ooc_resident_cols = n - o.c_res;
  if (k > 0) copy2d(st, Cd, m, B, ldb, m, k, is_device_ptr(B) ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice);
  factor_ooc(c, o, k > 0 ? Cd : nullptr, m, k, opt, &fv, dg);
  const int64_t r = finish_factor(c, n, dg, 0, opt.tau, true);              // ldt = 0: T_jj = dg[j]
  if (k > 0) {
    solve_z_ooc(c, o, r, Cd, m, k);
    solve_factored(c, n, r, nullptr, 0, nullptr, 0, k, Xd, n, fv, b, nullptr, true);
  }
  if (o.c_res < n) {                                                        // resident part of T
    UTV_CUDA(cudaEventRecord(h->ev_done, st));
    UTV_CUDA(cudaStreamWaitEvent(h->d2h, h->ev_done, 0));
    copy2d(h->d2h, A + cm(0, o.c_res, lda), lda, o.res, m, m, n - o.c_res, cudaMemcpyDeviceToHost);
    h->ooc_d2h += (n - o.c_res) * m * 8;
  }
  if (k > 0) {
    if (is_device_ptr(B)) copy2d(st, B, ldb, Cd, m, m, k, cudaMemcpyDeviceToDevice);
    copy2d(st, X, ldx, Xd, n, n, k, is_device_ptr(X) ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost);
  }
  UTV_CUDA(cudaStreamSynchronize(h->d2h));
  UTV_CUDA(cudaStreamSynchronize(st));
  return r;
}

// ------------------------------------------------------------------------------------------
// Multi-GPU randUTV least squares: 1D block-cyclic columns (block b, owner(blk) =
// blk mod P; each rank stores its blocks packed, in order); B / C and the small factors are
// replicated; the Philox sketch is counter-based, so every rank draws the same G.  Per step i
// (owner o = i mod P):
//   Z = sum_p A'_p Y_p                   AllReduce (m' x b), q times                 [a2]
//   Y rows of every rank                 AllGather; the same QR(Y) on every rank     [a3]
//   X = sum_p A_p W_V,p (all rows, R1)   AllReduce (m x b); local right update       [a4]
//   panel QR on o                        Broadcast (W_U, T_U)                        [a5]
//   fused two-sided update of the local blocks > i (K = 2b, as on one GPU); C := Q_U^T C [a6]
//   SVD on o                             Broadcast (U_s, V_s, sigma); local updates [a7]
// V stays factored and replicated (W_V, T_V, V_s are identical on every rank), so X = V z needs
// no communication; diag(T) is replicated through the sigma broadcasts (rank: no collective);
// the back substitution is block by block from the bottom with one AllReduce (partial sums of
// T_{blk, >blk} z) and one Broadcast (z_blk) per block.
// ------------------------------------------------------------------------------------------
int64_t dist_local_cols(int64_t n, int64_t b, int P, int p) {
  const int64_t nb = (n + b - 1) / b;
  int64_t c = 0;
  for (int64_t blk = p; blk < nb; blk += P) c += std::min(b, n - blk * b);
  return c;
}

size_t dist_dbuf_doubles(int64_t n, int64_t b, int P, int64_t k) {
  const int64_t nb = (n + b - 1) / b, Lmax = (nb + P - 1) / P * b;
  return (size_t)Lmax * b * (P + 1) + n + 64 + 2 * (size_t)b * (size_t)std::max<int64_t>(k, 1) + 64 +
         (size_t)(utv_handle_s::kLagMax + 1) * (size_t)(b * b + b);
}

// Every device allocation lstsq_dist makes, done up front (before the ranks agree on the call).
void dist_reserve(utv_handle h, int64_t m, int64_t n, int64_t k, const utv_opts& opt) {
  const int64_t b = opt.block, nsteps = (n + b - 1) / b;
  make_ctx(h, m, n, k, b);
  if (opt.flags & UTV_KEEP_FACTORS) {
    kept_prepare(h, m, n, b, true);
  } else {
    ensure_buf(&h->vbuf, &h->vbuf_doubles, factored_w_doubles(n, b) + 2 * (size_t)nsteps * b * b + 64);
  }
  ensure_buf(&h->dbuf, &h->dbuf_doubles, dist_dbuf_doubles(n, b, h->comm->nranks, k));
}

// The ranks of a multi-GPU handle agree on a call before its first collective: one AllReduce of
// "this rank failed its checks".  Any failure fails the call on every rank (no abort needed: no
// collective of the method was started, so the communicator stays usable).
void dist_agree(utv_handle h, utv_status local, const std::string& msg) {
  cudaStream_t st = h->stream;
  const double v = local != UTV_OK ? 1.0 : 0.0;
  double sum = 0.0;
  h->collective_phase = true;
  UTV_CUDA(cudaMemcpyAsync(h->agree, &v, sizeof(double), cudaMemcpyHostToDevice, st));
  h->comm->allreduce(h->agree, 1, st);
  UTV_CUDA(cudaMemcpyAsync(&sum, h->agree, sizeof(double), cudaMemcpyDeviceToHost, st));
  h->comm->wait(st);
  if (local != UTV_OK) { h->agreed_failure = true; fail(local, msg); }
  if (sum != 0.0) {
    h->agreed_failure = true;
    fail(UTV_ERR_ARG, "the call was rejected on " + std::to_string((int)sum) + " peer rank(s) (argument or "
                      "allocation error there); nothing was computed");
  }
}

// a9 on a block-cyclic T: z = T11^{-1} C(0:r, :) into the zsolve buffer (ld r), block by block from
// the bottom: one AllReduce of the partial sums T_{blk, >blk} z and one Broadcast of z_blk (from the
// block's owner) per block.  A = this rank's shard of T (lda), C replicated (ldc).
void dist_solve_z(const Ctx& c, Comm& comm, int64_t r, int64_t b, const double* A, int64_t lda, const double* Cm,
                  int64_t ldc, int64_t k) {
  if (r <= 0 || k <= 0) return;
  cudaStream_t st = c.st;
  const int P = comm.nranks, p = comm.rank;
  double* Zb = c.at(c.L.zsolve);
  double* Sp = c.at(c.L.nY);                                                             // my partial sums
  double* D = c.at(c.L.R);
  double* sbuf = c.at(c.L.tmp);                                                          // b x k
  double* zb = c.at(c.L.tmp2);                                                           // b x k
  launch_set_zero(st, r, k, Sp, r);
  for (int64_t blk = (r - 1) / b; blk >= 0; --blk) {
    const int64_t j0 = blk * b, j1 = std::min(r, j0 + b), w = j1 - j0;
    const int o = (int)(blk % P);
    launch_copy(st, w, k, Sp + j0, r, sbuf, w);
    comm.allreduce(sbuf, (size_t)w * k, st);                                             // sum_l T_blk,l z_l
    if (p == o) {
      const int64_t lc = (blk / P) * b;
      launch_copy(st, w, k, Cm + j0, ldc, zb, w);
      launch_axpy(st, w * k, -1.0, sbuf, zb);
      launch_copy(st, w, w, A + cm(j0, lc, lda), lda, D, b);
      launch_trsv_block(st, 0, w, D, b, zb, w, k);
      if (j0 > 0) c.gemm(false, false, j0, k, w, 1.0, A + cm(0, lc, lda), lda, zb, w, 1.0, Sp, r);
    }
    comm.bcast(zb, (size_t)w * k, o, st);
    launch_copy(st, w, k, zb, w, Zb + j0, r);
  }
}

// V's row block [v0, v0 + nrows) (nrows x n, ldv) from the factored V = Q_1 ... Q_s D (every rank
// holds the same factors): E^T V with the right multiplications applied in order, Q_1 first.
void factored_v_rows(const Ctx& c, const FactoredV& fv, int64_t n, int64_t b, int64_t v0, int64_t nrows, double* V,
                     int64_t ldv) {
  cudaStream_t st = c.st;
  if (nrows <= 0) return;
  launch_set_zero(st, nrows, n, V, ldv);
  launch_set_identity(st, nrows, nrows, V + cm(0, v0, ldv), ldv);
  double *t1 = c.at(c.L.X), *t2 = c.at(c.L.X2);
  for (size_t i = 0; i < fv.woff.size(); ++i) {                             // X := X Q_i
    const int64_t j0 = fv.j0[i], np = fv.np[i];
    const double* W = fv.W + fv.woff[i];
    double* Xc = V + cm(0, j0, ldv);
    c.gemm(false, false, nrows, b, np, 1.0, Xc, ldv, W, np, 0.0, t1, nrows);
    c.gemm(false, false, nrows, b, b, 1.0, t1, nrows, fv.T + (size_t)(j0 / b) * b * b, b, 0.0, t2, nrows);
    c.gemm(false, true, nrows, np, b, -1.0, t2, nrows, W, np, 1.0, Xc, ldv);
  }
  for (int64_t j0 = 0, step = 0; j0 < n; j0 += b, ++step) {                 // X := X D
    const int64_t bw = std::min(b, n - j0);
    c.gemm(false, false, nrows, bw, bw, 1.0, V + cm(0, j0, ldv), ldv, fv.Vs + (size_t)step * b * b, b, 0.0, t1, nrows);
    launch_copy(st, nrows, bw, t1, nrows, V + cm(0, j0, ldv), ldv);
  }
}

// Rows of V held by rank p (contiguous row blocks of ceil(n / P)).
void dist_v_rows(int64_t n, int P, int p, int64_t* v0, int64_t* nrows) {
  const int64_t per = (n + P - 1) / P;
  *v0 = std::min<int64_t>(n, (int64_t)p * per);
  *nrows = std::min<int64_t>(n, *v0 + per) - *v0;
}

int64_t lstsq_dist(utv_handle h, int64_t m, int64_t n, int64_t k, double* A, int64_t lda, double* B, int64_t ldb,
                   double* X, int64_t ldx, const utv_opts& opt, bool solve = true, double* Vrows = nullptr,
                   int64_t ldv = 0) {
  Comm& comm = *h->comm;
  const int P = comm.nranks, p = comm.rank;
  const int64_t b = opt.block, nb = (n + b - 1) / b;
  const int64_t nloc = dist_local_cols(n, b, P, p);
  cudaStream_t st = h->stream, cs = h->cst;
  h->dist_block = b;
  const int ns = h->num_sms;
  Ctx c = make_ctx(h, m, n, k, b);
  const Layout& L = c.L;
  const int64_t nsteps = nb;
  const size_t wdbl = factored_w_doubles(n, b), tdbl = (size_t)nsteps * b * b;
  const bool keep = (opt.flags & UTV_KEEP_FACTORS) != 0;
  Kept* kp = keep ? &kept_prepare(h, m, n, b, true) : nullptr;
  FactoredV fv_local;
  if (!keep) {
    ensure_buf(&h->vbuf, &h->vbuf_doubles, wdbl + 2 * tdbl + 64);
    fv_local.W = h->vbuf; fv_local.T = h->vbuf + wdbl; fv_local.Vs = fv_local.T + tdbl;
  }
  FactoredV& fv = keep ? kp->fv : fv_local;
  const int64_t Lmax = (nb + P - 1) / P * b;
  const size_t kk = (size_t)std::max<int64_t>(k, 1);
  ensure_buf(&h->dbuf, &h->dbuf_doubles, dist_dbuf_doubles(n, b, P, k));
  double* Ypad = h->dbuf;
  double* recv = Ypad + (size_t)Lmax * b;
  double* dg = recv + (size_t)P * Lmax * b;
  double* sbuf = dg + n + 64;
  double* zb = sbuf + (size_t)b * kk;
  double* flags = zb + (size_t)b * kk;
  double* usring = flags + 64;                                   // (kLagMax+1) x b^2: pending U_s
  double* sgring = usring + (size_t)(utv_handle_s::kLagMax + 1) * b * b;   // (kLagMax+1) x b: sigma
  UTV_CUDA(cudaMemsetAsync(h->info, 0, 4 * sizeof(int), st));
  UTV_CUDA(cudaMemsetAsync(h->flag, 0, sizeof(int), st));
  if (nloc > 0) launch_check_finite(st, m, nloc, A, lda, h->flag);
  if (k > 0) launch_check_finite(st, m, k, B, ldb, h->flag);
  double *G = c.at(L.G), *Y = c.at(L.Y), *Z = c.at(L.Z), *WP = c.at(L.Wv), *Xa = c.at(L.X), *LU = c.at(L.Wu);
  double *Tu = c.at(L.Tu), *tauu = c.at(L.tauu), *tauv = c.at(L.tauv), *S = c.at(L.S), *Z1 = c.at(L.Z1);
  double *Z2 = c.at(L.Z2), *Yl = c.at(L.tmp);

  // Column chunks of the b sketch columns: the power iteration is column-separable
  // (Y = (A'^T A')^q A'^T G, one column of G at a time), and so is X = A W_V, so chunk c's
  // AllReduce (communication stream) overlaps chunk c+1's GEMM (main stream).  SURVEY 8(e) overlap.
  const int nch = (int)std::max<int64_t>(1, std::min<int64_t>(g_dist_chunks > 0 ? g_dist_chunks : (P > 1 ? 2 : 1), b));
  auto chunk = [&](int q, int64_t* c0, int64_t* c1) {
    *c0 = b * q / nch; *c1 = b * (q + 1) / nch;
  };
  // comm stream joins the main stream's history once (buffers it reduces were written there)
  UTV_CUDA(cudaEventRecord(h->ev_panel, st));
  UTV_CUDA(cudaStreamWaitEvent(cs, h->ev_panel, 0));
  // produce(q) enqueues chunk q's product on the main stream; its AllReduce goes to the comm
  // stream; join() makes the main stream wait for every chunk's reduction.
  auto reduce_chunk = [&](int q, double* buf, size_t cnt) {
    UTV_CUDA(cudaEventRecord(h->ev_cq[q], st));
    UTV_CUDA(cudaStreamWaitEvent(cs, h->ev_cq[q], 0));
    comm.allreduce(buf, cnt, cs);
    UTV_CUDA(cudaEventRecord(h->ev_cd[q], cs));
  };
  auto wait_chunk = [&](int q) { UTV_CUDA(cudaStreamWaitEvent(st, h->ev_cd[q], 0)); };

  // a7 of block i runs on its owner's side stream right after block i's panel QR; everything it
  // changes in A (A11 := Sigma excepted), C and diag(T) is applied on the main stream `lag` steps
  // later, in block order, on every rank (broadcast from the owner).  Reading H5: U_s^T acts on
  // rows of block i that later steps only right-multiply (A12, and the top-row updates), and A01 V_s
  // on columns no later step reads, so left and right factors commute; applying them on the main
  // stream in block order keeps every read-modify-write of those rows / columns ordered.
  const int lag = (int)std::max<int64_t>(1, g_svd_lag > 0 ? g_svd_lag : (P > 1 ? utv_handle_s::kLagMax : 1));
  struct Pend { int64_t i, j0, bw, lt, lr, nrl; int owner; };
  std::vector<Pend> pend;                          // FIFO (front = oldest)
  size_t pend_head = 0;
  auto apply_front = [&]() {
    const Pend e = pend[pend_head++];
    const int slot = (int)(e.i % (utv_handle_s::kLagMax + 1));
    double* Usp = kp ? kp->Us + (size_t)e.i * b * b : usring + (size_t)slot * b * b;
    double* sgp = sgring + (size_t)slot * b;
    double* Vsp = fv.Vs + (size_t)e.i * b * b;
    if (p == e.owner) UTV_CUDA(cudaStreamWaitEvent(st, h->ev_svdq[slot], 0));
    comm.bcast(Usp, (size_t)b * b, e.owner, st);
    comm.bcast(Vsp, (size_t)b * b, e.owner, st);
    comm.bcast(sgp, (size_t)b, e.owner, st);
    launch_copy(st, e.bw, 1, sgp, e.bw, dg + e.j0, n);
    if (p == e.owner && e.j0 > 0) {                                                    // A01 := A01 V_s
      double* A01 = A + cm(0, e.lt, lda);
      c.gemm(false, false, e.j0, e.bw, e.bw, 1.0, A01, lda, Vsp, b, 0.0, Yl, e.j0);
      launch_copy(st, e.j0, e.bw, Yl, e.j0, A01, lda);
    }
    if (e.nrl > 0) {                                                                    // A12 := U_s^T A12
      double* A12 = A + cm(e.j0, e.lr, lda);
      c.gemm(true, false, e.bw, e.nrl, e.bw, 1.0, Usp, b, A12, lda, 0.0, Yl, e.bw);
      launch_copy(st, e.bw, e.nrl, Yl, e.bw, A12, lda);
    }
    if (k > 0) {                                                                        // C1 := U_s^T C1
      c.gemm(true, false, e.bw, k, e.bw, 1.0, Usp, b, B + e.j0, ldb, 0.0, Z1, e.bw);
      launch_copy(st, e.bw, k, Z1, e.bw, B + e.j0, ldb);
    }
  };
  for (int64_t i = 0, j0 = 0; i < nb; ++i, j0 += b) {
    const int64_t bw = std::min(b, n - j0), mp = m - j0, np = n - j0;
    const int owner = (int)(i % P);
    const bool own = p == owner;
    const int64_t first = i <= p ? 0 : (i - p + P - 1) / P;            // my first block >= i
    const int64_t lt = first * b, ncl = nloc - lt;                     // my trailing columns
    const int64_t lr = lt + (own ? bw : 0), nrl = ncl - (own ? bw : 0); // my columns > block i
    const int64_t ldwp = std::max<int64_t>(ncl, 1);
    const bool right = np > b;                                          // R5
    double* X2 = LU;
    double* Wu = LU + cm(j0, b, m);
    double* At = A + cm(j0, lt, lda);
    if (right) {
      double* Tvs = fv.T + (size_t)i * b * b;
      launch_sketch(st, opt.seed, i, j0, mp, b, G, mp, ns);                           // a1
      if (ncl) c.gemm(true, false, ncl, b, mp, 1.0, At, lda, G, mp, 0.0, Yl, ldwp);
      for (int32_t it = 0; it < opt.power_iters; ++it) {                              // a2 (R7)
        for (int q = 0; q < nch; ++q) {                                               // Z_q = A' Y_q
          int64_t c0, c1; chunk(q, &c0, &c1);
          double* Zq = Z + (size_t)mp * c0;
          if (ncl) c.gemm(false, false, mp, c1 - c0, ncl, 1.0, At, lda, Yl + c0 * ldwp, ldwp, 0.0, Zq, mp);
          else launch_set_zero(st, mp, c1 - c0, Zq, mp);
          reduce_chunk(q, Zq, (size_t)mp * (c1 - c0));                                // AllReduce(Z_q)
        }
        for (int q = 0; q < nch; ++q) {                                               // Y_q = A'^T Z_q
          int64_t c0, c1; chunk(q, &c0, &c1);
          wait_chunk(q);
          if (ncl) c.gemm(true, false, ncl, c1 - c0, mp, 1.0, At, lda, Z + (size_t)mp * c0, mp, 0.0, Yl + c0 * ldwp,
                          ldwp);
        }
      }
      launch_copy(st, ncl, b, Yl, ldwp, Ypad, Lmax);                                  // AllGather(Y)
      comm.allgather(Ypad, recv, (size_t)Lmax * b, st);
      launch_assemble_y(st, np, b, b, i, P, Lmax, recv, Y, np);
      fv.woff.push_back(fv.woff.empty() ? 0 : fv.woff.back() + (size_t)fv.np.back() * b);
      fv.j0.push_back(j0); fv.np.push_back(np); fv.has_q.push_back(1);
      double* Wv = fv.W + fv.woff.back();
      panel_qr(st, np, b, Y, np, Wv, np, tauv, Tvs, b, c.pw);                          // a3 (same on all)
      launch_gather_local(st, ncl, b, b, i, P, p, Wv, np, WP, ldwp);                   // my rows of W_V
      for (int q = 0; q < nch; ++q) {                                                 // X_q = A W_V,q
        int64_t c0, c1; chunk(q, &c0, &c1);
        double* Xq = Xa + (size_t)m * c0;
        if (ncl) c.gemm(false, false, m, c1 - c0, ncl, 1.0, A + cm(0, lt, lda), lda, WP + c0 * ldwp, ldwp, 0.0, Xq, m);
        else launch_set_zero(st, m, c1 - c0, Xq, m);
        reduce_chunk(q, Xq, (size_t)m * (c1 - c0));                                   // a4, R1: AllReduce
      }
      for (int q = 0; q < nch; ++q) wait_chunk(q);
      c.gemm(false, false, m, b, b, 1.0, Xa, m, Tvs, b, 0.0, X2, m);
      if (j0 > 0 && ncl) c.gemm(false, true, j0, ncl, b, -1.0, X2, m, WP, ldwp, 1.0, A + cm(0, lt, lda), lda);
      if (own) c.gemm(false, true, mp, bw, b, -1.0, X2 + j0, m, WP, ldwp, 1.0, At, lda);
    }
    // a5 on the owner; Broadcast(W_U) of the live rows j0:m only, packed (Xa is free here)
    if (own) {
      panel_qr(st, mp, bw, At, lda, Wu, m, tauu, Tu, b, c.pw);
      launch_copy(st, mp, bw, Wu, m, Xa, mp);
    }
    comm.bcast(Xa, (size_t)mp * bw, owner, st);
    if (!own) launch_copy(st, mp, bw, Xa, mp, Wu, m);
    comm.bcast(Tu, (size_t)b * b, owner, st);
    if (kp) kept_push_u(st, *kp, i, mp, bw, Wu, m, Tu);                                  // keep W_U, T_U
    if (nrl > 0) {                                                                      // a6, R3
      double* Ar = A + cm(j0, lr, lda);
      c.gemm(true, false, bw, nrl, mp, 1.0, Wu, m, Ar, lda, 0.0, Z1, bw);
      if (right) {
        double* Wr = WP + (own ? bw : 0);
        c.gemm(true, false, bw, b, mp, 1.0, Wu, m, X2 + j0, m, 0.0, S, bw);
        c.gemm(false, true, bw, nrl, b, -1.0, S, bw, Wr, ldwp, 1.0, Z1, bw);
        c.gemm(true, false, nrl, bw, bw, 1.0, Z1, bw, Tu, b, 0.0, Wr + cm(0, b, ldwp), ldwp);
        c.gemm(false, true, mp, nrl, 2 * b, -1.0, X2 + j0, m, Wr, ldwp, 1.0, Ar, lda);  // fused, K = 2b
      } else {
        c.gemm(true, false, bw, nrl, bw, 1.0, Tu, b, Z1, bw, 0.0, Z2, bw);
        c.gemm(false, false, mp, nrl, bw, -1.0, Wu, m, Z2, bw, 1.0, Ar, lda);
      }
    }
    if (k > 0) {                                                                        // C := Q_U^T C
      double* Cr = B + j0;
      c.gemm(true, false, bw, k, mp, 1.0, Wu, m, Cr, ldb, 0.0, Z1, bw);
      c.gemm(true, false, bw, k, bw, 1.0, Tu, b, Z1, bw, 0.0, Z2, bw);
      c.gemm(false, false, mp, k, bw, -1.0, Wu, m, Z2, bw, 1.0, Cr, ldb);
    }
    // a7: the owner's side stream computes (U_s, sigma, V_s) of R = A11 and writes A11 := Sigma
    // (nothing on the main stream touches A11 after the panel QR); the rest is applied `lag` steps
    // later (apply_front), at the same point of every rank's sequence of collectives.
    if (own) {
      const int slot = (int)(i % (utv_handle_s::kLagMax + 1));
      double* Vsi = fv.Vs + (size_t)i * b * b;
      double* Usi = kp ? kp->Us + (size_t)i * b * b : usring + (size_t)slot * b * b;
      double* sgi = sgring + (size_t)slot * b;
      UTV_CUDA(cudaEventRecord(h->ev_panel, st));
      UTV_CUDA(cudaStreamWaitEvent(c.side, h->ev_panel, 0));
      svd_small(c.side, bw, At, lda, Usi, b, sgi, Vsi, b, c.sw);
      launch_set_diag(c.side, bw, sgi, At, lda);
      UTV_CUDA(cudaEventRecord(h->ev_svdq[slot], c.side));
    }
    pend.push_back(Pend{i, j0, bw, lt, lr, nrl, owner});
    while (pend.size() - pend_head > (size_t)lag) apply_front();
  }
  while (pend_head < pend.size()) apply_front();
  // every rank fails alike: AllReduce the local NaN / Jacobi flags (the owners' side-stream SVDs
  // were all joined by apply_front)
  UTV_CUDA(cudaMemcpyAsync(h->h_info, h->info, 2 * sizeof(int), cudaMemcpyDeviceToHost, st));
  UTV_CUDA(cudaMemcpyAsync(h->h_info + 2, h->flag, sizeof(int), cudaMemcpyDeviceToHost, st));
  comm.wait(st);
  const double fl[2] = {(double)h->h_info[2], (double)h->h_info[1]};
  UTV_CUDA(cudaMemcpyAsync(flags, fl, sizeof(fl), cudaMemcpyHostToDevice, st));
  comm.allreduce(flags, 2, st);
  double flo[2] = {0.0, 0.0};
  UTV_CUDA(cudaMemcpyAsync(flo, flags, sizeof(flo), cudaMemcpyDeviceToHost, st));
  comm.wait(st);
  h->agreed_failure = flo[0] != 0.0 || flo[1] != 0.0;                                    // every rank fails alike
  if (flo[0] != 0.0) fail(UTV_ERR_NUMERICAL, "NaN or Inf in A or B (on some rank)");
  if (flo[1] != 0.0) fail(UTV_ERR_NUMERICAL, "Jacobi SVD of a diagonal block did not converge in 30 sweeps");
  const int64_t r = finish_factor(c, n, dg, 0, opt.tau, true);                          // a8 (replicated)
  if (kp) { kp->r = r; kp->valid = true; }
  if (!solve) {                                                                          // utv_factor
    if (Vrows) {
      int64_t v0, nv;
      dist_v_rows(n, P, p, &v0, &nv);
      factored_v_rows(c, fv, n, b, v0, nv, Vrows, ldv);
    }
    comm.wait(st);
    return r;
  }
  if (k <= 0) return r;
  dist_solve_z(c, comm, r, b, A, lda, B, ldb, k);                                        // a9
  solve_factored(c, n, r, nullptr, 0, nullptr, 0, k, X, ldx, fv, b, nullptr, true);      // X = V z (replicated)
  comm.wait(st);
  return r;
}

// ------------------------------------------------------------------------------------------
// Multi-GPU x out-of-core (SURVEY 8(e) with 8(f) #1; the north star's cfg5: "tiles streamed from
// pinned host memory across 8 x B200"): each rank's block-cyclic shard (m x nloc) stays in ITS
// pinned host memory and is overwritten by its shard of T there; HBM holds the rank's workspace,
// the replicated factored V, a staging ring and as many of its LAST local column blocks as the
// device budget allows (utv_set_device_budget), exactly as factor_ooc on one GPU.  The collectives
// are those of lstsq_dist (AllReduce Z / X, AllGather Y, Broadcast W_U / T_U / U_s / V_s / sigma);
// per step the rank streams its trailing columns 2q + 2 times and writes them back once (the
// right update of all rows, the deferred U_s^T of the previous block, Q_U^T, and the next step's
// local sketch product in one read+write pass).  The SVD of block i (owner's side stream) is
// applied one step later (lag 1, folded into the next step's pass, as on one GPU).
// ------------------------------------------------------------------------------------------

// The rank's out-of-core arena (two panel buffers, the staging ring, the resident last blocks),
// sized under the device budget; all device allocations happen here, before the ranks agree.
void dist_ooc_prepare(utv_handle h, Ooc& o, int64_t m, int64_t n, int64_t k, double* A, int64_t lda,
                      const utv_opts& opt) {
  const int P = h->comm->nranks, p = h->comm->rank;
  const int64_t b = opt.block, nloc = dist_local_cols(n, b, P, p);
  dist_reserve(h, m, n, k, opt);
  ooc_streams(h);
  h->ooc_h2d = h->ooc_d2h = 0;
  static const int64_t chunk_blocks = [] {
    const char* e = std::getenv("UTV_OOC_CHUNK_BLOCKS");
    return e ? std::max<int64_t>(1, std::atoll(e)) : (int64_t)4;
  }();
  const int64_t cw = std::max<int64_t>(b, std::min<int64_t>(chunk_blocks * b, (nloc + b - 1) / b * b));
  const size_t fixed = 2 * (size_t)m * b + (size_t)utv_handle_s::kStg * m * cw + 64;
  size_t free_b = 0, total_b = 0;
  UTV_CUDA(cudaMemGetInfo(&free_b, &total_b));
  const size_t used_b = (h->ws_doubles + h->vbuf_doubles + h->dbuf_doubles + h->ooc_doubles) * sizeof(double);
  size_t avail = free_b + h->ooc_doubles * sizeof(double);
  avail = avail > ((size_t)1 << 30) ? avail - ((size_t)1 << 30) : 0;
  if (h->dev_budget > 0) {
    const size_t base = used_b - h->ooc_doubles * sizeof(double);
    avail = std::min(avail, (size_t)h->dev_budget > base ? (size_t)h->dev_budget - base : (size_t)0);
  }
  if (avail < fixed * sizeof(double))
    fail(UTV_ERR_ALLOC, "device budget too small for the streamed working set of this rank");
  int64_t res_cols = (int64_t)((avail / sizeof(double) - fixed) / (size_t)m);
  if (const char* e = std::getenv("UTV_OOC_MAX_RESIDENT_COLS"))
    res_cols = std::min<int64_t>(res_cols, std::max<int64_t>(0, std::atoll(e)));
  o = Ooc{};
  o.h = h; o.m = m; o.n = nloc; o.b = b; o.hA = A; o.lda = lda; o.cw = cw;
  o.c_res = res_cols >= nloc ? 0 : std::min<int64_t>(nloc, (nloc - res_cols + b - 1) / b * b);
  const size_t total = fixed + (size_t)m * (nloc - o.c_res);
  if (h->ooc_doubles < total) {
    if (h->ooc) { UTV_CUDA(cudaFree(h->ooc)); h->ooc = nullptr; h->ooc_doubles = 0; }
    ensure_buf(&h->ooc, &h->ooc_doubles, total);
  }
  double* q = h->ooc;
  o.pb[0] = q; q += (size_t)m * b;
  o.pb[1] = q; q += (size_t)m * b;
  for (int s = 0; s < utv_handle_s::kStg; ++s) { o.stg[s] = q; q += (size_t)m * cw; }
  o.res = q;
  h->ooc_resident_cols = nloc - o.c_res;
}

// a9 on a block-cyclic T kept in the ranks' host memory: dist_solve_z with the owner's T column
// block fetched (rows 0:j1) through the out-of-core arena.
void dist_solve_z_ooc(const Ctx& c, Comm& comm, Ooc& o, int64_t r, int64_t b, const double* Cm, int64_t ldc,
                      int64_t k) {
  if (r <= 0 || k <= 0) return;
  cudaStream_t st = c.st;
  const int P = comm.nranks, p = comm.rank;
  double* Zb = c.at(c.L.zsolve);
  double* Sp = c.at(c.L.nY);
  double* D = c.at(c.L.R);
  double* sbuf = c.at(c.L.tmp);
  double* zb = c.at(c.L.tmp2);
  launch_set_zero(st, r, k, Sp, r);
  for (int64_t blk = (r - 1) / b; blk >= 0; --blk) {
    const int64_t j0 = blk * b, j1 = std::min(r, j0 + b), w = j1 - j0;
    const int o_ = (int)(blk % P);
    launch_copy(st, w, k, Sp + j0, r, sbuf, w);
    comm.allreduce(sbuf, (size_t)w * k, st);
    if (p == o_) {
      const int64_t lc = (blk / P) * b;
      int64_t ldt = o.m;
      const double* Tb = ooc_block(o, c, lc, w, j1, &ldt);
      launch_copy(st, w, k, Cm + j0, ldc, zb, w);
      launch_axpy(st, w * k, -1.0, sbuf, zb);
      launch_copy(st, w, w, Tb + j0, ldt, D, b);
      launch_trsv_block(st, 0, w, D, b, zb, w, k);
      if (j0 > 0) c.gemm(false, false, j0, k, w, 1.0, Tb, ldt, zb, w, 1.0, Sp, r);
    }
    comm.bcast(zb, (size_t)w * k, o_, st);
    launch_copy(st, w, k, zb, w, Zb + j0, r);
  }
}

int64_t lstsq_dist_ooc(utv_handle h, Ooc& o, int64_t m, int64_t n, int64_t k, double* B, int64_t ldb, double* X,
                       int64_t ldx, const utv_opts& opt) {
  Comm& comm = *h->comm;
  const int P = comm.nranks, p = comm.rank;
  const int64_t b = opt.block, nb = (n + b - 1) / b, nloc = o.n;
  cudaStream_t st = h->stream;
  h->dist_block = b;
  const int ns = h->num_sms;
  Ctx c = make_ctx(h, m, n, k, b);
  const Layout& L = c.L;
  const size_t wdbl = factored_w_doubles(n, b), tdbl = (size_t)nb * b * b;
  FactoredV fv;
  fv.W = h->vbuf; fv.T = h->vbuf + wdbl; fv.Vs = fv.T + tdbl;
  const int64_t Lmax = (nb + P - 1) / P * b;
  const size_t kk = (size_t)std::max<int64_t>(k, 1);
  double* Ypad = h->dbuf;
  double* recv = Ypad + (size_t)Lmax * b;
  double* dg = recv + (size_t)P * Lmax * b;
  double* sbuf = dg + n + 64;
  double* zb = sbuf + (size_t)b * kk;
  double* flags = zb + (size_t)b * kk;
  double* usring = flags + 64;
  double* sgring = usring + (size_t)(utv_handle_s::kLagMax + 1) * b * b;
  UTV_CUDA(cudaMemsetAsync(h->info, 0, 4 * sizeof(int), st));
  UTV_CUDA(cudaMemsetAsync(h->flag, 0, sizeof(int), st));
  if (k > 0) launch_check_finite(st, m, k, B, ldb, h->flag);
  double *G = c.at(L.G), *Y = c.at(L.Y), *Z = c.at(L.Z), *WP = c.at(L.Wv), *Xa = c.at(L.X), *LU = c.at(L.Wu);
  double *Tu = c.at(L.Tu), *tauu = c.at(L.tauu), *tauv = c.at(L.tauv), *Z1 = c.at(L.Z1), *Z2 = c.at(L.Z2);
  double *Yl = c.at(L.tmp), *tmp = c.at(L.tmp2);
  double* X2 = LU;
  if (o.c_res < nloc) {                                              // resident local blocks: loaded once
    UTV_CUDA(cudaEventRecord(h->ev_done, st));
    UTV_CUDA(cudaStreamWaitEvent(h->h2d, h->ev_done, 0));
    ooc_load(o, c, o.res, m, 0, m, o.c_res, nloc - o.c_res, h->ev_loaded[0]);
    launch_check_finite(st, m, nloc - o.c_res, o.res, m, h->flag);
  }
  bool y_ready = false;
  bool fin = false;                                                  // block i-1's SVD results pending
  int64_t f_i = 0, f_j0 = 0, f_bw = 0, f_lt = 0;
  int f_owner = 0;
  auto slot_us = [&](int64_t i) { return usring + (size_t)(i % (utv_handle_s::kLagMax + 1)) * b * b; };
  auto slot_sg = [&](int64_t i) { return sgring + (size_t)(i % (utv_handle_s::kLagMax + 1)) * b; };
  // the SVD results of block i-1 (f_*): broadcast; diag(T); C1 := U_s^T C1; on its owner the block
  // is finalised (A11 := Sigma, A01 := A01 V_s) and written back from panel buffer (f_i & 1)
  auto finalize = [&]() {
    double* Usp = slot_us(f_i);
    double* sgp = slot_sg(f_i);
    double* Vsp = fv.Vs + (size_t)f_i * b * b;
    if (p == f_owner) UTV_CUDA(cudaStreamWaitEvent(st, h->ev_svd, 0));
    comm.bcast(Usp, (size_t)b * b, f_owner, st);
    comm.bcast(Vsp, (size_t)b * b, f_owner, st);
    comm.bcast(sgp, (size_t)b, f_owner, st);
    launch_copy(st, f_bw, 1, sgp, f_bw, dg + f_j0, n);
    if (p == f_owner) {
      const bool resident = f_lt >= o.c_res;
      double* Af = resident ? o.res + cm(0, f_lt - o.c_res, m) : o.pb[f_i & 1];
      launch_set_diag(st, f_bw, sgp, Af + f_j0, m);
      if (f_j0 > 0) {
        c.gemm(false, false, f_j0, f_bw, f_bw, 1.0, Af, m, Vsp, b, 0.0, tmp, f_j0);
        launch_copy(st, f_j0, f_bw, tmp, f_j0, Af, m);
      }
      ooc_block_store(o, c, f_lt, f_bw, (int)(f_i & 1));
    }
    if (k > 0) {
      c.gemm(true, false, f_bw, k, f_bw, 1.0, Usp, b, B + f_j0, ldb, 0.0, Z1, f_bw);
      launch_copy(st, f_bw, k, Z1, f_bw, B + f_j0, ldb);
    }
  };
  for (int64_t i = 0, j0 = 0; i < nb; ++i, j0 += b) {
    const int64_t bw = std::min(b, n - j0), mp = m - j0, np = n - j0;
    const int owner = (int)(i % P);
    const bool own = p == owner;
    const int64_t first = i <= p ? 0 : (i - p + P - 1) / P;
    const int64_t lt = first * b, ncl = nloc - lt;
    const int64_t lr = lt + (own ? bw : 0), nrl = ncl - (own ? bw : 0);
    const int64_t ldwp = std::max<int64_t>(ncl, 1);
    const bool right = np > b;
    double* Wu = LU + cm(j0, b, m);
    double* Tvs = fv.T + (size_t)i * b * b;
    if (right) {
      if (!y_ready) {                                                  // a1 + local Y = A'^T G
        launch_sketch(st, opt.seed, i, j0, mp, b, G, mp, ns);
        ooc_pass(o, c, lt, j0, false, [&](double* d, int64_t ld, int64_t col, int64_t w) {
          if (i == 0 && col < o.c_res) launch_check_finite(st, mp, w, d, ld, h->flag);
          c.gemm(true, false, w, b, mp, 1.0, d, ld, G, mp, 0.0, Yl + (col - lt), ldwp);
        });
      }
      for (int32_t it = 0; it < opt.power_iters; ++it) {              // a2 (R7)
        launch_set_zero(st, mp, b, Z, mp);
        ooc_pass(o, c, lt, j0, false, [&](double* d, int64_t ld, int64_t col, int64_t w) {
          c.gemm(false, false, mp, b, w, 1.0, d, ld, Yl + (col - lt), ldwp, 1.0, Z, mp);
        });
        comm.allreduce(Z, (size_t)mp * b, st);
        ooc_pass(o, c, lt, j0, false, [&](double* d, int64_t ld, int64_t col, int64_t w) {
          c.gemm(true, false, w, b, mp, 1.0, d, ld, Z, mp, 0.0, Yl + (col - lt), ldwp);
        });
      }
      launch_copy(st, ncl, b, Yl, ldwp, Ypad, Lmax);                   // AllGather(Y)
      comm.allgather(Ypad, recv, (size_t)Lmax * b, st);
      launch_assemble_y(st, np, b, b, i, P, Lmax, recv, Y, np);
      fv.woff.push_back(fv.woff.empty() ? 0 : fv.woff.back() + (size_t)fv.np.back() * b);
      fv.j0.push_back(j0); fv.np.push_back(np); fv.has_q.push_back(1);
      double* Wv = fv.W + fv.woff.back();
      panel_qr(st, np, b, Y, np, Wv, np, tauv, Tvs, b, c.pw);          // a3 (same on every rank)
      launch_gather_local(st, ncl, b, b, i, P, p, Wv, np, WP, ldwp);
      launch_set_zero(st, m, b, Xa, m);                                // a4, R1: X = A W_V, all rows
      ooc_pass(o, c, lt, 0, false, [&](double* d, int64_t ld, int64_t col, int64_t w) {
        c.gemm(false, false, m, b, w, 1.0, d, ld, WP + (col - lt), ldwp, 1.0, Xa, m);
      });
      comm.allreduce(Xa, (size_t)m * b, st);
      c.gemm(false, false, m, b, b, 1.0, Xa, m, Tvs, b, 0.0, X2, m);
    }
    // block i on its owner: right update (all rows), the previous block's U_s^T on its rows
    int64_t lda_i = m;
    double* Ai = nullptr;
    if (own) {
      Ai = ooc_block(o, c, lt, bw, m, &lda_i, (int)(i & 1));
      if (i == 0 && !right && lt < o.c_res) launch_check_finite(st, m, bw, Ai, lda_i, h->flag);
      if (right) c.gemm(false, true, m, bw, b, -1.0, X2, m, WP, ldwp, 1.0, Ai, lda_i);
    }
    bool us_pend = false;
    const double* Usp = nullptr;
    int64_t pj0 = 0, pbw = 0;
    if (fin) {
      finalize();
      Usp = slot_us(f_i); pj0 = f_j0; pbw = f_bw;
      if (own) {                                                       // block i's part of A12(i-1)
        c.gemm(true, false, pbw, bw, pbw, 1.0, Usp, b, Ai + pj0, lda_i, 0.0, Z1, pbw);
        launch_copy(st, pbw, bw, Z1, pbw, Ai + pj0, lda_i);
      }
      us_pend = nrl > 0;
      fin = false;
    }
    // a5 on the owner; Broadcast(W_U) of the live rows (packed), T_U
    if (own) {
      panel_qr(st, mp, bw, Ai + j0, lda_i, Wu, m, tauu, Tu, b, c.pw);
      launch_copy(st, mp, bw, Wu, m, Xa, mp);
    }
    comm.bcast(Xa, (size_t)mp * bw, owner, st);
    if (!own) launch_copy(st, mp, bw, Xa, mp, Wu, m);
    comm.bcast(Tu, (size_t)b * b, owner, st);
    if (k > 0) {                                                       // C := Q_U^T C
      double* Cr = B + j0;
      c.gemm(true, false, bw, k, mp, 1.0, Wu, m, Cr, ldb, 0.0, Z1, bw);
      c.gemm(true, false, bw, k, bw, 1.0, Tu, b, Z1, bw, 0.0, Z2, bw);
      c.gemm(false, false, mp, k, bw, -1.0, Wu, m, Z2, bw, 1.0, Cr, ldb);
    }
    if (own) {                                                         // a7 on the side stream
      UTV_CUDA(cudaEventRecord(h->ev_panel, st));
      UTV_CUDA(cudaStreamWaitEvent(c.side, h->ev_panel, 0));
      svd_small(c.side, bw, Ai + j0, lda_i, slot_us(i), b, slot_sg(i), fv.Vs + (size_t)i * b * b, b, c.sw);
      UTV_CUDA(cudaEventRecord(h->ev_svd, c.side));
    }
    // one read+write pass over this rank's columns > block i (+ the next step's local sketch)
    const bool next_sketch = np - bw > b;                              // the same on every rank
    if (next_sketch) launch_sketch(st, opt.seed, i + 1, j0 + b, mp - b, b, G, mp - b, ns);
    const int64_t ldwn = std::max<int64_t>(nrl, 1);                    // next step's local Y
    if (nrl > 0) {
      ooc_pass(o, c, lr, 0, true, [&](double* d, int64_t ld, int64_t col, int64_t w) {
        if (right) c.gemm(false, true, m, w, b, -1.0, X2, m, WP + (col - lt), ldwp, 1.0, d, ld);
        if (us_pend) {                                                 // A12(i-1) := U_s^T A12
          c.gemm(true, false, pbw, w, pbw, 1.0, Usp, b, d + pj0, ld, 0.0, Z1, pbw);
          launch_copy(st, pbw, w, Z1, pbw, d + pj0, ld);
        }
        double* dr = d + j0;                                           // a6, R3
        c.gemm(true, false, bw, w, mp, 1.0, Wu, m, dr, ld, 0.0, Z1, bw);
        c.gemm(true, false, bw, w, bw, 1.0, Tu, b, Z1, bw, 0.0, Z2, bw);
        c.gemm(false, false, mp, w, bw, -1.0, Wu, m, Z2, bw, 1.0, dr, ld);
        if (next_sketch)
          c.gemm(true, false, w, b, mp - b, 1.0, d + j0 + b, ld, G, mp - b, 0.0, Yl + (col - lr), ldwn);
      });
    }
    y_ready = next_sketch;
    fin = true;
    f_i = i; f_j0 = j0; f_bw = bw; f_lt = lt; f_owner = owner;
  }
  if (fin) finalize();                                                 // the last block
  UTV_CUDA(cudaMemcpyAsync(h->h_info, h->info, 2 * sizeof(int), cudaMemcpyDeviceToHost, st));
  UTV_CUDA(cudaMemcpyAsync(h->h_info + 2, h->flag, sizeof(int), cudaMemcpyDeviceToHost, st));
  comm.wait(st);
  const double fl[2] = {(double)h->h_info[2], (double)h->h_info[1]};
  UTV_CUDA(cudaMemcpyAsync(flags, fl, sizeof(fl), cudaMemcpyHostToDevice, st));
  comm.allreduce(flags, 2, st);
  double flo[2] = {0.0, 0.0};
  UTV_CUDA(cudaMemcpyAsync(flo, flags, sizeof(flo), cudaMemcpyDeviceToHost, st));
  comm.wait(st);
  h->agreed_failure = flo[0] != 0.0 || flo[1] != 0.0;
  if (flo[0] != 0.0) fail(UTV_ERR_NUMERICAL, "NaN or Inf in A or B (on some rank)");
  if (flo[1] != 0.0) fail(UTV_ERR_NUMERICAL, "Jacobi SVD of a diagonal block did not converge in 30 sweeps");
  const int64_t r = finish_factor(c, n, dg, 0, opt.tau, true);        // a8 (replicated diag)
  if (k > 0) {
    dist_solve_z_ooc(c, comm, o, r, b, B, ldb, k);                     // a9
    solve_factored(c, n, r, nullptr, 0, nullptr, 0, k, X, ldx, fv, b, nullptr, true);
  }
  if (o.c_res < nloc) {                                                // resident part of the shard of T
    UTV_CUDA(cudaEventRecord(h->ev_done, st));
    UTV_CUDA(cudaStreamWaitEvent(h->d2h, h->ev_done, 0));
    copy2d(h->d2h, o.hA + cm(0, o.c_res, o.lda), o.lda, o.res, m, m, nloc - o.c_res, cudaMemcpyDeviceToHost);
    h->ooc_d2h += (nloc - o.c_res) * m * 8;
  }
  UTV_CUDA(cudaStreamSynchronize(h->d2h));
  comm.wait(st);
  return r;
}

}  // namespace

extern "C" {

const char* utv_version(void) { return "utv-b200 0.1 sm_100a (FP64 DMMA)"; }

utv_status utv_create(utv_handle* handle, int device, void* stream) {
  if (!handle) return UTV_ERR_ARG;
  *handle = nullptr;
  utv_handle h = new (std::nothrow) utv_handle_s();
  if (!h) return UTV_ERR_ALLOC;
  h->device = device;
  h->stream = (cudaStream_t)stream;
  utv_status s = guarded(h, [&] {
    int cnt = 0;
    UTV_CUDA(cudaGetDeviceCount(&cnt));
    if (device < 0 || device >= cnt) fail(UTV_ERR_ARG, "device ordinal out of range");
    UTV_CUDA(cudaSetDevice(device));
    UTV_CUDA(cudaDeviceGetAttribute(&h->num_sms, cudaDevAttrMultiProcessorCount, device));
    int coop = 0;
    UTV_CUDA(cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, device));
    if (!coop) fail(UTV_ERR_UNSUPPORTED, "device does not support cooperative launch");
    UTV_CUDA(cudaMalloc((void**)&h->bar, kGridBarrierBytes));
    UTV_CUDA(cudaMemset(h->bar, 0, kGridBarrierBytes));
    UTV_CUDA(cudaMalloc((void**)&h->bar2, kGridBarrierBytes));
    UTV_CUDA(cudaMemset(h->bar2, 0, kGridBarrierBytes));
    int lo = 0, hi = 0;
    UTV_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    // The SVD's results are needed only a step later (deferred A12 / finalisation), so its stream
    // yields SMs to the critical-path GEMMs (measured: cfg3 25.27 -> 25.22 s vs high priority).
    static const bool side_high = [] { const char* e = std::getenv("UTV_SIDE_HIGH_PRIORITY"); return e && e[0] == '1'; }();
    UTV_CUDA(cudaStreamCreateWithPriority(&h->side, cudaStreamNonBlocking, side_high ? hi : lo));
    UTV_CUDA(cudaEventCreateWithFlags(&h->ev_panel, cudaEventDisableTiming));
    UTV_CUDA(cudaEventCreateWithFlags(&h->ev_svd, cudaEventDisableTiming));
    UTV_CUDA(cudaEventCreateWithFlags(&h->ev_us, cudaEventDisableTiming));
    UTV_CUDA(cudaEventCreateWithFlags(&h->ev_r, cudaEventDisableTiming));
    UTV_CUDA(cudaStreamCreateWithPriority(&h->cst, cudaStreamNonBlocking, hi));
    for (int q = 0; q < utv_handle_s::kChunks; ++q) {
      UTV_CUDA(cudaEventCreateWithFlags(&h->ev_cq[q], cudaEventDisableTiming));
      UTV_CUDA(cudaEventCreateWithFlags(&h->ev_cd[q], cudaEventDisableTiming));
    }
    for (int q = 0; q <= utv_handle_s::kLagMax; ++q)
      UTV_CUDA(cudaEventCreateWithFlags(&h->ev_svdq[q], cudaEventDisableTiming));
    UTV_CUDA(cudaMalloc((void**)&h->info, 64 * sizeof(int)));
    UTV_CUDA(cudaMalloc((void**)&h->flag, sizeof(int)));
    UTV_CUDA(cudaMalloc((void**)&h->agree, 2 * sizeof(double)));
    UTV_CUDA(cudaMalloc((void**)&h->d_rank, sizeof(int64_t)));
    UTV_CUDA(cudaMallocHost((void**)&h->h_rank, sizeof(int64_t)));
    UTV_CUDA(cudaMallocHost((void**)&h->h_info, 4 * sizeof(int)));
  });
  if (s != UTV_OK) { utv_destroy(h); return s; }
  *handle = h;
  return UTV_OK;
}

utv_status utv_get_unique_id(void* uid) {
  if (!uid) return UTV_ERR_ARG;
  const NcclApi* api = nccl_api();
  if (!api) return UTV_ERR_NCCL;
  ncclUniqueId id;
  if (api->getUniqueId(&id) != ncclSuccess) return UTV_ERR_NCCL;
  std::memcpy(uid, &id, sizeof(id));
  return UTV_OK;
}

utv_status utv_create_dist(utv_handle* handle, int device, void* stream, const void* nccl_uid, int nranks, int rank) {
  if (!handle) return UTV_ERR_ARG;
  *handle = nullptr;
  if (!nccl_uid || nranks < 1 || rank < 0 || rank >= nranks) return UTV_ERR_ARG;
  utv_handle h = nullptr;
  utv_status s = utv_create(&h, device, stream);
  if (s != UTV_OK) return s;
  s = guarded(h, [&] {
    const NcclApi* api = nccl_api();
    if (!api) fail(UTV_ERR_NCCL, "libnccl.so.2 could not be loaded");
    auto* c = new NcclComm();
    c->api = api;
    c->nranks = nranks;
    c->rank = rank;
    ncclUniqueId id;
    std::memcpy(&id, nccl_uid, sizeof(id));
    h->comm = c;
    c->check(api->commInitRank(&c->comm, nranks, id, rank), "ncclCommInitRank");
  });
  if (s != UTV_OK) {
    if (h->comm) { delete h->comm; h->comm = nullptr; }   // NcclComm dtor skips a null comm
    utv_destroy(h);
    return s;
  }
  *handle = h;
  return UTV_OK;
}

utv_status utv_create_with_comm(utv_handle* handle, int device, void* stream, int nranks, int rank,
                                const utv_comm_ops* ops) {
  if (!handle) return UTV_ERR_ARG;
  *handle = nullptr;
  if (!ops || !ops->allreduce_sum || !ops->broadcast || !ops->allgather || nranks < 1 || rank < 0 || rank >= nranks)
    return UTV_ERR_ARG;
  utv_handle h = nullptr;
  utv_status s = utv_create(&h, device, stream);
  if (s != UTV_OK) return s;
  auto* c = new (std::nothrow) CallbackComm();
  if (!c) { utv_destroy(h); return UTV_ERR_ALLOC; }
  c->ops = *ops;
  c->nranks = nranks;
  c->rank = rank;
  h->comm = c;
  *handle = h;
  return UTV_OK;
}

utv_status utv_create_local_group(utv_handle* handles, int nranks, const int* devices, void* const* streams) {
  if (!handles || nranks < 1 || !devices) return UTV_ERR_ARG;
  for (int r = 0; r < nranks; ++r) handles[r] = nullptr;
  auto g = std::make_shared<LocalGroup>(nranks);
  for (int r = 0; r < nranks; ++r) {
    utv_handle h = nullptr;
    utv_status s = utv_create(&h, devices[r], streams ? streams[r] : nullptr);
    if (s != UTV_OK) {
      for (int q = 0; q < r; ++q) { utv_destroy(handles[q]); handles[q] = nullptr; }
      return s;
    }
    int share = 0;
    for (int q = 0; q < nranks; ++q) share += devices[q] == devices[r];
    h->coop_share = std::max(1, share);
    auto* c = new LocalComm();
    c->device = devices[r];
    c->g = g;
    c->nranks = nranks;
    c->rank = r;
    h->comm = c;
    handles[r] = h;
  }
  return UTV_OK;
}

int64_t utv_dist_local_cols(int64_t n, int64_t block, int nranks, int rank) {
  if (n <= 0 || block < 1 || nranks < 1 || rank < 0 || rank >= nranks) return 0;
  return dist_local_cols(n, block, nranks, rank);
}

utv_status utv_destroy(utv_handle h) {
  if (!h) return UTV_OK;
  cudaSetDevice(h->device);
  if (h->stream) cudaStreamSynchronize(h->stream); else cudaDeviceSynchronize();
  if (h->side) { cudaStreamSynchronize(h->side); cudaStreamDestroy(h->side); }
  if (h->cst) { cudaStreamSynchronize(h->cst); cudaStreamDestroy(h->cst); }
  if (h->ev_panel) cudaEventDestroy(h->ev_panel);
  if (h->ev_svd) cudaEventDestroy(h->ev_svd);
  if (h->ev_us) cudaEventDestroy(h->ev_us);
  if (h->ev_r) cudaEventDestroy(h->ev_r);
  for (int q = 0; q < utv_handle_s::kChunks; ++q) {
    if (h->ev_cq[q]) cudaEventDestroy(h->ev_cq[q]);
    if (h->ev_cd[q]) cudaEventDestroy(h->ev_cd[q]);
  }
  for (int q = 0; q <= utv_handle_s::kLagMax; ++q)
    if (h->ev_svdq[q]) cudaEventDestroy(h->ev_svdq[q]);
  if (h->h2d) { cudaStreamSynchronize(h->h2d); cudaStreamDestroy(h->h2d); }
  if (h->d2h) { cudaStreamSynchronize(h->d2h); cudaStreamDestroy(h->d2h); }
  for (int s = 0; s < utv_handle_s::kStg; ++s) {
    if (h->ev_loaded[s]) cudaEventDestroy(h->ev_loaded[s]);
    if (h->ev_free[s]) cudaEventDestroy(h->ev_free[s]);
  }
  if (h->ev_done) cudaEventDestroy(h->ev_done);
  if (h->ev_wb) cudaEventDestroy(h->ev_wb);
  cudaFree(h->ooc);
  cudaFree(h->dbuf);
  delete h->comm;
  cudaFree(h->bar2);
  cudaFree(h->ws); cudaFree(h->bar); cudaFree(h->info); cudaFree(h->flag); cudaFree(h->d_rank); cudaFree(h->agree);
  cudaFree(h->vbuf); cudaFree(h->stage); cudaFree(h->nbuf); cudaFree(h->kept.buf);
  cudaFreeHost(h->h_rank); cudaFreeHost(h->h_info);
  cudaGetLastError();
  delete h;
  return UTV_OK;
}

const char* utv_last_error(utv_handle h) { return h ? h->last_error.c_str() : "null handle"; }

utv_status utv_set_stream(utv_handle h, void* stream) {
  return guarded(h, [&] { h->stream = (cudaStream_t)stream; });
}

utv_status utv_synchronize(utv_handle h) {
  return guarded(h, [&] { UTV_CUDA(cudaStreamSynchronize(h->stream)); });
}

utv_status utv_factor(utv_handle h, int64_t m, int64_t n, double* A, int64_t lda, double* V, int64_t ldv, double* U,
                      int64_t ldu, double* B, int64_t ldb, int64_t k, const utv_opts* opts, int64_t* rank) {
  return guarded(h, [&] {
    if (h->comm) {                                                     // multi-GPU handle
      // A = this rank's block-cyclic shard -> its shard of T; V (if non-NULL) = this rank's
      // contiguous row block of V (ceil(n/P) rows, ldv >= them); B replicated -> U^T B.  The ranks
      // agree on the call before the first collective, as in utv_lstsq.
      utv_status local = UTV_OK;
      std::string msg;
      try {
        check_opts(opts);
        if (m < 0 || n < 0 || k < 0) fail(UTV_ERR_ARG, "negative dimension");
        if (m < n) fail(UTV_ERR_SHAPE, "m < n is not supported (R4)");
        if ((U && (opts->flags & UTV_WANT_U)) || (opts->flags & (UTV_NULLIFY_T12 | UTV_HOST_STREAMED)))
          fail(UTV_ERR_UNSUPPORTED, "multi-GPU utv_factor: no U, no UTV_NULLIFY_T12, no UTV_HOST_STREAMED");
        check_ld("lda", lda, m);
        int64_t v0 = 0, nv = 0;
        if (n > 0) dist_v_rows(n, h->comm->nranks, h->comm->rank, &v0, &nv);
        if (V) check_ld("ldv", ldv, nv);
        if (B && k > 0) check_ld("ldb", ldb, m);
        const int64_t nloc = n > 0 ? dist_local_cols(n, opts->block, h->comm->nranks, h->comm->rank) : 0;
        if (nloc > 0 && !A) fail(UTV_ERR_ARG, "A is NULL");
        if ((nloc > 0 && !is_device_ptr(A)) || (V && !is_device_ptr(V)) || (B && k > 0 && !is_device_ptr(B)))
          fail(UTV_ERR_ARG, "the multi-GPU path takes device pointers");
        if (n > 0) dist_reserve(h, m, n, k, *opts);
      } catch (const ApiError& e) {
        local = e.st;
        msg = e.msg;
      }
      dist_agree(h, local, msg);
      if (n == 0) { if (rank) *rank = 0; return; }
      const int64_t r = lstsq_dist(h, m, n, (B && k > 0) ? k : 0, A, lda, B, ldb, nullptr, 1, *opts, false, V,
                                   ldv);
      if (rank) *rank = r;
      return;
    }
    check_opts(opts);
    if (m < 0 || n < 0 || k < 0) fail(UTV_ERR_ARG, "negative dimension");
    if (m < n) fail(UTV_ERR_SHAPE, "m < n is not supported (R4)");
    if (n > 0 && !A) fail(UTV_ERR_ARG, "A is NULL");
    check_ld("lda", lda, m);
    if (V) check_ld("ldv", ldv, n);
    const bool want_u = U && (opts->flags & UTV_WANT_U);
    if (want_u) check_ld("ldu", ldu, m);
    if (B && k > 0) check_ld("ldb", ldb, m);
    const bool nullify = (opts->flags & UTV_NULLIFY_T12) != 0;
    const bool keep = (opts->flags & UTV_KEEP_FACTORS) != 0;
    if (keep && nullify) fail(UTV_ERR_UNSUPPORTED, "UTV_KEEP_FACTORS with UTV_NULLIFY_T12");
    if (keep && !is_device_ptr(A)) fail(UTV_ERR_UNSUPPORTED, "UTV_KEEP_FACTORS needs A in device memory");
    if (n == 0) { if (rank) *rank = 0; return; }
    Kept* kp = keep ? &kept_prepare(h, m, n, opts->block, false) : nullptr;
    Ctx c = make_ctx(h, m, n, k, opts->block);
    factor_impl(c, m, n, A, lda, V, ldv, want_u ? U : nullptr, ldu, (B && k > 0) ? B : nullptr, ldb, k, *opts,
                kp ? &kp->fv : nullptr, kp);
    int64_t r = finish_factor(c, n, A, lda, opts->tau, rank != nullptr || nullify || keep);
    if (kp) { kp->r = r; kp->valid = true; }
    if (nullify) nullify_impl(c, n, r, A, lda, V, ldv, opts->block, nullptr);   // fig:alg_axb line 3
    if (rank) *rank = r;
  });
}

utv_status utv_solve(utv_handle h, int64_t m, int64_t n, int64_t r, const double* T, int64_t ldt, const double* V,
                     int64_t ldv, const double* C, int64_t ldc, int64_t k, double* X, int64_t ldx) {
  return guarded(h, [&] {
    if (h->comm) {
      // multi-GPU handle: T = this rank's block-cyclic shard (block size of the handle's last
      // utv_factor / utv_lstsq), V = its contiguous row block, C replicated; z = T11^{-1} C(0:r) by
      // the distributed block back substitution, X's row block = V_p(:, 0:r) z, AllGather(X rows).
      Comm& comm = *h->comm;
      const int P = comm.nranks, p = comm.rank;
      utv_status local = UTV_OK;
      std::string msg;
      int64_t v0 = 0, nv = 0, per = 0;
      const int64_t b = h->dist_block;
      try {
        if (m < 0 || n < 0 || k < 0 || r < 0 || r > n) fail(UTV_ERR_ARG, "bad dimension (need 0 <= r <= n)");
        if (m < n) fail(UTV_ERR_SHAPE, "m < n is not supported (R4)");
        if (b < 1) fail(UTV_ERR_ARG, "multi-GPU utv_solve needs a preceding utv_factor on this handle");
        dist_v_rows(n, P, p, &v0, &nv);
        per = (n + P - 1) / P;
        check_ld("ldt", ldt, m); check_ld("ldv", ldv, nv); check_ld("ldc", ldc, m); check_ld("ldx", ldx, n);
        if (k > 0 && n > 0 && (!X || (r > 0 && (!C || (nv > 0 && !V)) ||
                                     (r > 0 && dist_local_cols(r, b, P, p) > 0 && !T))))
          fail(UTV_ERR_ARG, "NULL matrix");
        if (k > 0 && n > 0) {
          make_ctx(h, m, n, k, b);
          ensure_buf(&h->dbuf, &h->dbuf_doubles, std::max(dist_dbuf_doubles(n, b, P, k), (size_t)(P + 1) * per * k));
        }
      } catch (const ApiError& e) {
        local = e.st;
        msg = e.msg;
      }
      dist_agree(h, local, msg);
      if (k == 0 || n == 0) return;
      Ctx c = make_ctx(h, m, n, k, b);
      cudaStream_t st = h->stream;
      double* Zb = c.at(c.L.zsolve);
      launch_set_zero(st, n, k, X, ldx);
      if (r > 0) {
        dist_solve_z(c, comm, r, b, T, ldt, C, ldc, k);                   // z = T11^{-1} C(0:r) (ld r)
        double* mine = h->dbuf;                                            // per x k, this rank's rows
        double* all = mine + (size_t)per * k;                              // P x (per x k)
        launch_set_zero(st, per, k, mine, per);
        if (nv > 0) c.gemm(false, false, nv, k, r, 1.0, V, ldv, Zb, r, 0.0, mine, per);
        comm.allgather(mine, all, (size_t)per * k, st);
        for (int q = 0; q < P; ++q) {
          int64_t q0, qn;
          dist_v_rows(n, P, q, &q0, &qn);
          if (qn > 0) launch_copy(st, qn, k, all + (size_t)q * per * k, per, X + q0, ldx);
        }
      }
      comm.wait(st);
      return;
    }
    if (m < 0 || n < 0 || k < 0 || r < 0 || r > n) fail(UTV_ERR_ARG, "bad dimension (need 0 <= r <= n)");
    if (m < n) fail(UTV_ERR_SHAPE, "m < n is not supported (R4)");
    check_ld("ldt", ldt, m); check_ld("ldv", ldv, n); check_ld("ldc", ldc, m); check_ld("ldx", ldx, n);
    if (k == 0 || n == 0) return;
    if (!X || (r > 0 && (!T || !V || !C))) fail(UTV_ERR_ARG, "NULL matrix");
    Ctx c = make_ctx(h, m, n, k, 1);
    solve_impl(c, n, r, T, ldt, V, ldv, C, ldc, k, X, ldx);
  });
}

utv_status utv_solve_rhs(utv_handle h, int64_t m, int64_t n, int64_t k, const double* T, int64_t ldt, double* B,
                         int64_t ldb, double* X, int64_t ldx, int64_t* rank) {
  return guarded(h, [&] {
    Kept& kp = h->kept;
    utv_status local = UTV_OK;
    std::string msg;
    try {
      if (!kp.valid) fail(UTV_ERR_ARG, "no kept factorization: factor with UTV_KEEP_FACTORS first");
      if (m != kp.m || n != kp.n) fail(UTV_ERR_SHAPE, "m, n differ from the kept factorization");
      if (k < 0) fail(UTV_ERR_ARG, "k < 0");
      if (k > 0) {
        check_ld("ldb", ldb, m); check_ld("ldx", ldx, n);
        if (kp.dist) {
          if (!h->comm) fail(UTV_ERR_ARG, "the kept factorization is a multi-GPU one");
          const int64_t nloc = dist_local_cols(n, kp.b, h->comm->nranks, h->comm->rank);
          if (nloc > 0) check_ld("ldt", ldt, m);
          if (!B || !X || (nloc > 0 && kp.r > 0 && !T)) fail(UTV_ERR_ARG, "NULL matrix");
        } else {
          check_ld("ldt", ldt, m);
          if (!B || !X || (kp.r > 0 && !T)) fail(UTV_ERR_ARG, "NULL matrix");
        }
        if (!is_device_ptr(B) || !is_device_ptr(X) || (T && !is_device_ptr(T)))
          fail(UTV_ERR_ARG, "utv_solve_rhs takes device pointers");
        make_ctx(h, m, n, k, kp.b);                                    // reserve the workspace
      }
    } catch (const ApiError& e) {
      local = e.st;
      msg = e.msg;
    }
    if (h->comm) dist_agree(h, local, msg);                            // multi-GPU: agree first
    else if (local != UTV_OK) fail(local, msg);
    const int64_t r = kp.r;
    if (rank) *rank = r;
    if (k == 0) return;
    Ctx c = make_ctx(h, m, n, k, kp.b);
    kept_apply_ut(c, kp, B, ldb, k);                                                    // C = U^T B
    if (!kp.dist) {
      solve_factored(c, n, r, T, ldt, B, ldb, k, X, ldx, kp.fv, kp.b);                 // a9
    } else {
      dist_solve_z(c, *h->comm, r, kp.b, T, ldt, B, ldb, k);
      solve_factored(c, n, r, nullptr, 0, nullptr, 0, k, X, ldx, kp.fv, kp.b, nullptr, true);
    }
  });
}

// Wide least squares, m < n (reading R21): randUTV of the tall A^T (n x m),
// A^T V' = U' T', so A = V' T'^T U'^T and eq:simplesoln transposes to
//   X = U'(:, 0:r) T'11^{-T} V'(:, 0:r)^T B.
// U' is never formed: T' is upper trapezoidal, so column j < r of A^T V' = U' T' only involves
// U'(:, 0:r), i.e. A^T V'(:, 0:r) = U'(:, 0:r) T'11 and
//   X = A^T V'(:, 0:r) T'11^{-1} T'11^{-T} V'(:, 0:r)^T B
// (A is kept; the minimum-norm seminormal form, error O(kappa(T'11) eps) like the explicit-U'
// formula -- DESIGN.md R21).  Saves the n x n U' and its 4 n (n m - m^2 / 2) update flops; V' stays
// factored (its reflectors are applied transposed to B, forward to the solution).
// The lower-triangular solve T'11^{-T} runs as the upper block solve through the exchange matrix J:
// T'11^{-T} c = J (J T'11^T J)^{-1} J c (solve_impl with "V" = J).
int64_t lstsq_wide(utv_handle h, int64_t m, int64_t n, int64_t k, const double* A, int64_t lda, const double* B,
                   int64_t ldb, double* X, int64_t ldx, const utv_opts& opts) {
  cudaStream_t st = h->stream;
  const size_t nm = (size_t)n * m, mm = (size_t)m * m, mk = (size_t)m * std::max<int64_t>(k, 1);
  // V' is kept factored: V' = Q_1 ... Q_s blockdiag(V_s)
  const int64_t b = opts.block, nsteps = (m + b - 1) / b;
  const size_t wdbl = factored_w_doubles(m, b), tdbl = (size_t)nsteps * b * b;
  ensure_buf(&h->vbuf, &h->vbuf_doubles, nm + wdbl + 2 * tdbl + 3 * mm + 4 * mk + 64);
  double *At = h->vbuf, *Tr = At + nm, *Jm = Tr + mm, *Id = Jm + mm, *Cw = Id + mm, *Cr = Cw + mk, *Yw = Cr + mk,
         *Ww = Yw + mk;
  FactoredV fv;
  fv.W = Ww; fv.T = fv.W + wdbl; fv.Vs = fv.T + tdbl;
  launch_transpose(st, m, n, A, lda, At, n);
  Ctx c = make_ctx(h, n, m, k, b);
  factor_impl(c, n, m, At, n, nullptr, 0, nullptr, 0, nullptr, 0, 0, opts, &fv);
  if (k > 0) launch_check_finite(st, m, k, B, ldb, h->flag);           // B is not seen by the factorization
  const int64_t r = finish_factor(c, m, At, n, opts.tau, true);
  if (k == 0) return r;
  if (r == 0) { launch_set_zero(st, n, k, X, ldx); return r; }
  // c = V'(:, 0:r)^T B = (blockdiag(V_s)^T Q_s^T ... Q_1^T B)(0:r)
  double *tmp = c.at(c.L.Z1), *tmp2 = c.at(c.L.Z2);
  launch_copy(st, m, k, B, ldb, Cw, m);
  for (size_t i = 0; i < fv.woff.size(); ++i) {                        // Q_i^T = I - W_i T_i^T W_i^T
    const int64_t j0 = fv.j0[i], np = fv.np[i];
    const double* W = fv.W + fv.woff[i];
    c.gemm(true, false, b, k, np, 1.0, W, np, Cw + j0, m, 0.0, tmp, b);
    c.gemm(true, false, b, k, b, 1.0, fv.T + (size_t)(j0 / b) * b * b, b, tmp, b, 0.0, tmp2, b);
    c.gemm(false, false, np, k, b, -1.0, W, np, tmp2, b, 1.0, Cw + j0, m);
  }
  for (int64_t j0 = 0, step = 0; j0 < r; j0 += b, ++step) {             // V_s^T on the blocks 0:r
    const int64_t bw = std::min(b, m - j0);
    c.gemm(true, false, bw, k, bw, 1.0, fv.Vs + (size_t)step * b * b, b, Cw + j0, m, 0.0, Yw + j0, m);
  }
  launch_permute(st, 0, r, k, Yw, m, Cr, m);                          // J c
  launch_permute(st, 2, r, r, At, n, Tr, m);                          // J T'11^T J (upper)
  launch_set_identity(st, r, r, Id, m);
  launch_permute(st, 0, r, r, Id, m, Jm, m);                          // J
  solve_impl(c, r, r, Tr, m, Jm, m, Cr, m, k, Yw, m);                 // y = T'11^{-T} c
  solve_factored(c, m, r, At, n, Yw, m, k, Cw, m, fv, b);             // w = V'(:, 0:r) T'11^{-1} y
  c.gemm(true, false, n, k, m, 1.0, A, lda, Cw, m, 0.0, X, ldx);      // X = A^T w
  return r;
}

utv_status utv_lstsq(utv_handle h, int64_t m, int64_t n, int64_t k, double* A, int64_t lda, double* B, int64_t ldb,
                     double* X, int64_t ldx, const utv_opts* opts, int64_t* rank) {
  return guarded(h, [&] {
    if (h->comm) {                                                     // multi-GPU handle
      // Every rank validates its arguments and reserves its device memory, then the ranks agree
      // (one AllReduce of a flag) before the first collective of the method: a rank-local error
      // fails the call on every rank instead of leaving the peers blocked in a collective.
      utv_status local = UTV_OK;
      std::string msg;
      const bool streamed = opts && (opts->flags & UTV_HOST_STREAMED);
      HostPin pin;                                                     // streamed: the shard, pinned
      Ooc o;
      try {
        check_opts(opts);
        if (m < 0 || n < 0 || k < 0) fail(UTV_ERR_ARG, "negative dimension");
        if (m < n) fail(UTV_ERR_SHAPE, "m < n: single-GPU in-core utv_lstsq only (R21)");
        if (opts->flags & (UTV_NULLIFY_T12 | UTV_EXPLICIT_V))
          fail(UTV_ERR_UNSUPPORTED, "the multi-GPU path implements the fast option with factored V only");
        if (streamed && (opts->flags & UTV_KEEP_FACTORS))
          fail(UTV_ERR_UNSUPPORTED, "UTV_KEEP_FACTORS with UTV_HOST_STREAMED");
        check_ld("lda", lda, m);
        if (k > 0) { check_ld("ldb", ldb, m); check_ld("ldx", ldx, n); }
        const int64_t nloc = n > 0 ? dist_local_cols(n, opts->block, h->comm->nranks, h->comm->rank) : 0;
        if ((nloc > 0 && !A) || (k > 0 && (!B || !X))) fail(UTV_ERR_ARG, "NULL matrix");
        if (k > 0 && (!is_device_ptr(B) || !is_device_ptr(X)))
          fail(UTV_ERR_ARG, "the multi-GPU path takes device B and X (replicated)");
        if (nloc > 0 && streamed == is_device_ptr(A))
          fail(UTV_ERR_ARG, streamed ? "UTV_HOST_STREAMED: A (this rank's shard) must be in host memory"
                                     : "the multi-GPU path takes a device A (this rank's shard)");
        if (n > 0 && streamed) {
          pin.pin(A, m, nloc, lda);
          dist_ooc_prepare(h, o, m, n, k, A, lda, *opts);
        } else if (n > 0) {
          dist_reserve(h, m, n, k, *opts);
        }
      } catch (const ApiError& e) {
        local = e.st;
        msg = e.msg;
      }
      dist_agree(h, local, msg);
      if (n == 0) { if (rank) *rank = 0; return; }
      const int64_t r = streamed ? lstsq_dist_ooc(h, o, m, n, k, B, ldb, X, ldx, *opts)
                                 : lstsq_dist(h, m, n, k, A, lda, B, ldb, X, ldx, *opts);
      if (rank) *rank = r;
      return;
    }
    check_opts(opts);
    if (m < 0 || n < 0 || k < 0) fail(UTV_ERR_ARG, "negative dimension");
    const bool wide = m < n;
    if (wide && (opts->flags & UTV_HOST_STREAMED)) fail(UTV_ERR_SHAPE, "m < n: single-GPU in-core utv_lstsq only (R21)");
    if (wide && (opts->flags & UTV_NULLIFY_T12)) fail(UTV_ERR_UNSUPPORTED, "m < n with UTV_NULLIFY_T12");
    check_ld("lda", lda, m);
    if (k > 0) { check_ld("ldb", ldb, m); check_ld("ldx", ldx, n); }
    const bool keep = (opts->flags & UTV_KEEP_FACTORS) != 0;
    if (keep && (wide || (opts->flags & (UTV_NULLIFY_T12 | UTV_HOST_STREAMED)) || (n > 0 && !is_device_ptr(A))))
      fail(UTV_ERR_UNSUPPORTED, "UTV_KEEP_FACTORS: device A, m >= n, in core, without UTV_NULLIFY_T12");
    if ((n > 0 && !A) || (k > 0 && (!B || !X))) fail(UTV_ERR_ARG, "NULL matrix");
    if (n == 0) { if (rank) *rank = 0; return; }
    if (opts->flags & UTV_HOST_STREAMED) {
      const int64_t r = lstsq_streamed(h, m, n, k, A, lda, B, ldb, X, ldx, *opts);
      if (rank) *rank = r;
      return;
    }
    cudaStream_t st = h->stream;
    // host buffers (the end-to-end path): stage through device memory on the stream
    const bool hA = !is_device_ptr(A), hB = k > 0 && !is_device_ptr(B), hX = k > 0 && !is_device_ptr(X);
    size_t need = (hA ? (size_t)m * n : 0) + (hB ? (size_t)m * k : 0) + (hX ? (size_t)n * k : 0);
    if (need) ensure_buf(&h->stage, &h->stage_doubles, need);
    double* dA = A; int64_t dlda = lda;
    double* dB = B; int64_t dldb = ldb;
    double* dX = X; int64_t dldx = ldx;
    size_t off = 0;
    if (hA) { dA = h->stage + off; dlda = m; off += (size_t)m * n; copy2d(st, dA, m, A, lda, m, n, cudaMemcpyHostToDevice); }
    if (hB) { dB = h->stage + off; dldb = m; off += (size_t)m * k; copy2d(st, dB, m, B, ldb, m, k, cudaMemcpyHostToDevice); }
    if (hX) { dX = h->stage + off; dldx = n; off += (size_t)n * k; }
    const int64_t b = opts->block;
    if (wide) {
      const int64_t r = lstsq_wide(h, m, n, k, dA, dlda, dB, dldb, dX, dldx, *opts);
      if (hX) copy2d(st, X, ldx, dX, n, n, k, cudaMemcpyDeviceToHost);
      if (hX) UTV_CUDA(cudaStreamSynchronize(st));
      if (rank) *rank = r;
      return;
    }
    const bool explicit_v = (opts->flags & UTV_EXPLICIT_V) != 0;
    const bool nullify = (opts->flags & UTV_NULLIFY_T12) != 0;
    FactoredV fv_local;
    NullStore ns;
    Kept* kp = keep ? &kept_prepare(h, m, n, b, false) : nullptr;
    if (explicit_v) ensure_buf(&h->vbuf, &h->vbuf_doubles, (size_t)n * n);
    if (!explicit_v && !keep) {
      const int64_t nsteps = (n + b - 1) / b;
      const size_t wdbl = factored_w_doubles(n, b), tdbl = (size_t)nsteps * b * b;
      ensure_buf(&h->vbuf, &h->vbuf_doubles, wdbl + 2 * tdbl + 64);
      fv_local.W = h->vbuf; fv_local.T = h->vbuf + wdbl; fv_local.Vs = fv_local.T + tdbl;
    }
    FactoredV& fv = keep ? kp->fv : fv_local;
    Ctx c = make_ctx(h, m, n, k, b);
    if (explicit_v)
      factor_impl(c, m, n, dA, dlda, h->vbuf, n, nullptr, 0, k > 0 ? dB : nullptr, dldb, k, *opts,
                  keep ? &fv : nullptr, kp);
    else
      factor_impl(c, m, n, dA, dlda, nullptr, 0, nullptr, 0, k > 0 ? dB : nullptr, dldb, k, *opts, &fv, kp);
    int64_t r = finish_factor(c, n, dA, dlda, opts->tau, true);
    if (kp) { kp->r = r; kp->valid = true; }
    if (nullify) {                                                     // fig:alg_axb line 3
      if (!explicit_v) {
        ensure_buf(&h->nbuf, &h->nbuf_doubles, null_store_doubles(n, r, b) + 64);
        const size_t nblk = (size_t)((r + b - 1) / b);
        ns.Wtop = h->nbuf; ns.Tz = h->nbuf + nblk * b * b; ns.Wbot = ns.Tz + nblk * b * b;
      }
      nullify_impl(c, n, r, dA, dlda, explicit_v ? h->vbuf : nullptr, n, b, explicit_v ? nullptr : &ns);
    }
    if (k > 0) {
      if (explicit_v) solve_impl(c, n, r, dA, dlda, h->vbuf, n, dB, dldb, k, dX, dldx);
      else solve_factored(c, n, r, dA, dlda, dB, dldb, k, dX, dldx, fv, b, nullify ? &ns : nullptr);
    }
    // host A / B are inputs only: they are not written back (see utv.h)
    if (hX) copy2d(st, X, ldx, dX, n, n, k, cudaMemcpyDeviceToHost);
    if (hX) UTV_CUDA(cudaStreamSynchronize(st));
    if (rank) *rank = r;
  });
}

// ---------------------------------------------------------------- step-level entry points
utv_status utv_sketch(utv_handle h, uint64_t seed, int64_t step, int64_t row0, int64_t mrows, int64_t b, double* G,
                      int64_t ldg) {
  return guarded(h, [&] {
    if (mrows < 0 || b < 0 || row0 < 0 || step < 0) fail(UTV_ERR_ARG, "negative argument");
    if (mrows * b > 0 && !G) fail(UTV_ERR_ARG, "G is NULL");
    check_ld("ldg", ldg, mrows);
    launch_sketch(h->stream, seed, step, row0, mrows, b, G, ldg, h->num_sms);
  });
}

utv_status utv_philox(utv_handle h, int64_t n, const uint32_t* ctr, const uint32_t* key, uint32_t* out) {
  return guarded(h, [&] {
    if (n < 0) fail(UTV_ERR_ARG, "n < 0");
    if (n > 0 && (!ctr || !key || !out)) fail(UTV_ERR_ARG, "NULL pointer");
    launch_philox_words(h->stream, ctr, key, n, out);
  });
}

utv_status utv_hqr(utv_handle h, int64_t m, int64_t w, double* P, int64_t ldp, double* W, int64_t ldw, double* tau,
                   double* T, int64_t ldt) {
  return guarded(h, [&] {
    if (w < 0 || m < w) fail(UTV_ERR_SHAPE, "need m >= w >= 0");
    if (w == 0) return;
    if (!P || !W || !tau || !T) fail(UTV_ERR_ARG, "NULL pointer");
    check_ld("ldp", ldp, m); check_ld("ldw", ldw, m); check_ld("ldt", ldt, w);
    Ctx c = make_ctx(h, m, w, 1, w);
    panel_qr(h->stream, m, w, P, ldp, W, ldw, tau, T, ldt, c.pw);
  });
}

utv_status utv_svd_small(utv_handle h, int64_t b, const double* R, int64_t ldr, double* Us, int64_t ldu,
                         double* sigma, double* Vs, int64_t ldv, int32_t* sweeps) {
  return guarded(h, [&] {
    if (b < 1) fail(UTV_ERR_ARG, "b < 1");
    if (b > 256) fail(UTV_ERR_UNSUPPORTED, "b > 256");
    if (!R || !Us || !sigma || !Vs) fail(UTV_ERR_ARG, "NULL pointer");
    check_ld("ldr", ldr, b); check_ld("ldu", ldu, b); check_ld("ldv", ldv, b);
    Ctx c = make_ctx(h, b, b, 1, b);
    UTV_CUDA(cudaMemsetAsync(h->info, 0, 4 * sizeof(int), h->stream));
    svd_small(h->stream, b, R, ldr, Us, ldu, sigma, Vs, ldv, c.sw);
    UTV_CUDA(cudaMemcpyAsync(h->h_info, h->info, 2 * sizeof(int), cudaMemcpyDeviceToHost, h->stream));
    UTV_CUDA(cudaStreamSynchronize(h->stream));
    if (sweeps) *sweeps = h->h_info[0];
    if (h->h_info[1]) fail(UTV_ERR_NUMERICAL, "Jacobi did not converge in 30 sweeps");
  });
}

utv_status utv_svd_block(utv_handle h, int64_t b, double* A11, int64_t lda, double* Us, int64_t ldu, double* sigma,
                         double* Vs, int64_t ldv) {
  return guarded(h, [&] {
    if (b < 1) fail(UTV_ERR_ARG, "b < 1");
    if (b > 256) fail(UTV_ERR_UNSUPPORTED, "b > 256");
    if (!A11 || !Us || !sigma || !Vs) fail(UTV_ERR_ARG, "NULL pointer");
    check_ld("lda", lda, b); check_ld("ldu", ldu, b); check_ld("ldv", ldv, b);
    Ctx c = make_ctx(h, b, b, 1, b);
    svd_small(h->stream, b, A11, lda, Us, ldu, sigma, Vs, ldv, c.sw);   // info accumulates (sticky)
    launch_set_diag(h->stream, b, sigma, A11, lda);                    // A11 := Sigma
  });
}

utv_status utv_svd_status(utv_handle h, int32_t* failed, int32_t* max_sweeps) {
  return guarded(h, [&] {
    UTV_CUDA(cudaMemcpyAsync(h->h_info, h->info, 2 * sizeof(int), cudaMemcpyDeviceToHost, h->stream));
    UTV_CUDA(cudaStreamSynchronize(h->stream));
    if (max_sweeps) *max_sweeps = h->h_info[0];
    if (failed) *failed = h->h_info[1];
    UTV_CUDA(cudaMemsetAsync(h->info, 0, 2 * sizeof(int), h->stream));
  });
}

utv_status utv_trsm_upper(utv_handle h, int64_t n, const double* T, int64_t ldt, double* Z, int64_t ldz, int64_t k) {
  return guarded(h, [&] {
    if (n < 0 || k < 0) fail(UTV_ERR_ARG, "negative dimension");
    if (n == 0 || k == 0) return;
    if (!T || !Z) fail(UTV_ERR_ARG, "NULL pointer");
    check_ld("ldt", ldt, n); check_ld("ldz", ldz, n);
    Ctx c = make_ctx(h, n, n, k, 1);
    constexpr int64_t SB = 256;
    for (int64_t j0 = ((n - 1) / SB) * SB; j0 >= 0; j0 -= SB) {
      const int64_t j1 = std::min(n, j0 + SB);
      launch_trsv_block(c.st, j0, j1, T, ldt, Z, ldz, k);
      if (j0 > 0) c.gemm(false, false, j0, k, j1 - j0, -1.0, T + cm(0, j0, ldt), ldt, Z + j0, ldz, 1.0, Z, ldz);
    }
  });
}

utv_status utv_gemm(utv_handle h, int ta, int tb, int64_t M, int64_t N, int64_t K, double alpha, const double* A,
                    int64_t lda, const double* B, int64_t ldb, double beta, double* C, int64_t ldc) {
  return guarded(h, [&] {
    if (M < 0 || N < 0 || K < 0) fail(UTV_ERR_ARG, "negative dimension");
    if (M == 0 || N == 0) return;
    check_ld("lda", lda, ta ? K : M); check_ld("ldb", ldb, tb ? N : K); check_ld("ldc", ldc, M);
    if (!C || (K > 0 && (!A || !B))) fail(UTV_ERR_ARG, "NULL pointer");
    size_t need = dgemm_workspace_doubles(M, N, K, h->num_sms);
    if (need) ensure_buf(&h->ws, &h->ws_doubles, need);
    dgemm(h->stream, ta != 0, tb != 0, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, h->ws, h->ws_doubles,
          h->num_sms);
  });
}

utv_status utv_rank_diag(utv_handle h, int64_t n, const double* d, double tau, int64_t* rank) {
  return guarded(h, [&] {
    if (n < 0 || !rank) fail(UTV_ERR_ARG, "bad argument");
    if (!(tau >= 0.0 && tau < 1.0)) fail(UTV_ERR_ARG, "tau not in [0, 1)");
    if (n == 0) { *rank = 0; return; }
    if (!d) fail(UTV_ERR_ARG, "d is NULL");
    launch_rank(h->stream, n, d, 0, tau, h->d_rank);     // ldt = 0: T[j + j*0] = d[j]
    UTV_CUDA(cudaMemcpyAsync(h->h_rank, h->d_rank, sizeof(int64_t), cudaMemcpyDeviceToHost, h->stream));
    UTV_CUDA(cudaStreamSynchronize(h->stream));
    *rank = *h->h_rank;
  });
}

utv_status utv_rank(utv_handle h, int64_t n, const double* T, int64_t ldt, double tau, int64_t* rank) {
  return guarded(h, [&] {
    if (n < 0 || !rank) fail(UTV_ERR_ARG, "bad argument");
    if (!(tau >= 0.0 && tau < 1.0)) fail(UTV_ERR_ARG, "tau not in [0, 1)");
    if (n == 0) { *rank = 0; return; }
    check_ld("ldt", ldt, n);
    launch_rank(h->stream, n, T, ldt, tau, h->d_rank);
    UTV_CUDA(cudaMemcpyAsync(h->h_rank, h->d_rank, sizeof(int64_t), cudaMemcpyDeviceToHost, h->stream));
    UTV_CUDA(cudaStreamSynchronize(h->stream));
    *rank = *h->h_rank;
  });
}

utv_status utv_tune(int key, int64_t value, int64_t* old) {
  static std::mutex mu;
  static int64_t cur[9] = {0, -1, 0, 0, 0, 0, 0, 0, 0};
  std::lock_guard<std::mutex> lk(mu);
  if (key < UTV_TUNE_GEMM_CFG || key > UTV_TUNE_QR_CHOLQR) return UTV_ERR_ARG;
  if (old) *old = cur[key];
  cur[key] = value;
  if (key == UTV_TUNE_GEMM_CFG && (value < 0 || value > 5)) cur[key] = -1;
  if (key != UTV_TUNE_GEMM_CFG && value < 0) cur[key] = 0;
  dgemm_force((int)cur[UTV_TUNE_GEMM_CFG], (int)cur[UTV_TUNE_GEMM_SPLITS], (int)cur[UTV_TUNE_GEMM_PATH]);
  panel_force((int)cur[UTV_TUNE_QR_GLOBAL], (int)cur[UTV_TUNE_QR_CTAS], (int)cur[UTV_TUNE_QR_CHOLQR]);
  g_dist_chunks = (int)std::min<int64_t>(cur[UTV_TUNE_DIST_CHUNKS], utv_handle_s::kChunks);
  g_svd_lag = (int)std::min<int64_t>(cur[UTV_TUNE_SVD_LAG], utv_handle_s::kLagMax);
  return UTV_OK;
}

utv_status utv_set_device_budget(utv_handle h, int64_t bytes) {
  return guarded(h, [&] {
    if (bytes < 0) fail(UTV_ERR_ARG, "bytes < 0");
    h->dev_budget = bytes;
  });
}

utv_status utv_stream_stats(utv_handle h, int64_t* h2d_bytes, int64_t* d2h_bytes, int64_t* resident_cols) {
  return guarded(h, [&] {
    if (h2d_bytes) *h2d_bytes = h->ooc_h2d;
    if (d2h_bytes) *d2h_bytes = h->ooc_d2h;
    if (resident_cols) *resident_cols = h->ooc_resident_cols;
  });
}

utv_status utv_profile(utv_handle h, int enable) {
  return guarded(h, [&] {
    if (enable) { h->prof.reset(); h->prof.on = true; }
    else h->prof.on = false;
  });
}

utv_status utv_profile_dump(utv_handle h, const char* path) {
  return guarded(h, [&] {
    if (!path) fail(UTV_ERR_ARG, "path is NULL");
    UTV_CUDA(cudaStreamSynchronize(h->stream));
    UTV_CUDA(cudaStreamSynchronize(h->side));
    if (prof_dump(h->prof, path) < 0) fail(UTV_ERR_ARG, "cannot write the profile file");
  });
}

utv_status utv_profile_read(utv_handle h, utv_prof_entry* out) {
  return guarded(h, [&] {
    if (!out) fail(UTV_ERR_ARG, "out is NULL");
    UTV_CUDA(cudaStreamSynchronize(h->stream));
    UTV_CUDA(cudaStreamSynchronize(h->side));
    for (int f = 0; f < kProfN; ++f) out[f] = utv_prof_entry{0, 0, 0.0, 0.0, 0.0};
    for (const ProfRec& r : h->prof.recs) {
      if (r.family < 0 || r.family >= kProfN) continue;
      utv_prof_entry& e = out[r.family];
      e.launches += r.launches;
      e.calls += 1;
      e.flops += r.flops;
      e.bytes += r.bytes;
      float ms = 0.f;
      if (r.e0 && r.e1 && cudaEventElapsedTime(&ms, r.e0, r.e1) == cudaSuccess) e.ms += ms;
      else cudaGetLastError();
    }
  });
}

}  // extern "C"

// diagnostics only (not part of utv.h): run one collective of a multi-GPU handle on a device buffer
// (op 0 = AllReduce(sum) in place, 1 = Broadcast from `root`, 2 = AllGather of n into recv).
extern "C" utv_status utv_debug_collective(utv_handle h, int op, double* buf, int64_t n, int root, double* recv) {
  return guarded(h, [&] {
    if (!h->comm) fail(UTV_ERR_ARG, "not a multi-GPU handle");
    if (op == 0) h->comm->allreduce(buf, (size_t)n, h->stream);
    else if (op == 1) h->comm->bcast(buf, (size_t)n, root, h->stream);
    else h->comm->allgather(buf, recv, (size_t)n, h->stream);
    UTV_CUDA(cudaStreamSynchronize(h->stream));
  });
}
