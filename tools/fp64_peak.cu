// FP64 peak microbenchmark for B200 (sm_100a): DMMA (mma.sync f64) and DFMA.
// Measurement-only tool; its numbers are the FP64 roofline denominators.
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); exit(1);} } while (0)

template <int SHAPE_K>
__device__ __forceinline__ void mma_f64(double* d, const double* a, const double* b);

template <> __device__ __forceinline__ void mma_f64<4>(double* d, const double* a, const double* b) {
  asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
               : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3]) : "d"(a[0]), "d"(a[1]), "d"(b[0]));
}
template <> __device__ __forceinline__ void mma_f64<8>(double* d, const double* a, const double* b) {
  asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
               : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3]) : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
}
template <> __device__ __forceinline__ void mma_f64<16>(double* d, const double* a, const double* b) {
  asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
               : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3])
               : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                 "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
}
__device__ __forceinline__ void mma_m8n8k4(double* d, const double* a, const double* b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d[0]), "+d"(d[1]) : "d"(a[0]), "d"(b[0]));
}

template <int K, int CHAINS>
__global__ void dmma_loop(double* out, long iters, double seed) {
  double acc[CHAINS][4];
  double a[K / 2], b[K / 4];
  for (int i = 0; i < K / 2; ++i) a[i] = seed + threadIdx.x * 1e-3 + i;
  for (int i = 0; i < K / 4; ++i) b[i] = seed * 0.5 + i;
  for (int c = 0; c < CHAINS; ++c) for (int j = 0; j < 4; ++j) acc[c][j] = 0.0;
  for (long it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) mma_f64<K>(acc[c], a, b);
  }
  double s = 0; for (int c = 0; c < CHAINS; ++c) for (int j = 0; j < 4; ++j) s += acc[c][j];
  if (s == 1234.5) out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int CHAINS>
__global__ void dmma884_loop(double* out, long iters, double seed) {
  double acc[CHAINS][2]; double a = seed + threadIdx.x, b = seed * 0.5;
  for (int c = 0; c < CHAINS; ++c) acc[c][0] = acc[c][1] = 0.0;
  for (long it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) mma_m8n8k4(acc[c], &a, &b);
  }
  double s = 0; for (int c = 0; c < CHAINS; ++c) s += acc[c][0] + acc[c][1];
  if (s == 1234.5) out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int CHAINS>
__global__ void dfma_loop(double* out, long iters, double seed) {
  double acc[CHAINS]; double a = seed + threadIdx.x * 1e-9, b = 1.0 - 1e-12;
  for (int c = 0; c < CHAINS; ++c) acc[c] = c;
  for (long it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) acc[c] = fma(acc[c], b, a);
  }
  double s = 0; for (int c = 0; c < CHAINS; ++c) s += acc[c];
  if (s == 1234.5) out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <typename F>
double run(F launch, double flops_per_iter_total, long iters, int reps) {
  cudaEvent_t e0, e1; CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  launch(iters / 10); CK(cudaDeviceSynchronize());
  float best = 1e30f;
  for (int r = 0; r < reps; ++r) {
    CK(cudaEventRecord(e0)); launch(iters); CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
    float ms; CK(cudaEventElapsedTime(&ms, e0, e1)); if (ms < best) best = ms;
  }
  CK(cudaGetLastError());
  return flops_per_iter_total * iters / (best * 1e-3) / 1e12;
}

int main(int argc, char** argv) {
  int dev = 0; cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, dev));
  int sms = p.multiProcessorCount;
  printf("{\"gpu\": \"%s\", \"sms\": %d, \"cc\": \"%d.%d\"", p.name, sms, p.major, p.minor);
  double* out; CK(cudaMalloc(&out, 1 << 24));
  const int threads = 256; // 8 warps / CTA
  for (int ctas_per_sm = 1; ctas_per_sm <= 2; ++ctas_per_sm) {
    int grid = sms * ctas_per_sm;
    long warps = (long)grid * threads / 32;
    long it = 20000;
    double t4 = run([&](long n) { dmma_loop<4, 8><<<grid, threads>>>(out, n, 1.0); }, warps * 8 * 2.0 * 16 * 8 * 4, it, 3);
    double t8 = run([&](long n) { dmma_loop<8, 8><<<grid, threads>>>(out, n, 1.0); }, warps * 8 * 2.0 * 16 * 8 * 8, it / 2, 3);
    double t16 = run([&](long n) { dmma_loop<16, 8><<<grid, threads>>>(out, n, 1.0); }, warps * 8 * 2.0 * 16 * 8 * 16, it / 4, 3);
    double t884 = run([&](long n) { dmma884_loop<8><<<grid, threads>>>(out, n, 1.0); }, warps * 8 * 2.0 * 8 * 8 * 4, it, 3);
    double tf = run([&](long n) { dfma_loop<8><<<grid, threads>>>(out, n, 1.0); }, (double)grid * threads * 8 * 2.0, it * 4, 3);
    printf(", \"occ%d\": {\"dmma_m16n8k4_tflops\": %.2f, \"dmma_m16n8k8_tflops\": %.2f, \"dmma_m16n8k16_tflops\": %.2f, \"dmma_m8n8k4_tflops\": %.2f, \"dfma_tflops\": %.2f}",
           ctas_per_sm, t4, t8, t16, t884, tf);
  }
  // sustained: ~4 s of m16n8k8 back to back
  {
    int grid = sms; long warps = (long)grid * threads / 32;
    long it = 20000;
    double t = run([&](long n) { dmma_loop<8, 8><<<grid, threads>>>(out, n, 1.0); }, warps * 8 * 2.0 * 16 * 8 * 8, it / 2, 1);
    // scale iterations so one launch lasts ~4 s
    double sec_per_iter = (warps * 8 * 2.0 * 16 * 8 * 8) / (t * 1e12);
    long iters4 = (long)(4.0 / sec_per_iter);
    double ts = run([&](long n) { dmma_loop<8, 8><<<grid, threads>>>(out, n, 1.0); }, warps * 8 * 2.0 * 16 * 8 * 8, iters4, 1);
    printf(", \"dmma_m16n8k8_sustained_4s_tflops\": %.2f", ts);
  }
  printf("}\n");
  return 0;
}
