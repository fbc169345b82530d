// Latency of dependent FP64 / shared-memory / shuffle chains on one warp, in SM cycles.
#include <cstdio>
#include <cuda_runtime.h>
__device__ long long out[8];
__global__ void lat(double* g, int n) {
  __shared__ double s[1024];
  s[threadIdx.x] = g[threadIdx.x];
  __syncthreads();
  double x = g[threadIdx.x + 32], y = g[threadIdx.x + 64];
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = fma(x, y, 0.5);
  long long t1 = clock64();
  for (int i = 0; i < n; ++i) x = x * y;
  long long t2 = clock64();
  int idx = threadIdx.x;
  for (int i = 0; i < n; ++i) { double v = s[idx]; idx = ((int)v & 7) + threadIdx.x; }
  long long t3 = clock64();
  for (int i = 0; i < n; ++i) x = __shfl_sync(0xffffffffu, x, (threadIdx.x + 1) & 31);
  long long t4 = clock64();
  double z = x;
  for (int i = 0; i < n; ++i) z = 1.0 / z;
  long long t5 = clock64();
  for (int i = 0; i < n; ++i) __syncthreads();
  long long t6 = clock64();
  if (threadIdx.x == 0) { out[0] = t1 - t0; out[1] = t2 - t1; out[2] = t3 - t2; out[3] = t4 - t3; out[4] = t5 - t4; out[5] = t6 - t5; }
  g[threadIdx.x] = x + idx + z;
}
int main() {
  double* g; cudaMalloc(&g, 4096 * 8); cudaMemset(g, 0, 4096 * 8);
  const int n = 1000;
  lat<<<1, 32>>>(g, n); lat<<<1, 32>>>(g, n); cudaDeviceSynchronize();
  long long o[8]; cudaMemcpyFromSymbol(o, out, sizeof o);
  printf("per op cycles (1 warp): DFMA %.1f, DMUL %.1f, LDS %.1f, SHFL %.1f, DDIV %.1f, BAR %.1f\n", o[0] / (double)n, o[1] / (double)n,
         o[2] / (double)n, o[3] / (double)n, o[4] / (double)n, o[5] / (double)n);
  lat<<<1, 256>>>(g, n); cudaDeviceSynchronize(); cudaMemcpyFromSymbol(o, out, sizeof o);
  printf("per op cycles (8 warps): DFMA %.1f, DMUL %.1f, LDS %.1f, SHFL %.1f, DDIV %.1f, BAR %.1f\n", o[0] / (double)n, o[1] / (double)n,
         o[2] / (double)n, o[3] / (double)n, o[4] / (double)n, o[5] / (double)n);
  return 0;
}
