// Microbenchmark: latency of the single-CTA nb x nb building blocks of the CholeskyQR2 path
// (LU with one CTA barrier per column, barriers alone, the tiled product) in SM clock cycles.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o small_lu_bench small_lu_bench.cu
#include <cstdio>
#include <cuda_runtime.h>
constexpr int LD = 65, NB = 64, TH = 256;
__device__ long long out[8];

template <int MODE>   // 0 = full LU step, 1 = barrier only, 2 = no division, 3 = no FMA update, 5 = loads hoisted
__global__ void lu_k(double* g) {
  extern __shared__ double a[];
  const int tid = threadIdx.x, ty = tid >> 4, tx = tid & 15;
  for (int e = tid; e < NB * NB; e += TH) a[(e / NB) * LD + e % NB] = g[e];
  __syncthreads();
  long long t0 = clock64();
  double lprev[4] = {0, 0, 0, 0};
  for (int j = 0; j < NB; ++j) {
    if (MODE == 5) {
      if (tx == 0 && j > 0)
        for (int p = 0; p < 4; ++p) { const int i = j + ty + 16 * p; if (i < NB) a[i * LD + j - 1] = lprev[p]; }
      const double d = a[j * LD + j];
      double rj[4], ai[4], v[4][4];
#pragma unroll
      for (int q = 0; q < 4; ++q) { const int l = j + 1 + tx + 16 * q; rj[q] = l < NB ? a[j * LD + l] : 0.0; }
#pragma unroll
      for (int p = 0; p < 4; ++p) {
        const int i = j + 1 + ty + 16 * p;
        ai[p] = i < NB ? a[i * LD + j] : 0.0;
#pragma unroll
        for (int q = 0; q < 4; ++q) { const int l = j + 1 + tx + 16 * q; v[p][q] = (i < NB && l < NB) ? a[i * LD + l] : 0.0; }
      }
      const double pinv = 1.0 / d;
#pragma unroll
      for (int p = 0; p < 4; ++p) {
        const int i = j + 1 + ty + 16 * p;
        const double li = ai[p] * pinv;
        lprev[p] = li;
#pragma unroll
        for (int q = 0; q < 4; ++q) { const int l = j + 1 + tx + 16 * q; if (i < NB && l < NB) a[i * LD + l] = v[p][q] - li * rj[q]; }
      }
    } else if (MODE != 1) {
      if (tx == 0 && j > 0)
        for (int p = 0; p < 4; ++p) { const int i = j + ty + 16 * p; if (i < NB) a[i * LD + j - 1] = lprev[p]; }
      const double d = a[j * LD + j];
      const double pinv = MODE == 2 ? d : 1.0 / d;
#pragma unroll
      for (int p = 0; p < 4; ++p) {
        const int i = j + 1 + ty + 16 * p;
        if (i < NB) {
          const double li = a[i * LD + j] * pinv;
          lprev[p] = li;
          if (MODE != 3)
#pragma unroll
            for (int q = 0; q < 4; ++q) { const int l = j + 1 + tx + 16 * q; if (l < NB) a[i * LD + l] -= li * a[j * LD + l]; }
        }
      }
    }
    __syncthreads();
  }
  long long t1 = clock64();
  if (tid == 0) out[MODE] = t1 - t0;
  g[tid] = a[tid];
}

__global__ void mm_k(double* g) {
  extern __shared__ double s[];
  double *a = s, *b = s + NB * LD, *c = s + 2 * NB * LD;
  const int tid = threadIdx.x, ty = tid >> 4, tx = tid & 15;
  for (int e = tid; e < NB * NB; e += TH) { a[(e / NB) * LD + e % NB] = g[e]; b[(e / NB) * LD + e % NB] = g[e]; }
  __syncthreads();
  long long t0 = clock64();
  for (int rep = 0; rep < 4; ++rep) {
    double acc[4][4] = {};
    for (int k = 0; k < NB; ++k) {
      double av[4], bv[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) av[i] = a[(ty + 16 * i) * LD + k];
#pragma unroll
      for (int j = 0; j < 4; ++j) bv[j] = b[k * LD + tx + 16 * j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] += av[i] * bv[j];
    }
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) c[(ty + 16 * i) * LD + tx + 16 * j] = acc[i][j];
    __syncthreads();
  }
  long long t1 = clock64();
  if (tid == 0) out[4] = (t1 - t0) / 4;
  g[tid] = c[tid];
}

int main() {
  double* g; cudaMalloc(&g, NB * NB * 8);
  double h[NB * NB];
  for (int i = 0; i < NB; ++i) for (int j = 0; j < NB; ++j) h[i * NB + j] = (i == j ? NB : 0) + 1.0 / (1 + i + j);
  cudaMemcpy(g, h, sizeof h, cudaMemcpyHostToDevice);
  const int sm = NB * LD * 8;
  cudaFuncSetAttribute(mm_k, cudaFuncAttributeMaxDynamicSharedMemorySize, 3 * sm);
  for (int it = 0; it < 2; ++it) {
    lu_k<0><<<1, TH, sm>>>(g); lu_k<1><<<1, TH, sm>>>(g); lu_k<2><<<1, TH, sm>>>(g); lu_k<3><<<1, TH, sm>>>(g); lu_k<5><<<1, TH, sm>>>(g);
    cudaMemcpy(g, h, sizeof h, cudaMemcpyHostToDevice);
    mm_k<<<1, TH, 3 * sm>>>(g);
  }
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0); lu_k<0><<<1, TH, sm>>>(g); cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  long long o[8]; cudaMemcpyFromSymbol(o, out, sizeof o);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("hoisted LU %lld; cycles: LU %lld, barriers only %lld, LU without division %lld, LU without update %lld, mm %lld (clock %d kHz); LU kernel event %.1f us; err %s\n",
         o[5], o[0], o[1], o[2], o[3], o[4], clk, ms * 1e3, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
