// Microbenchmark: latency of the single-CTA nb x nb building blocks of the CholeskyQR2 path
// (LU with one CTA barrier per column, barriers alone, the tiled product) in SM clock cycles.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o small_lu_bench small_lu_bench.cu
#include <cstdio>
#include <cuda_runtime.h>
#include <cmath>
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


// register-tiled LU: thread (ty, tx) holds rows ty + 16 p, columns tx + 16 q; per step the pivot row
// and column go through shared memory (double-buffered), one barrier, branch-free updates.
__global__ void tile_lu_k(double* g) {
  __shared__ double xb[4 * NB];
  const int tid = threadIdx.x, ty = tid >> 4, tx = tid & 15;
  double v[4][4];
#pragma unroll
  for (int p = 0; p < 4; ++p)
#pragma unroll
    for (int q = 0; q < 4; ++q) v[p][q] = g[(ty + 16 * p) * NB + tx + 16 * q];
  __syncthreads();
  long long t0 = clock64();
  for (int j = 0; j < NB; ++j) {
    double* rb = xb + (j & 1) * 2 * NB;
    double* cb = rb + NB;
    const int jp = j >> 4, jr = j & 15;
    // publish row j / column j: select the register by an unrolled compare chain
    double rsel[4], csel[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) rsel[q] = jp == 0 ? v[0][q] : jp == 1 ? v[1][q] : jp == 2 ? v[2][q] : v[3][q];
#pragma unroll
    for (int p = 0; p < 4; ++p) csel[p] = jp == 0 ? v[p][0] : jp == 1 ? v[p][1] : jp == 2 ? v[p][2] : v[p][3];
    if (ty == jr) {
#pragma unroll
      for (int q = 0; q < 4; ++q) rb[tx + 16 * q] = rsel[q];
    }
    if (tx == jr) {
#pragma unroll
      for (int p = 0; p < 4; ++p) cb[ty + 16 * p] = csel[p];
    }
    __syncthreads();
    const double d = rb[j];
    const double pinv = 1.0 / d;
    double rv[4], li[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) rv[q] = rb[tx + 16 * q];
#pragma unroll
    for (int p = 0; p < 4; ++p) li[p] = cb[ty + 16 * p] * pinv;
#pragma unroll
    for (int p = 0; p < 4; ++p) {
      const bool below = ty + 16 * p > j;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int l = tx + 16 * q;
        const double upd = fma(-li[p], rv[q], v[p][q]);
        const double nv = (below && l > j) ? upd : ((below && l == j) ? li[p] : v[p][q]);
        v[p][q] = nv;
      }
    }
  }
  long long t1 = clock64();
  if (tid == 0) out[6] = t1 - t0;
#pragma unroll
  for (int p = 0; p < 4; ++p)
#pragma unroll
    for (int q = 0; q < 4; ++q) g[(ty + 16 * p) * NB + tx + 16 * q] = v[p][q];
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
    cudaMemcpy(g, h, sizeof h, cudaMemcpyHostToDevice);
    tile_lu_k<<<1, TH>>>(g);
  }
  {  // correctness of the tiled LU against the smem LU (MODE 0) on the same input
    static double r0[NB * NB], r1[NB * NB];
    cudaMemcpy(g, h, sizeof h, cudaMemcpyHostToDevice); tile_lu_k<<<1, TH>>>(g); cudaMemcpy(r1, g, sizeof r1, cudaMemcpyDeviceToHost);
    // reference LU on the host (row-major h)
    for (int i = 0; i < NB * NB; ++i) r0[i] = h[i];
    for (int j = 0; j < NB; ++j) for (int i = j + 1; i < NB; ++i) { r0[i * NB + j] /= r0[j * NB + j];
      for (int l = j + 1; l < NB; ++l) r0[i * NB + l] -= r0[i * NB + j] * r0[j * NB + l]; }
    double e = 0; for (int i = 0; i < NB * NB; ++i) e = fmax(e, fabs(r0[i] - r1[i]));
    printf("tile LU max |diff| vs host LU: %.2e\n", e);
  }
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0); lu_k<0><<<1, TH, sm>>>(g); cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  long long o[8]; cudaMemcpyFromSymbol(o, out, sizeof o);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("tiled LU %lld; hoisted LU %lld; cycles: LU %lld, barriers only %lld, LU without division %lld, LU without update %lld, mm %lld (clock %d kHz); LU kernel event %.1f us; err %s\n",
         o[6], o[5], o[0], o[1], o[2], o[3], o[4], clk, ms * 1e3, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
