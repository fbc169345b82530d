// sketch.cu -- a1: the Gaussian sketch G (P:634-636, P:783-785
// "generate_iid_stdnorm_matrix(m(A) - m(A00), n_b)").  The paper leaves the generator
// open; reading R6 fixes Philox4x32-10 with the counter layout
//   key = (lo32(seed), hi32(seed)), ctr = (lo32(g), hi32(g), c/2, step),  g = global row
// and Box-Muller on two 53-bit uniforms in (0, 1].  Counter-based, so every rank / every
// launch configuration produces identical integers (bit-exact) without any state.
// HBM-write bound: 8 bytes per entry.
#include "kernels.cuh"
#include "prof.cuh"

namespace utv {

__device__ __forceinline__ void philox4x32_10(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3, uint32_t k0,
                                              uint32_t k1, uint32_t (&o)[4]) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint32_t lo0 = 0xD2511F53u * c0, hi0 = __umulhi(0xD2511F53u, c0);
    const uint32_t lo1 = 0xCD9E8D57u * c2, hi1 = __umulhi(0xCD9E8D57u, c2);
    const uint32_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
    c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  o[0] = c0; o[1] = c1; o[2] = c2; o[3] = c3;
}

__device__ __forceinline__ double u01(uint32_t hi, uint32_t lo) {
  const uint64_t x = ((uint64_t)hi << 32) | lo;
  return (double)((x >> 11) + 1) * 0x1.0p-53;
}

// One thread per (row, column pair); consecutive threads -> consecutive rows (coalesced
// stores into both columns of the pair).
__global__ void sketch_kernel(uint64_t seed, int64_t step, int64_t row0, int64_t mrows, int64_t b, double* G,
                              int64_t ldg) {
  const int64_t npairs = (b + 1) / 2;
  const int64_t total = mrows * npairs;
  const uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
  const double two_pi = 6.283185307179586476925286766559;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e % mrows, p = e / mrows;
    const uint64_t gr = (uint64_t)(row0 + i);
    uint32_t x[4];
    philox4x32_10((uint32_t)gr, (uint32_t)(gr >> 32), (uint32_t)p, (uint32_t)step, k0, k1, x);
    const double rad = sqrt(-2.0 * log(u01(x[0], x[1])));
    const double ang = two_pi * u01(x[2], x[3]);
    G[cm(i, 2 * p, ldg)] = rad * cos(ang);
    if (2 * p + 1 < b) G[cm(i, 2 * p + 1, ldg)] = rad * sin(ang);
  }
}

__global__ void philox_words_kernel(const uint32_t* ctr, const uint32_t* key, int64_t n, uint32_t* out) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    uint32_t x[4];
    philox4x32_10(ctr[4 * e], ctr[4 * e + 1], ctr[4 * e + 2], ctr[4 * e + 3], key[2 * e], key[2 * e + 1], x);
    for (int c = 0; c < 4; ++c) out[4 * e + c] = x[c];
  }
}

void launch_sketch(cudaStream_t st, uint64_t seed, int64_t step, int64_t row0, int64_t mrows, int64_t b, double* G,
                   int64_t ldg, int num_sms) {
  const int64_t total = mrows * ((b + 1) / 2);
  if (total <= 0) return;
  const int blocks = (int)std::min<int64_t>((total + 255) / 256, (int64_t)num_sms * 16);
  ProfScope prof(st, kProfSketch, 1, 0.0, 8.0 * (double)mrows * b);
  sketch_kernel<<<blocks, 256, 0, st>>>(seed, step, row0, mrows, b, G, ldg);
  UTV_CUDA(cudaGetLastError());
}

void launch_philox_words(cudaStream_t st, const uint32_t* ctr, const uint32_t* key, int64_t n, uint32_t* out) {
  if (n <= 0) return;
  philox_words_kernel<<<(int)std::min<int64_t>((n + 255) / 256, 4096), 256, 0, st>>>(ctr, key, n, out);
  UTV_CUDA(cudaGetLastError());
}

}  // namespace utv
