// Microbenchmark: scatter writes whose destinations are a random permutation
// inside consecutive windows of W entries (the pass-B pattern of pscatter.cuh).
// Measures time per window size and element width; run under ncu for DRAM bytes.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__global__ void fill_perm(uint32_t* idx, long n, long W, uint64_t seed) {
  // affine permutation inside each window: j -> (a*j + c) mod W, W power of 2, a odd
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) {
    long w0 = i & ~(W - 1), j = i & (W - 1);
    uint64_t a = (seed * 2 + 1) | 1, c = seed * 7919;
    uint64_t x = (a * (uint64_t)j + c) & (W - 1);
    x = (x ^ (x >> 7)) & (W - 1);  // still a bijection? xor-shift right is bijective on W bits
    idx[i] = (uint32_t)(w0 + x);
  }
}
template <int MODE>
__global__ void scat4(const uint32_t* __restrict__ idx, uint32_t* out, long n) {
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) {
    uint32_t d = __ldcs(idx + i);
    out[d] = (uint32_t)i;
  }
}
__global__ void scat16(const uint32_t* __restrict__ idx, uint4* out, long n) {
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) {
    uint32_t d = __ldcs(idx + i);
    out[d] = make_uint4(i, i, i, i);
  }
}
int main() {
  long n = 1L << 28;
  uint32_t *idx, *out4; uint4* out16;
  cudaMalloc(&idx, n * 4); cudaMalloc(&out4, n * 4); cudaMalloc(&out16, n * 16);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  long wins[] = {1L << 16, 1L << 18, 1L << 20, 1L << 21, 1L << 22, 1L << 23, 1L << 24, 1L << 28};
  int grids[] = {1184, 2368, 4736};
  for (long W : wins) for (int g : grids) {
    fill_perm<<<1184, 256>>>(idx, n, W, 12345);
    float ms4, ms16;
    scat4<0><<<g, 256>>>(idx, out4, n);
    cudaEventRecord(a); scat4<0><<<g, 256>>>(idx, out4, n); cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms4, a, b);
    long n16 = n / 4;  // same bytes
    scat16<<<g, 256>>>(idx, out16, n16);
    cudaEventRecord(a); scat16<<<g, 256>>>(idx, out16, n16); cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms16, a, b);
    printf("window %8ld entries grid %5d: 4B %7.3f ms (%6.1f G/s)   16B(n/4) window %6.1f MB %7.3f ms\n", W, g, ms4,
           n / ms4 / 1e6, W * 16.0 / (1 << 20), ms16);
  }
  return 0;
}
