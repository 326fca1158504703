// Microbenchmark: random 4 B gathers from an array of S bytes (with and
// without a streaming companion read/write), to find the effective L2
// capacity for random-access targets on B200.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint64_t pol_last() { uint64_t p; asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p)); return p; }
__device__ __forceinline__ uint32_t ld_last(const uint32_t* a, uint64_t pol) { uint32_t r; asm volatile("ld.global.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(r) : "l"(a), "l"(pol)); return r; }
__global__ void gather(const uint32_t* idx, const uint32_t* tab, uint32_t* out, long n, int hint) {
  uint64_t pol = pol_last();
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) {
    uint32_t j = __ldcs(idx + i);
    uint32_t v = hint ? ld_last(tab + j, pol) : tab[j];
    __stcs(out + i, v);
  }
}
__global__ void fill_idx(uint32_t* idx, long n, uint32_t m, uint64_t seed) {
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) {
    uint64_t x = (i + 1) * 0x9E3779B97F4A7C15ull ^ seed; x ^= x >> 31; x *= 0xBF58476D1CE4E5B9ull; x ^= x >> 29;
    idx[i] = (uint32_t)(x % m);
  }
}
int main() {
  long n = 64L << 20;  // 64M gathers
  uint32_t *idx, *out, *tab; char* flush;
  cudaMalloc(&idx, n * 4); cudaMalloc(&out, n * 4); cudaMalloc(&tab, 512L << 20); cudaMalloc(&flush, 512L << 20);
  cudaMemset(tab, 1, 512L << 20);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  long sizes[] = {8, 16, 32, 48, 64, 80, 96, 112, 128, 192, 256, 512};
  for (int hint = 0; hint < 2; hint++)
  for (long mb : sizes) {
    uint32_t m = (uint32_t)((mb << 20) / 4);
    fill_idx<<<1184, 256>>>(idx, n, m, 12345);
    gather<<<1184 * 2, 256>>>(idx, tab, out, n, hint);  // warm
    cudaMemset(flush, 0, 512L << 20);
    cudaEventRecord(a);
    gather<<<1184 * 2, 256>>>(idx, tab, out, n, hint);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("hint=%d table %4ld MB: %.3f ms  %.1f Ggather/s\n", hint, mb, ms, n / ms / 1e6);
  }
  return 0;
}
