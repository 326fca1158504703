// scan.cuh -- device-wide exclusive scan with fused producer / consumer
// functors (reduce -> scan block sums -> apply).  This is the scan half of
// the paper's split primitive (parallel_sort.py:110-131 exclusive_scan,
// 150-163 split_by_bit) realised as warp-shuffle + shared-memory block scans.
//
//   In : __device__ u32 operator()(i64 i) const      value at i
//   Out: __device__ void operator()(i64 i, u32 excl, u32 v) const
//
// Values are staged striped (coalesced functor reads) into shared memory and
// scanned blocked, so both functors see coalesced index order.
#pragma once

#include "common.cuh"

namespace saix {

constexpr int SCAN_THREADS = 256;
constexpr int SCAN_ITEMS = 16;
constexpr int SCAN_TILE = SCAN_THREADS * SCAN_ITEMS;  // 4096

__device__ __forceinline__ u32 warp_inclusive_scan(u32 v) {
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        u32 y = __shfl_up_sync(0xffffffffu, v, o);
        if (lane_id() >= o) v += y;
    }
    return v;
}

// Block exclusive scan of one value per thread; returns the block total.
template <int THREADS>
__device__ __forceinline__ u32 block_exclusive_scan(u32 v, u32 &excl, u32 *sh_warp) {
    constexpr int WARPS = THREADS / 32;
    int w = threadIdx.x >> 5;
    u32 inc = warp_inclusive_scan(v);
    if (lane_id() == 31) sh_warp[w] = inc;
    __syncthreads();
    if (w == 0) {
        u32 x = lane_id() < WARPS ? sh_warp[lane_id()] : 0;
        u32 xi = warp_inclusive_scan(x);
        if (lane_id() < WARPS) sh_warp[lane_id()] = xi - x;
        if (lane_id() == WARPS - 1) sh_warp[WARPS] = xi;
    }
    __syncthreads();
    excl = sh_warp[w] + inc - v;
    u32 total = sh_warp[WARPS];
    __syncthreads();
    return total;
}

__device__ __forceinline__ int scan_smem_idx(int i) { return i + (i >> 5); }

template <class In>
__global__ void __launch_bounds__(SCAN_THREADS)
k_scan_reduce(In in, i64 n, u32 *block_sums) {
    __shared__ u32 sh_warp[SCAN_THREADS / 32 + 1];
    i64 base = (i64)blockIdx.x * SCAN_TILE;
    u32 s = 0;
#pragma unroll
    for (int r = 0; r < SCAN_ITEMS; r++) {
        i64 i = base + r * SCAN_THREADS + threadIdx.x;
        if (i < n) s += in(i);
    }
    u32 excl;
    u32 tot = block_exclusive_scan<SCAN_THREADS>(s, excl, sh_warp);
    if (threadIdx.x == 0) block_sums[blockIdx.x] = tot;
}

// Single CTA: exclusive scan of block sums in place, carrying across chunks.
static __global__ void __launch_bounds__(1024) k_scan_block_sums(u32 *sums, i64 nb, u32 *total) {
    __shared__ u32 sh_warp[1024 / 32 + 1];
    u32 carry = 0;
    for (i64 c = 0; c < nb; c += 1024) {
        i64 i = c + threadIdx.x;
        u32 v = i < nb ? sums[i] : 0;
        u32 excl;
        u32 tot = block_exclusive_scan<1024>(v, excl, sh_warp);
        if (i < nb) sums[i] = carry + excl;
        carry += tot;
    }
    if (threadIdx.x == 0 && total) *total = carry;
}

template <class In, class Out>
__global__ void __launch_bounds__(SCAN_THREADS)
k_scan_apply(In in, Out out, i64 n, const u32 *block_offsets) {
    __shared__ u32 sh[SCAN_TILE + SCAN_TILE / 32];
    __shared__ u32 sh_v[SCAN_TILE + SCAN_TILE / 32];
    __shared__ u32 sh_warp[SCAN_THREADS / 32 + 1];
    i64 base = (i64)blockIdx.x * SCAN_TILE;
#pragma unroll
    for (int r = 0; r < SCAN_ITEMS; r++) {
        int li = r * SCAN_THREADS + threadIdx.x;
        i64 i = base + li;
        sh_v[scan_smem_idx(li)] = i < n ? in(i) : 0u;
    }
    __syncthreads();
    u32 vals[SCAN_ITEMS];
    u32 s = 0;
#pragma unroll
    for (int r = 0; r < SCAN_ITEMS; r++) {
        vals[r] = sh_v[scan_smem_idx(threadIdx.x * SCAN_ITEMS + r)];
        s += vals[r];
    }
    u32 excl;
    block_exclusive_scan<SCAN_THREADS>(s, excl, sh_warp);
    excl += block_offsets[blockIdx.x];
#pragma unroll
    for (int r = 0; r < SCAN_ITEMS; r++) {
        sh[scan_smem_idx(threadIdx.x * SCAN_ITEMS + r)] = excl;
        excl += vals[r];
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < SCAN_ITEMS; r++) {
        int li = r * SCAN_THREADS + threadIdx.x;
        i64 i = base + li;
        if (i < n) out(i, sh[scan_smem_idx(li)], sh_v[scan_smem_idx(li)]);
    }
}

inline i64 scan_tmp_words(i64 n) { return ceil_div(n > 0 ? n : 1, SCAN_TILE) + 1; }

// Exclusive scan of in(0..n) fed to out(); *d_total (device, nullable) gets
// the sum.  tmp must hold scan_tmp_words(n) u32.
template <class In, class Out>
int scan_transform(In in, Out out, i64 n, u32 *tmp, u32 *d_total, cudaStream_t st,
                   const char *prof_name = "scan", double prof_bytes = 0) {
    Prof prof_(prof_name, prof_bytes, st);
    if (n <= 0) {
        if (d_total) SAIX_CUDA(cudaMemsetAsync(d_total, 0, sizeof(u32), st));
        return SAIX_OK;
    }
    i64 nb = ceil_div(n, SCAN_TILE);
    k_scan_reduce<In><<<(unsigned)nb, SCAN_THREADS, 0, st>>>(in, n, tmp);
    SAIX_LAUNCHED();
    k_scan_block_sums<<<1, 1024, 0, st>>>(tmp, nb, d_total);
    SAIX_LAUNCHED();
    k_scan_apply<In, Out><<<(unsigned)nb, SCAN_THREADS, 0, st>>>(in, out, n, tmp);
    SAIX_LAUNCHED();
    return SAIX_OK;
}

}  // namespace saix
