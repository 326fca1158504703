// radix.cuh -- stable LSD radix sort of (key, u32 value) pairs, 8-bit digits.
//
// The reference models DC3's sorting passes as a bulk-synchronous per-bit
// split (parallel_sort.py:150-203: stable 1-bit split, dest = b ? i - f +
// zeros : f, LSD digit passes).  On B200 one pass handles an 8-bit digit:
//   upsweep   per-tile digit histogram (shared-memory atomics)
//   scan      exclusive scan over the digit-major [digit][tile] table
//   downsweep per-warp stable ranking with __match_any_sync (the 256-way
//             generalisation of the ballot split), warp prefix per digit,
//             scatter.
// Stability: a tile is split into contiguous per-warp segments processed in
// index order, so equal digits keep their input order.
#pragma once

#include "scan.cuh"

namespace saix {

constexpr int RS_BITS = 8;
constexpr int RS_RADIX = 1 << RS_BITS;
constexpr int RS_THREADS = 256;
constexpr int RS_WARPS = RS_THREADS / 32;
constexpr int RS_ITEMS = 16;
constexpr int RS_TILE = RS_THREADS * RS_ITEMS;       // 4096
constexpr int RS_WARP_ITEMS = 32 * RS_ITEMS;         // 512 per warp

inline i64 radix_tiles(i64 n) { return ceil_div(n > 0 ? n : 1, RS_TILE); }
inline i64 radix_hist_words(i64 n) { return (i64)RS_RADIX * radix_tiles(n); }

template <typename K>
__global__ void __launch_bounds__(RS_THREADS)
k_radix_upsweep(const K *__restrict__ keys, i64 n, int shift, u32 *__restrict__ hist, i64 ntiles) {
    __shared__ u32 sh[RS_RADIX];
    for (int d = threadIdx.x; d < RS_RADIX; d += RS_THREADS) sh[d] = 0;
    __syncthreads();
    i64 base = (i64)blockIdx.x * RS_TILE;
#pragma unroll 4
    for (int r = 0; r < RS_ITEMS; r++) {
        i64 i = base + r * RS_THREADS + threadIdx.x;
        if (i < n) {
            u32 d = (u32)(keys[i] >> shift) & (RS_RADIX - 1);
            atomicAdd(&sh[d], 1u);
        }
    }
    __syncthreads();
    for (int d = threadIdx.x; d < RS_RADIX; d += RS_THREADS)
        hist[(i64)d * ntiles + blockIdx.x] = sh[d];
}

template <typename K>
__global__ void __launch_bounds__(RS_THREADS)
k_radix_downsweep(const K *__restrict__ keys, const u32 *__restrict__ vals, i64 n, int shift,
                  const u32 *__restrict__ offs, i64 ntiles, K *__restrict__ keys_out,
                  u32 *__restrict__ vals_out) {
    __shared__ u32 sh_cnt[RS_WARPS][RS_RADIX];
    __shared__ u32 sh_base[RS_RADIX];
    int w = threadIdx.x >> 5;
    int lane = lane_id();
    for (int d = lane; d < RS_RADIX; d += 32) sh_cnt[w][d] = 0;
    __syncwarp();
    i64 seg = (i64)blockIdx.x * RS_TILE + (i64)w * RS_WARP_ITEMS;
    K k[RS_ITEMS];
    u32 v[RS_ITEMS];
    u32 rank[RS_ITEMS];
    u32 dig[RS_ITEMS];
    u32 lt = lanemask_lt();
#pragma unroll
    for (int r = 0; r < RS_ITEMS; r++) {
        i64 i = seg + r * 32 + lane;
        bool ok = i < n;
        k[r] = ok ? keys[i] : (K)0;
        v[r] = ok ? vals[i] : 0u;
        u32 d = ok ? ((u32)(k[r] >> shift) & (RS_RADIX - 1)) : (u32)RS_RADIX;
        dig[r] = d;
        u32 peers = __match_any_sync(0xffffffffu, d);
        u32 before = __popc(peers & lt);
        u32 cur = ok ? sh_cnt[w][d] : 0u;
        __syncwarp();
        if (ok && before == 0) sh_cnt[w][d] = cur + __popc(peers);
        __syncwarp();
        rank[r] = cur + before;
    }
    __syncthreads();
    // per digit: exclusive prefix over warps, then the tile's global offset
    for (int d = threadIdx.x; d < RS_RADIX; d += RS_THREADS) {
        u32 run = 0;
#pragma unroll
        for (int q = 0; q < RS_WARPS; q++) {
            u32 c = sh_cnt[q][d];
            sh_cnt[q][d] = run;
            run += c;
        }
        sh_base[d] = offs[(i64)d * ntiles + blockIdx.x];
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < RS_ITEMS; r++) {
        u32 d = dig[r];
        if (d < RS_RADIX) {
            u32 dst = sh_base[d] + sh_cnt[w][d] + rank[r];
            keys_out[dst] = k[r];
            vals_out[dst] = v[r];
        }
    }
}

struct HistLoad {
    const u32 *h;
    __device__ u32 operator()(i64 i) const { return h[i]; }
};
struct HistStore {
    u32 *h;
    __device__ void operator()(i64 i, u32 excl, u32) const { h[i] = excl; }
};

// Scratch a sort of n pairs needs besides the alternate key/value buffers.
inline i64 radix_scratch_words(i64 n) {
    return radix_hist_words(n) + scan_tmp_words(radix_hist_words(n)) + 64;
}

// Sorts keys[0..n)/vals[0..n) on bits [begin_bit, end_bit).  Ping-pongs with
// keys_alt/vals_alt; on return `keys`/`vals` point at the sorted data.
template <typename K>
int radix_sort_pairs(K *&keys, u32 *&vals, K *keys_alt, u32 *vals_alt, i64 n, int begin_bit,
                     int end_bit, u32 *scratch, cudaStream_t st) {
    if (n <= 1) return SAIX_OK;
    i64 ntiles = radix_tiles(n);
    i64 hw = (i64)RS_RADIX * ntiles;
    u32 *hist = scratch;
    u32 *stmp = scratch + hw;
    for (int shift = begin_bit; shift < end_bit; shift += RS_BITS) {
        Prof prof_(sizeof(K) == 8 ? "radix.pass64" : "radix.pass32",
                   (double)n * (3 * sizeof(K) + 2 * 4), st);
        k_radix_upsweep<K><<<(unsigned)ntiles, RS_THREADS, 0, st>>>(keys, n, shift, hist, ntiles);
        SAIX_LAUNCHED();
        SAIX_TRY(scan_transform(HistLoad{hist}, HistStore{hist}, hw, stmp, nullptr, st, "radix.histscan",
                                8.0 * hw));
        k_radix_downsweep<K><<<(unsigned)ntiles, RS_THREADS, 0, st>>>(keys, vals, n, shift, hist,
                                                                      ntiles, keys_alt, vals_alt);
        SAIX_LAUNCHED();
        K *tk = keys;
        keys = keys_alt;
        keys_alt = tk;
        u32 *tv = vals;
        vals = vals_alt;
        vals_alt = tv;
    }
    return SAIX_OK;
}

}  // namespace saix
