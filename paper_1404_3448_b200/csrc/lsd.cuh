// lsd.cuh -- stable LSD radix partition of u32 payloads by a computed key,
// 8 bits per pass, as three streaming kernels per pass (no look-back chain);
// the stable counting pass of _counting_reorder (reference suffix_index.py:
// 157-171) at batch scale:
//
//   k_lsd_hist     per 4096-item tile, the digit histogram -> hist[d][tile]
//                  (digit-major, so one flat exclusive scan gives every
//                  (digit, tile) its global output offset)
//   scan           scan_transform over digits x tiles
//   k_lsd_scatter  per tile: warp-stable ranking (ballot peers + per-warp digit
//                  counters), tile staged digit-sorted in shared memory and
//                  written as per-digit runs at the scanned offsets
//
// The key is a functor of the payload (the batched-pairs partition keys a
// suffix position by its pair id), so only the 4 B payloads move.
//   struct Key { __device__ u32 operator()(u32 v) const; };
#pragma once

#include "scan.cuh"

namespace saix {

constexpr int LSD_THREADS = 512, LSD_WARPS = LSD_THREADS / 32, LSD_ITEMS = 8;
constexpr int LSD_TILE = LSD_THREADS * LSD_ITEMS;  // 4096

// one CTA per segment of LSD_SEG tiles (the per-CTA setup, histogram rows
// and scan length amortised over 32 K items)
constexpr int LSD_SEG = 8;

template <class Key>
__global__ void __launch_bounds__(LSD_THREADS)
k_lsd_hist(const u32 *__restrict__ in, i64 n, Key key, int shift, u32 mask, i64 segs, u32 *__restrict__ hist) {
    __shared__ u32 cnt[LSD_WARPS][256];  // warp-private: plain shared atomics, no peer votes
    const int wp = threadIdx.x >> 5;
    for (int d = threadIdx.x & 31; d < 256; d += 32) cnt[wp][d] = 0;
    __syncthreads();
    const i64 sgi = blockIdx.x;
    const i64 base = sgi * LSD_TILE * LSD_SEG;
    for (int x0 = 0; x0 < LSD_TILE * LSD_SEG; x0 += LSD_THREADS * 8) {
        u32 v[8];
#pragma unroll
        for (int q = 0; q < 8; q++) {  // 8 loads in flight per thread
            i64 i = base + x0 + q * LSD_THREADS + threadIdx.x;
            v[q] = i < n ? __ldcs(in + i) : 0u;
        }
#pragma unroll
        for (int q = 0; q < 8; q++) {
            i64 i = base + x0 + q * LSD_THREADS + threadIdx.x;
            if (i < n) atomicAdd(&cnt[wp][(key(v[q]) >> shift) & mask], 1u);
        }
    }
    __syncthreads();
    for (int d = threadIdx.x; d <= (int)mask; d += LSD_THREADS) {
        u32 c = 0;
#pragma unroll
        for (int q = 0; q < LSD_WARPS; q++) c += cnt[q][d];
        hist[(i64)d * segs + sgi] = c;
    }
}

template <class Key>
__global__ void __launch_bounds__(LSD_THREADS)
k_lsd_scatter(const u32 *__restrict__ in, i64 n, Key key, int shift, u32 mask, i64 segs,
              const u32 *__restrict__ offs, u32 *__restrict__ out) {
    __shared__ u32 sv[LSD_TILE];
    __shared__ u16 sd[LSD_TILE];
    __shared__ u32 cnt[LSD_WARPS][256];
    __shared__ u32 tile_excl[256], gbase[256], sh_warp[9];
    const int wp = threadIdx.x >> 5, lane = lane_id();
    const i64 sgi = blockIdx.x;
    const int d = threadIdx.x;
    if (d < 256) gbase[d] = d <= (int)mask ? offs[(i64)d * segs + sgi] : 0u;  // running output cursor per digit
    for (int tile = 0; tile < LSD_SEG; tile++) {
        const i64 t0 = (sgi * LSD_SEG + tile) * LSD_TILE;
        if (t0 >= n) break;  // block-uniform
        for (int dd = lane; dd < 256; dd += 32) cnt[wp][dd] = 0;
        __syncthreads();
        const i64 seg = t0 + (i64)wp * (32 * LSD_ITEMS);
        u32 v[LSD_ITEMS], pk[LSD_ITEMS];  // pk = digit | rank-in-warp-digit << 9
        const u32 lt = lanemask_lt();
#pragma unroll
        for (int r = 0; r < LSD_ITEMS; r++) {
            i64 i = seg + r * 32 + lane;
            pk[r] = 256u;
            if (i < n) {
                v[r] = __ldcs(in + i);
                pk[r] = (key(v[r]) >> shift) & mask;
            }
        }
#pragma unroll
        for (int r = 0; r < LSD_ITEMS; r++) {
            u32 dg = pk[r];
            bool ok = dg < 256u;
            u32 peers = digit_peers_w(dg, mask);
            u32 before = __popc(peers & lt);
            u32 cur = ok ? cnt[wp][dg] : 0u;
            __syncwarp();
            if (ok && before == 0) cnt[wp][dg] = cur + __popc(peers);
            __syncwarp();
            pk[r] |= (cur + before) << 9;
        }
        __syncthreads();
        u32 run = 0, inc = 0;
        if (d < 256) {
#pragma unroll
            for (int q = 0; q < LSD_WARPS; q++) {
                u32 c = cnt[q][d];
                cnt[q][d] = run;
                run += c;
            }
            inc = run;
            for (int o = 1; o < 32; o <<= 1) {
                u32 y = __shfl_up_sync(0xffffffffu, inc, o);
                if (lane >= o) inc += y;
            }
            if (lane == 31) sh_warp[wp] = inc;
        }
        __syncthreads();
        if (wp == 0) {
            u32 x = lane < 8 ? sh_warp[lane] : 0u, xi = x;
            for (int o = 1; o < 32; o <<= 1) {
                u32 y = __shfl_up_sync(0xffffffffu, xi, o);
                if (lane >= o) xi += y;
            }
            if (lane < 8) sh_warp[lane] = xi - x;
            if (lane == 7) sh_warp[8] = xi;
        }
        __syncthreads();
        if (d < 256) tile_excl[d] = sh_warp[wp] + inc - run;
        __syncthreads();
#pragma unroll
        for (int r = 0; r < LSD_ITEMS; r++) {
            u32 dg = pk[r] & 0x1FFu;
            if (dg < 256u) {
                u32 lp = tile_excl[dg] + cnt[wp][dg] + (pk[r] >> 9);
                sv[lp] = v[r];
                sd[lp] = (u16)dg;
            }
        }
        __syncthreads();
        const u32 valid = sh_warp[8];
        for (u32 x = threadIdx.x; x < valid; x += LSD_THREADS) {
            u32 dg = sd[x];
            __stcs(out + gbase[dg] + (x - tile_excl[dg]), sv[x]);
        }
        __syncthreads();
        if (d < 256) gbase[d] += run;  // this tile's items of digit d
        __syncthreads();
    }
}

struct LsdHistIn {
    const u32 *h;
    __device__ u32 operator()(i64 i) const { return h[i]; }
};
struct LsdStoreExcl {
    u32 *o;
    __device__ void operator()(i64 i, u32 excl, u32) const { o[i] = excl; }
};

inline i64 lsd_tiles(i64 n) { return ceil_div(n > 0 ? n : 1, (i64)LSD_TILE * LSD_SEG); }  // segments
// scratch words: hist (256 x segments) + scan temps
inline i64 lsd_scratch_words(i64 n) { return 256 * lsd_tiles(n) + scan_tmp_words(256 * lsd_tiles(n)) + 64; }

// Stable sort of the payloads by key bits [0, bits): ceil(bits/8) passes of
// equal digit width (7-bit digits for 14-bit keys keep the per-tile runs at
// >= 32 items), ping-pong between a and b; the result pointer is returned in
// `out`.
template <class Key>
int lsd_partition(Key key, u32 *a, u32 *b, i64 n, int bits, u32 *scratch, u32 *&out, cudaStream_t st,
                  const char *prof) {
    int passes = (bits + 7) / 8;
    int width = passes ? (bits + passes - 1) / passes : 0;
    Prof prof_(prof, 12.0 * n * passes, st);
    out = a;
    if (n <= 0 || passes == 0) return SAIX_OK;
    i64 tiles = lsd_tiles(n);
    u32 *hist = scratch, *tmp = hist + 256 * tiles;
    u32 *src = a, *dst = b;
    const u32 mask = (1u << width) - 1u;
    for (int p = 0; p < passes; p++) {
        k_lsd_hist<Key><<<(unsigned)tiles, LSD_THREADS, 0, st>>>(src, n, key, width * p, mask, tiles, hist);
        SAIX_LAUNCHED();
        SAIX_TRY(scan_transform(LsdHistIn{hist}, LsdStoreExcl{hist}, (i64)(mask + 1) * tiles, tmp, nullptr, st,
                                "lsd.scan", 0));
        k_lsd_scatter<Key><<<(unsigned)tiles, LSD_THREADS, 0, st>>>(src, n, key, width * p, mask, tiles, hist, dst);
        SAIX_LAUNCHED();
        u32 *x = src;
        src = dst;
        dst = x;
    }
    out = src;
    return SAIX_OK;
}

}  // namespace saix
