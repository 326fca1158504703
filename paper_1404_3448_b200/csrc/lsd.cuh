// lsd.cuh -- stable LSD radix partition of u32 payloads by a computed key,
// 8 bits per pass, as three streaming kernels per pass (no look-back chain):
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

template <class Key>
__global__ void __launch_bounds__(LSD_THREADS)
k_lsd_hist(const u32 *__restrict__ in, i64 n, Key key, int shift, i64 tiles, u32 *__restrict__ hist) {
    __shared__ u32 cnt[256];
    for (int d = threadIdx.x; d < 256; d += LSD_THREADS) cnt[d] = 0;
    __syncthreads();
    const i64 t = blockIdx.x;
    for (int x = threadIdx.x; x < LSD_TILE; x += LSD_THREADS) {
        i64 i = t * LSD_TILE + x;
        u32 d = i < n ? (key(__ldg(in + i)) >> shift) & 0xFFu : 0xFFFFFFFFu;
        u32 peers = digit_peers(d);
        if (d != 0xFFFFFFFFu && (peers & lanemask_lt()) == 0) atomicAdd(&cnt[d], (u32)__popc(peers));
    }
    __syncthreads();
    for (int d = threadIdx.x; d < 256; d += LSD_THREADS) hist[(i64)d * tiles + t] = cnt[d];
}

template <class Key>
__global__ void __launch_bounds__(LSD_THREADS)
k_lsd_scatter(const u32 *__restrict__ in, i64 n, Key key, int shift, i64 tiles, const u32 *__restrict__ offs,
              u32 *__restrict__ out) {
    __shared__ u32 sv[LSD_TILE];
    __shared__ u16 sd[LSD_TILE];
    __shared__ u32 cnt[LSD_WARPS][256];
    __shared__ u32 tile_excl[256], gbase[256], sh_warp[9];
    const int wp = threadIdx.x >> 5, lane = lane_id();
    for (int d = lane; d < 256; d += 32) cnt[wp][d] = 0;
    __syncthreads();
    const i64 t = blockIdx.x;
    const i64 seg = t * LSD_TILE + (i64)wp * (32 * LSD_ITEMS);
    u32 v[LSD_ITEMS], pk[LSD_ITEMS];  // pk = digit | rank-in-warp-digit << 9
    const u32 lt = lanemask_lt();
#pragma unroll
    for (int r = 0; r < LSD_ITEMS; r++) {
        i64 i = seg + r * 32 + lane;
        pk[r] = 256u;
        if (i < n) {
            v[r] = __ldcs(in + i);
            pk[r] = (key(v[r]) >> shift) & 0xFFu;
        }
    }
#pragma unroll
    for (int r = 0; r < LSD_ITEMS; r++) {
        u32 d = pk[r];
        bool ok = d < 256u;
        u32 peers = digit_peers(d);
        u32 before = __popc(peers & lt);
        u32 cur = ok ? cnt[wp][d] : 0u;
        __syncwarp();
        if (ok && before == 0) cnt[wp][d] = cur + __popc(peers);
        __syncwarp();
        pk[r] |= (cur + before) << 9;
    }
    __syncthreads();
    u32 run = 0, inc = 0;
    const int d = threadIdx.x;
    if (d < 256) {
#pragma unroll
        for (int q = 0; q < LSD_WARPS; q++) {
            u32 c = cnt[q][d];
            cnt[q][d] = run;
            run += c;
        }
        gbase[d] = run ? offs[(i64)d * tiles + t] : 0u;
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
}

struct LsdHistIn {
    const u32 *h;
    __device__ u32 operator()(i64 i) const { return h[i]; }
};
struct LsdStoreExcl {
    u32 *o;
    __device__ void operator()(i64 i, u32 excl, u32) const { o[i] = excl; }
};

inline i64 lsd_tiles(i64 n) { return ceil_div(n > 0 ? n : 1, LSD_TILE); }
// scratch words: hist (256 x tiles) + scan temps
inline i64 lsd_scratch_words(i64 n) { return 256 * lsd_tiles(n) + scan_tmp_words(256 * lsd_tiles(n)) + 64; }

// Stable sort of the payloads by key bits [0, 8*passes): ping-pong between
// a and b; the result pointer is returned in `out`.
template <class Key>
int lsd_partition(Key key, u32 *a, u32 *b, i64 n, int passes, u32 *scratch, u32 *&out, cudaStream_t st,
                  const char *prof) {
    Prof prof_(prof, 12.0 * n * passes, st);
    out = a;
    if (n <= 0) return SAIX_OK;
    i64 tiles = lsd_tiles(n);
    u32 *hist = scratch, *tmp = hist + 256 * tiles;
    u32 *src = a, *dst = b;
    for (int p = 0; p < passes; p++) {
        k_lsd_hist<Key><<<(unsigned)tiles, LSD_THREADS, 0, st>>>(src, n, key, 8 * p, tiles, hist);
        SAIX_LAUNCHED();
        SAIX_TRY(scan_transform(LsdHistIn{hist}, LsdStoreExcl{hist}, 256 * tiles, tmp, nullptr, st, "lsd.scan", 0));
        k_lsd_scatter<Key><<<(unsigned)tiles, LSD_THREADS, 0, st>>>(src, n, key, 8 * p, tiles, hist, dst);
        SAIX_LAUNCHED();
        u32 *x = src;
        src = dst;
        dst = x;
    }
    out = src;
    return SAIX_OK;
}

}  // namespace saix
