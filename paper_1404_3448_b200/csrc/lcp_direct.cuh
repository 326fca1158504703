// lcp_direct.cuh -- word-compare matching of two suffixes (lcp.cu direct
// LCP, and the batched-pairs LCP in overlap.cu): a 2-bit packed copy of the
// text (32 characters per 64-bit word, LSB first) or the byte text itself.
// lcp[r] = longest common prefix of suffixes sa[r-1], sa[r] -- the values
// _kasai_scan / build_lcp produce (reference suffix_index.py:461-506).
#pragma once

#include "common.cuh"

namespace saix {

constexpr u32 LCP_CAP = 256;

__device__ __forceinline__ u64 load2(const u64 *__restrict__ W, i64 p) {
    i64 q = p >> 5;
    u32 o = (u32)(p & 31) * 2;
    u64 lo = W[q];
    return o ? (lo >> o) | (W[q + 1] << (64 - o)) : lo;
}

// chars [p, p+32) -> 2-bit codes (c - base) & 3, LSB first; zero tail words
static __global__ void k_pack2(const u8 *__restrict__ T, i64 n, u32 base, u64 *__restrict__ W, i64 nw) {
    for (i64 w = (i64)blockIdx.x * blockDim.x + threadIdx.x; w < nw; w += (i64)gridDim.x * blockDim.x) {
        i64 p0 = w * 32;
        u64 x = 0;
        if (p0 + 32 <= n) {
            const uint4 *T16 = reinterpret_cast<const uint4 *>(T + p0);
            uint4 a = __ldcs(T16), b = __ldcs(T16 + 1);
            u32 v[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
#pragma unroll
            for (int q = 0; q < 8; q++)
#pragma unroll
                for (int c = 0; c < 4; c++) x |= (u64)((((v[q] >> (8 * c)) & 0xFFu) - base) & 3u) << (2 * (4 * q + c));
        } else {
            for (i64 p = p0; p < n && p < p0 + 32; p++) x |= (u64)(((u32)T[p] - base) & 3u) << (2 * (p - p0));
        }
        W[w] = x;
    }
}

struct Pack2Text {
    const u64 *W;
    __device__ __forceinline__ u32 match(i64 i, i64 j, u32 h, u32 stop) const {
        while (h < stop) {
            u64 d = load2(W, i + h) ^ load2(W, j + h);
            if (d) return min(h + ((u32)(__ffsll((long long)d) - 1) >> 1), stop);
            h += 32;
        }
        return stop;
    }
};
struct ByteText {
    const u8 *T;
    i64 n;
    __device__ __forceinline__ u32 match(i64 i, i64 j, u32 h, u32 stop) const {
        const u32 *W = reinterpret_cast<const u32 *>(T);
        while (h < stop) {
            i64 a = i + h, b = j + h;
            if (n - (a > b ? a : b) >= 8) {
                i64 aw = a >> 2, bw = b >> 2;
                u32 x = __funnelshift_r(W[aw], W[aw + 1], (u32)(a & 3) * 8);
                u32 y = __funnelshift_r(W[bw], W[bw + 1], (u32)(b & 3) * 8);
                u32 d = x ^ y;
                if (d) return min(h + (u32)(__ffs(d) - 1) / 8, stop);
                h += 4;
            } else {
                if (T[a] != T[b]) return h;
                h++;
            }
        }
        return stop;
    }
};

inline i64 lcp_list_cap(i64 n) { return n / 64 + 64; }
inline i64 pack2_words(i64 n) { return ceil_div(n > 0 ? n : 1, 32) + 2; }

}  // namespace saix
