// lcp.cu -- Kasai LCP (suffix_index.py:460-506 `_kasai_scan`) on sm_100a.
//
// The reference walks text positions in order so the matched length h drops
// by at most one per step.  Here every thread owns a contiguous chunk of
// LCP_CHUNK text positions and runs the same h-decrement walk inside it,
// starting from a seed; chunk seeds come from a sparse pass that computes
// the exact PLCP value at every chunk start (word-parallel compares), so the
// in-chunk walk never restarts from zero.  ISA is staged through shared
// memory in coalesced tiles; SA[r-1] and the partner text are gathers and
// lcp[r] is a scatter (one random access each).
#include "common.cuh"

namespace saix {

constexpr int LCP_THREADS = 256;
constexpr int LCP_CHUNK = 32;
constexpr int LCP_TILE = LCP_THREADS * LCP_CHUNK;

// Matched length of suffixes i and j starting from `h` already known equal.
template <typename TT>
__device__ __forceinline__ u32 extend_match(const TT *__restrict__ T, i64 n, i64 i, i64 j, u32 h) {
    while (i + h < n && j + h < n && T[i + h] == T[j + h]) h++;
    return h;
}

// u8 text: compare 4 characters at a time with funnel-shifted word loads.
template <>
__device__ __forceinline__ u32 extend_match<u8>(const u8 *__restrict__ T, i64 n, i64 i, i64 j, u32 h) {
    const u32 *W = reinterpret_cast<const u32 *>(T);
    while (true) {
        i64 a = i + h, b = j + h;
        i64 rem = n - (a > b ? a : b);
        if (rem <= 0) return h;
        if (rem >= 8) {
            // 4-byte windows at arbitrary offsets from two aligned words each
            i64 aw = a >> 2, bw = b >> 2;
            u32 as = (u32)(a & 3) * 8, bs = (u32)(b & 3) * 8;
            u32 x = __funnelshift_r(W[aw], W[aw + 1], as);
            u32 y = __funnelshift_r(W[bw], W[bw + 1], bs);
            u32 d = x ^ y;
            if (d) return h + (__ffs(d) - 1) / 8;
            h += 4;
        } else {
            if (T[a] != T[b]) return h;
            h++;
        }
    }
}

// Exact PLCP at every chunk start (seed of the in-chunk walk).
template <typename TT>
__global__ void k_lcp_seeds(const TT *__restrict__ T, i64 n, const u32 *__restrict__ sa,
                            const u32 *__restrict__ isa, u32 *__restrict__ seeds, i64 nchunks) {
    for (i64 c = (i64)blockIdx.x * blockDim.x + threadIdx.x; c < nchunks; c += (i64)gridDim.x * blockDim.x) {
        i64 i = c * LCP_CHUNK;
        u32 r = isa[i];
        seeds[c] = r == 0 ? 0u : extend_match<TT>(T, n, i, sa[r - 1], 0u);
    }
}

template <typename TT>
__global__ void __launch_bounds__(LCP_THREADS)
k_lcp_kasai(const TT *__restrict__ T, i64 n, const u32 *__restrict__ sa, const u32 *__restrict__ isa,
            const u32 *__restrict__ seeds, u32 *__restrict__ lcp) {
    __shared__ u32 sh[LCP_TILE + LCP_TILE / 32];
    i64 base = (i64)blockIdx.x * LCP_TILE;
    for (int x = threadIdx.x; x < LCP_TILE; x += LCP_THREADS) {
        i64 i = base + x;
        sh[x + (x >> 5)] = i < n ? isa[i] : 0u;
    }
    __syncthreads();
    i64 start = base + (i64)threadIdx.x * LCP_CHUNK;
    if (start >= n) return;
    u32 h = seeds[start / LCP_CHUNK];
    for (int c = 0; c < LCP_CHUNK; c++) {
        i64 i = start + c;
        if (i >= n) break;
        int x = threadIdx.x * LCP_CHUNK + c;
        u32 r = sh[x + (x >> 5)];
        if (r == 0) {
            lcp[0] = 0;
            h = 0;
            continue;
        }
        if (c > 0) h = extend_match<TT>(T, n, i, sa[r - 1], h);
        lcp[r] = h;
        if (h) h--;
    }
}

static int lcp_run(const void *text, int tb, i64 n, const u32 *sa, const u32 *isa, u32 *lcp, u32 *seeds,
                   cudaStream_t st) {
    i64 nchunks = ceil_div(n, LCP_CHUNK);
    int g = grid_for(nchunks, 256);
    unsigned tiles = (unsigned)ceil_div(n, LCP_TILE);
    if (tb == 1) {
        k_lcp_seeds<u8><<<g, 256, 0, st>>>((const u8 *)text, n, sa, isa, seeds, nchunks);
        SAIX_LAUNCHED();
        k_lcp_kasai<u8><<<tiles, LCP_THREADS, 0, st>>>((const u8 *)text, n, sa, isa, seeds, lcp);
    } else {
        k_lcp_seeds<u32><<<g, 256, 0, st>>>((const u32 *)text, n, sa, isa, seeds, nchunks);
        SAIX_LAUNCHED();
        k_lcp_kasai<u32><<<tiles, LCP_THREADS, 0, st>>>((const u32 *)text, n, sa, isa, seeds, lcp);
    }
    SAIX_LAUNCHED();
    return SAIX_OK;
}

}  // namespace saix

using namespace saix;

extern "C" size_t saix_lcp_workspace_bytes(int64_t n) {
    return (size_t)(ceil_div(n > 0 ? n : 1, LCP_CHUNK) + 64) * 4 + Arena::kAlign;
}

extern "C" int saix_lcp(const void *text, int text_bytes, int64_t n, const uint32_t *sa, const uint32_t *isa,
                        uint32_t *lcp, void *ws, size_t ws_bytes, void *stream) {
    if (n < 0 || (text_bytes != 1 && text_bytes != 4) || (n > 0 && (!text || !sa || !isa || !lcp))) {
        set_error("saix_lcp: invalid arguments");
        return SAIX_EINVAL;
    }
    if (ws_bytes < saix_lcp_workspace_bytes(n)) {
        set_error("saix_lcp: workspace too small");
        return SAIX_ENOSPC;
    }
    if (n == 0) return SAIX_OK;
    // u8 word compares need a 4-byte aligned text and only touch bytes < n.
    if (text_bytes == 1 && ((uintptr_t)text & 3)) {
        set_error("saix_lcp: u8 text must be 4-byte aligned");
        return SAIX_EINVAL;
    }
    return lcp_run(text, text_bytes, n, sa, isa, lcp, (u32 *)ws, (cudaStream_t)stream);
}
