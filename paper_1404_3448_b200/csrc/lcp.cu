// lcp.cu -- LCP array (suffix_index.py:460-506 `_kasai_scan`) on sm_100a.
//
// The reference walks text positions in order so the matched length h drops
// by at most one per step (Kasai).  The same walk is done here in the
// permuted-LCP (PLCP / Phi) formulation so every phase has exactly one
// random-access target:
//   k_phi         Phi[sa[r]] = sa[r-1]                   (scatter)
//   k_lcp_seeds   exact PLCP at every chunk start        (word compares)
//   k_plcp        per-thread h-decrement walk over a chunk of LCP_CHUNK text
//                 positions, Phi staged/overwritten in shared memory
//                 (partner text is the only gather)
//   k_lcp_permute lcp[r] = PLCP[sa[r]]                   (gather)
// At C2 size each random target (Phi/PLCP 80 MB, u8 text 20 MB) fits the
// 126 MB L2, so the scatter/gathers stay on chip.
#include "lcp_direct.cuh"

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

constexpr u32 kNone = 0xFFFFFFFFu;

// Phi[sa[r]] = sa[r-1]: the text-order predecessor map (one scatter).
__global__ void k_phi(const u32 *__restrict__ sa, i64 n, u32 *__restrict__ phi) {
    u64 pol = l2_evict_last();  // the scatter target stays on chip, SA streams through
    for (i64 r = (i64)blockIdx.x * blockDim.x + threadIdx.x; r < n; r += (i64)gridDim.x * blockDim.x)
        st_last(phi + __ldcs(sa + r), r ? sa[r - 1] : kNone, pol);
}

// Exact PLCP at every chunk start (seed of the in-chunk walk).
template <typename TT>
__global__ void k_lcp_seeds(const TT *__restrict__ T, i64 n, const u32 *__restrict__ phi,
                            u32 *__restrict__ seeds, i64 nchunks) {
    for (i64 c = (i64)blockIdx.x * blockDim.x + threadIdx.x; c < nchunks; c += (i64)gridDim.x * blockDim.x) {
        i64 i = c * LCP_CHUNK;
        u32 j = phi[i];
        seeds[c] = j == kNone ? 0u : extend_match<TT>(T, n, i, j, 0u);
    }
}

// PLCP in text order, Kasai's h-decrement walk per chunk (in place: the
// phi tile is staged in shared memory and overwritten with PLCP values).
template <typename TT>
__global__ void __launch_bounds__(LCP_THREADS)
k_plcp(const TT *__restrict__ T, i64 n, u32 *__restrict__ phi_plcp, const u32 *__restrict__ seeds,
       u8 *__restrict__ plcp8) {
    __shared__ u32 sh[LCP_TILE + LCP_TILE / 32];
    i64 base = (i64)blockIdx.x * LCP_TILE;
    for (int x = threadIdx.x; x < LCP_TILE; x += LCP_THREADS) {
        i64 i = base + x;
        sh[x + (x >> 5)] = i < n ? phi_plcp[i] : kNone;
    }
    __syncthreads();
    i64 start = base + (i64)threadIdx.x * LCP_CHUNK;
    if (start < n) {
        u32 h = seeds[start / LCP_CHUNK];
        for (int c = 0; c < LCP_CHUNK; c++) {
            i64 i = start + c;
            if (i >= n) break;
            int x = threadIdx.x * LCP_CHUNK + c;
            u32 j = sh[x + (x >> 5)];
            if (j == kNone) {
                h = 0;
            } else if (c > 0) {
                h = extend_match<TT>(T, n, i, j, h);
            }
            sh[x + (x >> 5)] = h;
            if (h) h--;
        }
    }
    __syncthreads();
    for (int x = threadIdx.x; x < LCP_TILE; x += LCP_THREADS) {
        i64 i = base + x;
        if (i < n) {
            u32 h = sh[x + (x >> 5)];
            phi_plcp[i] = h;
            plcp8[i] = (u8)(h < 255 ? h : 255);
        }
    }
}

// lcp[r] = PLCP[sa[r]] (one gather; lcp[0] = PLCP[sa[0]] = 0).  With
// best != nullptr it also folds in longest_overlap's first pass
// (overlap.py:129-136): max lcp over adjacent pairs on opposite sides of the
// separator at `boundary`.
// The gather reads a byte copy of PLCP (values >= 255 escape to the u32
// array): n bytes stay L2-resident where the 4n-byte array would not.
__global__ void k_lcp_permute(const u32 *__restrict__ sa, i64 n, const u32 *__restrict__ plcp,
                              const u8 *__restrict__ plcp8, u32 *__restrict__ lcp, u32 boundary, u32 *best) {
    u32 mx = 0;
    for (i64 r = (i64)blockIdx.x * blockDim.x + threadIdx.x; r < n; r += (i64)gridDim.x * blockDim.x) {
        u32 p = __ldcs(sa + r);
        u32 l = plcp8[p];
        if (l == 255) l = plcp[p];
        __stcs(lcp + r, l);
        if (best && r > 0) {
            u32 q = sa[r - 1];
            bool cross = p != boundary && q != boundary && ((p < boundary) != (q < boundary));
            if (cross && l > mx) mx = l;
        }
    }
    if (best) {
        for (int o = 16; o; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        if (lane_id() == 0 && mx) atomicMax(best, mx);
    }
}

// ------------------------------------------------------------ direct LCP
//
// lcp[r] straight from the two suffixes' text, 32 characters per 64-bit word
// compare on a 2-bit packed copy of the text (alphabet of <= 4 residues plus
// at most one unique separator, whose position bounds every match: two
// different suffixes can never both run through it), or 4 bytes per compare
// on a byte text.  In SA order every suffix pair is an independent thread:
// no Phi scatter, no PLCP walk, no permutation -- only random reads of the
// packed text, which at <= 64 MB (2^28 residues) stays L2-resident.
// Matches are capped at LCP_CAP characters; capped entries are listed and
// extended exactly by one warp each, and when more than n/64 + 64 entries
// hit the cap (highly repetitive text) the Kasai path above runs instead.
__device__ __forceinline__ u32 match_limit(i64 n, i64 sep, i64 i, i64 j) {
    i64 lim = n - (i > j ? i : j);
    if (sep >= 0) {
        if (i <= sep && sep - i < lim) lim = sep - i;
        if (j <= sep && sep - j < lim) lim = sep - j;
    }
    return (u32)(lim < 0 ? 0 : (lim > 0x7FFFFFFF ? 0x7FFFFFFF : lim));
}

__device__ __forceinline__ bool cross_pair(u32 p, u32 q, u32 boundary) {
    return p != boundary && q != boundary && ((p < boundary) != (q < boundary));
}

template <class Txt>
__global__ void k_lcp_direct(Txt tx, i64 n, i64 sep, const u32 *__restrict__ sa, u32 *__restrict__ lcp,
                             u32 *__restrict__ ncap, u32 *__restrict__ list, u32 list_cap, u32 boundary,
                             u32 *best) {
    u32 mx = 0;
    for (i64 r = (i64)blockIdx.x * blockDim.x + threadIdx.x; r < n; r += (i64)gridDim.x * blockDim.x) {
        u32 j = __ldcs(sa + r), h = 0;
        if (r > 0) {
            u32 i = sa[r - 1];
            u32 lim = match_limit(n, sep, i, j);
            u32 stop = lim < LCP_CAP ? lim : LCP_CAP;
            h = tx.match(i, j, 0, stop);
            if (h == LCP_CAP && lim > LCP_CAP) {
                u32 at = atomicAdd(ncap, 1u);
                if (at < list_cap) list[at] = (u32)r;
            }
            if (best && cross_pair(i, j, boundary) && h > mx) mx = h;
        }
        __stcs(lcp + r, h);
    }
    if (best) {
        for (int o = 16; o; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        if (lane_id() == 0 && mx) atomicMax(best, mx);
    }
}

// Packed-text direct LCP with instruction-level parallelism: every thread
// takes LD_ILP adjacent-suffix pairs of its CTA's chunk at once, so the SA
// loads and the first 32-character word compare of all of them are in flight
// together (the first word decides almost every pair of a DNA-like text).
constexpr int LD_ILP = 4;
__global__ void __launch_bounds__(256)
k_lcp_direct_p2(Pack2Text tx, i64 n, i64 sep, const u32 *__restrict__ sa, u32 *__restrict__ lcp,
                u32 *__restrict__ ncap, u32 *__restrict__ list, u32 list_cap, u32 boundary, u32 *best) {
    u32 mx = 0;
    const i64 step = (i64)gridDim.x * 256 * LD_ILP;
    for (i64 base = (i64)blockIdx.x * 256 * LD_ILP; base < n; base += step) {
        u32 iv[LD_ILP], jv[LD_ILP];
        u64 wi[LD_ILP], wj[LD_ILP];
        // rank r's predecessor SA[r-1] and its first text word are lane l-1's
        // own (ranks are consecutive across a warp): one random text load per
        // rank instead of two; lane 0 loads its predecessor itself
        const bool lane0 = (threadIdx.x & 31) == 0;
#pragma unroll
        for (int q = 0; q < LD_ILP; q++) {
            i64 r = base + q * 256 + threadIdx.x;
            jv[q] = r < n ? __ldcs(sa + r) : 0u;
            iv[q] = (lane0 && r > 0 && r < n) ? sa[r - 1] : 0u;
        }
#pragma unroll
        for (int q = 0; q < LD_ILP; q++) {
            wj[q] = load2(tx.W, jv[q]);
            wi[q] = lane0 ? load2(tx.W, iv[q]) : 0ull;
        }
#pragma unroll
        for (int q = 0; q < LD_ILP; q++) {
            const u32 up = __shfl_up_sync(0xffffffffu, jv[q], 1);
            const u64 wup = __shfl_up_sync(0xffffffffu, wj[q], 1);
            if (!lane0) {
                iv[q] = up;
                wi[q] = wup;
            }
        }
#pragma unroll
        for (int q = 0; q < LD_ILP; q++) {
            i64 r = base + q * 256 + threadIdx.x;
            if (r >= n) continue;
            u32 h = 0;
            if (r > 0) {
                u32 i = iv[q], j = jv[q];
                u32 lim = match_limit(n, sep, i, j);
                u32 stop = lim < LCP_CAP ? lim : LCP_CAP;
                u64 d = wi[q] ^ wj[q];
                if (d) h = min((u32)(__ffsll((long long)d) - 1) >> 1, stop);
                else h = tx.match(i, j, 32u < stop ? 32u : stop, stop);
                if (h == LCP_CAP && lim > LCP_CAP) {
                    u32 at = atomicAdd(ncap, 1u);
                    if (at < list_cap) list[at] = (u32)r;
                }
                if (best && cross_pair(i, j, boundary) && h > mx) mx = h;
            }
            __stcs(lcp + r, h);
        }
    }
    if (best) {
        for (int o = 16; o; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        if (lane_id() == 0 && mx) atomicMax(best, mx);
    }
}

// one warp per capped entry: 32 windows of 32 characters (2-bit) per step
template <class Txt>
__global__ void k_lcp_extend(Txt tx, i64 n, i64 sep, const u32 *__restrict__ sa, u32 *__restrict__ lcp,
                             const u32 *__restrict__ ncap, const u32 *__restrict__ list, u32 boundary, u32 *best) {
    const u32 cnt = *ncap;
    const int lane = lane_id();
    for (u32 e = ((i64)blockIdx.x * blockDim.x + threadIdx.x) >> 5; e < cnt; e += ((i64)gridDim.x * blockDim.x) >> 5) {
        u32 r = list[e];
        u32 i = sa[r - 1], j = sa[r];
        u32 lim = match_limit(n, sep, i, j);
        u32 h = LCP_CAP;
        while (h < lim) {
            u32 lo = h + 32u * lane;
            u32 got = lo < lim ? tx.match(i, j, lo, min(lo + 32u, lim)) : lo;
            u32 short_ = __ballot_sync(0xffffffffu, lo < lim && got < min(lo + 32u, lim));
            if (short_) {
                int l = __ffs(short_) - 1;
                h = __shfl_sync(0xffffffffu, got, l);
                break;
            }
            h = min(h + 32u * 32u, lim);
        }
        if (lane == 0) {
            lcp[r] = h;
            if (best && cross_pair(i, j, boundary)) atomicMax(best, h);
        }
    }
}


static int lcp_run(const void *text, int tb, i64 n, const u32 *sa, u32 *lcp, u32 *phi, u32 *seeds, u8 *plcp8,
                   cudaStream_t st, i64 boundary, u32 *best, bool phi_ready) {
    i64 nchunks = ceil_div(n, LCP_CHUNK);
    int g = grid_for(n, 256);
    unsigned tiles = (unsigned)ceil_div(n, LCP_TILE);
    if (!phi_ready) {
        Prof prof_("lcp.phi", 8.0 * n, st);
        k_phi<<<g, 256, 0, st>>>(sa, n, phi);
    }
    SAIX_LAUNCHED();
    {
        Prof prof_("lcp.seeds", 8.0 * nchunks, st);
        if (tb == 1)
            k_lcp_seeds<u8><<<grid_for(nchunks, 256), 256, 0, st>>>((const u8 *)text, n, phi, seeds, nchunks);
        else
            k_lcp_seeds<u32><<<grid_for(nchunks, 256), 256, 0, st>>>((const u32 *)text, n, phi, seeds, nchunks);
    }
    SAIX_LAUNCHED();
    {
        Prof prof_("lcp.plcp", (8.0 + tb) * n, st);
        if (tb == 1) k_plcp<u8><<<tiles, LCP_THREADS, 0, st>>>((const u8 *)text, n, phi, seeds, plcp8);
        else k_plcp<u32><<<tiles, LCP_THREADS, 0, st>>>((const u32 *)text, n, phi, seeds, plcp8);
    }
    SAIX_LAUNCHED();
    {
        Prof prof_("lcp.permute", 12.0 * n, st);
        k_lcp_permute<<<g, 256, 0, st>>>(sa, n, phi, plcp8, lcp, boundary >= 0 ? (u32)boundary : 0u,
                                         boundary >= 0 ? best : nullptr);
    }
    SAIX_LAUNCHED();
    return SAIX_OK;
}

size_t plcp_workspace_bytes(i64 n) {
    Arena ar;
    ar.alloc<u32>(ceil_div(n > 0 ? n : 1, LCP_CHUNK) + 1);
    ar.alloc<u8>(n);
    return ar.peak + Arena::kAlign;
}

int plcp_from_phi(const u8 *text, i64 n, u32 *phi_plcp, void *ws, size_t ws_bytes, cudaStream_t st) {
    Arena ar{(char *)ws, ws_bytes};
    i64 nchunks = ceil_div(n, LCP_CHUNK);
    u32 *seeds = ar.alloc<u32>(nchunks + 1);
    u8 *plcp8 = ar.alloc<u8>(n);
    SAIX_ARENA_OK(ar);
    {
        Prof prof_("lcp.seeds", 8.0 * nchunks, st);
        k_lcp_seeds<u8><<<grid_for(nchunks, 256), 256, 0, st>>>(text, n, phi_plcp, seeds, nchunks);
    }
    SAIX_LAUNCHED();
    {
        Prof prof_("lcp.plcp", 9.0 * n, st);
        k_plcp<u8><<<(unsigned)ceil_div(n, LCP_TILE), LCP_THREADS, 0, st>>>(text, n, phi_plcp, seeds, plcp8);
    }
    SAIX_LAUNCHED();
    return SAIX_OK;
}

int lcp_compute(const void *text, int text_bytes, i64 n, const u32 *sa, u32 *lcp, void *ws, size_t ws_bytes,
                cudaStream_t st, i64 boundary, u32 *best, u32 *phi_in, bool phi_ready, i64 sigma, i64 sep) {
    Arena ar{(char *)ws, ws_bytes};
    u32 *phi = phi_in ? phi_in : ar.alloc<u32>(n);
    u32 *seeds = ar.alloc<u32>(ceil_div(n, LCP_CHUNK) + 1);
    u8 *plcp8 = ar.alloc<u8>(n);
    u64 *W2 = ar.alloc<u64>(pack2_words(n));
    u32 *ncap = ar.alloc<u32>(2);
    u32 *list = ar.alloc<u32>(lcp_list_cap(n));
    SAIX_ARENA_OK(ar);
    // packed path: residues 1..4 (no separator) or 2..5 around a unique
    // separator 1 at `sep`; byte path for other small byte texts
    bool pack = text_bytes == 1 && sigma >= 1 && ((sep < 0 && sigma <= 4) || (sep >= 0 && sigma <= 5));
    bool bytes = !pack && text_bytes == 1 && n <= ((i64)48 << 20);
    if (n > 1 && (pack || bytes) && !phi_ready) {
        if (best) SAIX_CUDA(cudaMemsetAsync(best, 0, sizeof(u32), st));
        SAIX_CUDA(cudaMemsetAsync(ncap, 0, sizeof(u32), st));
        u32 lc = (u32)lcp_list_cap(n);
        u32 bd = boundary >= 0 ? (u32)boundary : 0u;
        u32 *bp = boundary >= 0 ? best : nullptr;
        int g = grid_for(n, 256);
        if (pack) {
            i64 nw = pack2_words(n);
            {
                Prof prof_("lcp.pack2", (double)n + 8.0 * nw, st);
                k_pack2<<<grid_for(nw, 256), 256, 0, st>>>((const u8 *)text, n, sep >= 0 ? 2u : 1u, W2, nw);
            }
            SAIX_LAUNCHED();
            Prof prof_("lcp.direct", 12.0 * n + 2.0 * n / 4, st);
            k_lcp_direct_p2<<<grid_for(ceil_div(n, LD_ILP), 256), 256, 0, st>>>(Pack2Text{W2}, n, sep, sa, lcp, ncap,
                                                                                list, lc, bd, bp);
        } else {
            Prof prof_("lcp.direct", 12.0 * n + 2.0 * n, st);
            k_lcp_direct<ByteText><<<g, 256, 0, st>>>(ByteText{(const u8 *)text, n}, n, sep, sa, lcp, ncap, list, lc,
                                                      bd, bp);
        }
        SAIX_LAUNCHED();
        u32 h = 0;
        SAIX_CUDA(cudaMemcpyAsync(&h, ncap, sizeof(u32), cudaMemcpyDeviceToHost, st));
        SAIX_CUDA(cudaStreamSynchronize(st));
        if (h == 0) return SAIX_OK;
        if (h <= lc) {
            Prof prof_("lcp.extend", 0.0, st);
            int ge = grid_for((i64)h * 32, 256);
            if (pack) k_lcp_extend<Pack2Text><<<ge, 256, 0, st>>>(Pack2Text{W2}, n, sep, sa, lcp, ncap, list, bd, bp);
            else k_lcp_extend<ByteText><<<ge, 256, 0, st>>>(ByteText{(const u8 *)text, n}, n, sep, sa, lcp, ncap, list,
                                                           bd, bp);
            SAIX_LAUNCHED();
            return SAIX_OK;
        }
        // highly repetitive text: Kasai below
        if (best) SAIX_CUDA(cudaMemsetAsync(best, 0, sizeof(u32), st));
    }
    return lcp_run(text, text_bytes, n, sa, lcp, phi, seeds, plcp8, st, boundary, best, phi_ready);
}

}  // namespace saix

using namespace saix;

extern "C" size_t saix_lcp_workspace_bytes(int64_t n) {
    Arena ar;
    ar.alloc<u32>(n);
    ar.alloc<u32>(ceil_div(n > 0 ? n : 1, LCP_CHUNK) + 1);
    ar.alloc<u8>(n);
    ar.alloc<u64>(pack2_words(n));
    ar.alloc<u32>(2);
    ar.alloc<u32>(lcp_list_cap(n));
    return ar.peak + Arena::kAlign;
}

extern "C" int saix_lcp(const void *text, int text_bytes, int64_t n, const uint32_t *sa, const uint32_t *isa,
                        uint32_t *lcp, void *ws, size_t ws_bytes, void *stream) {
    if (n < 0 || (text_bytes != 1 && text_bytes != 4) || (n > 0 && (!text || !sa || !lcp))) {
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
    (void)isa;  // the Phi formulation needs only SA
    return lcp_compute(text, text_bytes, n, sa, lcp, ws, ws_bytes, (cudaStream_t)stream, -1, nullptr);
}

extern "C" int saix_lcp_sigma(const void *text, int text_bytes, int64_t n, int64_t sigma, int64_t separator,
                              const uint32_t *sa, uint32_t *lcp, void *ws, size_t ws_bytes, void *stream) {
    if (n < 0 || (text_bytes != 1 && text_bytes != 4) || (n > 0 && (!text || !sa || !lcp)) || separator >= n) {
        set_error("saix_lcp_sigma: invalid arguments");
        return SAIX_EINVAL;
    }
    if (ws_bytes < saix_lcp_workspace_bytes(n)) {
        set_error("saix_lcp_sigma: workspace too small");
        return SAIX_ENOSPC;
    }
    if (n == 0) return SAIX_OK;
    if (text_bytes == 1 && ((uintptr_t)text & 15)) {
        set_error("saix_lcp_sigma: u8 text must be 16-byte aligned");
        return SAIX_EINVAL;
    }
    return lcp_compute(text, text_bytes, n, sa, lcp, ws, ws_bytes, (cudaStream_t)stream, -1, nullptr, nullptr, false,
                       sigma, separator);
}
