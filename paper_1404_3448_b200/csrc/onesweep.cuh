// onesweep.cuh -- stable LSD radix sort, one kernel per 8-bit digit pass with
// decoupled look-back (the B200 realisation of the reference's per-digit
// split passes, parallel_sort.py:150-203).
//
//   k_os_hist   one read of the source: privatised histograms of every digit
//               pass at once (all passes' counts are permutation-invariant)
//   k_os_scan   per-pass exclusive digit offsets (one CTA)
//   k_os_pass   per tile (in atomic-ticket order): load, warp-stable ranking
//               (8-ballot peer masks), publish the tile's per-digit counts,
//               look back over earlier tiles' status words for the digit's
//               global prefix, stage the tile digit-sorted in shared memory,
//               write runs out coalesced.
//
// Sources are functors so the first pass can build keys on the fly (DC3
// triple keys straight from the text; the mod-0 split straight from the
// sample order with an in-line filter) without materialising a key array:
//   struct Src { __device__ bool get(i64 i, K &key, u32 &val) const; };
// Items for which get() returns false are dropped (filter); the output holds
// the valid items only, in stable order.
#pragma once

#include <cstdlib>

#include "common.cuh"

namespace saix {

constexpr int OS_BITS = 8;
constexpr int OS_RADIX = 1 << OS_BITS;
constexpr int OS_THREADS = 256;
constexpr int OS_WARPS = OS_THREADS / 32;
constexpr int OS_ITEMS = 16;                    // default items per thread
constexpr int OS_MIN_ITEMS = 8;                 // smallest variant (scratch sizing)
constexpr int OS_TILE = OS_THREADS * OS_ITEMS;  // 4096
constexpr int OS_MAX_PASSES = 8;
constexpr u32 OS_FLAG_AGG = 1u << 30, OS_FLAG_PRE = 2u << 30, OS_MASK = (1u << 30) - 1;
static_assert(OS_THREADS == OS_RADIX, "one thread per digit in the look-back phase");

template <typename K>
struct ArraySrc {
    const K *keys;
    const u32 *vals;
    __device__ __forceinline__ bool get(i64 i, K &k, u32 &v) const {
        k = keys[i];
        v = vals[i];
        return true;
    }
};

inline i64 os_tiles(i64 n, int items = OS_MIN_ITEMS) { return ceil_div(n > 0 ? n : 1, (i64)OS_THREADS * items); }

// Scratch: hist [passes][256] + offsets + status [tiles][256] + ticket.
inline i64 os_scratch_words(i64 n) { return 2 * OS_MAX_PASSES * OS_RADIX + 64 + os_tiles(n) * OS_RADIX + 64; }

// Digit histograms of every pass in one read.  Few distinct digits per warp
// are the common case (small alphabets, high key bits), so counts are
// warp-aggregated when the digit is uniform across the warp (vote only).
template <typename K, class Src>
__global__ void __launch_bounds__(OS_THREADS)
k_os_hist(Src src, i64 n, int shift0, int passes, u32 *__restrict__ hist) {
    __shared__ u32 sh[OS_MAX_PASSES][OS_RADIX];
    for (int x = threadIdx.x; x < OS_MAX_PASSES * OS_RADIX; x += OS_THREADS) (&sh[0][0])[x] = 0;
    __syncthreads();
    const u32 lt = lanemask_lt();
    const i64 stride = (i64)gridDim.x * blockDim.x;
    for (i64 base = (i64)blockIdx.x * blockDim.x; base < n; base += stride) {  // warp-uniform trip count
        i64 i = base + threadIdx.x;
        K k = 0;
        u32 v;
        bool ok = i < n && src.get(i, k, v);
        u32 okm = __ballot_sync(0xffffffffu, ok);
        for (int p = 0; p < passes; p++) {
            u32 d = ok ? ((u32)(k >> (shift0 + OS_BITS * p)) & (OS_RADIX - 1)) : (u32)OS_RADIX;
            // uniform digit across the valid lanes (high key bits, small
            // alphabets): one atomic for the warp; else one per lane
            u32 d0 = __shfl_sync(0xffffffffu, d, __ffs(okm ? okm : 1u) - 1);
            bool uni = __all_sync(0xffffffffu, !ok || d == d0);
            if (uni) {
                if (okm && (okm & lt) == 0 && ok) atomicAdd(&sh[p][d], (u32)__popc(okm));
            } else if (ok) {
                atomicAdd(&sh[p][d], 1u);
            }
        }
    }
    __syncthreads();
    for (int x = threadIdx.x; x < passes * OS_RADIX; x += OS_THREADS)
        if ((&sh[0][0])[x]) atomicAdd(&hist[x], (&sh[0][0])[x]);
}

// One CTA of 256 threads: exclusive scan over digits of every pass.
static __global__ void __launch_bounds__(OS_RADIX) k_os_scan(const u32 *__restrict__ hist, int passes, u32 *__restrict__ offs,
                                                       u32 *__restrict__ total) {
    __shared__ u32 sh[OS_RADIX];
    for (int p = 0; p < passes; p++) {
        u32 v = hist[p * OS_RADIX + threadIdx.x];
        sh[threadIdx.x] = v;
        __syncthreads();
        // Hillis-Steele inclusive scan over 256 digits
        for (int o = 1; o < OS_RADIX; o <<= 1) {
            u32 y = threadIdx.x >= o ? sh[threadIdx.x - o] : 0u;
            __syncthreads();
            sh[threadIdx.x] += y;
            __syncthreads();
        }
        offs[p * OS_RADIX + threadIdx.x] = sh[threadIdx.x] - v;
        if (p == 0 && threadIdx.x == OS_RADIX - 1 && total) *total = sh[threadIdx.x];
        __syncthreads();
    }
}

// V: payload type (u32 sample index, or a 16 B DC3 record); keys_out may be
// null when only the payloads are wanted (single-pass stable partitions).
template <typename K, class Src, int ITEMS, typename V = u32>
__global__ void __launch_bounds__(OS_THREADS, 2)
k_os_pass(Src src, i64 n, int shift, const u32 *__restrict__ offs, u32 *__restrict__ status, u32 *__restrict__ ticket,
          K *__restrict__ keys_out, V *__restrict__ vals_out) {
    constexpr int TILE = OS_THREADS * ITEMS;
    extern __shared__ __align__(16) unsigned char smem[];
    V *sv = reinterpret_cast<V *>(smem);
    K *sk = reinterpret_cast<K *>(sv + TILE);
    u32(*cnt)[OS_RADIX] = reinterpret_cast<u32(*)[OS_RADIX]>(sk + TILE);
    u32 *tile_excl = &cnt[OS_WARPS][0];
    u32 *gbase = tile_excl + OS_RADIX;
    __shared__ u32 sh_tile, sh_warp[OS_WARPS + 1];

    if (threadIdx.x == 0) sh_tile = atomicAdd(ticket, 1u);
    int w = threadIdx.x >> 5, lane = lane_id();
    for (int d = lane; d < OS_RADIX; d += 32) cnt[w][d] = 0;
    __syncthreads();
    const u32 tile = sh_tile;
    i64 seg = (i64)tile * TILE + (i64)w * (32 * ITEMS);
    K k[ITEMS];
    V v[ITEMS];
    u32 rank[ITEMS], dig[ITEMS];
    u32 lt = lanemask_lt();
    // all loads first (16 in flight per thread), then the ranking rounds
#pragma unroll
    for (int r = 0; r < ITEMS; r++) {
        i64 i = seg + r * 32 + lane;
        bool ok = i < n && src.get(i, k[r], v[r]);
        dig[r] = ok ? ((u32)(k[r] >> shift) & (OS_RADIX - 1)) : (u32)OS_RADIX;
    }
#pragma unroll
    for (int r = 0; r < ITEMS; r++) {
        u32 d = dig[r];
        bool ok = d < OS_RADIX;
        u32 peers = digit_peers(d);
        u32 before = __popc(peers & lt);
        u32 cur = ok ? cnt[w][d] : 0u;
        __syncwarp();
        if (ok && before == 0) cnt[w][d] = cur + __popc(peers);
        __syncwarp();
        rank[r] = cur + before;
    }
    __syncthreads();
    // thread d owns digit d: warp-exclusive prefixes, tile count, look-back
    {
        const int d = threadIdx.x;
        u32 run = 0;
#pragma unroll
        for (int q = 0; q < OS_WARPS; q++) {
            u32 c = cnt[q][d];
            cnt[q][d] = run;
            run += c;
        }
        u32 *my = status + (i64)tile * OS_RADIX + d;
        u32 excl = 0;
        if (tile == 0) {
            *(volatile u32 *)my = OS_FLAG_PRE | run;
        } else {
            *(volatile u32 *)my = OS_FLAG_AGG | run;
            // windowed look-back: 32 predecessors per round trip, so a chain
            // of aggregate-only tiles costs 1/32 of the serial L2 latency
            constexpr int WIN = 32;
            i64 t = (i64)tile - 1;
            while (true) {
                u32 s[WIN];
#pragma unroll
                for (int q = 0; q < WIN; q++)
                    s[q] = (t - q >= 0) ? *(volatile const u32 *)(status + (t - q) * OS_RADIX + d) : OS_FLAG_PRE;
                int q = 0;
                bool done = false;
#pragma unroll
                for (; q < WIN; q++) {
                    if ((s[q] & ~OS_MASK) == 0) break;  // not published yet: resume here
                    excl += s[q] & OS_MASK;
                    if (s[q] & OS_FLAG_PRE) {
                        done = true;
                        break;
                    }
                }
                if (done) break;
                t -= q;
            }
            *(volatile u32 *)my = OS_FLAG_PRE | (excl + run);
        }
        gbase[d] = offs[d] + excl;
        // exclusive scan of tile counts over digits (tile-local staging offsets)
        u32 inc = run;
        for (int o = 1; o < 32; o <<= 1) {
            u32 y = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += y;
        }
        if (lane == 31) sh_warp[w] = inc;
        __syncthreads();
        if (w == 0) {
            u32 x = lane < OS_WARPS ? sh_warp[lane] : 0u;
            u32 xi = x;
            for (int o = 1; o < 32; o <<= 1) {
                u32 y = __shfl_up_sync(0xffffffffu, xi, o);
                if (lane >= o) xi += y;
            }
            if (lane < OS_WARPS) sh_warp[lane] = xi - x;
            if (lane == OS_WARPS - 1) sh_warp[OS_WARPS] = xi;
        }
        __syncthreads();
        tile_excl[d] = sh_warp[w] + inc - run;
    }
    __syncthreads();
    const u32 valid = sh_warp[OS_WARPS];
#pragma unroll
    for (int r = 0; r < ITEMS; r++) {
        u32 d = dig[r];
        if (d < OS_RADIX) {
            u32 lp = tile_excl[d] + cnt[w][d] + rank[r];
            sk[lp] = k[r];
            sv[lp] = v[r];
        }
    }
    __syncthreads();
    for (u32 x = threadIdx.x; x < valid; x += OS_THREADS) {
        K kk = sk[x];
        u32 d = (u32)(kk >> shift) & (OS_RADIX - 1);
        u32 dst = gbase[d] + (x - tile_excl[d]);
        if (keys_out) keys_out[dst] = kk;
        vals_out[dst] = sv[x];
    }
}

template <typename K, int ITEMS, typename V = u32>
constexpr size_t os_pass_smem() {
    return (size_t)OS_THREADS * ITEMS * (sizeof(K) + sizeof(V)) + (size_t)(OS_WARPS + 2) * OS_RADIX * 4;
}

inline int os_items_choice() {
    static int v = [] {
        const char *e = getenv("SAIX_OS_ITEMS");
        int x = e ? atoi(e) : OS_ITEMS;
        return (x == 8 || x == 12 || x == 16) ? x : OS_ITEMS;
    }();
    return v;
}

template <typename K, class Src, int ITEMS, typename V = u32>
static int os_launch_pass(Src src, i64 np, int shift, const u32 *offs, u32 *status, u32 *ticket, K *dk, V *dv,
                          cudaStream_t st) {
    static DeviceFlags attr;
    constexpr size_t smem = os_pass_smem<K, ITEMS, V>();
    if (attr.need()) {
        SAIX_CUDA(cudaFuncSetAttribute(k_os_pass<K, Src, ITEMS, V>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem));
        attr.set();
    }
    i64 ntiles = os_tiles(np, ITEMS);
    SAIX_CUDA(cudaMemsetAsync(status, 0, (size_t)ntiles * OS_RADIX * 4, st));
    k_os_pass<K, Src, ITEMS, V><<<(unsigned)ntiles, OS_THREADS, smem, st>>>(src, np, shift, offs, status, ticket, dk,
                                                                            dv);
    SAIX_LAUNCHED();
    return SAIX_OK;
}

template <typename K, class Src>
static int os_pass_any(Src src, i64 np, int shift, const u32 *offs, u32 *status, u32 *ticket, K *dk, u32 *dv,
                       cudaStream_t st) {
    switch (os_items_choice()) {
        case 8: return os_launch_pass<K, Src, 8>(src, np, shift, offs, status, ticket, dk, dv, st);
        case 12: return os_launch_pass<K, Src, 12>(src, np, shift, offs, status, ticket, dk, dv, st);
        default: return os_launch_pass<K, Src, 16>(src, np, shift, offs, status, ticket, dk, dv, st);
    }
}

// Sort `n` source items on bits [shift0, shift0 + 8*passes).  Pass 0 reads
// `src` (which may filter); n_out is the number of valid items, which the
// caller must know on the host when passes > 1.  Later passes ping-pong
// between (k0,v0) and (k1,v1); out_k/out_v receive the result buffers.
//
// `hsrc` (n_h items) must enumerate the same multiset of valid keys as `src`
// in any order (digit counts are permutation-invariant); it lets the
// histogram stream over a cheaper source than pass 0's gather.
template <typename K, class Src, class HSrc>
int onesweep_sort(Src src, i64 n, HSrc hsrc, i64 n_h, i64 n_out, int shift0, int passes, K *k0, u32 *v0, K *k1,
                  u32 *v1, u32 *scratch, K *&out_k, u32 *&out_v, u32 *d_count, cudaStream_t st,
                  const char *prof = "onesweep") {
    if (passes < 1 || passes > OS_MAX_PASSES || n >= ((i64)1 << 30)) {
        set_error("onesweep_sort: unsupported passes=%d n=%lld", passes, (long long)n);
        return SAIX_EINVAL;
    }
    u32 *hist = scratch;
    u32 *offs = hist + OS_MAX_PASSES * OS_RADIX;
    u32 *ticket = offs + OS_MAX_PASSES * OS_RADIX;  // 32 words, one per pass
    u32 *status = ticket + 64;
    Prof prof_(prof, ((double)n + (double)n_out * (2 * passes - 1)) * (sizeof(K) + 4), st);
    if (n <= 0) return SAIX_OK;
    SAIX_CUDA(cudaMemsetAsync(hist, 0, (size_t)(OS_MAX_PASSES * OS_RADIX) * 4, st));
    SAIX_CUDA(cudaMemsetAsync(ticket, 0, 64 * 4, st));
    k_os_hist<K, HSrc><<<grid_for(n_h, OS_THREADS, kNumSMs * 8), OS_THREADS, 0, st>>>(hsrc, n_h, shift0, passes, hist);
    SAIX_LAUNCHED();
    k_os_scan<<<1, OS_RADIX, 0, st>>>(hist, passes, offs, d_count);
    SAIX_LAUNCHED();
    K *ok = k0;
    u32 *ov = v0;
    for (int p = 0; p < passes; p++) {
        i64 np = p == 0 ? n : n_out;
        K *dk = (p % 2 == 0) ? k0 : k1;
        u32 *dv = (p % 2 == 0) ? v0 : v1;
        if (p == 0) {
            SAIX_TRY((os_pass_any<K, Src>(src, n, shift0, offs, status, ticket, dk, dv, st)));
        } else {
            SAIX_TRY((os_pass_any<K, ArraySrc<K>>(ArraySrc<K>{ok, ov}, np, shift0 + OS_BITS * p, offs + OS_RADIX * p,
                                                  status, ticket + p, dk, dv, st)));
        }
        ok = dk;
        ov = dv;
    }
    out_k = ok;
    out_v = ov;
    return SAIX_OK;
}

// Single-pass stable partition of `src`'s valid items by an 8-bit key
// (bits [shift, shift+8)), payloads only: out receives the n_out valid
// payloads grouped by key, input order kept within a key.  `hsrc` enumerates
// the same key multiset (see onesweep_sort).
template <typename V, class Src, class HSrc>
int onesweep_partition(Src src, i64 n, HSrc hsrc, i64 n_h, int shift, V *out, u32 *scratch, cudaStream_t st,
                       const char *prof, double bytes) {
    if (n >= ((i64)1 << 30)) {
        set_error("onesweep_partition: n=%lld too large", (long long)n);
        return SAIX_EINVAL;
    }
    Prof prof_(prof, bytes, st);
    if (n <= 0) return SAIX_OK;
    u32 *hist = scratch;
    u32 *offs = hist + OS_MAX_PASSES * OS_RADIX;
    u32 *ticket = offs + OS_MAX_PASSES * OS_RADIX;
    u32 *status = ticket + 64;
    SAIX_CUDA(cudaMemsetAsync(hist, 0, (size_t)OS_RADIX * 4, st));
    SAIX_CUDA(cudaMemsetAsync(ticket, 0, 64 * 4, st));
    k_os_hist<u32, HSrc><<<grid_for(n_h, OS_THREADS, kNumSMs * 8), OS_THREADS, 0, st>>>(hsrc, n_h, shift, 1, hist);
    SAIX_LAUNCHED();
    k_os_scan<<<1, OS_RADIX, 0, st>>>(hist, 1, offs, nullptr);
    SAIX_LAUNCHED();
    constexpr int kItems = sizeof(V) > 4 ? 8 : 16;  // 16 B payloads: keep the tile in registers
    return os_launch_pass<u32, Src, kItems, V>(src, n, shift, offs, status, ticket, (u32 *)nullptr, out, st);
}

}  // namespace saix
