// bsort.cuh -- MSD bucket sort for wide keys (large-alphabet DC3 levels):
// the sort behind _name_triples' lexicographic triple order (reference
// suffix_index.py:221-253, via _lexsort_keys / _pack_keys, 57-82).
//
// Deep DC3 levels sort items whose keys span a large range (level-2 triples
// of DNA: 3 x 18-bit names); LSD radix needs 7 passes of 8 bits there.  Here
// the key range is cut into ~n/8 equal buckets (bucket = key >> shift, a
// monotone function of the key), so buckets hold a handful of items each:
//   count    histogram of bucket ids (global atomics, L2-resident counters)
//   scan     exclusive bucket starts; buckets of > 32 items are listed
//   scatter  item -> its bucket's next slot (atomic cursor; order inside a
//            bucket is arbitrary and fixed by the segment sort)
//   segsort  <= 32 items: one warp, register bitonic via shuffles;
//            <= 1024: one warp, bitonic in shared memory;
//            <= 4096: one CTA; larger buckets are reported so the caller can
//            fall back to a full LSD sort.
// Sources: struct { __device__ void get(i64 i, u64 &key, u32 &val) const;
//                   __device__ u64 dense(u64 key) const; }
// where dense() is a monotone map of the keys onto [0, span] that spreads
// them evenly (e.g. the mixed-radix value of the leading key fields); the
// result is sorted by key (ties in any order).
#pragma once

#include "pscatter.cuh"
#include "scan.cuh"

namespace saix {

constexpr int BS_TINY = 32;     // register bitonic limit
constexpr int BS_SMALL = 1024;  // warp-per-bucket (shared memory) limit
constexpr int BS_LARGE = 4096;  // CTA-per-bucket limit
constexpr int BS_WARPS = 8;

// key, value and dense bucket coordinate of item i; sources that can derive
// the dense value more cheaply than from the key overload this (ADL)
template <class Src>
__device__ __forceinline__ u64 bs_get(const Src &src, i64 i, u64 &k, u32 &v) {
    src.get(i, k, v);
    return src.dense(k);
}

template <class Src>
__global__ void k_bs_count(Src src, i64 n, int shift, u32 *__restrict__ cnt) {
    for (i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x) {
        u64 k;
        u32 v;
        const u64 d = bs_get(src, i, k, v);
        atomicAdd(&cnt[d >> shift], 1u);
    }
}

struct BsCntIn {
    const u32 *cnt;
    __device__ u32 operator()(i64 i) const { return cnt[i]; }
};
// bucket starts + cursor copy; buckets beyond BS_TINY are listed (medium /
// large) and the largest size is recorded
struct BsStartOut {
    u32 *start, *cursor, *mid_list, *big_list, *scal;  // scal: [0] mid count, [1] big count, [2] max size
    __device__ void operator()(i64 i, u32 excl, u32 v) const {
        start[i] = excl;
        cursor[i] = excl;
        if (v > BS_TINY) {
            if (v <= BS_SMALL) mid_list[atomicAdd(&scal[0], 1u)] = (u32)i;
            else big_list[atomicAdd(&scal[1], 1u)] = (u32)i;
            atomicMax(&scal[2], v);
        }
    }
};

template <class Src>
__global__ void k_bs_scatter(Src src, i64 n, int shift, u32 *__restrict__ cursor, u64 *__restrict__ keys,
                             u32 *__restrict__ vals) {
    for (i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x) {
        u64 k;
        u32 v;
        const u64 d = bs_get(src, i, k, v);
        u32 at = atomicAdd(&cursor[d >> shift], 1u);
        keys[at] = k;
        vals[at] = v;
    }
}

// Large inputs: the same scatter, its writes through the bucketed scatter
// (pscatter.cuh) instead of random 12 B stores -- pass A item
// {slot, val, key lo, key hi}; pass B writes keys/vals windows as full lines.
constexpr int BSE_ITEMS = 8;
template <class Src>
__global__ void __launch_bounds__(256, 4)
k_bs_scatter_emit(Src src, i64 n, int shift, u32 *__restrict__ cursor, PsPlan plan, uint4 *__restrict__ stage) {
    extern __shared__ __align__(16) unsigned char bse_smem[];
    uint4 *sh_items = reinterpret_cast<uint4 *>(bse_smem);
    u32 *sh_cnt = reinterpret_cast<u32 *>(sh_items + 256 * BSE_ITEMS);
    u32 *sh_base = sh_cnt + plan.a.buckets;
    const i64 i0 = (i64)blockIdx.x * (256 * BSE_ITEMS);
    uint4 it[BSE_ITEMS];
    bool ok[BSE_ITEMS];
#pragma unroll
    for (int q = 0; q < BSE_ITEMS; q++) {
        i64 i = i0 + q * 256 + threadIdx.x;
        ok[q] = i < n;
        if (ok[q]) {
            u64 k;
            u32 v;
            const u64 d = bs_get(src, i, k, v);
            u32 at = atomicAdd(&cursor[d >> shift], 1u);
            it[q] = make_uint4(at, v, (u32)k, (u32)(k >> 32));
        }
    }
    ps_block_emit<uint4, 256, BSE_ITEMS>(it, ok, plan.a, stage, sh_items, sh_cnt, sh_base);
}

__global__ void __launch_bounds__(PS_THREADS)
k_bs_window(const uint4 *__restrict__ stage2, PsPlan plan, u64 *__restrict__ keys, u32 *__restrict__ vals) {
    extern __shared__ __align__(16) unsigned char ps_smem[];
    uint4 *win = reinterpret_cast<uint4 *>(ps_smem);
    const i64 w = blockIdx.x;
    const i64 d0 = w << plan.s2;
    const i64 len = (d0 + ((i64)1 << plan.s2) < plan.n_dest ? d0 + ((i64)1 << plan.s2) : plan.n_dest) - d0;
    const i64 cnt = plan.cursor2[w];
    const uint4 *src = stage2 + d0;
    if (cnt == len) {
        for (i64 x = threadIdx.x; x < cnt; x += PS_THREADS) {
            uint4 v = ld_stream(src + x);
            win[(i64)v.x - d0] = v;
        }
        __syncthreads();
        for (i64 x = threadIdx.x; x < len; x += PS_THREADS) {
            uint4 v = win[x];
            keys[d0 + x] = ((u64)v.w << 32) | v.z;
            vals[d0 + x] = v.y;
        }
    } else {
        for (i64 x = threadIdx.x; x < cnt; x += PS_THREADS) {
            uint4 v = ld_stream(src + x);
            keys[v.x] = ((u64)v.w << 32) | v.z;
            vals[v.x] = v.y;
        }
    }
}
// bytes of arena space bucket_sort takes for the bucketed scatter
inline size_t bs_ps_bytes(i64 n) {
    if (n < kDirectScatterItems) return 0;
    PsPlan p = PsPlan::of(n, 16);
    return (size_t)(p.stage1_items() + p.stage2_items()) * 16 + (size_t)p.cursor_words() * 4 + 4 * Arena::kAlign;
}

// ascending bitonic sort of one (key, val) per lane inside aligned segments
// of W lanes (W = 8, 16, 32)
template <int W>
__device__ __forceinline__ void seg_bitonic(u64 &k, u32 &v) {
    const int lane = lane_id();
#pragma unroll
    for (int size = 2; size <= W; size <<= 1) {
#pragma unroll
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            u64 ok = __shfl_xor_sync(0xffffffffu, k, stride);
            u32 ov = __shfl_xor_sync(0xffffffffu, v, stride);
            bool up = (lane & size) == 0 || size == W;
            bool lower = (lane & stride) == 0;
            bool take = (lower == up) ? (ok < k) : (ok > k);
            if (take) {
                k = ok;
                v = ov;
            }
        }
    }
}

// sort the buckets flagged in `todo` (lane q of the warp holds bucket q's
// length / start), 32/W buckets per round, one W-lane segment each
template <int W>
__device__ __forceinline__ void tiny_round(u32 todo, u32 my_len, u32 my_s0, u64 *__restrict__ keys,
                                           u32 *__restrict__ vals) {
    const int lane = lane_id();
    const int g = lane / W, sl = lane & (W - 1);
    while (todo) {
        // the g-th set bit of todo belongs to segment g
        u32 t = todo;
        int q = -1;
        for (int x = 0; x < 32 / W; x++) {
            int f = t ? __ffs(t) - 1 : -1;
            if (x == g) q = f;
            if (t) t &= t - 1;
        }
        todo = t;
        u32 len = __shfl_sync(0xffffffffu, my_len, q < 0 ? 0 : q);
        u32 s0 = __shfl_sync(0xffffffffu, my_s0, q < 0 ? 0 : q);
        if (q < 0) len = 0;
        u64 k = ~0ull;
        u32 v = 0xFFFFFFFFu;
        if ((u32)sl < len) {
            k = keys[s0 + sl];
            v = vals[s0 + sl];
        }
        seg_bitonic<W>(k, v);
        if ((u32)sl < len) {
            keys[s0 + sl] = k;
            vals[s0 + sl] = v;
        }
    }
}

// buckets of <= 32 items: a warp takes 32 consecutive buckets (coalesced
// count/start reads) and sorts them in register segments of 8/16/32 lanes
__global__ void __launch_bounds__(256)
k_bs_tiny(const u32 *__restrict__ start, const u32 *__restrict__ cnt, i64 nb, u64 *__restrict__ keys,
          u32 *__restrict__ vals) {
    const int lane = lane_id();
    const i64 warps = ((i64)gridDim.x * blockDim.x) >> 5;
    for (i64 b0 = (((i64)blockIdx.x * blockDim.x + threadIdx.x) >> 5) * 32; b0 < nb; b0 += warps * 32) {
        u32 my_len = b0 + lane < nb ? cnt[b0 + lane] : 0u;
        u32 my_s0 = b0 + lane < nb ? start[b0 + lane] : 0u;
        tiny_round<8>(__ballot_sync(0xffffffffu, my_len > 1 && my_len <= 8), my_len, my_s0, keys, vals);
        tiny_round<16>(__ballot_sync(0xffffffffu, my_len > 8 && my_len <= 16), my_len, my_s0, keys, vals);
        tiny_round<32>(__ballot_sync(0xffffffffu, my_len > 16 && my_len <= BS_TINY), my_len, my_s0, keys, vals);
    }
}

// bitonic sort of `len` (key, val) pairs in shared memory, padded to the
// next power of two with +inf keys, by `nthr` cooperating threads (tid)
__device__ __forceinline__ void bitonic_smem(u64 *sk, u32 *sv, int len, int tid, int nthr, bool warp_only) {
    int p2 = 1;
    while (p2 < len) p2 <<= 1;
    for (int x = len + tid; x < p2; x += nthr) {
        sk[x] = ~0ull;
        sv[x] = 0xFFFFFFFFu;
    }
    if (warp_only) __syncwarp();
    else __syncthreads();
    for (int size = 2; size <= p2; size <<= 1) {
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            for (int t = tid; t < (p2 >> 1); t += nthr) {
                int lo = 2 * t - (t & (stride - 1));
                int hi = lo + stride;
                bool up = (lo & size) == 0;
                u64 a = sk[lo], b = sk[hi];
                if ((a > b) == up) {
                    sk[lo] = b;
                    sk[hi] = a;
                    u32 tv = sv[lo];
                    sv[lo] = sv[hi];
                    sv[hi] = tv;
                }
            }
            if (warp_only) __syncwarp();
            else __syncthreads();
        }
    }
}

// one warp per listed bucket of BS_TINY < size <= BS_SMALL items
__global__ void __launch_bounds__(32 * BS_WARPS)
k_bs_small(const u32 *__restrict__ start, const u32 *__restrict__ cnt, const u32 *__restrict__ list,
           const u32 *__restrict__ list_len, u64 *__restrict__ keys, u32 *__restrict__ vals) {
    extern __shared__ __align__(16) unsigned char bs_small_smem[];
    int w = threadIdx.x >> 5, lane = lane_id();
    u64 *sk = reinterpret_cast<u64 *>(bs_small_smem) + (size_t)w * BS_SMALL;
    u32 *sv = reinterpret_cast<u32 *>(reinterpret_cast<u64 *>(bs_small_smem) + (size_t)BS_WARPS * BS_SMALL) +
              (size_t)w * BS_SMALL;
    const u32 nl = *list_len;
    for (u32 q = blockIdx.x * BS_WARPS + w; q < nl; q += gridDim.x * BS_WARPS) {
        u32 b = list[q];
        u32 len = cnt[b], s0 = start[b];
        for (u32 x = lane; x < len; x += 32) {
            sk[x] = keys[s0 + x];
            sv[x] = vals[s0 + x];
        }
        __syncwarp();
        bitonic_smem(sk, sv, (int)len, lane, 32, true);
        for (u32 x = lane; x < len; x += 32) {
            keys[s0 + x] = sk[x];
            vals[s0 + x] = sv[x];
        }
        __syncwarp();
    }
}
constexpr size_t BS_SMALL_SMEM = (size_t)BS_WARPS * BS_SMALL * 12;

// one CTA per listed bucket of BS_SMALL < size <= BS_LARGE items
__global__ void __launch_bounds__(256)
k_bs_large(const u32 *__restrict__ start, const u32 *__restrict__ cnt, const u32 *__restrict__ list,
           const u32 *__restrict__ list_len, u64 *__restrict__ keys, u32 *__restrict__ vals) {
    extern __shared__ __align__(16) unsigned char bs_smem[];
    u64 *sk = reinterpret_cast<u64 *>(bs_smem);
    u32 *sv = reinterpret_cast<u32 *>(sk + BS_LARGE);
    u32 nl = *list_len;
    for (u32 q = blockIdx.x; q < nl; q += gridDim.x) {
        u32 b = list[q];
        u32 len = cnt[b], s0 = start[b];
        if (len > BS_LARGE) continue;  // caller falls back to a full sort
        for (u32 x = threadIdx.x; x < len; x += blockDim.x) {
            sk[x] = keys[s0 + x];
            sv[x] = vals[s0 + x];
        }
        __syncthreads();
        bitonic_smem(sk, sv, (int)len, threadIdx.x, blockDim.x, false);
        for (u32 x = threadIdx.x; x < len; x += blockDim.x) {
            keys[s0 + x] = sk[x];
            vals[s0 + x] = sv[x];
        }
        __syncthreads();
    }
}

// Bucket geometry: ~n/8 buckets (at most 2^23) over [0, max_key].
struct BsGeom {
    int shift;
    i64 nb;
};
inline BsGeom bs_geom(u64 max_key, i64 n, int per_bucket = 8, int max_bits = 23) {
    i64 want = n / per_bucket > 1 ? n / per_bucket : 1;
    if (want > ((i64)1 << max_bits)) want = (i64)1 << max_bits;
    int shift = 0;
    while ((i64)(max_key >> shift) + 1 > want) shift++;
    return BsGeom{shift, (i64)(max_key >> shift) + 1};
}

// scratch words: cnt, start, cursor, mid list, big list (nb + 1 each), scalars, scan tmp
inline i64 bs_scratch_words(i64 nb) { return 5 * (nb + 1) + 8 + scan_tmp_words(nb) + 64; }
inline i64 bs_scratch_words_for(u64 max_key, i64 n) { return bs_scratch_words(bs_geom(max_key, n).nb); }

// Returns ok = false (after the count pass only) when some bucket exceeds
// BS_LARGE; the caller then sorts with onesweep instead.  One host sync.
template <class Src>
int bucket_sort(Src src, i64 n, u64 span, u64 *keys, u32 *vals, u32 *scratch, bool &ok, cudaStream_t st,
                const char *prof = "bsort", Arena *ar = nullptr, int per_bucket = 8, int max_bits = 23) {
    ok = true;
    if (n <= 0) return SAIX_OK;
    BsGeom g = bs_geom(span, n, per_bucket, max_bits);
    const i64 nb = g.nb;
    Prof prof_(prof, 24.0 * n + 16.0 * nb, st);
    u32 *cnt = scratch, *start = cnt + (nb + 1), *cursor = start + (nb + 1), *mid = cursor + (nb + 1);
    u32 *big = mid + (nb + 1);
    u32 *scal = big + (nb + 1);  // [0] mid count, [1] big count, [2] max size
    u32 *tmp = scal + 8;
    SAIX_CUDA(cudaMemsetAsync(cnt, 0, (size_t)(nb + 1) * 4, st));
    SAIX_CUDA(cudaMemsetAsync(scal, 0, 8 * 4, st));
    int gr = grid_for(n, 256);
    k_bs_count<Src><<<gr, 256, 0, st>>>(src, n, g.shift, cnt);
    SAIX_LAUNCHED();
    SAIX_TRY(scan_transform(BsCntIn{cnt}, BsStartOut{start, cursor, mid, big, scal}, nb, tmp, nullptr, st,
                            "bsort.scan", 16.0 * nb));
    u32 h[3];
    SAIX_CUDA(cudaMemcpyAsync(h, scal, 12, cudaMemcpyDeviceToHost, st));
    SAIX_CUDA(cudaStreamSynchronize(st));
    if (h[2] > (u32)BS_LARGE) {
        ok = false;
        return SAIX_OK;
    }
    if (ar && bs_ps_bytes(n)) {
        size_t mark = ar->mark();
        PsPlan pp = PsPlan::of(n, 16);
        pp.set_cursors(ar->alloc<u32>(pp.cursor_words()));
        uint4 *s1 = ar->alloc<uint4>(pp.stage1_items()), *s2 = ar->alloc<uint4>(pp.stage2_items());
        SAIX_ARENA_OK(*ar);
        SAIX_CUDA(cudaMemsetAsync(pp.a.cursor, 0, (size_t)pp.cursor_words() * 4, st));
        static DeviceFlags attr;
        if (attr.need()) {
            SAIX_CUDA(cudaFuncSetAttribute(k_bs_scatter_emit<Src>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           256 * BSE_ITEMS * 16 + 8 * PS_MAX_BUCKETS));
            SAIX_CUDA(cudaFuncSetAttribute(k_ps_refine<uint4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)(PS_REFINE_TILE * 16 + 8 * 256)));
            SAIX_CUDA(cudaFuncSetAttribute(k_bs_window, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)PS_WINDOW_BYTES));
            attr.set();
        }
        size_t smem = (size_t)256 * BSE_ITEMS * 16 + 8 * (size_t)pp.a.buckets;
        k_bs_scatter_emit<Src><<<(unsigned)ceil_div(n, 256 * BSE_ITEMS), 256, smem, st>>>(src, n, g.shift, cursor, pp,
                                                                                          s1);
        SAIX_LAUNCHED();
        SAIX_TRY(ps_refine_launch(s1, pp, s2, st));
        k_bs_window<<<(unsigned)pp.windows, PS_THREADS, (size_t)16 << pp.s2, st>>>(s2, pp, keys, vals);
        SAIX_LAUNCHED();
        ar->reset(mark);
    } else {
        k_bs_scatter<Src><<<gr, 256, 0, st>>>(src, n, g.shift, cursor, keys, vals);
        SAIX_LAUNCHED();
    }
    k_bs_tiny<<<grid_for(ceil_div(nb, 32) * 32, 256, kNumSMs * 16), 256, 0, st>>>(start, cnt, nb, keys, vals);
    SAIX_LAUNCHED();
    if (h[0]) {
        static DeviceFlags attr;
        if (attr.need()) {
            SAIX_CUDA(cudaFuncSetAttribute(k_bs_small, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)BS_SMALL_SMEM));
            attr.set();
        }
        u32 blocks = (h[0] + BS_WARPS - 1) / BS_WARPS;
        k_bs_small<<<blocks < 2 * kNumSMs ? blocks : 2 * kNumSMs, 32 * BS_WARPS, BS_SMALL_SMEM, st>>>(start, cnt, mid,
                                                                                                   scal, keys, vals);
        SAIX_LAUNCHED();
    }
    if (h[1]) {
        static DeviceFlags attr;
        size_t smem = (size_t)BS_LARGE * 12;
        if (attr.need()) {
            SAIX_CUDA(cudaFuncSetAttribute(k_bs_large, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            attr.set();
        }
        k_bs_large<<<h[1] < 4 * kNumSMs ? h[1] : 4 * kNumSMs, 256, smem, st>>>(start, cnt, big, scal + 1, keys, vals);
        SAIX_LAUNCHED();
    }
    return SAIX_OK;
}

}  // namespace saix
