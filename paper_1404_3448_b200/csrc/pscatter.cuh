// pscatter.cuh -- bucketed scatter for permutation-like writes.
//
// A random 4-16 B scatter into an array larger than the ~64 MB that B200's L2
// holds for random targets runs at ~25-60 G/s, and B200's L2 does not merge
// scattered partial-line writes even inside a small window: a 4 B scatter
// confined to 256 KB windows still moves ~4x its bytes through DRAM
// (tools/wprobe.cu, profiles/r1_window_scatter_probe.txt).  Every DC3 level
// has such permutations (ISA = SuffixArray.from_order, reference
// suffix_index.py:96-101; the rank_of tables of _sort_samples / _merge,
// 256-271 / 362-378; Kasai's Phi, 461-476), so they are done as three
// streaming passes whose global writes are all contiguous runs:
//
//   pass A  (inside the producing kernel, ps_block_emit): a CTA's items are
//           bucketed in shared memory by dest >> s1 and each bucket's run is
//           written contiguously into that coarse bucket's staging region
//           (one global atomic per (tile, bucket) reserves the run);
//   pass A2 (k_ps_refine): each coarse region is re-bucketed the same way by
//           dest >> s2 into shared-memory-sized windows;
//   pass B  (k_ps_window): one CTA per window scatters its items into shared
//           memory and writes the window out as full lines.
//
// Bucket b's region starts at b << shift and holds at most 2^shift items:
// destinations are distinct (a permutation or an injective map into
// [0, n_dest)), so no count pass is needed.  A window that did not receive
// all of its 2^s2 destinations (injective, non-surjective maps) is written
// item by item instead, so untouched destinations keep their contents.
#pragma once

#include "common.cuh"

namespace saix {

constexpr int PS_MAX_BUCKETS = 4096;
constexpr int PS_THREADS = 256;
constexpr int PS_REFINE_THREADS = 512;
constexpr int PS_REFINE_ITEMS = 8;                             // pass A2 tile: 4096 items
constexpr int PS_REFINE_TILE = PS_REFINE_THREADS * PS_REFINE_ITEMS;
constexpr i64 PS_WINDOW_BYTES = 64 << 10;                      // pass B window in shared memory

// staging traffic streams past L2 (evict-first)
__device__ __forceinline__ uint4 ld_stream(const uint4 *p) { return __ldcs(p); }
__device__ __forceinline__ uint2 ld_stream(const uint2 *p) { return __ldcs(p); }
__device__ __forceinline__ void st_stream(uint4 *p, const uint4 &v) { __stcs(p, v); }
__device__ __forceinline__ void st_stream(uint2 *p, const uint2 &v) { __stcs(p, v); }
__device__ __forceinline__ void st_stream(u32 *p, const u32 &v) { __stcs(p, v); }

// One level of bucketing: bucket = (dest >> shift) - base, region of bucket
// q at stage + (q << shift), items written so far in cursor[q].
struct PsLevel {
    int shift = 0;
    i64 buckets = 0;
    u32 base = 0;
    u32 *cursor = nullptr;
};

struct PsPlan {
    i64 n_dest = 0;  // destinations are in [0, n_dest)
    PsLevel a;       // coarse (pass A)
    int s2 = 0;      // window shift (pass A2 / B)
    i64 windows = 0;
    u32 *cursor2 = nullptr;

    // payload of `out_bytes` per destination; coarse regions of <= 256
    // windows, at most PS_MAX_BUCKETS of them
    static PsPlan of(i64 n_dest, int out_bytes, i64 window_bytes = PS_WINDOW_BYTES) {
        PsPlan p;
        p.n_dest = n_dest > 0 ? n_dest : 1;
        int s2 = 6;
        while (((i64)out_bytes << (s2 + 1)) <= window_bytes && ((i64)1 << s2) < p.n_dest) s2++;
        int s1 = s2;
        while (s1 < s2 + 8 && ((i64)1 << s1) < p.n_dest) s1++;
        while (ceil_div(p.n_dest, (i64)1 << s1) > PS_MAX_BUCKETS) s1++;
        p.s2 = s2;
        p.a.shift = s1;
        p.a.buckets = ceil_div(p.n_dest, (i64)1 << s1);
        p.windows = ceil_div(p.n_dest, (i64)1 << s2);
        return p;
    }
    i64 stage1_items() const { return a.buckets << a.shift; }
    i64 stage2_items() const { return windows << s2; }
    i64 cursor_words() const { return a.buckets + windows; }
    void set_cursors(u32 *c) {
        a.cursor = c;
        cursor2 = c + a.buckets;
    }
};

// Pass A/A2, block level.  Every thread offers ITEMS items (dest in .x, ok
// flags); the block stages them by bucket in shared memory and writes each
// bucket's run contiguously.  smem: THREADS*ITEMS items (sh_items) + 2 *
// buckets u32 (sh_cnt, sh_base).  All threads of the block must call it.
template <class P, int THREADS, int ITEMS, int MAXB = PS_MAX_BUCKETS>
__device__ __forceinline__ void ps_block_emit(const P (&it)[ITEMS], const bool (&ok)[ITEMS], const PsLevel &lv,
                                              P *__restrict__ stage, P *__restrict__ sh_items, u32 *__restrict__ sh_cnt,
                                              u32 *__restrict__ sh_base) {
    const int nb = (int)lv.buckets;
    for (int b = threadIdx.x; b < nb; b += THREADS) sh_cnt[b] = 0;
    __syncthreads();
    u32 slot[ITEMS];
#pragma unroll
    for (int r = 0; r < ITEMS; r++)
        if (ok[r]) slot[r] = atomicAdd(&sh_cnt[(u32)(it[r].x >> lv.shift) - lv.base], 1u);
    __syncthreads();
    // bucket starts: exclusive scan over buckets in chunks of THREADS (one
    // bucket per thread), and one independent global atomic per non-empty
    // (tile, bucket) to reserve the run inside the bucket's region.  The
    // reservations stay in registers until after the staging loop, so their
    // L2 round trip overlaps it.
    constexpr int MAXC = (MAXB + THREADS - 1) / THREADS;
    u32 res[MAXC];
    __shared__ u32 sh_warp[THREADS / 32 + 1];
    __shared__ u32 sh_total;
    u32 carry = 0;
#pragma unroll
    for (int k = 0; k < MAXC; k++) {
        const int c0 = k * THREADS;
        if (c0 >= nb) break;  // block-uniform
        int b = c0 + threadIdx.x;
        u32 c = b < nb ? sh_cnt[b] : 0u;
        u32 inc = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            u32 y = __shfl_up_sync(0xffffffffu, inc, o);
            if ((threadIdx.x & 31) >= o) inc += y;
        }
        if ((threadIdx.x & 31) == 31) sh_warp[threadIdx.x >> 5] = inc;
        __syncthreads();
        if (threadIdx.x < 32) {
            u32 x = threadIdx.x < THREADS / 32 ? sh_warp[threadIdx.x] : 0u, xi = x;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                u32 y = __shfl_up_sync(0xffffffffu, xi, o);
                if ((int)threadIdx.x >= o) xi += y;
            }
            if (threadIdx.x < THREADS / 32) sh_warp[threadIdx.x] = xi - x;
            if (threadIdx.x == THREADS / 32 - 1) sh_warp[THREADS / 32] = xi;
        }
        __syncthreads();
        res[k] = (b < nb && c) ? atomicAdd(&lv.cursor[b], c) : 0u;  // run base inside the region
        if (b < nb) sh_cnt[b] = carry + sh_warp[threadIdx.x >> 5] + inc - c;  // local start of the bucket
        carry += sh_warp[THREADS / 32];
        __syncthreads();
    }
    if (threadIdx.x == 0) sh_total = carry;
#pragma unroll
    for (int r = 0; r < ITEMS; r++)
        if (ok[r]) sh_items[sh_cnt[(u32)(it[r].x >> lv.shift) - lv.base] + slot[r]] = it[r];
#pragma unroll
    for (int k = 0; k < MAXC; k++) {
        const int b = k * THREADS + threadIdx.x;
        if (k * THREADS >= nb) break;
        if (b < nb) sh_base[b] = res[k];
    }
    __syncthreads();
    const u32 tot = sh_total;
    for (u32 x = threadIdx.x; x < tot; x += THREADS) {
        P v = sh_items[x];
        u32 q = (u32)(v.x >> lv.shift) - lv.base;
        st_stream(stage + ((i64)q << lv.shift) + sh_base[q] + (x - sh_cnt[q]), v);
    }
    __syncthreads();
}

// Pass A2: tile t covers stage1[t*TILE, (t+1)*TILE) inside one coarse region.
template <class P>
__global__ void __launch_bounds__(PS_REFINE_THREADS, sizeof(P) <= 8 ? 3 : 2)
k_ps_refine(const P *__restrict__ stage1, PsPlan plan, P *__restrict__ stage2) {
    extern __shared__ __align__(16) unsigned char ps_smem[];
    P *sh_items = reinterpret_cast<P *>(ps_smem);
    u32 *sh_cnt = reinterpret_cast<u32 *>(sh_items + PS_REFINE_TILE);
    u32 *sh_base = sh_cnt + ((i64)1 << (plan.a.shift - plan.s2));
    const i64 i0 = (i64)blockIdx.x * PS_REFINE_TILE;
    const i64 b = i0 >> plan.a.shift;
    const i64 fill = plan.a.cursor[b];
    const i64 off = i0 - (b << plan.a.shift);
    if (off >= fill) return;  // whole tile beyond the region's items (block-uniform)
    PsLevel lv;
    lv.shift = plan.s2;
    lv.base = (u32)(b << (plan.a.shift - plan.s2));
    lv.buckets = ((i64)1 << (plan.a.shift - plan.s2));
    if ((i64)lv.base + lv.buckets > plan.windows) lv.buckets = plan.windows - lv.base;
    lv.cursor = plan.cursor2 + lv.base;
    P it[PS_REFINE_ITEMS];
    bool ok[PS_REFINE_ITEMS];
#pragma unroll
    for (int r = 0; r < PS_REFINE_ITEMS; r++) {
        i64 x = off + r * PS_REFINE_THREADS + threadIdx.x;
        ok[r] = x < fill;
        if (ok[r]) it[r] = ld_stream(stage1 + (b << plan.a.shift) + x);
    }
    ps_block_emit<P, PS_REFINE_THREADS, PS_REFINE_ITEMS, 256>(it, ok, lv, stage2 + ((i64)lv.base << plan.s2), sh_items,
                                                        sh_cnt, sh_base);
}

template <class P>
int ps_refine_launch(const P *stage1, const PsPlan &plan, P *stage2, cudaStream_t st) {
    static DeviceFlags attr;
    if (attr.need()) {
        SAIX_CUDA(cudaFuncSetAttribute(k_ps_refine<P>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)(PS_REFINE_TILE * sizeof(P) + 8 * 256)));
        attr.set();
    }
    size_t smem = (size_t)PS_REFINE_TILE * sizeof(P) + 8 * ((size_t)1 << (plan.a.shift - plan.s2));
    i64 tiles = ceil_div(plan.stage1_items(), PS_REFINE_TILE);
    k_ps_refine<P><<<(unsigned)tiles, PS_REFINE_THREADS, smem, st>>>(stage1, plan, stage2);
    SAIX_LAUNCHED();
    return SAIX_OK;
}

// Pass B: one CTA per window.  Apply provides `using Out = ...;`, the
// destination array `out` and  __device__ Out value(const P &) const.
template <class P, class Apply>
__global__ void __launch_bounds__(PS_THREADS)
k_ps_window(const P *__restrict__ stage2, PsPlan plan, Apply ap) {
    using Out = typename Apply::Out;
    extern __shared__ __align__(16) unsigned char ps_smem[];
    Out *win = reinterpret_cast<Out *>(ps_smem);
    const i64 w = blockIdx.x;
    const i64 d0 = w << plan.s2;
    const i64 len = (d0 + ((i64)1 << plan.s2) < plan.n_dest ? d0 + ((i64)1 << plan.s2) : plan.n_dest) - d0;
    const i64 cnt = plan.cursor2[w];
    const P *src = stage2 + d0;
    if (cnt == len) {
        for (i64 x = threadIdx.x; x < cnt; x += PS_THREADS) {
            P v = ld_stream(src + x);
            win[(i64)v.x - d0] = ap.value(v);
        }
        __syncthreads();
        for (i64 x = threadIdx.x; x < len; x += PS_THREADS) st_stream(ap.out + d0 + x, win[x]);
    } else {
        for (i64 x = threadIdx.x; x < cnt; x += PS_THREADS) {
            P v = ld_stream(src + x);
            ap.out[v.x] = ap.value(v);
        }
    }
}

// Pass A is the caller's kernel (ps_block_emit over plan.a into stage1, with
// the cursors zeroed beforehand); ps_finish runs A2 and B.
template <class P, class Apply>
int ps_finish(const P *stage1, P *stage2, const PsPlan &plan, Apply ap, cudaStream_t st, const char *prof,
              double bytes) {
    using Out = typename Apply::Out;
    Prof prof_(prof, bytes, st);
    SAIX_TRY(ps_refine_launch(stage1, plan, stage2, st));
    {
        static DeviceFlags attr;
        if (attr.need()) {
            SAIX_CUDA(cudaFuncSetAttribute(k_ps_window<P, Apply>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)PS_WINDOW_BYTES));
            attr.set();
        }
        size_t smem = (size_t)sizeof(Out) << plan.s2;
        k_ps_window<P, Apply><<<(unsigned)plan.windows, PS_THREADS, smem, st>>>(stage2, plan, ap);
        SAIX_LAUNCHED();
    }
    return SAIX_OK;
}

// ------------------------------------------------ generic u32 scatter

struct U32Apply {
    using Out = u32;
    u32 *out;
    __device__ __forceinline__ u32 value(const uint2 &p) const { return p.y; }
};

// generic pass A of a u32 scatter dst[idx[i]] = val[i] (val == nullptr: i)
constexpr int PE_ITEMS = 8;
template <int ITEMS = PE_ITEMS>
__global__ void __launch_bounds__(256)
k_pairs_emit(const u32 *__restrict__ idx, const u32 *__restrict__ val, i64 n, PsPlan plan, uint2 *__restrict__ stage) {
    extern __shared__ __align__(16) unsigned char pe_smem[];
    uint2 *sh_items = reinterpret_cast<uint2 *>(pe_smem);
    u32 *sh_cnt = reinterpret_cast<u32 *>(sh_items + 256 * PE_ITEMS);
    u32 *sh_base = sh_cnt + plan.a.buckets;
    const i64 i0 = (i64)blockIdx.x * (256 * PE_ITEMS);
    uint2 it[ITEMS];
    bool ok[ITEMS];
#pragma unroll
    for (int q = 0; q < PE_ITEMS; q++) {
        i64 i = i0 + q * 256 + threadIdx.x;
        ok[q] = i < n;
        if (ok[q]) it[q] = make_uint2(__ldcs(idx + i), val ? __ldcs(val + i) : (u32)i);
    }
    ps_block_emit<uint2, 256, PE_ITEMS>(it, ok, plan.a, stage, sh_items, sh_cnt, sh_base);
}

// dst[idx[i]] = val[i] for a permutation-like idx, through the bucketed
// scatter (small n: direct)
template <int UNUSED = 0>
__global__ void k_scatter_direct(const u32 *__restrict__ idx, const u32 *__restrict__ val, i64 n, u32 *__restrict__ dst) {
    for (i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x)
        dst[idx[i]] = val ? val[i] : (u32)i;
}
static inline int scatter_u32(Arena &ar, const u32 *idx, const u32 *val, i64 n, i64 n_dest, u32 *dst, cudaStream_t st,
                       const char *prof) {
    if (n <= 0) return SAIX_OK;
    if (n < kDirectScatterItems) {
        Prof prof_(prof, 12.0 * n, st);
        k_scatter_direct<><<<grid_for(n, 256), 256, 0, st>>>(idx, val, n, dst);
        SAIX_LAUNCHED();
        return SAIX_OK;
    }
    size_t mark = ar.mark();
    PsPlan pp = PsPlan::of(n_dest, 4);
    pp.set_cursors(ar.alloc<u32>(pp.cursor_words()));
    uint2 *s1 = ar.alloc<uint2>(pp.stage1_items()), *s2 = ar.alloc<uint2>(pp.stage2_items());
    SAIX_ARENA_OK(ar);
    SAIX_CUDA(cudaMemsetAsync(pp.a.cursor, 0, (size_t)pp.cursor_words() * 4, st));
    {
        Prof prof_(prof, 16.0 * n, st);
        static DeviceFlags attr;
        if (attr.need()) {
            SAIX_CUDA(cudaFuncSetAttribute(k_pairs_emit<>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           256 * PE_ITEMS * 8 + 8 * PS_MAX_BUCKETS));
            attr.set();
        }
        size_t smem = (size_t)256 * PE_ITEMS * 8 + 8 * (size_t)pp.a.buckets;
        k_pairs_emit<><<<(unsigned)ceil_div(n, 256 * PE_ITEMS), 256, smem, st>>>(idx, val, n, pp, s1);
    }
    SAIX_LAUNCHED();
    SAIX_TRY(ps_finish(s1, s2, pp, U32Apply{dst}, st, prof, 28.0 * n));
    ar.reset(mark);
    return SAIX_OK;
}
inline size_t scatter_u32_bytes(i64 n_dest) {
    PsPlan pp = PsPlan::of(n_dest, 4);
    return (size_t)(pp.stage1_items() + pp.stage2_items()) * 8 + (size_t)pp.cursor_words() * 4 + 4 * Arena::kAlign;
}

}  // namespace saix
