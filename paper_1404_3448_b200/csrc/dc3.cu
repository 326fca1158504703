// dc3.cu -- DC3 / skew suffix array construction on sm_100a.
//
// Restates the reference recursion (suffix_index.py:381-392 `_dc3`) level by
// level as HBM-streaming kernels; the recursion driver stays on the host and
// reads back one u32 (`distinct`) per level.
//
// Level layout (text T of length N, ranks 0..sigma, virtual zero padding):
//   sample index s in [0, m): s < m1 -> position 3s+1 (mod-1 block),
//                             else  -> position 3(s-m1)+2 (mod-2 block)
//   tt[s]    triple name of sample s  (the recursion string, `triple_text`)
//   SAc, ISAc  suffix array / inverse of tt (sample indices, 0-based ranks);
//            the reference's 1-based `rank_of[pos(s)]` is ISAc[s] + 1.
// Steps per level (reference lines):
//   1 naming  (_name_triples 221-253): dense names of sample triples, either
//             by a presence bitmap over the (sigma+1)^3 code space when that
//             is small (levels 0-1 on DNA: no sort at all) or by an onesweep
//             LSD radix sort of packed triple keys + adjacent-difference scan.
//   2 recurse (_sort_samples 256-271) iff distinct < m.
//   3 mod-0   (_sort_nonsamples 274-290): mod-1 samples in rank order, one
//             position left, stably split by first character.
//   4 merge   (_merge_walk 173-218): merge-path partition with the DC3
//             comparator, ISA scattered in the same kernel.
#include <vector>

#include "bsort.cuh"
#include "onesweep.cuh"
#include "pscatter.cuh"
#include "scan.cuh"
#include "wsort.cuh"

namespace saix {

template <typename TT>
struct Text {
    const TT *t;
    i64 n;
    __device__ __forceinline__ u32 operator()(i64 p) const { return p < n ? (u32)t[p] : 0u; }
    __host__ __device__ static constexpr int bytes() { return (int)sizeof(TT); }
};

// ------------------------------------------------------------ naming
// Triple naming of the samples: _name_triples (suffix_index.py:221-253), the
// sample positions of _sample_positions (149-155) over _padded (143-147).
// A tile of a byte text staged in shared memory with aligned 4-byte loads
// (coalesced; the per-character loads of the triple kernels hit shared
// memory instead of issuing one global byte load each).  Covers absolute
// positions [b0, b0 + len); positions >= n read as the virtual zero padding.
struct SmemText {
    const u8 *sh;  // sh[p - a0]
    i64 a0;
    __device__ __forceinline__ u32 operator()(i64 p) const { return sh[p - a0]; }
};
__device__ __forceinline__ SmemText stage_text(const u8 *__restrict__ T, i64 n, i64 b0, int len, u32 *sh_words,
                                               int nthreads) {
    i64 a0 = b0 & ~(i64)3;
    int nw = (int)((b0 - a0 + len + 3) >> 2);
    const u32 *W = reinterpret_cast<const u32 *>(T);
    for (int w = threadIdx.x; w < nw; w += nthreads) {
        i64 q = a0 + 4 * (i64)w;
        u32 x = 0;
        if (q + 4 <= n) x = __ldg(W + (q >> 2));
        else
            for (int c = 0; c < 4; c++)
                if (q + c < n) x |= (u32)T[q + c] << (8 * c);
        sh_words[w] = x;
    }
    __syncthreads();
    return SmemText{reinterpret_cast<const u8 *>(sh_words), a0};
}
constexpr int TT_TILE = 2048;  // triplets per CTA in the staged byte-text kernels
constexpr int TT_WORDS = (3 * TT_TILE + 8) / 4 + 2;


template <typename TT>
__global__ void k_bitmap_set(Text<TT> T, SampleLayout L, u64 s1, u32 *__restrict__ bm,
                             u32 nwords, int use_smem) {
    extern __shared__ u32 shb[];
    if (use_smem) {
        for (u32 w = threadIdx.x; w < nwords; w += blockDim.x) shb[w] = 0;
        __syncthreads();
    }
    for (i64 s = (i64)blockIdx.x * blockDim.x + threadIdx.x; s < L.m; s += (i64)gridDim.x * blockDim.x) {
        i64 p = L.pos(s);
        u64 code = ((u64)T(p) * s1 + T(p + 1)) * s1 + T(p + 2);
        u32 w = (u32)(code >> 5), bit = 1u << (code & 31);
        u32 *dst = use_smem ? shb : bm;
        if (!(dst[w] & bit)) atomicOr(&dst[w], bit);
    }
    if (use_smem) {
        __syncthreads();
        for (u32 w = threadIdx.x; w < nwords; w += blockDim.x)
            if (shb[w]) atomicOr(&bm[w], shb[w]);
    }
}

// Byte-text versions: one CTA per TT_TILE triplets j, samples 3j+1 (mod-1,
// s = j) and 3j+2 (mod-2, s = m1 + j) read from the staged tile.
__global__ void __launch_bounds__(256)
k_bitmap_set_u8(const u8 *__restrict__ T, SampleLayout L, u64 s1, u32 *__restrict__ bm, u32 nwords, int use_smem) {
    extern __shared__ u32 shb[];
    __shared__ u32 shw[TT_WORDS];
    if (use_smem) {
        for (u32 w = threadIdx.x; w < nwords; w += blockDim.x) shb[w] = 0;
    }
    u32 *dst = use_smem ? shb : bm;
    const i64 ntiles = ceil_div(L.m1 > 0 ? L.m1 : 1, TT_TILE);
    // grid-stride over tiles: a large private bitmap is merged once per CTA
    for (i64 tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const i64 j0 = tile * TT_TILE;
        SmemText t = stage_text(T, L.n, 3 * j0, 3 * TT_TILE + 4, shw, 256);
        for (int x = threadIdx.x; x < TT_TILE; x += 256) {
            i64 j = j0 + x;
            if (j >= L.m1) break;
            i64 p = 3 * j;
            u32 c1 = t(p + 1), c2 = t(p + 2), c3 = t(p + 3), c4 = t(p + 4);
            u64 code = ((u64)c1 * s1 + c2) * s1 + c3;
            u32 w = (u32)(code >> 5), bit = 1u << (code & 31);
            if (!(dst[w] & bit)) atomicOr(&dst[w], bit);
            if (j < L.m2) {
                code = ((u64)c2 * s1 + c3) * s1 + c4;
                w = (u32)(code >> 5);
                bit = 1u << (code & 31);
                if (!(dst[w] & bit)) atomicOr(&dst[w], bit);
            }
        }
        __syncthreads();  // the staged tile is reused by the next iteration
    }
    if (use_smem) {
        __syncthreads();
        for (u32 w = threadIdx.x; w < nwords; w += blockDim.x)
            if (shb[w]) atomicOr(&bm[w], shb[w]);
    }
}

template <typename OT>
__global__ void __launch_bounds__(256)
k_bitmap_name_u8(const u8 *__restrict__ T, SampleLayout L, u64 s1, const u32 *__restrict__ bm,
                 const u32 *__restrict__ wp, OT *__restrict__ tt) {
    __shared__ u32 shw[TT_WORDS];
    const i64 j0 = (i64)blockIdx.x * TT_TILE;
    SmemText t = stage_text(T, L.n, 3 * j0, 3 * TT_TILE + 4, shw, 256);
    for (int x = threadIdx.x; x < TT_TILE; x += 256) {
        i64 j = j0 + x;
        if (j >= L.m1) break;
        i64 p = 3 * j;
        u32 c1 = t(p + 1), c2 = t(p + 2), c3 = t(p + 3), c4 = t(p + 4);
        u64 code = ((u64)c1 * s1 + c2) * s1 + c3;
        u32 w = (u32)(code >> 5);
        tt[j] = (OT)(wp[w] + __popc(bm[w] & ((1u << (code & 31)) - 1u)) + 1u);
        if (j < L.m2) {
            code = ((u64)c2 * s1 + c3) * s1 + c4;
            w = (u32)(code >> 5);
            tt[L.m1 + j] = (OT)(wp[w] + __popc(bm[w] & ((1u << (code & 31)) - 1u)) + 1u);
        }
    }
}

struct PopcIn {
    const u32 *bm;
    __device__ u32 operator()(i64 i) const { return __popc(bm[i]); }
};
struct StoreExcl {
    u32 *out;
    __device__ void operator()(i64 i, u32 excl, u32) const { out[i] = excl; }
};

// OT = u8 when the names fit a byte: the recursion string is then a u8 text
template <typename TT, typename OT>
__global__ void k_bitmap_name(Text<TT> T, SampleLayout L, u64 s1, const u32 *__restrict__ bm,
                              const u32 *__restrict__ wp, OT *__restrict__ tt) {
    for (i64 s = (i64)blockIdx.x * blockDim.x + threadIdx.x; s < L.m; s += (i64)gridDim.x * blockDim.x) {
        i64 p = L.pos(s);
        u64 code = ((u64)T(p) * s1 + T(p + 1)) * s1 + T(p + 2);
        u32 w = (u32)(code >> 5);
        u32 below = bm[w] & ((1u << (code & 31)) - 1u);
        tt[s] = (OT)(wp[w] + __popc(below) + 1u);
    }
}

// onesweep sources: packed triple keys of the samples, read from the text
// Mixed-radix triple key ((c0 s1 + c1) s1 + c2), s1 = sigma + 1: order-
// preserving and 3 log2(s1) bits instead of 3 ceil(log2(s1)).
template <typename TT>
struct TripleSrc {
    Text<TT> T;
    SampleLayout L;
    u64 s1;
    __device__ __forceinline__ bool get(i64 s, u64 &k, u32 &v) const {
        i64 p = L.pos(s);
        k = ((u64)T(p) * s1 + T(p + 1)) * s1 + T(p + 2);
        v = (u32)s;
        return true;
    }
};
// mod-0 split source: mod-1 samples in rank order (s < m1), keyed by the
// first character of the mod-0 suffix 3s (suffix_index.py:274-290)
template <typename TT>
struct Mod0Src {
    Text<TT> T;
    const u32 *sac;
    u32 m1;
    __device__ __forceinline__ bool get(i64 i, u32 &k, u32 &v) const {
        u32 s = __ldcs(sac + i);
        if (s >= m1) return false;
        k = T(3 * (i64)s);
        v = s;
        return true;
    }
};
// Small-alphabet mod-0 split without a sort.  Mod-0 suffix 3j sorts by
// (T(3j), R(3j+1)); bit isac[j] of the per-character bitmap B[T(3j)] marks
// it in sample-rank order.  One flattened popcount scan over the bitmaps
// (character-major) gives every suffix its output slot:
//   slot(j) = prefix[c][r >> 5] + popc(B[c][r >> 5] & below(r)),  r = isac[j].
// bitmap word and its exclusive popcount prefix interleaved: one 8 B gather
// per mod-0 suffix in the placement pass
template <typename TT>
__global__ void k_mod0_bits(Text<TT> T, const u32 *__restrict__ isac, i64 k, i64 words_per_char,
                            uint2 *__restrict__ pb) {
    for (i64 j = (i64)blockIdx.x * blockDim.x + threadIdx.x; j < k; j += (i64)gridDim.x * blockDim.x) {
        u32 r = __ldcs(isac + j);
        u32 c = T(3 * j);
        atomicOr(&pb[(i64)c * words_per_char + (r >> 5)].x, 1u << (r & 31));
    }
}
template <typename TT>
__global__ void k_mod0_place(Text<TT> T, const u32 *__restrict__ isac, i64 k, i64 words_per_char,
                             const uint2 *__restrict__ pb, u32 *__restrict__ out) {
    for (i64 j = (i64)blockIdx.x * blockDim.x + threadIdx.x; j < k; j += (i64)gridDim.x * blockDim.x) {
        u32 r = __ldcs(isac + j);
        u32 c = T(3 * j);
        uint2 e = pb[(i64)c * words_per_char + (r >> 5)];
        out[e.y + __popc(e.x & ((1u << (r & 31)) - 1u))] = (u32)j;
    }
}
struct PbPopc {
    const uint2 *pb;
    __device__ u32 operator()(i64 i) const { return __popc(pb[i].x); }
};
struct PbStore {
    uint2 *pb;
    __device__ void operator()(i64 i, u32 excl, u32) const { pb[i].y = excl; }
};
// (sigma+1) * m/32 bitmap words: only worth it for tiny alphabets (level 0 of
// DNA: 5-7 symbols); at sigma ~ 66 (level 1) and C3 size the bitmaps alone
// would be 2 GB, so larger alphabets take the onesweep split.
static bool mod0_use_bitmaps(u64 sigma) { return sigma + 1 <= 8; }
inline i64 mod0_bitmap_words(u64 sigma, i64 m) { return (i64)(sigma + 1) * (ceil_div(m, 32) + 1); }

// the same multiset of mod-0 first characters, streamed in text order
template <typename TT>
struct Mod0HistSrc {
    Text<TT> T;
    __device__ __forceinline__ bool get(i64 j, u32 &k, u32 &v) const {
        k = T(3 * j);
        v = 0;
        return true;
    }
};

// bucket-sort sources (wide keys, bsort.cuh): mixed-radix keys, bucketed by
// their top bits
template <typename TT>
struct TripleBucketSrc {  // key = c0 << 2b | c1 << b | c2 (b = bits(sigma)); dense = c0 * s1 + c1
    Text<TT> T;
    SampleLayout L;
    int b;
    u64 s1;
    __device__ __forceinline__ void get(i64 s, u64 &k, u32 &v) const {
        i64 p = L.pos(s);
        k = ((u64)T(p) << (2 * b)) | ((u64)T(p + 1) << b) | T(p + 2);
        v = (u32)s;
    }
    __device__ __forceinline__ u64 dense(u64 k) const {
        return (k >> (2 * b)) * s1 + ((k >> b) & (((u64)1 << b) - 1));
    }
};
// mod-0 suffix 3j keyed by (T(3j), R(3j+1)) = T(3j) << rb | ISAc[j] + 1;
// streamed in text order (the keys are distinct)
template <typename TT>
struct Mod0BucketSrc {
    Text<TT> T;
    const u32 *isac;
    int rb;  // bits(m)
    u64 m1;  // m + 1
    __device__ __forceinline__ void get(i64 j, u64 &k, u32 &v) const {
        k = ((u64)T(3 * j) << rb) | (__ldcs(isac + j) + 1u);
        v = (u32)j;
    }
    __device__ __forceinline__ u64 dense(u64 k) const { return (k >> rb) * m1 + (k & (((u64)1 << rb) - 1)); }
};
// bucket sort replaces LSD radix when the keys are wide
static bool use_bsort(u64 max_key, i64 n) { return n >= 4096 && bits_for(max_key) > 24; }

// wide-alphabet naming sources (3 bits(sigma) > 64)
template <typename TT>
struct ThirdSrc {
    Text<TT> T;
    SampleLayout L;
    __device__ __forceinline__ bool get(i64 s, u64 &k, u32 &v) const {
        k = T(L.pos(s) + 2);
        v = (u32)s;
        return true;
    }
};
template <typename TT>
struct PairGatherSrc {  // (c0, c1) of the sample at sorted slot i
    Text<TT> T;
    SampleLayout L;
    const u32 *order;
    u64 s1;
    __device__ __forceinline__ bool get(i64 i, u64 &k, u32 &v) const {
        v = order[i];
        i64 p = L.pos(v);
        k = (u64)T(p) * s1 + T(p + 1);
        return true;
    }
};
template <typename TT>
struct PairStreamSrc {  // the same keys in sample order (histogram)
    Text<TT> T;
    SampleLayout L;
    u64 s1;
    __device__ __forceinline__ bool get(i64 s, u64 &k, u32 &v) const {
        i64 p = L.pos(s);
        k = (u64)T(p) * s1 + T(p + 1);
        v = 0;
        return true;
    }
};
template <typename TT>
struct FlagWide {  // new name iff (c0, c1) key or c2 differs from the predecessor
    Text<TT> T;
    SampleLayout L;
    const u64 *keys;
    const u32 *vals;
    __device__ u32 operator()(i64 i) const {
        if (i == 0 || keys[i] != keys[i - 1]) return 1u;
        return T(L.pos(vals[i]) + 2) != T(L.pos(vals[i - 1]) + 2) ? 1u : 0u;
    }
};

struct FlagPacked {
    const u64 *keys;
    __device__ u32 operator()(i64 i) const { return (i == 0 || keys[i] != keys[i - 1]) ? 1u : 0u; }
};
// number of distinct keys in a sorted array (heads of equal-key runs)
__global__ void k_count_distinct(const u64 *__restrict__ keys, i64 m, u32 *__restrict__ count) {
    u32 c = 0;
    for (i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (i64)gridDim.x * blockDim.x)
        c += (i == 0 || keys[i] != keys[i - 1]) ? 1u : 0u;
    for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if (lane_id() == 0 && c) atomicAdd(count, c);
}

struct ScatterName {
    const u32 *vals;
    u32 *tt;
    __device__ void operator()(i64 i, u32 excl, u32 v) const { tt[vals[i]] = excl + v; }
};

// all names distinct: the names are the 1-based sample ranks
__global__ void k_unique_from_names(const u32 *__restrict__ tt, i64 m, u32 *__restrict__ sac,
                                    u32 *__restrict__ isac) {
    for (i64 s = (i64)blockIdx.x * blockDim.x + threadIdx.x; s < m; s += (i64)gridDim.x * blockDim.x) {
        u32 r = tt[s] - 1u;
        isac[s] = r;
        sac[r] = (u32)s;
    }
}
__global__ void k_unique_from_sorted(const u32 *__restrict__ vals, i64 m, u32 *__restrict__ sac,
                                     u32 *__restrict__ isac) {
    for (i64 r = (i64)blockIdx.x * blockDim.x + threadIdx.x; r < m; r += (i64)gridDim.x * blockDim.x) {
        u32 s = vals[r];
        if (sac) sac[r] = s;
        isac[s] = (u32)r;
    }
}

// ------------------------------------------------------------ mod-0 order
// _sort_nonsamples (suffix_index.py:274-290): non-samples 3j ordered by
// (T[3j], rank of 3j+1).

// ------------------------------------------------------------ merge

// Comparator of the merge step (suffix_index.py:192-202, `_merge_walk`):
// suffix(a) < suffix(b) for sample position a and non-sample position b.
template <typename TT, class Rank>
__device__ __forceinline__ bool dc3_a_first(const Text<TT> &T, const Rank &R, i64 a, i64 b) {
    u32 ca = T(a), cb = T(b);
    if (ca != cb) return ca < cb;
    if (a % 3 == 1) return R(a + 1) < R(b + 1);
    u32 ca2 = T(a + 1), cb2 = T(b + 1);
    if (ca2 != cb2) return ca2 < cb2;
    return R(a + 2) < R(b + 2);
}

// 1-based sample rank by position from the child's 0-based ISA over sample
// indices (the reference's `rank_of`, 0 at non-sample / beyond-limit spots).
struct RankFromIsa {
    SampleLayout L;
    const u32 *isac;
    __device__ __forceinline__ u32 operator()(i64 p) const {
        i64 j = p / 3;
        i64 r = p - 3 * j;
        if (r == 1) return j < L.m1 ? isac[j] + 1u : 0u;
        if (r == 2) return j < L.m2 ? isac[L.m1 + j] + 1u : 0u;
        return 0u;
    }
};
struct RankByPos {
    const u32 *rank;
    __device__ __forceinline__ u32 operator()(i64 p) const { return rank[p]; }
};

// Comparison record of one suffix p: the two leading characters and the
// 1-based sample ranks one and two positions on.  Everything the DC3
// comparator can ask about p, fetched once.
struct MRec {
    u32 pos, c0, c1, r1, r2;
};

template <typename TT, class Rank>
__device__ __forceinline__ MRec make_rec(const Text<TT> &T, const Rank &R, i64 p) {
    MRec m;
    m.pos = (u32)p;
    m.c0 = T(p);
    m.c1 = T(p + 1);
    m.r1 = (p % 3 == 2) ? 0u : R(p + 1);  // mod-2 samples never use r1
    m.r2 = (p % 3 == 1) ? 0u : R(p + 2);  // mod-1 samples never use r2
    return m;
}

// suffix(a) < suffix(b), a a sample, b a non-sample (suffix_index.py:192-202)
__device__ __forceinline__ bool rec_a_first(const MRec &a, const MRec &b) {
    if (a.c0 != b.c0) return a.c0 < b.c0;
    if (a.pos % 3 == 1) return a.r1 < b.r1;
    if (a.c1 != b.c1) return a.c1 < b.c1;
    return a.r2 < b.r2;
}

// Per-triplet comparison block E[j] (j in [0, k)) built by one streaming
// pass over the text and the child's ISA: the four characters T(3j..3j+3)
// and the sample ranks R(3j+1), R(3j+2), R(3j+4).  Every suffix p the merge
// compares (non-sample 3j, mod-1 3j+1, mod-2 3j+2) finds its whole DC3
// comparison record in E[p / 3], so the merge does one 16 B (u8 text) or
// 32 B (wider text) gather per element instead of 2-3 dependent ones.
struct EBlock8 {  // u8 text
    u32 chars, r1, r2, r4;
};
struct EBlock32 {  // u32 text
    u32 c0, c1, c2, c3, r1, r2, r4, pad;
};
template <typename TT>
struct EBlockOf {
    using type = EBlock32;
};
template <>
struct EBlockOf<u8> {
    using type = EBlock8;
};

template <typename TT>
__global__ void k_build_eblocks(Text<TT> T, RankFromIsa R, i64 k, typename EBlockOf<TT>::type *__restrict__ E) {
    for (i64 j = (i64)blockIdx.x * blockDim.x + threadIdx.x; j < k; j += (i64)gridDim.x * blockDim.x) {
        i64 p = 3 * j;
        u32 r1 = R(p + 1), r2 = R(p + 2), r4 = R(p + 4);
        if constexpr (sizeof(TT) == 1) {
            u32 ch = T(p) | (T(p + 1) << 8) | (T(p + 2) << 16) | (T(p + 3) << 24);
            __stcs(reinterpret_cast<uint4 *>(E + j), make_uint4(ch, r1, r2, r4));
        } else {
            uint4 *dst = reinterpret_cast<uint4 *>(E + j);
            __stcs(dst, make_uint4(T(p), T(p + 1), T(p + 2), T(p + 3)));
            __stcs(dst + 1, make_uint4(r1, r2, r4, 0u));
        }
    }
}

template <typename TT>
__device__ __forceinline__ MRec rec_from_eblock(const typename EBlockOf<TT>::type *__restrict__ E, i64 p, u64 pol) {
    i64 j = p / 3;
    int r = (int)(p - 3 * j);
    u32 c[4], r1, r2, r4;
    if constexpr (sizeof(TT) == 1) {
        uint4 e = ldg_last(reinterpret_cast<const uint4 *>(E + j), pol);
        c[0] = e.x & 0xFF;
        c[1] = (e.x >> 8) & 0xFF;
        c[2] = (e.x >> 16) & 0xFF;
        c[3] = e.x >> 24;
        r1 = e.y;
        r2 = e.z;
        r4 = e.w;
    } else {
        uint4 a = ldg_last(reinterpret_cast<const uint4 *>(E + j), pol);
        uint4 b = ldg_last(reinterpret_cast<const uint4 *>(E + j) + 1, pol);
        c[0] = a.x;
        c[1] = a.y;
        c[2] = a.z;
        c[3] = a.w;
        r1 = b.x;
        r2 = b.y;
        r4 = b.z;
    }
    MRec m;
    m.pos = (u32)p;
    if (r == 0) {  // non-sample 3j: (c0, c1, R(3j+1), R(3j+2))
        m.c0 = c[0];
        m.c1 = c[1];
        m.r1 = r1;
        m.r2 = r2;
    } else if (r == 1) {  // mod-1 sample: (c0, R(p+1))
        m.c0 = c[1];
        m.c1 = 0;
        m.r1 = r2;
        m.r2 = 0;
    } else {  // mod-2 sample: (c0, c1, R(p+2))
        m.c0 = c[2];
        m.c1 = c[3];
        m.r1 = 0;
        m.r2 = r4;
    }
    return m;
}

// Compact 8-byte block when 2 bits(m) + 3 bits(sigma) <= 64:
//   r1 | r2 << rb | c0 << 2rb | c1 << 2rb+cb | c2 << 2rb+2cb
// (R(3j+4) and T(3j+3) are the next block's r1 and c0, so they are not
// stored).  Random gathers on B200 only stay in L2 while the target is
// below ~64 MB (profiles/r1_l2_random_gather_probe.txt); at C2 level 0 the
// compact blocks are 53 MB instead of 107 MB.  E[k] is a zero sentinel.
__global__ void k_build_ecompact_u8(Text<u8> T, RankFromIsa R, i64 k, int rb, int cb, u64 *__restrict__ E) {
    for (i64 j = (i64)blockIdx.x * blockDim.x + threadIdx.x; j <= k; j += (i64)gridDim.x * blockDim.x) {
        u64 x = 0;
        if (j < k) {
            i64 p = 3 * j;
            x = (u64)R(p + 1) | ((u64)R(p + 2) << rb) | ((u64)T(p) << (2 * rb)) | ((u64)T(p + 1) << (2 * rb + cb)) |
                ((u64)T(p + 2) << (2 * rb + 2 * cb));
        }
        __stcs(E + j, x);
    }
}

struct ECompact {
    const u64 *E;
    int rb, cb;
    __device__ __forceinline__ MRec rec(i64 p) const {
        i64 j = p / 3;
        int r = (int)(p - 3 * j);
        u64 rm = ((u64)1 << rb) - 1, cm = ((u64)1 << cb) - 1;
        u64 x = __ldg(E + j);
        MRec m;
        m.pos = (u32)p;
        if (r == 0) {
            m.c0 = (u32)((x >> (2 * rb)) & cm);
            m.c1 = (u32)((x >> (2 * rb + cb)) & cm);
            m.r1 = (u32)(x & rm);
            m.r2 = (u32)((x >> rb) & rm);
        } else if (r == 1) {
            m.c0 = (u32)((x >> (2 * rb + cb)) & cm);
            m.c1 = 0;
            m.r1 = (u32)((x >> rb) & rm);
            m.r2 = 0;
        } else {
            u64 y = __ldg(E + j + 1);
            m.c0 = (u32)((x >> (2 * rb + 2 * cb)) & cm);
            m.c1 = (u32)((y >> (2 * rb)) & cm);
            m.r1 = 0;
            m.r2 = (u32)(y & rm);
        }
        return m;
    }
};

// Merge inputs: sorted samples as sample indices / sorted mod-0 as indices.
template <typename TT>
struct MergeIdx {
    Text<TT> T;
    RankFromIsa R;
    const u32 *A, *B;
    const typename EBlockOf<TT>::type *E;
    ECompact EC;  // used when EC.E != nullptr
    __device__ __forceinline__ i64 apos(i64 i) const { return R.L.pos(A[i]); }
    __device__ __forceinline__ i64 bpos(i64 j) const { return 3 * (i64)B[j]; }
    __device__ __forceinline__ i64 apos_cs(i64 i) const { return R.L.pos(__ldcs(A + i)); }
    __device__ __forceinline__ i64 bpos_cs(i64 j) const { return 3 * (i64)__ldcs(B + j); }
    __device__ __forceinline__ MRec rec(i64 p) const {
        return EC.E ? EC.rec(p) : rec_from_eblock<TT>(E, p, l2_evict_last());
    }
    __device__ __forceinline__ MRec reca(i64 i) const { return rec(apos(i)); }
    __device__ __forceinline__ MRec recb(i64 j) const { return rec(bpos(j)); }
};
// Merge inputs given as positions with a by-position rank array
// (merge_sample_nonsample, suffix_index.py:452-457).
template <typename TT>
struct MergePos {
    Text<TT> T;
    RankByPos R;
    const u32 *A, *B;
    __device__ __forceinline__ i64 apos(i64 i) const { return A[i]; }
    __device__ __forceinline__ i64 bpos(i64 j) const { return B[j]; }
    __device__ __forceinline__ i64 apos_cs(i64 i) const { return A[i]; }
    __device__ __forceinline__ i64 bpos_cs(i64 j) const { return B[j]; }
    __device__ __forceinline__ MRec rec(i64 p) const { return make_rec(T, R, p); }
    __device__ __forceinline__ MRec reca(i64 i) const { return rec(apos(i)); }
    __device__ __forceinline__ MRec recb(i64 j) const { return rec(bpos(j)); }
};

// Merge path in two kernels.  k_merge_partition splits the output into
// MT_TILE-sized diagonals with one global binary search per tile;
// k_merge_tile stages the tile's samples and non-samples as comparison
// records in shared memory, merges them with per-thread merge paths in
// shared memory, writes SA coalesced and scatters ISA.
constexpr int MT_THREADS = 256;
constexpr int MT_ITEMS = 8;
constexpr int MT_TILE = MT_THREADS * MT_ITEMS;  // 2048 outputs per CTA

// One warp per tile boundary: a 33-ary search (each lane probes one split
// candidate per round) so a split costs ~log_32(n) dependent gather rounds.
template <class V, int TILE = MT_TILE>
__global__ void k_merge_partition(V v, i64 na, i64 nb, i64 ntiles, u32 *__restrict__ split, i64 stride = 1,
                                  const u32 *__restrict__ coarse = nullptr) {
    i64 total = na + nb;
    int lane = lane_id();
    i64 warps = ((i64)gridDim.x * blockDim.x) >> 5;
    i64 nsplit = ceil_div(ntiles, stride);
    for (i64 t = ((i64)blockIdx.x * blockDim.x + threadIdx.x) >> 5; t <= nsplit; t += warps) {
        i64 d = t * stride * TILE < total ? t * stride * TILE : total;
        // invariant: answer in [lo, hi]; P(x) = a_first(A[x], B[d-1-x]) is
        // true for x < answer and false from answer on
        i64 lo = d > nb ? d - nb : 0, hi = d < na ? d : na;
        if (coarse) {  // inside the coarse window (see k_merge_partition_rec)
            i64 c = t / 32;
            i64 clo = coarse[c], chi = coarse[c + 1 <= ceil_div(ntiles, 32) ? c + 1 : c];
            if (clo > lo) lo = clo;
            if (chi < hi && t % 32) hi = chi;
            if (t % 32 == 0) lo = hi = clo;
        }
        while (lo < hi) {
            i64 span = hi - lo;
            i64 x = lo + (span * (lane + 1)) / 33;  // candidates in [lo, hi)
            bool p = x < hi && rec_a_first(v.reca(x), v.recb(d - 1 - x));
            u32 tr = __ballot_sync(0xffffffffu, p);
            u32 fl = __ballot_sync(0xffffffffu, x < hi && !p);
            // last true candidate -> lo = x+1; first false candidate -> hi = x
            if (tr) {
                int lt = 31 - __clz(tr);
                lo = __shfl_sync(0xffffffffu, x, lt) + 1;
            }
            if (fl) {
                int lf = __ffs(fl) - 1;
                hi = __shfl_sync(0xffffffffu, x, lf);
            }
            if (span <= 32) {
                // every candidate in [lo, hi) was probed this round
                break;
            }
        }
        if (lane == 0) split[t] = (u32)lo;
    }
}

template <class V>
__global__ void __launch_bounds__(MT_THREADS)
k_merge_tile(V v, i64 na, i64 nb, const u32 *__restrict__ split, u32 *__restrict__ sa, u32 *__restrict__ isa) {
    __shared__ MRec sh[MT_TILE];
    __shared__ u32 out[MT_TILE];
    i64 total = na + nb;
    i64 d0 = (i64)blockIdx.x * MT_TILE;
    i64 d1 = d0 + MT_TILE < total ? d0 + MT_TILE : total;
    i64 i0 = split[blockIdx.x], i1 = split[blockIdx.x + 1];
    i64 j0 = d0 - i0;
    int nat = (int)(i1 - i0), cnt = (int)(d1 - d0), nbt = cnt - nat;
#pragma unroll
    for (int q = 0; q < MT_ITEMS; q++) {
        int x = threadIdx.x + q * MT_THREADS;
        if (x < cnt) sh[x].pos = (u32)(x < nat ? v.apos_cs(i0 + x) : v.bpos_cs(j0 + (x - nat)));
    }
#pragma unroll
    for (int q = 0; q < MT_ITEMS; q++) {
        int x = threadIdx.x + q * MT_THREADS;
        if (x < cnt) sh[x] = v.rec(sh[x].pos);
    }
    __syncthreads();
    const MRec *A = sh, *B = sh + nat;
    int dt = threadIdx.x * MT_ITEMS;
    if (dt < cnt) {
        int lo = dt > nbt ? dt - nbt : 0, hi = dt < nat ? dt : nat;
        while (lo < hi) {
            int mid = (lo + hi) >> 1;
            if (rec_a_first(A[mid], B[dt - 1 - mid])) lo = mid + 1;
            else hi = mid;
        }
        int i = lo, j = dt - lo;
#pragma unroll
        for (int r = 0; r < MT_ITEMS; r++) {
            if (dt + r >= cnt) break;
            bool takeA = j >= nbt || (i < nat && rec_a_first(A[i], B[j]));
            out[dt + r] = takeA ? A[i++].pos : B[j++].pos;
        }
    }
    __syncthreads();
    for (int x = threadIdx.x; x < cnt; x += MT_THREADS) {
        u32 p = out[x];
        __stcs(sa + d0 + x, p);
        if (isa) isa[p] = (u32)(d0 + x);
    }
}

template <class V>
static int merge_run(V v, i64 na, i64 nb, u32 *split, u32 *sa, u32 *isa, cudaStream_t st) {
    i64 total = na + nb;
    if (total == 0) return SAIX_OK;
    i64 ntiles = ceil_div(total, MT_TILE);
    {
        Prof prof_("dc3.merge_partition", 4.0 * (ntiles + 1), st);
        k_merge_partition<V><<<grid_for((ntiles + 1) * 32, 128), 128, 0, st>>>(v, na, nb, ntiles, split);
    }
    SAIX_LAUNCHED();
    {
        // indices 4 + chars 2w + ranks (4 per sample, 8 per non-sample) + SA 4 + ISA 4
        double w = (double)v.T.bytes();
        Prof prof_("dc3.merge_tile", total * (4 + 2 * w + 4) + 4.0 * (na + 2 * nb) + (isa ? 4.0 * total : 0), st);
        k_merge_tile<V><<<(unsigned)ntiles, MT_THREADS, 0, st>>>(v, na, nb, split, sa, isa);
    }
    SAIX_LAUNCHED();
    return SAIX_OK;
}

inline i64 merge_split_words(i64 total) { return ceil_div(total > 0 ? total : 1, MT_TILE) + 2; }

// ------------------------------------------------------------ streaming level (u8 text)
// One level of _dc3 (suffix_index.py:381-392) after the sample sort:
// _sort_nonsamples (274-290) and _merge / _merge_walk (362-378, 173-218).
//
// Levels with a byte text (sigma < 256: DNA levels 0-1) avoid every random
// gather of the merge and of the mod-0 split.  Each suffix the merge needs is
// described by one 16 B record, laid out the same for samples and non-samples:
//   {pos, R(pos+1), R(pos+2), c0 | c1 << 8 | cprev << 16}
// (1-based sample ranks, 0 where the reference's rank_of is 0; a mod-1 sample
// carries only R(pos+1) and c0, a mod-2 sample only R(pos+2), c0, c1; cprev =
// T(pos-1) rides along on mod-1 samples for the mod-0 split).
//   1 k_srec_emit   stream the text and ISAc in triplet order; every sample's
//                   record goes, via the bucketed scatter (pscatter.cuh), to
//                   RS[rank] -- the samples' records in sorted order.
//   2 mod-0 split   RS streamed in rank order; every mod-1 sample 3j+1 yields
//                   the record of non-sample 3j, stably partitioned by
//                   cprev = T(3j) (one onesweep pass): the non-samples sorted
//                   by (T(3j), R(3j+1)) (suffix_index.py:274-290).
//   3 merge         both sides are contiguous record runs per tile; output SA
//                   (top level) and the bucketed ISA (inner levels, the
//                   parent's ranks) or Phi pairs (top level, for the LCP).
// Random traffic left: none outside the L2-windowed scatter passes.
__device__ __forceinline__ bool recq_a_first(const uint4 &a, const uint4 &b) {
    u32 ca = a.w & 0xFFu, cb = b.w & 0xFFu;
    if (ca != cb) return ca < cb;
    if (a.x % 3 == 1) return a.y < b.y;
    u32 ca1 = (a.w >> 8) & 0xFFu, cb1 = (b.w >> 8) & 0xFFu;
    if (ca1 != cb1) return ca1 < cb1;
    return a.z < b.z;
}

constexpr int SR_THREADS = 256;
constexpr int SR_J = 4;                      // triplets per thread
constexpr int SR_TILE = SR_THREADS * SR_J;   // 2048 triplets -> <= 4096 records

// pass A of the record scatter: item {dest = 0-based sample rank, pos, nb, chars}
__global__ void __launch_bounds__(SR_THREADS, 4)
k_srec_emit(Text<u8> T, SampleLayout L, const u32 *__restrict__ isac, PsPlan plan, uint4 *__restrict__ stage) {
    extern __shared__ __align__(16) unsigned char smem[];
    uint4 *sh_items = reinterpret_cast<uint4 *>(smem);
    u32 *sh_cnt = reinterpret_cast<u32 *>(sh_items + 2 * SR_TILE);
    u32 *sh_base = sh_cnt + plan.a.buckets;
    __shared__ u32 shw[(3 * SR_TILE + 8) / 4 + 2];
    const i64 j0 = (i64)blockIdx.x * SR_TILE;
    SmemText t = stage_text(T.t, T.n, 3 * j0, 3 * SR_TILE + 4, shw, SR_THREADS);
    uint4 it[2 * SR_J];
    bool ok[2 * SR_J];
#pragma unroll
    for (int r = 0; r < SR_J; r++) {
        i64 j = j0 + r * SR_THREADS + threadIdx.x;
        ok[2 * r] = j < L.m1;
        ok[2 * r + 1] = j < L.m2;
        if (ok[2 * r]) {
            i64 p = 3 * j;
            u32 cp = t(p), c0 = t(p + 1), c1 = t(p + 2), c2 = t(p + 3);
            u32 r1 = isac[j];
            u32 r2 = j < L.m2 ? isac[L.m1 + j] : 0xFFFFFFFFu;
            u32 r4 = j + 1 < L.m1 ? isac[j + 1] + 1u : 0u;
            it[2 * r] = make_uint4(r1, (u32)(p + 1), r2 + 1u, c0 | (c1 << 8) | (cp << 16));
            if (ok[2 * r + 1]) it[2 * r + 1] = make_uint4(r2, (u32)(p + 2), r4, c1 | (c2 << 8));
        }
    }
    ps_block_emit<uint4, SR_THREADS, 2 * SR_J>(it, ok, plan.a, stage, sh_items, sh_cnt, sh_base);
}

// pass B: RS[rank] = record
struct RsApply {
    using Out = uint4;
    uint4 *out;
    __device__ __forceinline__ uint4 value(const uint4 &p) const {
        return (p.y % 3 == 1) ? make_uint4(p.y, p.z, 0u, p.w) : make_uint4(p.y, 0u, p.z, p.w);
    }
};

// mod-0 split source: RS in rank order; mod-1 sample 3j+1 at rank r gives
// non-sample 3j = {3j, r+1, R(3j+2), T(3j) | T(3j+1) << 8} keyed by T(3j)
struct Mod0RecSrc {
    const uint4 *rs;
    __device__ __forceinline__ bool get(i64 r, u32 &k, uint4 &v) const {
        uint4 e = rs[r];
        if (e.x % 3 != 1) return false;
        u32 cp = (e.w >> 16) & 0xFFu;
        k = cp;
        v = make_uint4(e.x - 1, (u32)r + 1u, e.y, cp | ((e.w & 0xFFu) << 8));
        return true;
    }
};

// Pass B of the record scatter, specialised: writes RS window w (2048 ranks)
// and counts its mod-1 samples per cprev digit into hist[d * windows + w]
// (digit-major, so one flat exclusive scan gives every (digit, window) its
// output offset in the mod-0 order).
constexpr int RW_SHIFT = 11;  // 2048 records = 32 KB window
__global__ void __launch_bounds__(PS_THREADS)
k_rs_window(const uint4 *__restrict__ stage2, PsPlan plan, uint4 *__restrict__ rs, u32 *__restrict__ hist, int D1) {
    extern __shared__ __align__(16) unsigned char ps_smem[];
    uint4 *win = reinterpret_cast<uint4 *>(ps_smem);
    __shared__ u32 cnt[PS_THREADS / 32][256];  // warp-private digit counters (plain shared atomics)
    const i64 w = blockIdx.x;
    const i64 d0 = w << RW_SHIFT;
    const i64 len = (d0 + (1 << RW_SHIFT) < plan.n_dest ? d0 + (1 << RW_SHIFT) : plan.n_dest) - d0;
    const i64 n_in = plan.cursor2[w];
    const uint4 *src = stage2 + d0;
    RsApply ap{rs};
    for (int d = threadIdx.x; d < (PS_THREADS / 32) * 256; d += PS_THREADS) (&cnt[0][0])[d] = 0;
    __syncthreads();
    const bool full = n_in == len;
    for (i64 x = threadIdx.x; x < n_in; x += PS_THREADS) {
        uint4 p = ld_stream(src + x);
        uint4 e = ap.value(p);
        if (full) win[(i64)p.x - d0] = e;
        else rs[p.x] = e;
    }
    __syncthreads();
    // count digits over the window's records (window order when full)
    const i64 nc = full ? len : n_in;
    for (i64 x0 = 0; x0 < nc; x0 += PS_THREADS) {
        i64 x = x0 + threadIdx.x;
        u32 d = 0xFFFFFFFFu;
        if (x < nc) {
            uint4 e;
            if (full) {
                e = win[x];
                st_stream(rs + d0 + x, e);
            } else {
                e = ap.value(ld_stream(src + x));
            }
            if (e.x % 3 == 1) d = (e.w >> 16) & 0xFFu;
        }
        if (d != 0xFFFFFFFFu) atomicAdd(&cnt[threadIdx.x >> 5][d], 1u);
    }
    __syncthreads();
    for (int d = threadIdx.x; d < D1; d += PS_THREADS) {
        u32 c = 0;
#pragma unroll
        for (int q = 0; q < PS_THREADS / 32; q++) c += cnt[q][d];
        hist[(i64)d * plan.windows + w] = c;
    }
}

// Small levels (text + ISAc <= 128 MB: random reads mostly L2 hits; C2 level
// 0 at 73 MB measured 0.17 ms vs 0.36 ms for the scatter passes): RS by
// gathers in rank order from the child's SAc instead of the bucketed
// scatter -- one CTA per 2048-rank window, also counting the window's mod-1
// samples per cprev digit (as k_rs_window does).
constexpr i64 RS_GATHER_BYTES = (i64)128 << 20;
constexpr int RG_THREADS = 256, RG_ITEMS = 8;  // 2048 = 1 << RW_SHIFT
__global__ void __launch_bounds__(RG_THREADS)
k_rs_gather(const u32 *__restrict__ sac, Text<u8> T, SampleLayout L, const u32 *__restrict__ isac,
            uint4 *__restrict__ rs, u32 *__restrict__ hist, int D1, u32 dmask, i64 windows) {
    __shared__ u32 cnt[256];
    for (int d = threadIdx.x; d < 256; d += RG_THREADS) cnt[d] = 0;
    __syncthreads();
    const i64 w = blockIdx.x;
    const i64 r0 = w << RW_SHIFT;
    u32 sv[RG_ITEMS];
#pragma unroll
    for (int q = 0; q < RG_ITEMS; q++) {
        i64 r = r0 + q * RG_THREADS + threadIdx.x;
        sv[q] = r < L.m ? __ldcs(sac + r) : 0u;
    }
#pragma unroll
    for (int q = 0; q < RG_ITEMS; q++) {
        i64 r = r0 + q * RG_THREADS + threadIdx.x;
        u32 d = 256u;
        if (r < L.m) {
            u32 sidx = sv[q];
            uint4 e;
            if (sidx < L.m1) {  // mod-1 sample 3s+1: {pos, R(pos+1), 0, c0 | c1 << 8 | cprev << 16}
                i64 p = 3 * (i64)sidx + 1;
                u32 nb = sidx < L.m2 ? isac[L.m1 + sidx] + 1u : 0u;
                u32 cp = T(p - 1);
                e = make_uint4((u32)p, nb, 0u, T(p) | (T(p + 1) << 8) | (cp << 16));
                d = cp;
            } else {  // mod-2 sample 3j+2: {pos, 0, R(pos+2), c0 | c1 << 8}
                i64 j = sidx - L.m1;
                i64 p = 3 * j + 2;
                u32 nb = j + 1 < L.m1 ? isac[j + 1] + 1u : 0u;
                e = make_uint4((u32)p, 0u, nb, T(p) | (T(p + 1) << 8));
            }
            __stcs(rs + r, e);
        }
        u32 peers = digit_peers_w(d, dmask);
        if (d < 256u && (peers & lanemask_lt()) == 0) atomicAdd(&cnt[d], (u32)__popc(peers));
    }
    __syncthreads();
    for (int d = threadIdx.x; d < D1; d += RG_THREADS) hist[(i64)d * windows + w] = cnt[d];
}

// Mod-0 records of RS window w, stably partitioned by cprev: one tile of
// 2048 ranks per CTA (256 threads x 8), warp-stable ranking (as in
// k_os_pass) with the global per-(digit, window) offsets already known, so
// no look-back; the tile is staged digit-sorted in shared memory and written
// as runs.
constexpr int M0_THREADS = 256, M0_WARPS = M0_THREADS / 32;
constexpr int M0_ITEMS = 8;  // 256 x 8 = 2048 = 1 << RW_SHIFT
struct RsRecSrc {  // 16 B records RS[rank]; fetch / decode split so all loads issue first
    const uint4 *rs;
    using Raw = uint4;
    static constexpr int kMinBlocks = 4;  // k_mod0_window residency
    __device__ __forceinline__ Raw fetch(i64 i) const { return __ldcs(rs + i); }
    __device__ __forceinline__ uint4 decode(const Raw &e) const { return e; }
    __device__ __forceinline__ uint4 operator()(i64 i) const { return fetch(i); }
};
template <class Src>
__global__ void __launch_bounds__(M0_THREADS, Src::kMinBlocks)
k_mod0_window(Src rs, i64 m, i64 windows, const u32 *__restrict__ offs, uint4 *__restrict__ M0, u32 dmask) {
    extern __shared__ __align__(16) unsigned char m0_smem[];
    uint4 *sv = reinterpret_cast<uint4 *>(m0_smem);
    u32(*cnt)[256] = reinterpret_cast<u32(*)[256]>(sv + (1 << RW_SHIFT));
    __shared__ u32 tile_excl[256], gbase[256], sh_warp[9];
    const int wp = threadIdx.x >> 5, lane = lane_id();
    for (int d = lane; d < 256; d += 32) cnt[wp][d] = 0;
    __syncthreads();
    const i64 w = blockIdx.x;
    const i64 seg = (w << RW_SHIFT) + (i64)wp * (32 * M0_ITEMS);
    // per item: pos, nb, and c0 | digit << 8 | rank-in-digit << 17
    u32 pos[M0_ITEMS], nb[M0_ITEMS], pk[M0_ITEMS];
    const u32 lt = lanemask_lt();
    typename Src::Raw raw[M0_ITEMS];
#pragma unroll
    for (int r = 0; r < M0_ITEMS; r++) {
        const i64 i = seg + r * 32 + lane;
        if (i < m) raw[r] = rs.fetch(i);
    }
#pragma unroll
    for (int r = 0; r < M0_ITEMS; r++) {
        i64 i = seg + r * 32 + lane;
        pk[r] = 256u << 8;
        if (i < m) {
            uint4 e = rs.decode(raw[r]);
            if (e.x % 3 == 1) {
                pos[r] = e.x;
                nb[r] = e.y;
                pk[r] = (e.w & 0xFFu) | (((e.w >> 16) & 0xFFu) << 8);
            }
        }
    }
#pragma unroll
    for (int r = 0; r < M0_ITEMS; r++) {
        u32 d = (pk[r] >> 8) & 0x1FFu;
        bool ok = d < 256u;
        u32 peers = digit_peers_w(d, dmask);
        u32 before = __popc(peers & lt);
        u32 cur = ok ? cnt[wp][d] : 0u;
        __syncwarp();
        if (ok && before == 0) cnt[wp][d] = cur + __popc(peers);
        __syncwarp();
        pk[r] |= (cur + before) << 17;
    }
    __syncthreads();
    // threads 0..255 own one digit each: warp-exclusive prefixes, tile counts
    u32 run = 0, inc = 0;
    const int d = threadIdx.x;
    if (d < 256) {
#pragma unroll
        for (int q = 0; q < M0_WARPS; q++) {
            u32 c = cnt[q][d];
            cnt[q][d] = run;
            run += c;
        }
        gbase[d] = run ? offs[(i64)d * windows + w] : 0u;
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
    for (int r = 0; r < M0_ITEMS; r++) {
        u32 dg = (pk[r] >> 8) & 0x1FFu;
        if (dg < 256u) {
            u32 lp = tile_excl[dg] + cnt[wp][dg] + (pk[r] >> 17);
            i64 rk = seg + r * 32 + lane;  // 0-based sample rank of 3j+1
            sv[lp] = make_uint4(pos[r] - 1, (u32)rk + 1u, nb[r], dg | ((pk[r] & 0xFFu) << 8));
        }
    }
    __syncthreads();
    const u32 valid = sh_warp[8];
    for (u32 x = threadIdx.x; x < valid; x += M0_THREADS) {
        uint4 v = sv[x];
        u32 dg = v.w & 0xFFu;
        __stcs(M0 + gbase[dg] + (x - tile_excl[dg]), v);
    }
}
constexpr size_t M0_SMEM = ((size_t)16 << RW_SHIFT) + (size_t)M0_WARPS * 256 * 4;

// ---- compact byte-level records (levels named by the DNA window sort)
// The window sort leaves the samples' rank order SR (= SAc, sample indices)
// and their first two characters CH (c0 | c1 << 4, from the window key) in
// rank order; only the rank of the next sample (+ cprev of mod-1 samples)
// travels through the bucketed scatter, 8 B items instead of 16 B records:
//   NX[rank] = R(next sample) (1-based, 0 past the end) | cprev << 29
// (cprev field 7 marks a mod-2 sample).  The record of the mod-0 and merge
// passes ({pos, R(pos+1), R(pos+2), c0 | c1 << 8 | cprev << 16}) is rebuilt
// from (SR, NX, CH): 9 B read per rank instead of 16.
constexpr u32 NX_MASK = (1u << 29) - 1;
constexpr u32 NX_MOD2 = 7u;
struct CompactRecSrc {
    const u32 *sr, *nx;
    const u8 *ch;
    u32 m1;
    using Raw = uint3;  // {SR, NX, CH}
    static constexpr int kMinBlocks = 4;  // k_mod0_window residency (5 measured slower: 1.20 vs 0.83 ms at C3)
    __device__ __forceinline__ Raw fetch(i64 i) const {
        return make_uint3(__ldcs(sr + i), __ldcs(nx + i), (u32)__ldcs(ch + i));
    }
    __device__ __forceinline__ uint4 decode(const Raw &w) const {
        const u32 s = w.x, x = w.y, c = w.z;
        const u32 r = x & NX_MASK;
        const u32 cc = (c & 15u) | ((c >> 4) << 8);
        if (s < m1) return make_uint4(3u * s + 1u, r, 0u, cc | ((x >> 29) << 16));
        return make_uint4(3u * (s - m1) + 2u, 0u, r, cc);
    }
    __device__ __forceinline__ uint4 operator()(i64 i) const { return decode(fetch(i)); }
};
struct CompactMergeView {
    CompactRecSrc a;
    i64 off;  // the padding sample (rank 0) is not a suffix
    const uint4 *B;
    // cached loads: the partition's probes are random, the tile's loads contiguous
    __device__ __forceinline__ uint4 ra(i64 i) const {
        i += off;
        const u32 s = __ldg(a.sr + i), x = __ldg(a.nx + i), c = __ldg(a.ch + i);
        const u32 r = x & NX_MASK;
        const u32 cc = (c & 15u) | ((c >> 4) << 8);
        if (s < a.m1) return make_uint4(3u * s + 1u, r, 0u, cc | ((x >> 29) << 16));
        return make_uint4(3u * (s - a.m1) + 2u, 0u, r, cc);
    }
    __device__ __forceinline__ uint4 rb(i64 j) const { return B[j]; }
};

// pass A of the NX scatter: triplet j -> mod-1 sample 3j+1 and mod-2 sample 3j+2
constexpr int NX_THREADS = 256, NX_J = 4;
__global__ void __launch_bounds__(NX_THREADS, 4)
k_nx_emit(const u8 *__restrict__ t, SampleLayout L, const u32 *__restrict__ isac, PsPlan plan,
          uint2 *__restrict__ stage) {
    extern __shared__ __align__(16) unsigned char smem[];
    uint2 *sh_items = reinterpret_cast<uint2 *>(smem);
    u32 *sh_cnt = reinterpret_cast<u32 *>(sh_items + 2 * NX_THREADS * NX_J);
    u32 *sh_base = sh_cnt + plan.a.buckets;
    const i64 j0 = (i64)blockIdx.x * (NX_THREADS * NX_J);
    uint2 it[2 * NX_J];
    bool ok[2 * NX_J];
    // all loads first (the kernel is load-latency bound), then the items
    u32 a1[NX_J], a2[NX_J], a3[NX_J], cp[NX_J];
#pragma unroll
    for (int r = 0; r < NX_J; r++) {
        const i64 j = j0 + r * NX_THREADS + threadIdx.x;
        a1[r] = j < L.m1 ? __ldcs(isac + j) : 0u;
        a2[r] = j < L.m2 ? __ldg(isac + L.m1 + j) : 0xFFFFFFFFu;
        a3[r] = j + 1 < L.m1 ? __ldg(isac + j + 1) : 0xFFFFFFFFu;
        cp[r] = j < L.m1 ? (u32)__ldg(t + 3 * j) : 0u;
    }
#pragma unroll
    for (int r = 0; r < NX_J; r++) {
        const i64 j = j0 + r * NX_THREADS + threadIdx.x;
        ok[2 * r] = j < L.m1;
        ok[2 * r + 1] = j < L.m2;
        it[2 * r] = make_uint2(a1[r], (a2[r] + 1u) | (cp[r] << 29));        // 0xFFFFFFFF + 1 = 0: no next
        it[2 * r + 1] = make_uint2(a2[r], (a3[r] + 1u) | (NX_MOD2 << 29));
    }
    ps_block_emit<uint2, NX_THREADS, 2 * NX_J>(it, ok, plan.a, stage, sh_items, sh_cnt, sh_base);
}
constexpr size_t NX_EMIT_SMEM = (size_t)2 * NX_THREADS * NX_J * 8 + 8 * PS_MAX_BUCKETS;

// pass B: NX window w (2048 ranks) + its mod-1 samples per cprev digit into
// hist[d * windows + w] (the mod-0 offsets, as k_rs_window)
__global__ void __launch_bounds__(PS_THREADS)
k_nx_window(const uint2 *__restrict__ stage2, PsPlan plan, u32 *__restrict__ nx, u32 *__restrict__ hist, int D1) {
    __shared__ u32 win[1 << RW_SHIFT];
    __shared__ u32 cnt[8];
    const i64 w = blockIdx.x;
    const i64 d0 = w << RW_SHIFT;
    const i64 len = (d0 + (1 << RW_SHIFT) < plan.n_dest ? d0 + (1 << RW_SHIFT) : plan.n_dest) - d0;
    const i64 n_in = plan.cursor2[w];
    const uint2 *src = stage2 + d0;
    if (threadIdx.x < 8) cnt[threadIdx.x] = 0;
    const bool full = n_in == len;
    // a window holds at most 2048 items: all loads of a thread in flight at once
    constexpr int NW_ITEMS = (1 << RW_SHIFT) / PS_THREADS;
    uint2 v[NW_ITEMS];
#pragma unroll
    for (int r = 0; r < NW_ITEMS; r++) {
        const int x = r * PS_THREADS + threadIdx.x;
        if (x < n_in) v[r] = ld_stream(src + x);
    }
#pragma unroll
    for (int r = 0; r < NW_ITEMS; r++) {
        const int x = r * PS_THREADS + threadIdx.x;
        if (x < n_in) {
            if (full) win[(i64)v[r].x - d0] = v[r].y;
            else nx[v[r].x] = v[r].y;
        }
    }
    __syncthreads();
    const int nc = (int)(full ? len : n_in);
    u32 c[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
    for (int r = 0; r < NW_ITEMS; r++) {
        const int x = r * PS_THREADS + threadIdx.x;
        u32 dg = NX_MOD2;
        if (x < nc) {
            const u32 e = full ? win[x] : v[r].y;  // not full: item x is this thread's v[r]
            if (full) st_stream(nx + d0 + x, e);
            dg = e >> 29;
        }
#pragma unroll
        for (int d = 0; d < 7; d++) c[d] += __popc(__ballot_sync(0xffffffffu, dg == (u32)d));
    }
    if (lane_id() == 0)
#pragma unroll
        for (int d = 0; d < 7; d++)
            if (c[d]) atomicAdd(&cnt[d], c[d]);
    __syncthreads();
    for (int d = threadIdx.x; d < D1; d += PS_THREADS) hist[(i64)d * plan.windows + w] = cnt[d];
}

struct HistIn {
    const u32 *h;
    __device__ u32 operator()(i64 i) const { return h[i]; }
};

struct RecMergeView {
    const uint4 *A, *B;
    __device__ __forceinline__ uint4 ra(i64 i) const { return A[i]; }
    __device__ __forceinline__ uint4 rb(i64 j) const { return B[j]; }
};

// record merge tile: 4096 outputs per CTA (one merge-path search per 16
// outputs); shared keys + positions 24 B per output
constexpr int RM_THREADS = 256, RM_ITEMS = 4, RM_TILE = RM_THREADS * RM_ITEMS;

// Split search at every `stride`-th tile boundary (stride = 1: every tile).
// With `coarse` (splits at RM_COARSE x coarser boundaries) each search starts
// inside its coarse window: ~half the probe rounds, and the probes of
// neighbouring tiles share the window's lines.
constexpr int RM_COARSE = 32;
template <class View>
__global__ void k_merge_partition_rec(View v, i64 na, i64 nb, i64 ntiles, u32 *__restrict__ split,
                                      i64 stride, const u32 *__restrict__ coarse) {
    // G lanes per search, 32/G searches per warp: each round probes G+1-ary
    // (fewer random record loads per split than one 33-ary search per warp)
    constexpr int G = 8;
    i64 total = na + nb;
    const int lane = lane_id(), grp = lane / G, sl = lane % G;
    const u32 gmask = ((1u << G) - 1u) << (grp * G);
    i64 groups = ((i64)gridDim.x * blockDim.x) / G;
    i64 nsplit = ceil_div(ntiles, stride);  // boundaries 0 .. nsplit (the last = total)
    const i64 g0 = ((i64)blockIdx.x * blockDim.x + threadIdx.x) / G;
    const i64 rounds = ceil_div(nsplit + 1, groups);
    for (i64 rr = 0; rr < rounds; rr++) {  // warp-uniform trip count (shuffles below)
        const i64 t = g0 + rr * groups;
        const bool act = t <= nsplit;
        i64 d = 0, lo = 0, hi = 0;
        if (act) {
            d = t * stride * RM_TILE < total ? t * stride * RM_TILE : total;
            lo = d > nb ? d - nb : 0;
            hi = d < na ? d : na;
            if (coarse) {
                i64 c = t / RM_COARSE;
                i64 clo = coarse[c], chi = coarse[c + 1 <= ceil_div(ntiles, RM_COARSE) ? c + 1 : c];
                if (clo > lo) lo = clo;
                if (chi < hi && t % RM_COARSE) hi = chi;
                if (t % RM_COARSE == 0) lo = hi = clo;  // a coarse boundary: already known
            }
        }
        bool live = act && lo < hi;
        while (__any_sync(0xffffffffu, live)) {
            const i64 span = hi - lo;
            const i64 x = lo + (span * (sl + 1)) / (G + 1);
            const bool p = live && x < hi && recq_a_first(v.ra(x), v.rb(d - 1 - x));
            const bool f = live && x < hi && !p;
            const u32 tr = (__ballot_sync(0xffffffffu, p) & gmask) >> (grp * G);
            const u32 fl = (__ballot_sync(0xffffffffu, f) & gmask) >> (grp * G);
            const i64 xt = __shfl_sync(0xffffffffu, x, tr ? grp * G + 31 - __clz(tr) : lane);
            const i64 xf = __shfl_sync(0xffffffffu, x, fl ? grp * G + __ffs(fl) - 1 : lane);
            if (live) {
                if (tr) lo = xt + 1;
                if (fl) hi = xf;
                if (span <= G || lo >= hi) live = false;
            }
        }
        if (act && sl == 0) split[t] = (u32)lo;
    }
}

// Comparison keys of the record merge (byte text): a non-sample b gets
//   K1 = c0 << 32 | R(b+1)            (against mod-1 samples)
//   K2 = (c0 << 8 | c1) << 32 | R(b+2) (against mod-2 samples)
// and a sample its own form, mod-2 samples flagged in bit 63; then
// recq_a_first(a, b) == keys_a_first(key(a), K1(b), K2(b)).
constexpr u64 kMod2Flag = 1ull << 63;
__device__ __forceinline__ u64 merge_key1(const uint4 &e) { return ((u64)(e.w & 0xFFu) << 32) | e.y; }
__device__ __forceinline__ u64 merge_key2(const uint4 &e) {
    return ((u64)(((e.w & 0xFFu) << 8) | ((e.w >> 8) & 0xFFu)) << 32) | e.z;
}
__device__ __forceinline__ u64 merge_key_sample(const uint4 &e) {
    if (e.x % 3 == 1) return ((u64)(e.w & 0xFFu) << 32) | e.y;
    u32 c01 = ((e.w & 0xFFu) << 8) | ((e.w >> 8) & 0xFFu);
    return kMod2Flag | ((u64)c01 << 32) | e.z;
}
__device__ __forceinline__ bool keys_a_first(u64 ka, const u64 *B1, const u64 *B2, int j) {
    return (ka & kMod2Flag) ? (ka & ~kMod2Flag) < B2[j] : ka < B1[j];
}

enum { EMIT_NONE = 0, EMIT_ISA = 1, EMIT_PHI = 2 };
constexpr u32 kNoPred = 0xFFFFFFFFu;

// Merge of record runs; MODE selects the bucketed side output:
//   EMIT_ISA  {pos, rank}           -> ISA[pos] = rank
//   EMIT_PHI  {pos, pos of rank-1}  -> Phi[pos]  (kNoPred at rank 0)
template <int MODE, class View>
__global__ void __launch_bounds__(RM_THREADS)
k_merge_tile_rec(View v, i64 na, i64 nb, const u32 *__restrict__ split, u32 *__restrict__ sa, PsPlan plan,
                 uint2 *__restrict__ stage, u32 *__restrict__ isa_direct) {
    // shared tile as comparison keys (merge_key_*) + positions: one 8 B key
    // pair per comparison instead of two 16 B records
    extern __shared__ __align__(16) unsigned char smem[];
    u64 *k1 = reinterpret_cast<u64 *>(smem);
    u64 *k2 = k1 + RM_TILE;
    u32 *pos = reinterpret_cast<u32 *>(k2 + RM_TILE);
    u32 *out = pos + RM_TILE;
    u32 *sh_cnt = out + RM_TILE;
    u32 *sh_base = sh_cnt + plan.a.buckets;
    __shared__ u32 sh_pred;
    i64 total = na + nb;
    i64 d0 = (i64)blockIdx.x * RM_TILE;
    i64 d1 = d0 + RM_TILE < total ? d0 + RM_TILE : total;
    i64 i0 = split[blockIdx.x], i1 = split[blockIdx.x + 1];
    i64 j0 = d0 - i0;
    int nat = (int)(i1 - i0), cnt = (int)(d1 - d0), nbt = cnt - nat;
#pragma unroll
    for (int q = 0; q < RM_ITEMS; q++) {
        int x = threadIdx.x + q * RM_THREADS;
        if (x < cnt) {
            if (x < nat) {
                uint4 e = v.ra(i0 + x);
                k1[x] = merge_key_sample(e);
                pos[x] = e.x;
            } else {
                uint4 e = v.rb(j0 + (x - nat));
                k1[x] = merge_key1(e);
                k2[x] = merge_key2(e);
                pos[x] = e.x;
            }
        }
    }
    if (MODE == EMIT_PHI && threadIdx.x == 0) {
        // the suffix at rank d0-1 is the larger of the two run predecessors
        u32 pr = kNoPred;
        if (d0 > 0) {
            if (i0 == 0) pr = v.rb(j0 - 1).x;
            else if (j0 == 0) pr = v.ra(i0 - 1).x;
            else {
                uint4 a = v.ra(i0 - 1), b = v.rb(j0 - 1);
                pr = recq_a_first(a, b) ? b.x : a.x;
            }
        }
        sh_pred = pr;
    }
    __syncthreads();
    const u64 *B1 = k1 + nat, *B2 = k2 + nat;
    int dt = threadIdx.x * RM_ITEMS;
    if (dt < cnt) {
        int lo = dt > nbt ? dt - nbt : 0, hi = dt < nat ? dt : nat;
        while (lo < hi) {
            int mid = (lo + hi) >> 1;
            if (keys_a_first(k1[mid], B1, B2, dt - 1 - mid)) lo = mid + 1;
            else hi = mid;
        }
        int i = lo, j = dt - lo;
        u32 o[RM_ITEMS];
#pragma unroll
        for (int r = 0; r < RM_ITEMS; r++) {
            o[r] = 0;
            if (dt + r < cnt) {
                bool takeA = j >= nbt || (i < nat && keys_a_first(k1[i], B1, B2, j));
                o[r] = takeA ? pos[i++] : pos[nat + j++];
            }
        }
        static_assert(RM_ITEMS == 4, "one 16-byte store per thread");
        if (dt + RM_ITEMS <= cnt) *reinterpret_cast<uint4 *>(out + dt) = make_uint4(o[0], o[1], o[2], o[3]);
        else
#pragma unroll
            for (int r = 0; r < RM_ITEMS; r++)
                if (dt + r < cnt) out[dt + r] = o[r];
    }
    __syncthreads();
    if (sa)
        for (int x = threadIdx.x; x < cnt; x += RM_THREADS) __stcs(sa + d0 + x, out[x]);
    if (isa_direct)  // small levels: the ISA target is L2-resident
        for (int x = threadIdx.x; x < cnt; x += RM_THREADS) isa_direct[out[x]] = (u32)(d0 + x);
    if (MODE != EMIT_NONE) {
        uint2 it[RM_ITEMS];
        bool ok[RM_ITEMS];
#pragma unroll
        for (int q = 0; q < RM_ITEMS; q++) {
            int x = threadIdx.x + q * RM_THREADS;
            ok[q] = x < cnt;
            if (ok[q]) {
                if (MODE == EMIT_ISA) it[q] = make_uint2(out[x], (u32)(d0 + x));
                else it[q] = make_uint2(out[x], x > 0 ? out[x - 1] : sh_pred);
            }
        }
        ps_block_emit<uint2, RM_THREADS, RM_ITEMS>(it, ok, plan.a, stage, reinterpret_cast<uint2 *>(k1), sh_cnt,
                                                   sh_base);
    }
}

template <int MODE, class View>
static int merge_rec_launch(View v, i64 na, i64 nb, const u32 *split, u32 *sa, const PsPlan &plan,
                            uint2 *stage, cudaStream_t st, u32 *isa_direct = nullptr) {
    static DeviceFlags attr;
    size_t smem = (size_t)RM_TILE * 24 + 8 * (size_t)PS_MAX_BUCKETS;
    if (attr.need()) {
        SAIX_CUDA(cudaFuncSetAttribute(k_merge_tile_rec<MODE, View>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem));
        attr.set();
    }
    size_t use = (size_t)RM_TILE * 24 + 8 * (size_t)(MODE == EMIT_NONE ? 1 : plan.a.buckets);
    k_merge_tile_rec<MODE, View><<<(unsigned)ceil_div(na + nb, RM_TILE), RM_THREADS, use, st>>>(
        v, na, nb, split, sa, plan, stage, isa_direct);
    SAIX_LAUNCHED();
    return SAIX_OK;
}

// all names distinct (bitmap naming): ISAc[s] = name - 1
__global__ void k_isa_from_names(const u32 *__restrict__ tt, i64 m, u32 *__restrict__ isac) {
    for (i64 s = (i64)blockIdx.x * blockDim.x + threadIdx.x; s < m; s += (i64)gridDim.x * blockDim.x)
        isac[s] = __ldcs(tt + s) - 1u;
}

// all names distinct after a sort: SAc = the sorted sample order (streamed
// copy) and ISAc through the bucketed scatter (pass A here)
constexpr int UE_ITEMS = 8;
__global__ void __launch_bounds__(256)
k_unique_emit(const u32 *__restrict__ vals, i64 m, u32 *__restrict__ sac, PsPlan plan, uint2 *__restrict__ stage) {
    extern __shared__ __align__(16) unsigned char ue_smem[];
    uint2 *sh_items = reinterpret_cast<uint2 *>(ue_smem);
    u32 *sh_cnt = reinterpret_cast<u32 *>(sh_items + 256 * UE_ITEMS);
    u32 *sh_base = sh_cnt + plan.a.buckets;
    const i64 r0 = (i64)blockIdx.x * (256 * UE_ITEMS);
    uint2 it[UE_ITEMS];
    bool ok[UE_ITEMS];
#pragma unroll
    for (int q = 0; q < UE_ITEMS; q++) {
        i64 r = r0 + q * 256 + threadIdx.x;
        ok[q] = r < m;
        if (ok[q]) {
            u32 sidx = __ldcs(vals + r);
            if (sac) __stcs(sac + r, sidx);
            it[q] = make_uint2(sidx, (u32)r);
        }
    }
    ps_block_emit<uint2, 256, UE_ITEMS>(it, ok, plan.a, stage, sh_items, sh_cnt, sh_base);
}

inline bool stream_level_ok(int text_bytes, u64 sigma, i64 N, const saix_dc3_probe *probe) {
    return text_bytes == 1 && sigma + 1 <= 256 && probe == nullptr && N < ((i64)3 << 29);
}

// ------------------------------------------------------------ probes

__global__ void k_probe_rank(RankFromIsa R, i64 n3, u32 *__restrict__ out) {
    for (i64 p = (i64)blockIdx.x * blockDim.x + threadIdx.x; p < n3; p += (i64)gridDim.x * blockDim.x)
        out[p] = R(p);
}
__global__ void k_probe_samples(SampleLayout L, const u32 *__restrict__ sac, i64 from,
                                u32 *__restrict__ out) {
    for (i64 r = from + (i64)blockIdx.x * blockDim.x + threadIdx.x; r < L.m; r += (i64)gridDim.x * blockDim.x)
        out[r - from] = (u32)L.pos(sac[r]);
}
__global__ void k_times3(const u32 *__restrict__ in, i64 k, u32 *__restrict__ out) {
    for (i64 j = (i64)blockIdx.x * blockDim.x + threadIdx.x; j < k; j += (i64)gridDim.x * blockDim.x)
        out[j] = 3u * in[j];
}
__global__ void k_iota_pair(u32 *sa, u32 *isa, i64 n) {
    for (i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x) {
        sa[i] = (u32)i;
        if (isa) isa[i] = (u32)i;
    }
}

// ------------------------------------------------------------ driver
// _dc3 (suffix_index.py:381-392) / build_sa_dc3 (395-399): per level, name the
// samples, recurse (_sort_samples, 256-271) unless the names are unique,
// order the non-samples, merge; SuffixArray.from_order (96-101) is the ISA.

constexpr int K_THREADS = 256;
constexpr u64 kBitmapMaxCodes = (u64)1 << 31;

struct Dc3Ctx {
    Arena *ar;
    cudaStream_t st;
    int max_depth;
};

// Level trace of the last saix_dc3 / dc3_compute on this host thread
// (saix_dc3_trace): (N, sigma, m, distinct names) per level, top first.
struct LevelRec {
    i64 n, sigma, m, names;
};
static thread_local std::vector<LevelRec> g_trace;
// level-0 naming of the last DC3 on this thread: 0 triples (+ recursion),
// 1 generic window sort, 2 DNA window sort (wsort.cuh)
static thread_local int g_naming = 0;

// Level-0 window naming switch: SAIX_WINDOW_NAMING=0 or saix_dc3_set_window_naming(0)
// turns it off (the reference recursion runs; A/B measurement and the
// reference level trace for the section 8(d) model)
static int g_window_naming = -1;
static thread_local int g_window_override = -1;
int dc3_window_naming_override(int v) {
    const int old = g_window_override;
    g_window_override = v;
    return old;
}
static bool window_naming_on() {
    if (g_window_override >= 0) return g_window_override != 0;
    if (g_window_naming < 0) {
        const char *e = getenv("SAIX_WINDOW_NAMING");
        g_window_naming = (e && e[0] == '0') ? 0 : 1;
    }
    return g_window_naming != 0;
}

// SAIX_TRACE=1: one stderr line per level (development aid)
static bool trace_on() {
    static int v = [] {
        const char *e = getenv("SAIX_TRACE");
        return e && *e == '1' ? 1 : 0;
    }();
    return v != 0;
}

static bool use_bitmap(u64 sigma, i64 m) {
    u64 s1 = sigma + 1;
    if (s1 >= ((u64)1 << 21)) return false;
    u64 codes = s1 * s1 * s1;
    if (codes > kBitmapMaxCodes) return false;
    u64 words = codes / 32 + 1;
    u64 lim = (u64)(2 * m) > ((u64)1 << 16) ? (u64)(2 * m) : ((u64)1 << 16);
    return words <= lim;
}

static int read_u32(const u32 *d, u32 *h, cudaStream_t st) {
    SAIX_CUDA(cudaMemcpyAsync(h, d, sizeof(u32), cudaMemcpyDeviceToHost, st));
    SAIX_CUDA(cudaStreamSynchronize(st));
    return SAIX_OK;
}

template <typename TT>
static int dc3_level(Dc3Ctx &c, const TT *text, i64 N, u64 sigma, u32 *SA, u32 *ISA,
                     saix_dc3_probe *probe, int depth, u32 *Phi = nullptr, bool *phi_done = nullptr);

// ------------------------------------------------------------ wide-level finish
// (the _sort_nonsamples / _merge steps, suffix_index.py:274-290, 362-378, of a
// u32 level)
//
// A u32 level whose sample triples are all distinct (the deepest level of
// DNA-like texts) gets its merge inputs as records built in sorted order,
// with one random read per item instead of the merge's per-element gathers:
//   RA[r] = {pos, R(pos+1) | R(pos+2), c0, c1} of the sample at rank r, from
//           the bucket-sorted triple keys (chars) and one ISAc read;
//   RB[q] = {3j, R(3j+1), R(3j+2), c0} (+ c1) of the q-th non-sample, from
//           the bucket-sorted (T(3j), R(3j+1)) keys and RA[R(3j+1) - 1] --
//           the mod-1 sample 3j+1, whose record holds R(3j+2) and T(3j+1).
// RA from a sample order (recursion case / wide naming): chars and the
// neighbour rank by two random reads per sample
template <typename TT>
__global__ void k_arec_sa(const u32 *__restrict__ sac, Text<TT> T, SampleLayout L, const u32 *__restrict__ isac,
                          uint4 *__restrict__ ra) {
    for (i64 r = (i64)blockIdx.x * blockDim.x + threadIdx.x; r < L.m; r += (i64)gridDim.x * blockDim.x) {
        u32 sidx = __ldcs(sac + r);
        u32 nb;
        i64 pos;
        if (sidx < L.m1) {
            pos = 3 * (i64)sidx + 1;
            nb = sidx < L.m2 ? isac[L.m1 + sidx] + 1u : 0u;
        } else {
            i64 j = sidx - L.m1;
            pos = 3 * j + 2;
            nb = j + 1 < L.m1 ? isac[j + 1] + 1u : 0u;
        }
        __stcs(ra + r, make_uint4((u32)pos, nb, T(pos), T(pos + 1)));
    }
}

// Wide naming (3 bits(sigma) > 64): bucket sort by the dense pair
// c0 * s1 + c1, then every run of equal pairs (rare: repeats) is ordered by
// c2 in place; runs longer than FR_MAX are reported (caller falls back).
template <typename TT>
struct PairDenseSrc {
    Text<TT> T;
    SampleLayout L;
    u64 s1;
    __device__ __forceinline__ void get(i64 s, u64 &k, u32 &v) const {
        i64 p = L.pos(s);
        k = (u64)T(p) * s1 + T(p + 1);
        v = (u32)s;
    }
    __device__ __forceinline__ u64 dense(u64 k) const { return k; }
};
constexpr int FR_MAX = 64;
template <typename TT>
__global__ void k_fix_runs(const u64 *__restrict__ keys, u32 *__restrict__ vals, i64 m, Text<TT> T, SampleLayout L,
                           u32 *__restrict__ overflow) {
    for (i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x; i + 1 < m; i += (i64)gridDim.x * blockDim.x) {
        u64 k = keys[i];
        if (keys[i + 1] != k || (i > 0 && keys[i - 1] == k)) continue;  // not a run head
        i64 e = i + 2;
        while (e < m && keys[e] == k && e - i <= FR_MAX) e++;
        if (e - i > FR_MAX) {
            atomicMax(overflow, 1u);
            continue;
        }
        u32 v[FR_MAX], c[FR_MAX];
        int len = (int)(e - i);
        for (int x = 0; x < len; x++) {
            v[x] = vals[i + x];
            c[x] = T(L.pos(v[x]) + 2);
        }
        for (int x = 1; x < len; x++) {  // insertion sort by c2
            u32 cv = c[x], vv = v[x];
            int y = x - 1;
            while (y >= 0 && c[y] > cv) {
                c[y + 1] = c[y];
                v[y + 1] = v[y];
                y--;
            }
            c[y + 1] = cv;
            v[y + 1] = vv;
        }
        for (int x = 0; x < len; x++) vals[i + x] = v[x];
    }
}
struct StoreName {
    u32 *names;
    __device__ void operator()(i64 i, u32 excl, u32 v) const { names[i] = excl + v; }
};

__global__ void k_arec(const u64 *__restrict__ keys, const u32 *__restrict__ vals, SampleLayout L, int b,
                       const u32 *__restrict__ isac, uint4 *__restrict__ ra) {
    const u64 cm = ((u64)1 << b) - 1;
    for (i64 r = (i64)blockIdx.x * blockDim.x + threadIdx.x; r < L.m; r += (i64)gridDim.x * blockDim.x) {
        u64 key = __ldcs(keys + r);
        u32 sidx = __ldcs(vals + r);
        u32 nb;
        i64 pos;
        if (sidx < L.m1) {  // mod-1 sample 3s+1: R(3s+2)
            pos = 3 * (i64)sidx + 1;
            nb = sidx < L.m2 ? isac[L.m1 + sidx] + 1u : 0u;
        } else {  // mod-2 sample 3j+2: R(3j+4)
            i64 j = sidx - L.m1;
            pos = 3 * j + 2;
            nb = j + 1 < L.m1 ? isac[j + 1] + 1u : 0u;
        }
        __stcs(ra + r, make_uint4((u32)pos, nb, (u32)(key >> (2 * b)), (u32)((key >> b) & cm)));
    }
}

// Large wide levels: the neighbour ranks reach rank order by the bucketed
// scatter instead of a random ISAc gather per sample -- nbv[s] (sample order,
// streamed reads of ISAc) is scattered to NB[ISAc[s]].
__global__ void k_nb_by_sample(SampleLayout L, const u32 *__restrict__ isac, u32 *__restrict__ nbv) {
    for (i64 sidx = (i64)blockIdx.x * blockDim.x + threadIdx.x; sidx < L.m; sidx += (i64)gridDim.x * blockDim.x) {
        u32 nb;
        if (sidx < L.m1) nb = sidx < L.m2 ? isac[L.m1 + sidx] + 1u : 0u;  // R(3s+2)
        else nb = sidx - L.m1 + 1 < L.m1 ? isac[sidx - L.m1 + 1] + 1u : 0u;  // R(3j+4)
        __stcs(nbv + sidx, nb);
    }
}
__global__ void k_arec_nb(const u64 *__restrict__ keys, const u32 *__restrict__ vals, SampleLayout L, int b,
                          const u32 *__restrict__ nb_by_rank, uint4 *__restrict__ ra) {
    const u64 cm = ((u64)1 << b) - 1;
    for (i64 r = (i64)blockIdx.x * blockDim.x + threadIdx.x; r < L.m; r += (i64)gridDim.x * blockDim.x) {
        u64 key = __ldcs(keys + r);
        u32 sidx = __ldcs(vals + r);
        i64 pos = sidx < L.m1 ? 3 * (i64)sidx + 1 : 3 * (i64)(sidx - L.m1) + 2;
        __stcs(ra + r, make_uint4((u32)pos, __ldcs(nb_by_rank + r), (u32)(key >> (2 * b)), (u32)((key >> b) & cm)));
    }
}

__global__ void k_brec(const u64 *__restrict__ keys, const u32 *__restrict__ vals, i64 k, int rb,
                       const uint4 *__restrict__ ra, uint4 *__restrict__ rb4, u32 *__restrict__ rbc1) {
    const u64 rm = ((u64)1 << rb) - 1;
    for (i64 q = (i64)blockIdx.x * blockDim.x + threadIdx.x; q < k; q += (i64)gridDim.x * blockDim.x) {
        u64 key = __ldcs(keys + q);
        u32 j = __ldcs(vals + q);
        u32 r1 = (u32)(key & rm);
        uint4 e = ra[r1 - 1];  // mod-1 sample 3j+1
        __stcs(rb4 + q, make_uint4(3u * j, r1, e.y, (u32)(key >> rb)));
        __stcs(rbc1 + q, e.z);
    }
}

struct MergeRA {
    const uint4 *A, *B;
    const u32 *Bc1;
    __device__ __forceinline__ MRec reca(i64 i) const {
        uint4 e = A[i];
        MRec m;
        m.pos = e.x;
        m.c0 = e.z;
        if (e.x % 3 == 1) {
            m.c1 = 0;
            m.r1 = e.y;
            m.r2 = 0;
        } else {
            m.c1 = e.w;
            m.r1 = 0;
            m.r2 = e.y;
        }
        return m;
    }
    __device__ __forceinline__ MRec recb(i64 j) const {
        uint4 e = B[j];
        MRec m;
        m.pos = e.x;
        m.c0 = e.w;
        m.c1 = Bc1[j];
        m.r1 = e.y;
        m.r2 = e.z;
        return m;
    }
};

// Wide merge tile on comparison keys (as k_merge_tile_rec): a non-sample b
// holds K1 = c0 << 32 | R(b+1), K2 = c0 << 32 | c1 and R(b+2); a mod-1
// sample its K1 form, a mod-2 sample its K2 form + R(a+2).  1024 outputs per
// CTA, 28 B of shared memory per output.
constexpr int WT_THREADS = 256, WT_ITEMS = 4, WT_TILE = WT_THREADS * WT_ITEMS;
template <int MODE>
__global__ void __launch_bounds__(WT_THREADS)
k_merge_tile_w(MergeRA v, i64 na, i64 nb, const u32 *__restrict__ split, u32 *__restrict__ sa, PsPlan plan,
               uint2 *__restrict__ stage, u32 *__restrict__ isa_direct) {
    extern __shared__ __align__(16) unsigned char smem[];
    u64 *ka = reinterpret_cast<u64 *>(smem);
    u64 *kb = ka + WT_TILE;
    u32 *rr = reinterpret_cast<u32 *>(kb + WT_TILE);
    u32 *pos = rr + WT_TILE;
    u32 *out = pos + WT_TILE;
    u32 *sh_cnt = out + WT_TILE;
    u32 *sh_base = sh_cnt + plan.a.buckets;
    i64 total = na + nb;
    i64 d0 = (i64)blockIdx.x * WT_TILE;
    i64 d1 = d0 + WT_TILE < total ? d0 + WT_TILE : total;
    i64 i0 = split[blockIdx.x], i1 = split[blockIdx.x + 1];
    i64 j0 = d0 - i0;
    int nat = (int)(i1 - i0), cnt = (int)(d1 - d0), nbt = cnt - nat;
#pragma unroll
    for (int q = 0; q < WT_ITEMS; q++) {
        int x = threadIdx.x + q * WT_THREADS;
        if (x < cnt) {
            if (x < nat) {  // RA: {pos, nb, c0, c1}
                uint4 e = v.A[i0 + x];
                pos[x] = e.x;
                if (e.x % 3 == 1) {
                    ka[x] = ((u64)e.z << 32) | e.y;
                } else {
                    ka[x] = ((u64)e.z << 32) | e.w;
                    rr[x] = e.y;
                }
            } else {  // RB: {3j, r1, r2, c0} + c1
                i64 jj = j0 + (x - nat);
                uint4 e = v.B[jj];
                pos[x] = e.x;
                ka[x] = ((u64)e.w << 32) | e.y;
                kb[x] = ((u64)e.w << 32) | v.Bc1[jj];
                rr[x] = e.z;
            }
        }
    }
    __syncthreads();
    auto a_first = [&](int i, int j) -> bool {  // sample i vs non-sample nat + j
        int b = nat + j;
        if (pos[i] % 3 == 1) return ka[i] < ka[b];
        u64 x = ka[i], y = kb[b];
        return x < y || (x == y && rr[i] < rr[b]);
    };
    int dt = threadIdx.x * WT_ITEMS;
    if (dt < cnt) {
        int lo = dt > nbt ? dt - nbt : 0, hi = dt < nat ? dt : nat;
        while (lo < hi) {
            int mid = (lo + hi) >> 1;
            if (a_first(mid, dt - 1 - mid)) lo = mid + 1;
            else hi = mid;
        }
        int i = lo, j = dt - lo;
#pragma unroll
        for (int r = 0; r < WT_ITEMS; r++) {
            if (dt + r >= cnt) break;
            bool takeA = j >= nbt || (i < nat && a_first(i, j));
            out[dt + r] = takeA ? pos[i++] : pos[nat + j++];
        }
    }
    __syncthreads();
    if (sa)
        for (int x = threadIdx.x; x < cnt; x += WT_THREADS) __stcs(sa + d0 + x, out[x]);
    if (isa_direct)
        for (int x = threadIdx.x; x < cnt; x += WT_THREADS) isa_direct[out[x]] = (u32)(d0 + x);
    if (MODE == EMIT_ISA) {
        uint2 it[WT_ITEMS];
        bool ok[WT_ITEMS];
#pragma unroll
        for (int q = 0; q < WT_ITEMS; q++) {
            int x = threadIdx.x + q * WT_THREADS;
            ok[q] = x < cnt;
            if (ok[q]) it[q] = make_uint2(out[x], (u32)(d0 + x));
        }
        ps_block_emit<uint2, WT_THREADS, WT_ITEMS>(it, ok, plan.a, stage, reinterpret_cast<uint2 *>(ka), sh_cnt,
                                                   sh_base);
    }
}

template <typename TT>
static int dc3_wide_finish(Dc3Ctx &c, Text<TT> T, const SampleLayout &L, u64 sigma, const u32 *ISAc,
                           const uint4 *RA, u32 *SA, u32 *ISA, bool &fin) {
    Arena &ar = *c.ar;
    cudaStream_t st = c.st;
    fin = false;
    const i64 m = L.m, k = L.k, N = L.n;
    size_t mark = ar.mark();
    int rbm = bits_for((u64)m);
    u64 mk = ((u64)sigma << rbm) | (u64)m;
    if (bits_for(sigma) + rbm > 64) return SAIX_OK;
    // mod-0 order: bucket sort of (T(3j), R(3j+1))
    uint4 *RB = ar.alloc<uint4>(k);
    u32 *RBc1 = ar.alloc<u32>(k);
    size_t mark_b = ar.mark();
    u64 *k64 = ar.alloc<u64>(k);
    u32 *v0 = ar.alloc<u32>(k);
    u32 *scratch = ar.alloc<u32>(bs_scratch_words(N / 8 + 2));
    SAIX_ARENA_OK(ar);
    bool ok = false;
    SAIX_TRY(bucket_sort(Mod0BucketSrc<TT>{T, ISAc, rbm, (u64)m + 1}, k, sigma * ((u64)m + 1) + m, k64, v0, scratch,
                         ok, st, "dc3.mod0_split", &ar));
    if (!ok) {
        ar.reset(mark);
        return SAIX_OK;
    }
    {
        Prof prof_("dc3.brec", 12.0 * k + 16.0 * k + 20.0 * k, st);
        k_brec<<<grid_for(k, 256), 256, 0, st>>>(k64, v0, k, rbm, RA, RB, RBc1);
    }
    SAIX_LAUNCHED();
    ar.reset(mark_b);
    // merge
    i64 pad = L.pad ? 1 : 0;
    i64 na = m - pad, total = na + k;
    MergeRA V{RA + pad, RB, RBc1};
    i64 ntiles = ceil_div(total, WT_TILE);
    u32 *split = ar.alloc<u32>(ntiles + 2);
    u32 *coarse = ar.alloc<u32>(ceil_div(ntiles, 32) + 2);
    u32 *isa_direct = (ISA && total < 2 * kDirectScatterItems) ? ISA : nullptr;
    if (isa_direct) ISA = nullptr;  // written by the tiles directly
    PsPlan pm = PsPlan::of(ISA ? total : 1, 4);
    pm.set_cursors(ar.alloc<u32>(pm.cursor_words()));
    uint2 *pst1 = ISA ? ar.alloc<uint2>(pm.stage1_items()) : nullptr;
    uint2 *pst2 = ISA ? ar.alloc<uint2>(pm.stage2_items()) : nullptr;
    SAIX_ARENA_OK(ar);
    SAIX_CUDA(cudaMemsetAsync(pm.a.cursor, 0, (size_t)pm.cursor_words() * 4, st));
    {
        Prof prof_("dc3.merge_partition", 32.0 * (ntiles + 1), st);
        i64 nc = ceil_div(ntiles, 32);
        k_merge_partition<MergeRA, WT_TILE><<<grid_for((nc + 1) * 32, 128), 128, 0, st>>>(V, na, k, ntiles, coarse, 32,
                                                                                          nullptr);
        SAIX_LAUNCHED();
        k_merge_partition<MergeRA, WT_TILE><<<grid_for((ntiles + 1) * 32, 128), 128, 0, st>>>(V, na, k, ntiles, split,
                                                                                             1, coarse);
    }
    SAIX_LAUNCHED();
    {
        Prof prof_("dc3.merge_tile", 16.0 * na + 20.0 * k + (SA ? 4.0 * total : 0) + (ISA ? 8.0 * total : 0), st);
        static DeviceFlags attr;
        size_t smax = (size_t)WT_TILE * 28 + 8 * (size_t)PS_MAX_BUCKETS;
        if (attr.need()) {
            SAIX_CUDA(cudaFuncSetAttribute(k_merge_tile_w<EMIT_ISA>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)smax));
            SAIX_CUDA(cudaFuncSetAttribute(k_merge_tile_w<EMIT_NONE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)smax));
            attr.set();
        }
        size_t smem = (size_t)WT_TILE * 28 + 8 * (size_t)(ISA ? pm.a.buckets : 1);
        if (ISA)
            k_merge_tile_w<EMIT_ISA><<<(unsigned)ntiles, WT_THREADS, smem, st>>>(V, na, k, split, SA, pm, pst1, nullptr);
        else
            k_merge_tile_w<EMIT_NONE><<<(unsigned)ntiles, WT_THREADS, smem, st>>>(V, na, k, split, SA, pm, pst1,
                                                                                  isa_direct);
    }
    SAIX_LAUNCHED();
    if (ISA) SAIX_TRY(ps_finish(pst1, pst2, pm, U32Apply{ISA}, st, "dc3.isa_apply", 28.0 * total));
    ar.reset(mark);
    fin = true;
    return SAIX_OK;
}

static int dc3_level_stream(Dc3Ctx &c, const u8 *text, i64 N, u64 sigma, u32 *SA, u32 *ISA, u32 *Phi,
                            bool *phi_done, int depth);

// ------------------------------------------------------------ tie resolution
// (replaces the recursion of _sort_samples, suffix_index.py:256-271, when only
// a few sample names repeat; the order is the one the recursion returns)
//
// When a level's sample names are almost all distinct (m - names <= m/32;
// e.g. the deep levels of DNA pairs with planted repeats), the recursion
// would re-run a full DC3 level only to order the few samples that share a
// name.  Those ties are resolved instead by prefix doubling on the recursion
// string R = tt (whose suffix order is exactly what the recursion returns,
// suffix_index.py:256-271): G[s] = head of s's group in the sorted order;
// each round sorts every tied group by G[s + h] (0 past the end) and splits
// it, h doubling, until all groups are singletons -- then G = ISAc and the
// sorted order = SAc.  Work is proportional to the tied samples only.
struct EqPacked {
    const u64 *keys;
    __device__ __forceinline__ bool operator()(i64 a, i64 b) const { return keys[a] == keys[b]; }
};
template <typename TT>
struct EqWide {  // (c0, c1) dense key + third character
    Text<TT> T;
    SampleLayout L;
    const u64 *keys;
    const u32 *vals;
    __device__ __forceinline__ bool operator()(i64 a, i64 b) const {
        return keys[a] == keys[b] && T(L.pos(vals[a]) + 2) == T(L.pos(vals[b]) + 2);
    }
};
constexpr i64 TIE_MAX_RUN = 4096;

template <class Eq>
__global__ void k_tie_init(Eq eq, i64 m, u32 *__restrict__ head, u32 *__restrict__ rs, u32 *__restrict__ rl,
                           u32 *__restrict__ nruns, u32 cap, u32 *__restrict__ overflow) {
    for (i64 r = (i64)blockIdx.x * blockDim.x + threadIdx.x; r < m; r += (i64)gridDim.x * blockDim.x) {
        i64 h = r;
        while (h > 0 && r - h <= TIE_MAX_RUN && eq(h - 1, h)) h--;
        if (r - h > TIE_MAX_RUN) {
            atomicMax(overflow, 1u);
            h = r;
        }
        head[r] = (u32)h;
        if (h == r && r + 1 < m && eq(r, r + 1)) {  // head of a tied group
            i64 e = r + 2;
            while (e < m && e - r <= TIE_MAX_RUN && eq(r, e)) e++;
            u32 at = atomicAdd(nruns, 1u);
            if (at < cap) {
                rs[at] = (u32)r;
                rl[at] = (u32)(e - r);
            } else {
                atomicMax(overflow, 1u);
            }
        }
    }
}

// one thread per run: doubling key of every member (G read only)
__global__ void k_tie_keys(const u32 *__restrict__ rs, const u32 *__restrict__ rl, const u32 *__restrict__ nruns,
                           const u32 *__restrict__ S, const u32 *__restrict__ G, i64 m, i64 h, u64 *__restrict__ kk) {
    const u32 nr = *nruns;
    for (u32 q = (u32)((i64)blockIdx.x * blockDim.x + threadIdx.x); q < nr; q += gridDim.x * blockDim.x) {
        u32 s0 = rs[q], len = rl[q];
        for (u32 x = s0; x < s0 + len; x++) {
            i64 sidx = (i64)S[x] + h;
            kk[x] = sidx < m ? (u64)G[sidx] + 1u : 0ull;
        }
    }
}

// runs of 33..4096 members for the shared-memory sorts
__global__ void k_tie_lists(const u32 *__restrict__ rl, const u32 *__restrict__ nruns, u32 *__restrict__ mid,
                            u32 *__restrict__ big, u32 *__restrict__ scal) {
    const u32 nr = *nruns;
    for (u32 q = (u32)((i64)blockIdx.x * blockDim.x + threadIdx.x); q < nr; q += gridDim.x * blockDim.x) {
        u32 len = rl[q];
        if (len > BS_SMALL) big[atomicAdd(&scal[1], 1u)] = q;
        else if (len > BS_TINY) mid[atomicAdd(&scal[0], 1u)] = q;
    }
}

// split every sorted run where the key changes: members get their sub-run's
// head as group id; sub-runs of > 1 member go to the next round's list
__global__ void k_tie_split(const u32 *__restrict__ rs, const u32 *__restrict__ rl, const u32 *__restrict__ nruns,
                            const u32 *__restrict__ S, const u64 *__restrict__ kk, u32 *__restrict__ G,
                            u32 *__restrict__ rs2, u32 *__restrict__ rl2, u32 *__restrict__ nruns2) {
    const u32 nr = *nruns;
    for (u32 q = (u32)((i64)blockIdx.x * blockDim.x + threadIdx.x); q < nr; q += gridDim.x * blockDim.x) {
        u32 s0 = rs[q], e = s0 + rl[q];
        u32 sub = s0;
        for (u32 x = s0; x < e; x++) {
            if (x > s0 && kk[x] != kk[x - 1]) {
                if (x - sub > 1) {
                    u32 at = atomicAdd(nruns2, 1u);
                    rs2[at] = sub;
                    rl2[at] = x - sub;
                }
                sub = x;
            }
            G[S[x]] = sub;
        }
        if (e - sub > 1) {
            u32 at = atomicAdd(nruns2, 1u);
            rs2[at] = sub;
            rl2[at] = e - sub;
        }
    }
}

// One pass over sorted keys: distinct count and the tied runs (head, length)
// of <= TIE_MAX_RUN members (longer runs or more than cap -> overflow)
__global__ void k_count_runs(const u64 *__restrict__ keys, i64 m, u32 *__restrict__ count, u32 *__restrict__ rs,
                             u32 *__restrict__ rl, u32 *__restrict__ nruns, u32 cap, u32 *__restrict__ overflow) {
    u32 c = 0;
    for (i64 r = (i64)blockIdx.x * blockDim.x + threadIdx.x; r < m; r += (i64)gridDim.x * blockDim.x) {
        const u64 k = keys[r];
        const bool head = r == 0 || keys[r - 1] != k;
        c += head;
        if (head && r + 1 < m && keys[r + 1] == k) {
            i64 e = r + 2;
            while (e < m && e - r <= TIE_MAX_RUN && keys[e] == k) e++;
            if (e - r > TIE_MAX_RUN) {
                atomicMax(overflow, 1u);
                continue;
            }
            const u32 at = atomicAdd(nruns, 1u);
            if (at < cap) {
                rs[at] = (u32)r;
                rl[at] = (u32)(e - r);
            } else {
                atomicMax(overflow, 1u);
            }
        }
    }
    for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if (lane_id() == 0 && c) atomicAdd(count, c);
}
// members of every tied run take the run head as group id
__global__ void k_tie_groups(const u32 *__restrict__ rs, const u32 *__restrict__ rl, const u32 *__restrict__ nruns,
                             const u32 *__restrict__ S, u32 *__restrict__ G) {
    const u32 nr = *nruns;
    for (u32 q = (u32)((i64)blockIdx.x * blockDim.x + threadIdx.x); q < nr; q += gridDim.x * blockDim.x) {
        const u32 s0 = rs[q], len = rl[q];
        for (u32 x = s0 + 1; x < s0 + len; x++) G[S[x]] = s0;
    }
}

// Prefix-doubling rounds over the tied runs (rsA/rlA, nr0 of them; G holds
// every sample's group id = its run head or its own rank): each round keys
// the members by G[s + h], sorts every run, and splits it where keys change.
static int tie_rounds(Dc3Ctx &c, i64 m, i64 ties, u32 *S, u64 *kk, u32 *ISAc, u32 *rsA, u32 *rlA, u32 *rsB,
                      u32 *rlB, u32 *mid, u32 *big, u32 *scal, u32 nr0) {
    cudaStream_t st = c.st;
    u32 nr = nr0;
    u32 *rs = rsA, *rl = rlA, *rs2 = rsB, *rl2 = rlB;
    u32 *cnt_cur = scal + 2, *cnt_next = scal + 3;
    Prof prof_("dc3.tie_resolve", 24.0 * ties, st);
    for (i64 h = 1; nr > 0; h <<= 1) {
        if (h > 2 * m) {
            set_error("dc3: tie resolution did not converge");
            return SAIX_EINVAL;
        }
        int g = grid_for(nr, 128);
        k_tie_keys<<<g, 128, 0, st>>>(rs, rl, cnt_cur, S, ISAc, m, h, kk);
        SAIX_LAUNCHED();
        // sort every run by its key (runs are buckets for the bucket-sort kernels)
        k_bs_tiny<<<grid_for(ceil_div(nr, 32) * 32, 256, kNumSMs * 16), 256, 0, st>>>(rs, rl, nr, kk, S);
        SAIX_LAUNCHED();
        SAIX_CUDA(cudaMemsetAsync(scal, 0, 8, st));
        k_tie_lists<<<g, 128, 0, st>>>(rl, cnt_cur, mid, big, scal);
        SAIX_LAUNCHED();
        u32 hl[2];
        SAIX_CUDA(cudaMemcpyAsync(hl, scal, 8, cudaMemcpyDeviceToHost, st));
        SAIX_CUDA(cudaStreamSynchronize(st));
        if (hl[0]) {
            static DeviceFlags attr;
            if (attr.need()) {
                SAIX_CUDA(cudaFuncSetAttribute(k_bs_small, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                               (int)BS_SMALL_SMEM));
                attr.set();
            }
            u32 blocks = (hl[0] + BS_WARPS - 1) / BS_WARPS;
            k_bs_small<<<blocks < 2 * kNumSMs ? blocks : 2 * kNumSMs, 32 * BS_WARPS, BS_SMALL_SMEM, st>>>(
                rs, rl, mid, scal, kk, S);
            SAIX_LAUNCHED();
        }
        if (hl[1]) {
            static DeviceFlags attr;
            size_t smem = (size_t)BS_LARGE * 12;
            if (attr.need()) {
                SAIX_CUDA(cudaFuncSetAttribute(k_bs_large, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
                attr.set();
            }
            k_bs_large<<<hl[1] < 4 * kNumSMs ? hl[1] : 4 * kNumSMs, 256, smem, st>>>(rs, rl, big, scal + 1, kk, S);
            SAIX_LAUNCHED();
        }
        SAIX_CUDA(cudaMemsetAsync(cnt_next, 0, 4, st));
        k_tie_split<<<g, 128, 0, st>>>(rs, rl, cnt_cur, S, kk, ISAc, rs2, rl2, cnt_next);
        SAIX_LAUNCHED();
        SAIX_CUDA(cudaMemcpyAsync(&nr, cnt_next, 4, cudaMemcpyDeviceToHost, st));
        SAIX_CUDA(cudaStreamSynchronize(st));
        u32 *t;
        t = rs; rs = rs2; rs2 = t;
        t = rl; rl = rl2; rl2 = t;
        t = cnt_cur; cnt_cur = cnt_next; cnt_next = t;
    }
    return SAIX_OK;
}

// Resolve the tied groups of the sorted samples (keys/S from the naming sort)
// into ISAc (and SAc when asked).  ok = false: too many / too long ties, the
// caller recurses instead (nothing has been written to ISAc / SAc then).
template <class Eq>
static int resolve_ties(Dc3Ctx &c, Eq eq, i64 m, i64 ties, u32 *S, u64 *kk, u32 *SAc, u32 *ISAc, bool &ok) {
    Arena &ar = *c.ar;
    cudaStream_t st = c.st;
    ok = false;
    size_t mark = ar.mark();
    u32 cap = (u32)(ties + 64);
    u32 *head = ar.alloc<u32>(m);
    u32 *rsA = ar.alloc<u32>(cap), *rlA = ar.alloc<u32>(cap), *rsB = ar.alloc<u32>(cap), *rlB = ar.alloc<u32>(cap);
    u32 *mid = ar.alloc<u32>(cap), *big = ar.alloc<u32>(cap);
    u32 *scal = ar.alloc<u32>(16);  // [0] mid, [1] big, [2] runs A, [3] runs B, [4] overflow
    SAIX_ARENA_OK(ar);
    SAIX_CUDA(cudaMemsetAsync(scal, 0, 16 * 4, st));
    {
        Prof prof_("dc3.tie_resolve", 8.0 * m, st);
        k_tie_init<Eq><<<grid_for(m, 256), 256, 0, st>>>(eq, m, head, rsA, rlA, scal + 2, cap, scal + 4);
    }
    SAIX_LAUNCHED();
    u32 h2[3];
    SAIX_CUDA(cudaMemcpyAsync(h2, scal + 2, 12, cudaMemcpyDeviceToHost, st));
    SAIX_CUDA(cudaStreamSynchronize(st));
    if (h2[2]) {
        ar.reset(mark);
        return SAIX_OK;
    }
    // G[S[r]] = head(r): the (mostly unique) group ids through the bucketed scatter
    SAIX_TRY(scatter_u32(ar, S, head, m, m, ISAc, st, "dc3.tie_scatter"));
    SAIX_TRY(tie_rounds(c, m, ties, S, kk, ISAc, rsA, rlA, rsB, rlB, mid, big, scal, h2[0]));
    if (SAc) SAIX_CUDA(cudaMemcpyAsync(SAc, S, (size_t)m * 4, cudaMemcpyDeviceToDevice, st));
    ar.reset(mark);
    ok = true;
    return SAIX_OK;
}

// RA (sample records in rank order) from the sorted triple keys: neighbour
// ranks gathered (small levels) or scattered to rank order (large levels)
static int build_ra(Dc3Ctx &c, const u64 *keys, const u32 *vals, const SampleLayout &L, int kbits, const u32 *ISAc,
                    uint4 *RA) {
    Arena &ar = *c.ar;
    cudaStream_t st = c.st;
    const i64 m = L.m;
    if (m < kDirectScatterItems) {
        Prof prof_("dc3.arec", 36.0 * m, st);
        k_arec<<<grid_for(m, 256), 256, 0, st>>>(keys, vals, L, kbits, ISAc, RA);
        SAIX_LAUNCHED();
        return SAIX_OK;
    }
    size_t mark = ar.mark();
    u32 *nbv = ar.alloc<u32>(m), *nbr = ar.alloc<u32>(m);
    SAIX_ARENA_OK(ar);
    {
        Prof prof_("dc3.arec", 16.0 * m, st);
        k_nb_by_sample<<<grid_for(m, 256), 256, 0, st>>>(L, ISAc, nbv);
    }
    SAIX_LAUNCHED();
    SAIX_TRY(scatter_u32(ar, ISAc, nbv, m, m, nbr, st, "dc3.nb_scatter"));
    {
        Prof prof_("dc3.arec", 32.0 * m, st);
        k_arec_nb<<<grid_for(m, 256), 256, 0, st>>>(keys, vals, L, kbits, nbr, RA);
    }
    SAIX_LAUNCHED();
    ar.reset(mark);
    return SAIX_OK;
}

// Steps 1-2: names of the sample triples, then SAc/ISAc (recursing if needed).
template <typename TT>
static int sort_samples(Dc3Ctx &c, Text<TT> T, const SampleLayout &L, u64 sigma, u32 *tt,
                        u32 *SAc, u32 *ISAc, u32 *d_scal, int depth, bool keep_u32, uint4 **RA_out) {
    Arena &ar = *c.ar;
    cudaStream_t st = c.st;
    size_t mark = ar.mark();
    i64 m = L.m;
    int g = grid_for(m, K_THREADS);
    u32 D = 0;
    bool narrow = false;  // recursion string stored as u8
    u32 *sorted_vals = nullptr;
    u64 *sorted_keys = nullptr;
    bool bsorted = false;  // keys are shift-packed triples (bucket sort)
    int kbits = 0;
    bool wide_names = false;                        // keys hold (c0, c1) only; c2 from the text
    u64 *k0_keep = nullptr, *k1_keep = nullptr;     // the sort's key buffers (tie resolution scratch)
    bool keep_arena = false;  // RA built: the caller releases the sort temps
    if (RA_out) *RA_out = nullptr;
    if (use_bitmap(sigma, m)) {
        u64 s1 = sigma + 1;
        u64 codes = s1 * s1 * s1;
        u32 nwords = (u32)(codes / 32 + 1);
        u32 *bm = ar.alloc<u32>(nwords);
        u32 *wp = ar.alloc<u32>(nwords);
        u32 *tmp = ar.alloc<u32>(scan_tmp_words(nwords));
        SAIX_ARENA_OK(ar);
        SAIX_CUDA(cudaMemsetAsync(bm, 0, (size_t)nwords * 4, st));
        // private bitmap in shared memory when it fits beside the kernels' 6 KB
        // text tile under the default 48 KB dynamic + static limit
        int use_smem = nwords * 4 <= 40 * 1024;
        // tiny bitmaps (level 0: <= 216 codes) merge cheaply from every CTA;
        // larger ones are privatised in fewer, longer-lived CTAs
        int gs = (use_smem && nwords > 1024) ? (g < 2 * kNumSMs ? g : 2 * kNumSMs) : g;
        {
            Prof prof_("dc3.bitmap_set", (double)sizeof(TT) * L.n, st);
            if (sizeof(TT) == 1 && ((uintptr_t)T.t & 3) == 0) {
                i64 gt = ceil_div(L.m1 > 0 ? L.m1 : 1, TT_TILE);
                i64 gcap = (use_smem && nwords > 1024) ? 2 * kNumSMs : 8 * kNumSMs;  // few long-lived CTAs
                if (gt > gcap) gt = gcap;
                k_bitmap_set_u8<<<(unsigned)gt, 256, use_smem ? nwords * 4 : 0, st>>>((const u8 *)T.t, L, s1, bm,
                                                                                     nwords, use_smem);
            } else {
                k_bitmap_set<TT><<<gs, K_THREADS, use_smem ? nwords * 4 : 0, st>>>(T, L, s1, bm, nwords, use_smem);
            }
        }
        SAIX_LAUNCHED();
        SAIX_TRY(scan_transform(PopcIn{bm}, StoreExcl{wp}, nwords, tmp, d_scal, st, "dc3.bitmap_scan", 8.0 * nwords));
        SAIX_TRY(read_u32(d_scal, &D, st));
        narrow = !keep_u32 && D <= 255 && (i64)D < m;
        {
            Prof prof_("dc3.bitmap_name", (double)sizeof(TT) * L.n + (narrow ? 1.0 : 4.0) * m, st);
            if (sizeof(TT) == 1 && ((uintptr_t)T.t & 3) == 0) {
                unsigned gt = (unsigned)ceil_div(L.m1 > 0 ? L.m1 : 1, TT_TILE);
                if (narrow) k_bitmap_name_u8<u8><<<gt, 256, 0, st>>>((const u8 *)T.t, L, s1, bm, wp, (u8 *)tt);
                else k_bitmap_name_u8<u32><<<gt, 256, 0, st>>>((const u8 *)T.t, L, s1, bm, wp, tt);
            } else if (narrow) {
                k_bitmap_name<TT, u8><<<g, K_THREADS, 0, st>>>(T, L, s1, bm, wp, (u8 *)tt);
            } else {
                k_bitmap_name<TT, u32><<<g, K_THREADS, 0, st>>>(T, L, s1, bm, wp, tt);
            }
        }
        SAIX_LAUNCHED();
    } else {
        int b = bits_for(sigma);
        u64 *k0 = ar.alloc<u64>(m), *k1 = ar.alloc<u64>(m);
        u32 *v0 = ar.alloc<u32>(m), *v1 = ar.alloc<u32>(m);
        u32 *scratch = ar.alloc<u32>(os_scratch_words(m) > bs_scratch_words(L.n / 8 + 2) ? os_scratch_words(m)
                                                                                  : bs_scratch_words(L.n / 8 + 2));
        u32 *tmp = ar.alloc<u32>(scan_tmp_words(m));
        SAIX_ARENA_OK(ar);
        u64 *keys = k0;
        u32 *vals = v0;
        k0_keep = k0;
        k1_keep = k1;
        if (3 * b <= 64) {
            u64 s1 = sigma + 1;
            int kb = bits_for(s1 * s1 * s1 - 1);
            int passes = (kb + OS_BITS - 1) / OS_BITS;
            TripleSrc<TT> src{T, L, s1};
            bool done = false;
            u64 bmax = (sigma << (2 * b)) | (sigma << b) | sigma;
            if (use_bsort(bmax, m)) {
                SAIX_TRY(bucket_sort(TripleBucketSrc<TT>{T, L, b, s1}, m, sigma * s1 + sigma, k0, v0, scratch, done,
                                     st, "dc3.triple_sort", &ar));
                bsorted = done;
                keys = k0;
                vals = v0;
            }
            if (!done)
                SAIX_TRY(onesweep_sort<u64>(src, m, src, m, m, 0, passes, k0, v0, k1, v1, scratch, keys, vals,
                                            nullptr, st, "dc3.triple_sort"));
            // count distinct triples first: when all are distinct (the last
            // recursion level) the sorted order already is the rank order and
            // the recursion string is never needed
            SAIX_CUDA(cudaMemsetAsync(d_scal, 0, sizeof(u32), st));
            {
                Prof prof_("dc3.count_names", 8.0 * m, st);
                k_count_distinct<<<grid_for(m, K_THREADS, kNumSMs * 8), K_THREADS, 0, st>>>(keys, m, d_scal);
            }
            SAIX_LAUNCHED();
            SAIX_TRY(read_u32(d_scal, &D, st));
            if ((i64)D < m || keep_u32) {
                u32 *names = reinterpret_cast<u32 *>(keys == k0 ? k1 : k0);
                SAIX_TRY(scan_transform(FlagPacked{keys}, StoreName{names}, m, tmp, nullptr, st, "dc3.name_scan",
                                        16.0 * m));
                SAIX_TRY(scatter_u32(ar, vals, names, m, m, tt, st, "dc3.name_scatter"));
            }
        } else {
            // wide alphabet: bucket sort by (c0, c1), repeats ordered by c2
            wide_names = true;
            u64 s1 = sigma + 1;
            bool done = false;
            if (sigma < ((u64)1 << 32) && m >= 4096) {
                SAIX_TRY(bucket_sort(PairDenseSrc<TT>{T, L, s1}, m, sigma * s1 + sigma, k0, v0, scratch, done, st,
                                     "dc3.triple_sort", &ar));
                if (done) {
                    SAIX_CUDA(cudaMemsetAsync(d_scal, 0, sizeof(u32), st));
                    {
                        Prof prof_("dc3.fix_runs", 12.0 * m, st);
                        k_fix_runs<TT><<<grid_for(m, 256), 256, 0, st>>>(k0, v0, m, T, L, d_scal);
                    }
                    SAIX_LAUNCHED();
                    u32 of = 0;
                    SAIX_TRY(read_u32(d_scal, &of, st));
                    done = of == 0;
                    keys = k0;
                    vals = v0;
                }
            }
            if (!done) {
                // LSD over components: stably by the third character, then by
                // the mixed-radix pair of the first two
                ThirdSrc<TT> src1{T, L};
                SAIX_TRY(onesweep_sort<u64>(src1, m, src1, m, m, 0, (b + OS_BITS - 1) / OS_BITS, k0, v0, k1, v1,
                                            scratch, keys, vals, nullptr, st, "dc3.triple_sort"));
                PairGatherSrc<TT> src2{T, L, vals, s1};
                PairStreamSrc<TT> hsrc2{T, L, s1};
                int kb2 = bits_for(s1 * s1 - 1);
                u64 *ok0 = keys == k0 ? k1 : k0;  // pass 0 must not overwrite its source
                u32 *ov0 = vals == v0 ? v1 : v0;
                SAIX_TRY(onesweep_sort<u64>(src2, m, hsrc2, m, m, 0, (kb2 + OS_BITS - 1) / OS_BITS, ok0, ov0, keys,
                                            vals, scratch, keys, vals, nullptr, st, "dc3.triple_sort"));
            }
            // names in sorted order (into the free key buffer), then scattered
            u32 *names = reinterpret_cast<u32 *>(keys == k0 ? k1 : k0);
            SAIX_TRY(scan_transform(FlagWide<TT>{T, L, keys, vals}, StoreName{names}, m, tmp, d_scal, st,
                                    "dc3.name_scan", 24.0 * m));
            SAIX_TRY(read_u32(d_scal, &D, st));
            if ((i64)D < m || keep_u32) SAIX_TRY(scatter_u32(ar, vals, names, m, m, tt, st, "dc3.name_scatter"));
        }
        sorted_vals = vals;
        sorted_keys = keys;
        kbits = b;
    }
    if ((size_t)depth >= g_trace.size()) g_trace.resize((size_t)depth + 1);
    g_trace[(size_t)depth] = LevelRec{L.n, (i64)sigma, m, (i64)D};
    if (trace_on())
        fprintf(stderr, "[saix dc3] depth %d: N=%lld text=u%d sigma=%llu m=%lld names=%u naming=%s%s\n", depth,
                (long long)L.n, (int)sizeof(TT) * 8, (unsigned long long)sigma, (long long)m, D,
                sorted_vals ? (bsorted ? "bucket-sort" : "radix") : "bitmap", (i64)D == m ? " (unique)" : "");
    if ((i64)D == m) {
        if (sorted_vals && m >= kDirectScatterItems) {
            PsPlan pu = PsPlan::of(m, 4);
            pu.set_cursors(ar.alloc<u32>(pu.cursor_words()));
            uint2 *s1 = ar.alloc<uint2>(pu.stage1_items()), *s2 = ar.alloc<uint2>(pu.stage2_items());
            SAIX_ARENA_OK(ar);
            SAIX_CUDA(cudaMemsetAsync(pu.a.cursor, 0, (size_t)pu.cursor_words() * 4, st));
            {
                Prof prof_("dc3.unique_ranks", (SAc ? 16.0 : 12.0) * m, st);
                static DeviceFlags attr;
                if (attr.need()) {
                    SAIX_CUDA(cudaFuncSetAttribute(k_unique_emit, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                   256 * UE_ITEMS * 8 + 8 * PS_MAX_BUCKETS));
                    attr.set();
                }
                size_t smem = (size_t)256 * UE_ITEMS * 8 + 8 * (size_t)pu.a.buckets;
                k_unique_emit<<<(unsigned)ceil_div(m, 256 * UE_ITEMS), 256, smem, st>>>(sorted_vals, m, SAc, pu, s1);
            }
            SAIX_LAUNCHED();
            SAIX_TRY(ps_finish(s1, s2, pu, U32Apply{ISAc}, st, "dc3.unique_isa", 28.0 * m));
        } else {
            Prof prof_("dc3.unique_ranks", 12.0 * m, st);
            if (sorted_vals) k_unique_from_sorted<<<g, K_THREADS, 0, st>>>(sorted_vals, m, SAc, ISAc);
            else if (SAc) k_unique_from_names<<<g, K_THREADS, 0, st>>>(tt, m, SAc, ISAc);
            else k_isa_from_names<<<g, K_THREADS, 0, st>>>(tt, m, ISAc);
            SAIX_LAUNCHED();
        }
        if (RA_out && bsorted) {
            // the wide-level finish (dc3_wide_finish) merges from sample
            // records in rank order: build them while the keys are alive
            uint4 *RA = ar.alloc<uint4>(m);
            SAIX_ARENA_OK(ar);
            SAIX_TRY(build_ra(c, sorted_keys, sorted_vals, L, kbits, ISAc, RA));
            *RA_out = RA;
            keep_arena = true;
        }
        if (!keep_arena) ar.reset(mark);
    } else {
        bool resolved = false;
        if (sorted_vals && !keep_u32 && m >= 4096 && (i64)(m - D) <= m / 32) {
            // almost all names distinct: order the tied samples by prefix
            // doubling instead of a full recursion level
            u64 *kk = sorted_keys == k0_keep ? k1_keep : k0_keep;
            if (wide_names)
                SAIX_TRY(resolve_ties(c, EqWide<TT>{T, L, sorted_keys, sorted_vals}, m, m - D, sorted_vals, kk, SAc,
                                      ISAc, resolved));
            else
                SAIX_TRY(resolve_ties(c, EqPacked{sorted_keys}, m, m - D, sorted_vals, kk, SAc, ISAc, resolved));
        }
        if (resolved && RA_out && bsorted) {
            // the keys still describe the (tie-reordered) sorted samples: RA
            // for the wide-level finish without text gathers
            uint4 *RA = ar.alloc<uint4>(m);
            SAIX_ARENA_OK(ar);
            SAIX_TRY(build_ra(c, sorted_keys, sorted_vals, L, kbits, ISAc, RA));
            *RA_out = RA;
        } else {
            ar.reset(mark);
        }
        if (!resolved) {
            if (narrow) SAIX_TRY(dc3_level<u8>(c, (const u8 *)tt, m, (u64)D, SAc, ISAc, nullptr, depth + 1));
            else SAIX_TRY(dc3_level<u32>(c, tt, m, (u64)D, SAc, ISAc, nullptr, depth + 1));
        }
    }
    return SAIX_OK;
}

template <typename TT>
static int dc3_level(Dc3Ctx &c, const TT *text, i64 N, u64 sigma, u32 *SA, u32 *ISA,
                     saix_dc3_probe *probe, int depth, u32 *Phi, bool *phi_done) {
    Arena &ar = *c.ar;
    cudaStream_t st = c.st;
    if (depth > c.max_depth) c.max_depth = depth;
    if (N <= 1) {
        if (N == 1) {
            if (SA) k_iota_pair<<<1, 32, 0, st>>>(SA, ISA, 1);
            else if (ISA) k_iota_pair<<<1, 32, 0, st>>>(ISA, nullptr, 1);
            SAIX_LAUNCHED();
        }
        return SAIX_OK;
    }
    if constexpr (sizeof(TT) == 1) {
        if (stream_level_ok(1, sigma, N, probe) && ((uintptr_t)text & 3) == 0)
            return dc3_level_stream(c, text, N, sigma, SA, ISA, Phi, phi_done, depth);
    }
    SampleLayout L = SampleLayout::of(N);
    size_t mark0 = ar.mark();
    u32 *tt = ar.alloc<u32>(L.m);
    u32 *SAc = ar.alloc<u32>(L.m);
    u32 *ISAc = ar.alloc<u32>(L.m);
    u32 *d_scal = ar.alloc<u32>(8);
    if (!SA) SA = ar.alloc<u32>(N);  // a streaming parent needs only the ranks
    SAIX_ARENA_OK(ar);
    Text<TT> T{text, N};

    // wide levels whose names all differ take the record finish below
    uint4 *RA = nullptr;
    size_t mark_s = ar.mark();
    bool want_ra = sizeof(TT) == 4 && probe == nullptr && L.m >= 4096;
    SAIX_TRY(sort_samples<TT>(c, T, L, sigma, tt, SAc, ISAc, d_scal, depth, probe != nullptr,
                              want_ra ? &RA : nullptr));
    if (!RA && want_ra) {
        // recursion case: sample records from the child's order
        RA = ar.alloc<uint4>(L.m);
        SAIX_ARENA_OK(ar);
        Prof prof_("dc3.arec", 36.0 * L.m, st);
        k_arec_sa<TT><<<grid_for(L.m, 256), 256, 0, st>>>(SAc, T, L, ISAc, RA);
        SAIX_LAUNCHED();
    }
    if (RA) {
        bool fin = false;
        SAIX_TRY(dc3_wide_finish<TT>(c, T, L, sigma, ISAc, RA, SA, ISA, fin));
        if (fin) {
            ar.reset(mark0);
            return SAIX_OK;
        }
        ar.reset(mark_s);  // sort temps + RA
    }

    // step 3: mod-0 suffixes = mod-1 samples in rank order, minus one,
    // stably split by their first character
    size_t mark1 = ar.mark();
    i64 k = L.k;
    u32 *k0 = ar.alloc<u32>(k), *k1 = ar.alloc<u32>(k);
    u32 *v0 = ar.alloc<u32>(k), *v1 = ar.alloc<u32>(k);
    u32 *scratch = ar.alloc<u32>(os_scratch_words(L.m) > bs_scratch_words(N / 8 + 2) ? os_scratch_words(L.m)
                                                                                  : bs_scratch_words(N / 8 + 2));
    u32 *split = ar.alloc<u32>(merge_split_words(N));
    SAIX_ARENA_OK(ar);
    u32 *keys = k0, *vals = v0;
    if (mod0_use_bitmaps(sigma)) {
        i64 wpc = ceil_div(L.m, 32) + 1;
        i64 nw = mod0_bitmap_words(sigma, L.m);
        uint2 *pb = ar.alloc<uint2>(nw);
        u32 *tmp = ar.alloc<u32>(scan_tmp_words(nw));
        SAIX_ARENA_OK(ar);
        Prof prof_("dc3.mod0_split", (8.0 + 2 * sizeof(TT)) * k + 4.0 * k + 8.0 * nw, st);
        SAIX_CUDA(cudaMemsetAsync(pb, 0, (size_t)nw * 8, st));
        int g = grid_for(k, K_THREADS);
        k_mod0_bits<TT><<<g, K_THREADS, 0, st>>>(T, ISAc, k, wpc, pb);
        SAIX_LAUNCHED();
        SAIX_TRY(scan_transform(PbPopc{pb}, PbStore{pb}, nw, tmp, nullptr, st, "dc3.mod0_scan", 12.0 * nw));
        k_mod0_place<TT><<<g, K_THREADS, 0, st>>>(T, ISAc, k, wpc, pb, v0);
        SAIX_LAUNCHED();
    } else {
        bool done = false;
        int rbm = bits_for((u64)L.m);
        u64 mk = ((u64)sigma << rbm) | (u64)L.m;
        if (sigma + 1 > 256 && bits_for(sigma) + rbm <= 64 && use_bsort(mk, k)) {
            // the (char, rank) keys are distinct, so an unstable bucket split
            // followed by in-bucket sorts gives the exact order
            u64 *k64 = ar.alloc<u64>(k);
            SAIX_ARENA_OK(ar);
            SAIX_TRY(bucket_sort(Mod0BucketSrc<TT>{T, ISAc, rbm, (u64)L.m + 1}, k, sigma * ((u64)L.m + 1) + L.m,
                                 k64, v0, scratch, done, st, "dc3.mod0_split", &ar));
            vals = v0;
        }
        if (!done) {
            int passes = (bits_for(sigma) + OS_BITS - 1) / OS_BITS;
            SAIX_TRY(onesweep_sort<u32>(Mod0Src<TT>{T, SAc, (u32)L.m1}, L.m, Mod0HistSrc<TT>{T}, k, k, 0, passes,
                                        k0, v0, k1, v1, scratch, keys, vals, nullptr, st, "dc3.mod0_split"));
        }
    }

    // step 4: merge real samples (skip the padding sample at rank 1) with mod-0
    RankFromIsa R{L, ISAc};
    i64 pad = L.pad ? 1 : 0;
    i64 na = L.m - pad;
    using EB = typename EBlockOf<TT>::type;
    int rb = bits_for((u64)L.m), cb = bits_for(sigma);
    bool compact = sizeof(TT) == 1 && 2 * rb + 3 * cb <= 64;
    EB *E = nullptr;
    ECompact EC{nullptr, rb, cb};
    if (compact) {
        u64 *E64 = ar.alloc<u64>(k + 1);
        SAIX_ARENA_OK(ar);
        Prof prof_("dc3.eblocks", (double)sizeof(TT) * N + 8.0 * L.m + 8.0 * k, st);
        k_build_ecompact_u8<<<grid_for(k + 1, K_THREADS), K_THREADS, 0, st>>>(
            Text<u8>{(const u8 *)text, N}, R, k, rb, cb, E64);
        EC.E = E64;
    } else {
        E = ar.alloc<EB>(k);
        SAIX_ARENA_OK(ar);
        Prof prof_("dc3.eblocks", (double)sizeof(TT) * N + 8.0 * L.m + (double)sizeof(EB) * k, st);
        k_build_eblocks<TT><<<grid_for(k, K_THREADS), K_THREADS, 0, st>>>(T, R, k, E);
    }
    SAIX_LAUNCHED();
    MergeIdx<TT> V{T, R, SAc + pad, vals, E, EC};
    SAIX_TRY(merge_run(V, na, k, split, SA, ISA, st));

    if (probe) {
        int g = grid_for(N + 3, K_THREADS);
        if (probe->triple_text)
            SAIX_CUDA(cudaMemcpyAsync(probe->triple_text, tt, (size_t)L.m * 4, cudaMemcpyDeviceToDevice, st));
        if (probe->sample_rank) {
            k_probe_rank<<<g, K_THREADS, 0, st>>>(R, N + 3, probe->sample_rank);
            SAIX_LAUNCHED();
        }
        if (probe->sorted_samples) {
            k_probe_samples<<<g, K_THREADS, 0, st>>>(L, SAc, pad, probe->sorted_samples);
            SAIX_LAUNCHED();
        }
        if (probe->sorted_nonsamples) {
            k_times3<<<g, K_THREADS, 0, st>>>(vals, k, probe->sorted_nonsamples);
            SAIX_LAUNCHED();
        }
        probe->n_samples = L.m;
        probe->n_sorted_samples = na;
        probe->n_sorted_nonsamples = k;
    }
    (void)mark1;
    ar.reset(mark0);
    return SAIX_OK;
}

// Streaming level (see "streaming level" above).  SA / ISA / Phi nullable;
// Phi is produced only when ISA is not requested (*phi_done tells).
// ------------------------------------------------ level-0 window naming
// (replaces _name_triples + the recursion of _sort_samples, suffix_index.py:
// 221-271, on level 0 of byte texts; same sample order)
// Byte levels with sigma <= 7: name every sample by its 21-character window
// (3 bits per character, u64 key, 0 past the end) instead of its triple.  The
// reduced string's suffix order is unchanged -- equal names mean equal 21
// characters, a comparison continued at the next name (3 characters on)
// re-reads what is already equal, and windows reaching past the end hold the
// sentinel at distinct offsets, so they are unique and no comparison runs
// across the end of a sample block (the same property DC3's padding triples
// give).  On non-repetitive text almost all windows are distinct: the tied
// samples are ordered by the prefix doubling of resolve_ties and the
// recursion below this level disappears.  Too many ties -> the caller runs
// the triple naming + recursion as before.
constexpr int WN_CHARS = 21;
struct WindowSrc {
    const u8 *t;
    i64 N;
    SampleLayout L;
    u32 lo, r;  // dense digits: c - lo in [0, r) for c >= lo
    int j;      // leading characters in the dense map
    int rb;     // log2(r) when r is a power of two, else 0
    __device__ __forceinline__ void get(i64 s, u64 &k, u32 &v) const {
        const i64 p = L.pos(s);
        u64 key = 0;
        const i64 a = p & ~(i64)3;
        if (a + 28 <= N) {
            const u32 *w = reinterpret_cast<const u32 *>(t + a);
            const int sh = 8 * (int)(p - a);
            u32 x[7];
#pragma unroll
            for (int q = 0; q < 7; q++) x[q] = __ldg(w + q);
            u32 y[6];
#pragma unroll
            for (int q = 0; q < 6; q++) y[q] = __funnelshift_r(x[q], x[q + 1], sh);
#pragma unroll
            for (int q = 0; q < WN_CHARS; q++) key = (key << 3) | ((y[q >> 2] >> (8 * (q & 3))) & 7u);
        } else {
            for (int q = 0; q < WN_CHARS; q++) key = (key << 3) | (p + q < N ? (u64)(t[p + q] & 7u) : 0ull);
        }
        k = key;
        v = (u32)s;
    }
    // monotone: mixed radix of the leading j characters; a character below lo
    // (sentinel / separator) zeroes itself and everything after it
    __device__ __forceinline__ u64 dense(u64 k) const {
        u64 d = 0;
        bool low = false;
        for (int q = 0; q < j; q++) {
            const u32 c = (u32)(k >> (3 * (WN_CHARS - 1 - q))) & 7u;
            low = low || c < lo;
            d = d * r + (low ? 0u : c - lo);
        }
        return d;
    }
};

// key + dense value from the same loaded bytes (bucket-sort hook, bs_get).
// SWAR: byte-reverse each 4-character word (__byte_perm) and compress its
// 8-bit lanes to 3-bit key fields / 2-bit dense digits with two shifts; the
// per-character loop only runs for windows with a low character (sentinel /
// separator) among the dense digits, or for alphabets without 2-bit digits.
__device__ __forceinline__ u64 wn_dense_loop(const WindowSrc &w, const u32 *y) {
    u64 d = 0;
    bool low = false;
    for (int q = 0; q < w.j; q++) {
        const u32 c = (y[q >> 2] >> (8 * (q & 3))) & 0xFFu;
        low = low || c < w.lo;
        const u32 dig = low ? 0u : c - w.lo;
        d = w.rb ? ((d << w.rb) | dig) : d * w.r + dig;
    }
    return d;
}

__device__ __forceinline__ u64 bs_get(const WindowSrc &w, i64 s, u64 &k, u32 &v) {
    const i64 p = w.L.pos(s);
    const i64 a = p & ~(i64)3;
    u32 y[6];
    if (a + 28 <= w.N) {
        const u32 *wp = reinterpret_cast<const u32 *>(w.t + a);
        const int sh = 8 * (int)(p - a);
        u32 x[7];
#pragma unroll
        for (int q = 0; q < 7; q++) x[q] = __ldg(wp + q);
#pragma unroll
        for (int q = 0; q < 6; q++) y[q] = __funnelshift_r(x[q], x[q + 1], sh);
    } else {
#pragma unroll
        for (int q = 0; q < 6; q++) {
            u32 word = 0;
            for (int b = 0; b < 4; b++) {
                const i64 at = p + 4 * q + b;
                word |= (at < w.N ? (u32)w.t[at] : 0u) << (8 * b);
            }
            y[q] = word;
        }
    }
    // key: 5 words of 4 characters -> 12 bits each, then character 20
    u64 key = 0;
#pragma unroll
    for (int q = 0; q < 5; q++) {
        const u32 r = __byte_perm(y[q], 0, 0x0123) & 0x07070707u;
        const u32 pp = r | (r >> 5);
        key = (key << 12) | (((pp >> 10) & 0xFC0u) | (pp & 0x3Fu));
    }
    key = (key << 3) | (y[5] & 7u);
    k = key;
    v = (u32)s;
    // dense: 2-bit digits of the first 14 characters when no low character is among them
    if (w.rb == 2 && w.j == 14) {
        const u32 lo4 = w.lo * 0x01010101u;
        const u32 lowm = __vcmpltu4(y[0], lo4) | __vcmpltu4(y[1], lo4) | __vcmpltu4(y[2], lo4) |
                         (__vcmpltu4(y[3], lo4) & 0x0000FFFFu);
        if (!lowm) {
            u64 d = 0;
#pragma unroll
            for (int q = 0; q < 3; q++) {
                const u32 r = (__byte_perm(y[q], 0, 0x0123) - lo4) & 0x03030303u;
                const u32 pp = r | (r >> 6);
                d = (d << 8) | (((pp >> 12) & 0xF0u) | (pp & 0xFu));
            }
            d = (d << 2) | ((y[3] & 0xFFu) - w.lo);
            d = (d << 2) | (((y[3] >> 8) & 0xFFu) - w.lo);
            return d;
        }
    }
    return wn_dense_loop(w, y);
}

static int window_rank_generic(Dc3Ctx &c, const u8 *text, i64 N, u64 sigma, const SampleLayout &L, u32 *SAc,
                               u32 *ISAc, u32 *d_scal, int depth, bool &handled) {
    Arena &ar = *c.ar;
    cudaStream_t st = c.st;
    handled = false;
    const i64 m = L.m;
    const size_t mark = ar.mark();
    if (ar.cap - mark < (size_t)m * 96 + ((size_t)64 << 20)) return SAIX_OK;  // no room: recurse instead
    WindowSrc src;
    src.t = text;
    src.N = N;
    src.L = L;
    src.lo = sigma <= 4 ? 1u : 2u;
    src.r = (u32)sigma - src.lo + 1u;
    src.j = 0;
    src.rb = (src.r & (src.r - 1)) == 0 ? __builtin_ctz(src.r) : 0;
    u64 span = 1;
    while (src.j < WN_CHARS && span * src.r <= ((u64)1 << 28)) {
        span *= src.r;
        src.j++;
    }
    constexpr int WN_PER_BUCKET = 6, WN_MAX_BITS = 24;  // counters stay L2-resident (64 MB)
    const BsGeom g = bs_geom(span - 1, m, WN_PER_BUCKET, WN_MAX_BITS);
    u64 *k0 = ar.alloc<u64>(m), *k1 = ar.alloc<u64>(m);
    u32 *v0 = ar.alloc<u32>(m);
    u32 *scratch = ar.alloc<u32>(bs_scratch_words(g.nb));
    SAIX_ARENA_OK(ar);
    bool done = false;
    SAIX_TRY(bucket_sort(src, m, span - 1, k0, v0, scratch, done, st, "dc3.window_sort", &ar, WN_PER_BUCKET,
                         WN_MAX_BITS));
    if (!done) {
        ar.reset(mark);
        return SAIX_OK;
    }
    // distinct windows and the tied runs in one pass
    const u32 cap = (u32)(m / 32 + 64);
    u32 *rsA = ar.alloc<u32>(cap), *rlA = ar.alloc<u32>(cap), *rsB = ar.alloc<u32>(cap), *rlB = ar.alloc<u32>(cap);
    u32 *mid = ar.alloc<u32>(cap), *big = ar.alloc<u32>(cap);
    u32 *scal = ar.alloc<u32>(16);  // [0] mid, [1] big, [2] runs A, [3] runs B, [4] overflow, [5] distinct
    SAIX_ARENA_OK(ar);
    SAIX_CUDA(cudaMemsetAsync(scal, 0, 16 * 4, st));
    {
        Prof prof_("dc3.count_names", 8.0 * m, st);
        k_count_runs<<<grid_for(m, K_THREADS, kNumSMs * 8), K_THREADS, 0, st>>>(k0, m, scal + 5, rsA, rlA, scal + 2,
                                                                               cap, scal + 4);
    }
    SAIX_LAUNCHED();
    u32 h6[6];
    SAIX_CUDA(cudaMemcpyAsync(h6, scal, 24, cudaMemcpyDeviceToHost, st));
    SAIX_CUDA(cudaStreamSynchronize(st));
    const u32 D = h6[5];
    const bool tie_ok = (i64)D < m && (i64)(m - D) <= m / 32 && !h6[4];
    if ((i64)D == m || tie_ok) {
        // ranks = sorted positions (the ties' order is fixed below)
        if (m >= kDirectScatterItems) {
            PsPlan pu = PsPlan::of(m, 4);
            pu.set_cursors(ar.alloc<u32>(pu.cursor_words()));
            uint2 *s1 = ar.alloc<uint2>(pu.stage1_items()), *s2 = ar.alloc<uint2>(pu.stage2_items());
            SAIX_ARENA_OK(ar);
            SAIX_CUDA(cudaMemsetAsync(pu.a.cursor, 0, (size_t)pu.cursor_words() * 4, st));
            {
                Prof prof_("dc3.unique_ranks", (SAc ? 16.0 : 12.0) * m, st);
                static DeviceFlags attr;
                if (attr.need()) {
                    SAIX_CUDA(cudaFuncSetAttribute(k_unique_emit, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                   256 * UE_ITEMS * 8 + 8 * PS_MAX_BUCKETS));
                    attr.set();
                }
                size_t smem = (size_t)256 * UE_ITEMS * 8 + 8 * (size_t)pu.a.buckets;
                k_unique_emit<<<(unsigned)ceil_div(m, 256 * UE_ITEMS), 256, smem, st>>>(v0, m, SAc, pu, s1);
            }
            SAIX_LAUNCHED();
            SAIX_TRY(ps_finish(s1, s2, pu, U32Apply{ISAc}, st, "dc3.unique_isa", 28.0 * m));
        } else {
            Prof prof_("dc3.unique_ranks", 12.0 * m, st);
            k_unique_from_sorted<<<grid_for(m, K_THREADS), K_THREADS, 0, st>>>(v0, m, SAc, ISAc);
            SAIX_LAUNCHED();
        }
        if (tie_ok) {
            {
                Prof prof_("dc3.tie_resolve", 12.0 * (m - D), st);
                k_tie_groups<<<grid_for(h6[2], 128), 128, 0, st>>>(rsA, rlA, scal + 2, v0, ISAc);
            }
            SAIX_LAUNCHED();
            SAIX_TRY(tie_rounds(c, m, m - D, v0, k1, ISAc, rsA, rlA, rsB, rlB, mid, big, scal, h6[2]));
            if (SAc) SAIX_CUDA(cudaMemcpyAsync(SAc, v0, (size_t)m * 4, cudaMemcpyDeviceToDevice, st));
        }
        handled = true;
    }
    if (handled) {
        if (depth == 0) g_naming = 1;
        if ((size_t)depth >= g_trace.size()) g_trace.resize((size_t)depth + 1);
        g_trace[(size_t)depth] = LevelRec{L.n, (i64)sigma, m, (i64)D};
        g_trace.resize((size_t)depth + 1);
        if (trace_on())
            fprintf(stderr, "[saix dc3] depth %d: N=%lld text=u8 sigma=%llu m=%lld names=%u naming=window%d%s\n",
                    depth, (long long)L.n, (unsigned long long)sigma, (long long)m, D, WN_CHARS,
                    (i64)D == m ? " (unique)" : " (ties resolved)");
    }
    ar.reset(mark);
    return SAIX_OK;
}

// Level-0 window naming of DNA texts by the MSD record sort (wsort.cuh).
// tried = false: preconditions not met (caller runs the generic window
// sort); tried && !handled: too many ties -> the triple-naming recursion.
static bool ws_dna_on() {
    static int v = [] {
        const char *e = getenv("SAIX_WS_DNA");
        return e && e[0] == '0' ? 0 : 1;
    }();
    return v != 0;
}
// SAIX_COMPACT_RECORDS=0: the 16 B record path after the DNA window sort (A/B)
static bool compact_records_on() {
    static int v = [] {
        const char *e = getenv("SAIX_COMPACT_RECORDS");
        return e && e[0] == '0' ? 0 : 1;
    }();
    return v != 0;
}
template <bool SEP>
static int ws_sort_attrs() {
    SAIX_CUDA(cudaFuncSetAttribute(k_ws_sort<0, SEP>, cudaFuncAttributeMaxDynamicSharedMemorySize, 224 << 10));
    SAIX_CUDA(cudaFuncSetAttribute(k_ws_sort<2, SEP>, cudaFuncAttributeMaxDynamicSharedMemorySize, 224 << 10));
    SAIX_CUDA(cudaFuncSetAttribute(k_ws_sort<4, SEP>, cudaFuncAttributeMaxDynamicSharedMemorySize, 224 << 10));
    SAIX_CUDA(cudaFuncSetAttribute(k_ws_sort<6, SEP>, cudaFuncAttributeMaxDynamicSharedMemorySize, 224 << 10));
    SAIX_CUDA(cudaFuncSetAttribute(k_ws_sort<8, SEP>, cudaFuncAttributeMaxDynamicSharedMemorySize, 224 << 10));
    return SAIX_OK;
}
static int window_rank_dna(Dc3Ctx &c, const u8 *text, i64 N, const SampleLayout &L, const WsAlpha &A, u32 *SAc,
                           u32 *ISAc, int depth, bool &handled, bool &tried, u8 *CH) {
    Arena &ar = *c.ar;
    cudaStream_t st = c.st;
    handled = tried = false;
    const i64 m = L.m;
    PsPlan pu = PsPlan::of(m, 4);
    i64 stage_items = m;
    if (pu.stage1_items() > stage_items) stage_items = pu.stage1_items();
    if (pu.stage2_items() > stage_items) stage_items = pu.stage2_items();
    const u32 cap = (u32)(m / 32 + 64);
    const size_t need = (size_t)stage_items * 16 + (SAc ? 0 : (size_t)m * 4) + (size_t)cap * 24 +
                        ((size_t)3 * WS_FINE + 2 * WS_COARSE + scan_tmp_words(WS_FINE) + pu.cursor_words() + 32) * 4 +
                        24 * Arena::kAlign;
    const size_t mark = ar.mark();
    if (ar.cap - mark < need) return SAIX_OK;
    u64 *SA_ = ar.alloc<u64>(stage_items), *SB = ar.alloc<u64>(stage_items);
    u32 *sorted = SAc ? SAc : ar.alloc<u32>(m);
    u32 *hist = ar.alloc<u32>(WS_FINE), *off = ar.alloc<u32>(WS_FINE + 1), *curF = ar.alloc<u32>(WS_FINE);
    u32 *curC = ar.alloc<u32>(WS_COARSE), *tstart = ar.alloc<u32>(WS_COARSE + 1);
    u32 *tmp = ar.alloc<u32>(scan_tmp_words(WS_FINE));
    u32 *scal = ar.alloc<u32>(16);  // resolve_ties layout; [6] P1 overflow, [7] largest bucket
    u32 *rsA = ar.alloc<u32>(cap), *rlA = ar.alloc<u32>(cap), *rsB = ar.alloc<u32>(cap), *rlB = ar.alloc<u32>(cap);
    u32 *mid = ar.alloc<u32>(cap), *big = ar.alloc<u32>(cap);
    pu.set_cursors(ar.alloc<u32>(pu.cursor_words()));
    SAIX_ARENA_OK(ar);
    const i64 ntiles = ceil_div(N + 1, (i64)WS_TP);
    static DeviceFlags attr;
    if (attr.need()) {
        SAIX_CUDA(cudaFuncSetAttribute(k_ws_count<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, WS_COUNT_SMEM));
        SAIX_CUDA(cudaFuncSetAttribute(k_ws_count<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, WS_COUNT_SMEM));
        SAIX_CUDA(cudaFuncSetAttribute(k_ws_part1<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)WS_P2_SMEM));
        SAIX_CUDA(cudaFuncSetAttribute(k_ws_part1<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)WS_P2_SMEM));
        SAIX_CUDA(cudaFuncSetAttribute(k_ws_part2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)WS_P2B_SMEM));
        SAIX_TRY(ws_sort_attrs<false>());
        SAIX_TRY(ws_sort_attrs<true>());
        attr.set();
    }
    SAIX_CUDA(cudaMemsetAsync(hist, 0, (size_t)WS_FINE * 4, st));
    SAIX_CUDA(cudaMemsetAsync(scal, 0, 16 * 4, st));
    {
        Prof prof_("dc3.ws_count", (double)N, st);
        if (A.sep >= 0) k_ws_count<true><<<kNumSMs, 1024, WS_COUNT_SMEM, st>>>(text, L, A, ntiles, hist, scal + 6);
        else k_ws_count<false><<<kNumSMs, 1024, WS_COUNT_SMEM, st>>>(text, L, A, ntiles, hist, scal + 6);
        SAIX_LAUNCHED();
    }
    SAIX_TRY(scan_transform(WsHistIn{hist}, WsOffOut{off, curF, curC, scal + 7}, WS_FINE, tmp, off + WS_FINE, st,
                            "dc3.ws_scan", 16.0 * WS_FINE));
    k_ws_tiles<<<1, WS_COARSE, 0, st>>>(off, m, tstart);
    SAIX_LAUNCHED();
    // P3 unit: 2^G fine buckets -- ~3 k records on average, or fewer
    // buckets per unit where a skewed text makes some unit too large
    const i64 mean = m >> 16;
    const int Gmean = mean >= 1024 ? 0 : mean >= 256 ? 2 : mean >= 64 ? 4 : mean >= 16 ? 6 : 8;
    for (int g = 0; g <= Gmean; g += 2) {
        k_ws_unit_max<<<(WS_FINE >> g) / 256 + 1, 256, 0, st>>>(off, m, g, scal + 9 + g / 2);
        SAIX_LAUNCHED();
    }
    u32 h[8];
    SAIX_CUDA(cudaMemcpyAsync(h, scal + 6, 32, cudaMemcpyDeviceToHost, st));
    SAIX_CUDA(cudaStreamSynchronize(st));
    int G = 0;
    for (int g = Gmean; g > 0; g -= 2)
        if (h[3 + g / 2] <= (u32)WS_CAP_MAX) {
            G = g;
            break;
        }
    h[1] = h[3 + G / 2];  // the largest unit bounds P3's shared buffers
    if (h[0] || h[1] > (u32)WS_CAP_MAX) {  // skewed text: the generic window sort
        ar.reset(mark);
        return SAIX_OK;
    }
    if (pu.a.buckets > WS_ST) {  // P3 reserves one ISA run per coarse bucket and thread
        ar.reset(mark);
        return SAIX_OK;
    }
    tried = true;
    const int capA = (int)(h[1] <= (u32)WS_CAP_MIN ? WS_CAP_MIN : ceil_div((i64)h[1], (i64)256) * 256);
    // (the largest bucket fits; emit staging reuses S)
    {
        Prof prof_("dc3.ws_part1", (double)N + 8.0 * m, st);
        if (A.sep >= 0) k_ws_part1<true><<<(unsigned)ntiles, WS_PT, WS_P2_SMEM, st>>>(text, L, A, curC, SA_);
        else k_ws_part1<false><<<(unsigned)ntiles, WS_PT, WS_P2_SMEM, st>>>(text, L, A, curC, SA_);
        SAIX_LAUNCHED();
    }
    {
        Prof prof_("dc3.ws_part2", 16.0 * m, st);
        k_ws_part2<<<(unsigned)(ceil_div(m, (i64)WS_PTILE2) + WS_COARSE), WS_PT, WS_P2B_SMEM, st>>>(SA_, off, tstart, m,
                                                                                                  curF, SB);
        SAIX_LAUNCHED();
    }
    SAIX_CUDA(cudaMemsetAsync(pu.a.cursor, 0, (size_t)pu.cursor_words() * 4, st));
    {
        Prof prof_("dc3.ws_sort", 8.0 * m + 4.0 * m + 8.0 * m, st);
        const size_t smem = ws_sort_smem(capA, pu, 4096);
        const int per_sm = smem <= (74u << 10) ? 3 : smem <= (112u << 10) ? 2 : 1;
        const unsigned grid = (unsigned)(kNumSMs * per_sm);
        uint2 *st1 = reinterpret_cast<uint2 *>(SA_);
#define WS_SORT_G(g)                                                                                            \
    (A.sep >= 0 ? k_ws_sort<g, true><<<grid, WS_ST, smem, st>>>(SB, off, m, L.m1, capA, sorted, pu, st1, rsA, rlA,  \
                                                                cap, scal, CH, N, A)                               \
                : k_ws_sort<g, false><<<grid, WS_ST, smem, st>>>(SB, off, m, L.m1, capA, sorted, pu, st1, rsA, rlA, \
                                                                 cap, scal, CH, N, A))
        switch (G) {
            case 0: WS_SORT_G(0); break;
            case 2: WS_SORT_G(2); break;
            case 4: WS_SORT_G(4); break;
            case 6: WS_SORT_G(6); break;
            default: WS_SORT_G(8); break;
        }
#undef WS_SORT_G
        SAIX_LAUNCHED();
    }
    u32 h6[9];
    SAIX_CUDA(cudaMemcpyAsync(h6, scal, 36, cudaMemcpyDeviceToHost, st));
    SAIX_CUDA(cudaStreamSynchronize(st));
    if (h6[8]) {  // low-complexity sub-bucket: the generic window sort
        tried = false;
        ar.reset(mark);
        return SAIX_OK;
    }
    const u32 D = h6[5];
    const bool tie_ok = (i64)D < m && (i64)(m - D) <= m / 32 && !h6[4];
    if ((i64)D == m || tie_ok) {
        SAIX_TRY(ps_finish(reinterpret_cast<uint2 *>(SA_), reinterpret_cast<uint2 *>(SB), pu, U32Apply{ISAc}, st,
                           "dc3.unique_isa", 28.0 * m));
        if (tie_ok) {
            {
                Prof prof_("dc3.tie_resolve", 12.0 * (m - D), st);
                k_tie_groups<<<grid_for(h6[2], 128), 128, 0, st>>>(rsA, rlA, scal + 2, sorted, ISAc);
            }
            SAIX_LAUNCHED();
            SAIX_TRY(tie_rounds(c, m, m - D, sorted, SA_, ISAc, rsA, rlA, rsB, rlB, mid, big, scal, h6[2]));
        }
        handled = true;
        if (depth == 0) g_naming = 2;
        if ((size_t)depth >= g_trace.size()) g_trace.resize((size_t)depth + 1);
        g_trace[(size_t)depth] = LevelRec{L.n, A.lo == 2 ? 5 : 4, m, (i64)D};
        g_trace.resize((size_t)depth + 1);
        if (trace_on())
            fprintf(stderr, "[saix dc3] depth %d: N=%lld text=u8 sigma<=4 m=%lld names=%u naming=window21/msd%s\n",
                    depth, (long long)L.n, (long long)m, D, (i64)D == m ? " (unique)" : " (ties resolved)");
    }
    ar.reset(mark);
    return SAIX_OK;
}

// smallest level the DNA window sort takes (below, the generic sort's few
// launches win); SAIX_WS_MIN_M lowers it for compute-sanitizer runs on small
// texts (tools/sanitize_run.py)
static i64 ws_min_m() {
    static i64 v = [] {
        const char *e = getenv("SAIX_WS_MIN_M");
        return e && *e ? (i64)atoll(e) : ((i64)1 << 20);
    }();
    return v;
}
static bool ws_dna_eligible(const u8 *text, i64 N, u64 sigma, const SampleLayout &L) {
    return (sigma <= 4 || sigma == 5) && N + 1 < (i64)WS_POS_MASK && L.m >= ws_min_m() &&
           ((uintptr_t)text & 15) == 0 && ws_dna_on();
}
// sigma 5: the DNA window sort applies when rank 1 occurs exactly once (the
// generalized text's separator); out[0] = count, out[1] = first position
__global__ void k_ws_find_sep(const u8 *__restrict__ t, i64 N, unsigned long long *__restrict__ out) {
    u32 c = 0;
    unsigned long long first = ~0ull;
    for (i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x; i < N; i += (i64)gridDim.x * blockDim.x)
        if (t[i] == 1) {
            c++;
            first = first < (unsigned long long)i ? first : (unsigned long long)i;
        }
    for (int o = 16; o; o >>= 1) {
        c += __shfl_xor_sync(0xffffffffu, c, o);
        const unsigned long long y = __shfl_xor_sync(0xffffffffu, first, o);
        first = y < first ? y : first;
    }
    if (lane_id() == 0 && c) {
        atomicAdd(&out[0], (unsigned long long)c);
        atomicMin(&out[1], first);
    }
}
__global__ void k_ws_sep_init(unsigned long long *out) {
    out[0] = 0;
    out[1] = ~0ull;
}
static int ws_alpha(Dc3Ctx &c, const u8 *text, i64 N, u64 sigma, WsAlpha &A, bool &ok) {
    ok = true;
    A = WsAlpha{1u, -1};
    if (sigma <= 4) return SAIX_OK;
    ok = false;
    if (sigma != 5) return SAIX_OK;
    Arena &ar = *c.ar;
    const size_t mark = ar.mark();
    unsigned long long *d = ar.alloc<unsigned long long>(2);
    SAIX_ARENA_OK(ar);
    k_ws_sep_init<<<1, 1, 0, c.st>>>(d);
    k_ws_find_sep<<<grid_for(N, 256, kNumSMs * 4), 256, 0, c.st>>>(text, N, d);
    SAIX_LAUNCHED();
    unsigned long long h[2];
    SAIX_CUDA(cudaMemcpyAsync(h, d, 16, cudaMemcpyDeviceToHost, c.st));
    SAIX_CUDA(cudaStreamSynchronize(c.st));
    ar.reset(mark);
    if (h[0] != 1) return SAIX_OK;
    A = WsAlpha{2u, (i64)h[1]};
    ok = true;
    return SAIX_OK;
}
// compact: the DNA window sort named the level and wrote SAc (rank order)
// and CH (first two characters per rank) -- the records can be compact
static int window_rank(Dc3Ctx &c, const u8 *text, i64 N, u64 sigma, const SampleLayout &L, u32 *SAc, u32 *ISAc,
                       u32 *d_scal, int depth, bool &handled, u8 *CH = nullptr, bool *compact = nullptr) {
    if (compact) *compact = false;
    WsAlpha A;
    bool alpha_ok = false;
    if (ws_dna_eligible(text, N, sigma, L)) SAIX_TRY(ws_alpha(c, text, N, sigma, A, alpha_ok));
    if (alpha_ok) {
        bool tried = false;
        SAIX_TRY(window_rank_dna(c, text, N, L, A, SAc, ISAc, depth, handled, tried, CH));
        if (compact) *compact = handled && SAc && CH;
        if (tried) return SAIX_OK;
    }
    return window_rank_generic(c, text, N, sigma, L, SAc, ISAc, d_scal, depth, handled);
}

// Steps 1-3 of a streaming level over compact records (levels named by the
// DNA window sort, which left SR = SAc and CH in rank order).
static int stream_finish_compact(Dc3Ctx &c, const u8 *text, u64 sigma, const SampleLayout &L, const u32 *SR,
                                 const u32 *ISAc, const u8 *CH, u32 *SA, u32 *ISA, u32 *Phi, bool *phi_done) {
    Arena &ar = *c.ar;
    cudaStream_t st = c.st;
    const i64 m = L.m, k = L.k;
    const int D1 = (int)sigma + 1;
    u32 *NX = ar.alloc<u32>(m);
    uint4 *M0 = ar.alloc<uint4>(k);
    SAIX_ARENA_OK(ar);
    const size_t mark_s1 = ar.mark();
    PsPlan pn = PsPlan::of(m, 4, (i64)4 << RW_SHIFT);
    if (pn.windows > 1 && pn.s2 != RW_SHIFT) {
        set_error("dc3: NX window %d != %d", pn.s2, RW_SHIFT);
        return SAIX_EINVAL;
    }
    pn.set_cursors(ar.alloc<u32>(pn.cursor_words()));
    uint2 *s1 = ar.alloc<uint2>(pn.stage1_items()), *s2 = ar.alloc<uint2>(pn.stage2_items());
    u32 *hist = ar.alloc<u32>((i64)D1 * pn.windows + 1);
    u32 *hscan = ar.alloc<u32>(scan_tmp_words((i64)D1 * pn.windows));
    SAIX_ARENA_OK(ar);
    SAIX_CUDA(cudaMemsetAsync(pn.a.cursor, 0, (size_t)pn.cursor_words() * 4, st));
    {
        Prof prof_("dc3.nx_emit", 12.0 * m + (double)k + 8.0 * m, st);
        static DeviceFlags attr;
        if (attr.need()) {
            SAIX_CUDA(cudaFuncSetAttribute(k_nx_emit, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)NX_EMIT_SMEM));
            attr.set();
        }
        const size_t smem = (size_t)2 * NX_THREADS * NX_J * 8 + 8 * (size_t)pn.a.buckets;
        k_nx_emit<<<(unsigned)ceil_div(L.m1, (i64)NX_THREADS * NX_J), NX_THREADS, smem, st>>>(text, L, ISAc, pn, s1);
    }
    SAIX_LAUNCHED();
    {
        Prof prof_("dc3.nx_apply", 28.0 * m, st);
        SAIX_TRY(ps_refine_launch(s1, pn, s2, st));
        k_nx_window<<<(unsigned)pn.windows, PS_THREADS, 0, st>>>(s2, pn, NX, hist, D1);
        SAIX_LAUNCHED();
    }
    SAIX_TRY(scan_transform(HistIn{hist}, StoreExcl{hist}, (i64)D1 * pn.windows, hscan, nullptr, st,
                            "dc3.mod0_scan", 8.0 * D1 * pn.windows));
    const CompactRecSrc src{SR, NX, CH, (u32)L.m1};
    {
        Prof prof_("dc3.mod0_split", 9.0 * m + 16.0 * k, st);
        static DeviceFlags attr;
        if (attr.need()) {
            SAIX_CUDA(cudaFuncSetAttribute(k_mod0_window<CompactRecSrc>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)M0_SMEM));
            attr.set();
        }
        u32 dmask = 1;
        while (dmask < (u32)D1 - 1) dmask = dmask * 2 + 1;
        k_mod0_window<CompactRecSrc><<<(unsigned)pn.windows, M0_THREADS, M0_SMEM, st>>>(src, m, pn.windows, hist, M0,
                                                                                        dmask);
    }
    SAIX_LAUNCHED();
    ar.reset(mark_s1);

    // 3: merge (the padding sample has rank 0 and is not a suffix)
    const i64 pad = L.pad ? 1 : 0;
    const i64 na = m - pad;
    const CompactMergeView V{src, pad, M0};
    const i64 total = na + k;
    const i64 ntiles = ceil_div(total, RM_TILE);
    u32 *split = ar.alloc<u32>(ceil_div(total, RM_TILE) + 2);
    const bool isa_direct = ISA && total < 2 * kDirectScatterItems;
    const int mode = (ISA && !isa_direct) ? EMIT_ISA : (ISA ? EMIT_NONE : (Phi ? EMIT_PHI : EMIT_NONE));
    PsPlan pm = PsPlan::of(mode == EMIT_NONE ? 1 : total, 4);
    pm.set_cursors(ar.alloc<u32>(pm.cursor_words()));
    uint2 *pst1 = mode == EMIT_NONE ? nullptr : ar.alloc<uint2>(pm.stage1_items());
    uint2 *pst2 = mode == EMIT_NONE ? nullptr : ar.alloc<uint2>(pm.stage2_items());
    SAIX_ARENA_OK(ar);
    SAIX_CUDA(cudaMemsetAsync(pm.a.cursor, 0, (size_t)pm.cursor_words() * 4, st));
    {
        Prof prof_("dc3.merge_partition", 18.0 * (ntiles + 1), st);
        const i64 nc = ceil_div(ntiles, RM_COARSE);
        u32 *coarse = ar.alloc<u32>(nc + 2);
        SAIX_ARENA_OK(ar);
        k_merge_partition_rec<<<grid_for((nc + 1) * 8, 128), 128, 0, st>>>(V, na, k, ntiles, coarse, RM_COARSE,
                                                                            nullptr);
        SAIX_LAUNCHED();
        k_merge_partition_rec<<<grid_for((ntiles + 1) * 8, 128), 128, 0, st>>>(V, na, k, ntiles, split, 1, coarse);
    }
    SAIX_LAUNCHED();
    {
        Prof prof_("dc3.merge_tile", 9.0 * na + 16.0 * k + (SA ? 4.0 * total : 0) + (mode ? 8.0 * total : 0), st);
        if (mode == EMIT_ISA) SAIX_TRY(merge_rec_launch<EMIT_ISA>(V, na, k, split, SA, pm, pst1, st));
        else if (mode == EMIT_PHI) SAIX_TRY(merge_rec_launch<EMIT_PHI>(V, na, k, split, SA, pm, pst1, st));
        else SAIX_TRY(merge_rec_launch<EMIT_NONE>(V, na, k, split, SA, pm, pst1, st, isa_direct ? ISA : nullptr));
    }
    if (mode != EMIT_NONE)
        SAIX_TRY(ps_finish(pst1, pst2, pm, U32Apply{mode == EMIT_ISA ? ISA : Phi}, st,
                           mode == EMIT_ISA ? "dc3.isa_apply" : "dc3.phi_apply", 28.0 * total));
    if (phi_done) *phi_done = mode == EMIT_PHI;
    return SAIX_OK;
}

static int dc3_level_stream(Dc3Ctx &c, const u8 *text, i64 N, u64 sigma, u32 *SA, u32 *ISA, u32 *Phi,
                            bool *phi_done, int depth) {
    Arena &ar = *c.ar;
    cudaStream_t st = c.st;
    if (depth > c.max_depth) c.max_depth = depth;
    SampleLayout L = SampleLayout::of(N);
    const i64 m = L.m, k = L.k;
    size_t mark0 = ar.mark();
    u32 *tt = ar.alloc<u32>(m);
    u32 *ISAc = ar.alloc<u32>(m);
    u32 *d_scal = ar.alloc<u32>(8);
    SAIX_ARENA_OK(ar);
    Text<u8> T{text, N};
    // small level: the child also returns its order, and RS is gathered
    const bool gather = N + 4 * m <= RS_GATHER_BYTES;
    u32 *SAc = gather ? ar.alloc<u32>(m) : nullptr;
    SAIX_ARENA_OK(ar);
    bool windowed = false, compact = false;
    if (depth == 0) g_naming = 0;
    if (sigma <= 7 && m >= 4096 && window_naming_on()) {
        // the DNA window sort can also leave SAc and CH: compact records below
        u32 *SAw = SAc;
        u8 *CH = nullptr;
        if (!gather && ws_dna_eligible(text, N, sigma, L) && compact_records_on()) {
            SAw = ar.alloc<u32>(m);
            CH = ar.alloc<u8>(m);
            SAIX_ARENA_OK(ar);
        }
        SAIX_TRY(window_rank(c, text, N, sigma, L, SAw, ISAc, d_scal, depth, windowed, CH, &compact));
        if (compact) {
            SAIX_TRY(stream_finish_compact(c, text, sigma, L, SAw, ISAc, CH, SA, ISA, Phi, phi_done));
            ar.reset(mark0);
            return SAIX_OK;
        }
    }
    if (!windowed) SAIX_TRY(sort_samples<u8>(c, T, L, sigma, tt, SAc, ISAc, d_scal, depth, false, nullptr));

    // 1: sample records in rank order
    uint4 *RS = ar.alloc<uint4>(m);
    size_t mark1 = ar.mark();
    PsPlan pr = PsPlan::of(m, 16, (i64)16 << RW_SHIFT);
    const int D1 = (int)sigma + 1;
    if (pr.windows > 1 && pr.s2 != RW_SHIFT) {
        set_error("dc3: record window %d != %d", pr.s2, RW_SHIFT);
        return SAIX_EINVAL;
    }
    u32 *hist = nullptr, *hscan = nullptr;
    uint4 *stage1 = nullptr;
    size_t mark_s1 = 0;
    if (gather) {
        stage1 = ar.alloc<uint4>(k);  // M0
        mark_s1 = ar.mark();
        hist = ar.alloc<u32>((i64)D1 * pr.windows + 1);
        hscan = ar.alloc<u32>(scan_tmp_words((i64)D1 * pr.windows));
        SAIX_ARENA_OK(ar);
        u32 dmask = 1;
        while (dmask < (u32)D1 - 1) dmask = dmask * 2 + 1;
        Prof prof_("dc3.srec_gather", 4.0 * m + 2.0 * 32 * m + 16.0 * m, st);
        k_rs_gather<<<(unsigned)pr.windows, RG_THREADS, 0, st>>>(SAc, T, L, ISAc, RS, hist, D1, dmask, pr.windows);
        SAIX_LAUNCHED();
    } else {

    pr.set_cursors(ar.alloc<u32>(pr.cursor_words()));
    stage1 = ar.alloc<uint4>(pr.stage1_items() > k ? pr.stage1_items() : k);  // later: M0
    mark_s1 = ar.mark();
    uint4 *stage2 = ar.alloc<uint4>(pr.stage2_items());
    SAIX_ARENA_OK(ar);
    SAIX_CUDA(cudaMemsetAsync(pr.a.cursor, 0, (size_t)pr.cursor_words() * 4, st));
    {
        Prof prof_("dc3.srec_emit", (double)N + 12.0 * m + 16.0 * m, st);
        size_t smem = (size_t)2 * SR_TILE * 16 + 8 * (size_t)pr.a.buckets;
        static DeviceFlags attr;
        if (attr.need()) {
            SAIX_CUDA(cudaFuncSetAttribute(k_srec_emit, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           2 * SR_TILE * 16 + 8 * PS_MAX_BUCKETS));
            attr.set();
        }
        k_srec_emit<<<(unsigned)ceil_div(k, SR_TILE), SR_THREADS, smem, st>>>(T, L, ISAc, pr, stage1);
    }
    SAIX_LAUNCHED();
    // A2 + the specialised pass B (RS windows + per-window cprev histogram)
    hist = ar.alloc<u32>((i64)D1 * pr.windows + 1);
    hscan = ar.alloc<u32>(scan_tmp_words((i64)D1 * pr.windows));
    SAIX_ARENA_OK(ar);
    {
        Prof prof_("dc3.srec_apply", 48.0 * m, st);
        static DeviceFlags attr;
        if (attr.need()) {
            SAIX_CUDA(cudaFuncSetAttribute(k_ps_refine<uint4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)(PS_REFINE_TILE * 16 + 8 * 256)));
            SAIX_CUDA(cudaFuncSetAttribute(k_rs_window, cudaFuncAttributeMaxDynamicSharedMemorySize, 16 << RW_SHIFT));
            attr.set();
        }
        SAIX_TRY(ps_refine_launch(stage1, pr, stage2, st));
        k_rs_window<<<(unsigned)pr.windows, PS_THREADS, 16 << RW_SHIFT, st>>>(stage2, pr, RS, hist, D1);
        SAIX_LAUNCHED();
    }
    }  // scatter path
    // 2: non-sample records in sorted order: per-(digit, window) offsets,
    // then one CTA per RS window
    uint4 *M0 = (uint4 *)stage1;  // stage1 is free again and holds >= m records
    SAIX_TRY(scan_transform(HistIn{hist}, StoreExcl{hist}, (i64)D1 * pr.windows, hscan, nullptr, st,
                            "dc3.mod0_scan", 8.0 * D1 * pr.windows));
    {
        Prof prof_("dc3.mod0_split", 16.0 * m + 16.0 * k, st);
        static DeviceFlags attr;
        if (attr.need()) {
            SAIX_CUDA(cudaFuncSetAttribute(k_mod0_window<RsRecSrc>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)M0_SMEM));
            attr.set();
        }
        u32 dmask = 1;
        while (dmask < (u32)D1 - 1) dmask = dmask * 2 + 1;
        k_mod0_window<<<(unsigned)pr.windows, M0_THREADS, M0_SMEM, st>>>(RsRecSrc{RS}, m, pr.windows, hist, M0,
                                                                         dmask);
    }
    SAIX_LAUNCHED();
    ar.reset(mark_s1);  // stage2, histogram and scan temps are dead

    // 3: merge (the padding sample has rank 0 and is not a suffix)
    i64 pad = L.pad ? 1 : 0;
    i64 na = m - pad;
    RecMergeView V{RS + pad, M0};
    i64 total = na + k;
    i64 ntiles = ceil_div(total, RM_TILE);
    u32 *split = ar.alloc<u32>(ceil_div(total, RM_TILE) + 2);
    const bool isa_direct = ISA && total < 2 * kDirectScatterItems;
    int mode = (ISA && !isa_direct) ? EMIT_ISA : (ISA ? EMIT_NONE : (Phi ? EMIT_PHI : EMIT_NONE));
    PsPlan pm = PsPlan::of(mode == EMIT_NONE ? 1 : total, 4);
    pm.set_cursors(ar.alloc<u32>(pm.cursor_words()));
    uint2 *pst1 = mode == EMIT_NONE ? nullptr : ar.alloc<uint2>(pm.stage1_items());
    uint2 *pst2 = mode == EMIT_NONE ? nullptr : ar.alloc<uint2>(pm.stage2_items());
    SAIX_ARENA_OK(ar);
    SAIX_CUDA(cudaMemsetAsync(pm.a.cursor, 0, (size_t)pm.cursor_words() * 4, st));
    {
        Prof prof_("dc3.merge_partition", 32.0 * (ntiles + 1), st);
        i64 nc = ceil_div(ntiles, RM_COARSE);
        u32 *coarse = ar.alloc<u32>(nc + 2);
        SAIX_ARENA_OK(ar);
        k_merge_partition_rec<<<grid_for((nc + 1) * 8, 128), 128, 0, st>>>(V, na, k, ntiles, coarse, RM_COARSE,
                                                                            nullptr);
        SAIX_LAUNCHED();
        k_merge_partition_rec<<<grid_for((ntiles + 1) * 8, 128), 128, 0, st>>>(V, na, k, ntiles, split, 1, coarse);
    }
    SAIX_LAUNCHED();
    {
        Prof prof_("dc3.merge_tile", 16.0 * total + (SA ? 4.0 * total : 0) + (mode ? 8.0 * total : 0), st);
        if (mode == EMIT_ISA) SAIX_TRY(merge_rec_launch<EMIT_ISA>(V, na, k, split, SA, pm, pst1, st));
        else if (mode == EMIT_PHI) SAIX_TRY(merge_rec_launch<EMIT_PHI>(V, na, k, split, SA, pm, pst1, st));
        else SAIX_TRY(merge_rec_launch<EMIT_NONE>(V, na, k, split, SA, pm, pst1, st, isa_direct ? ISA : nullptr));
    }
    if (mode != EMIT_NONE)
        SAIX_TRY(ps_finish(pst1, pst2, pm, U32Apply{mode == EMIT_ISA ? ISA : Phi}, st,
                           mode == EMIT_ISA ? "dc3.isa_apply" : "dc3.phi_apply", 28.0 * total));
    if (phi_done) *phi_done = mode == EMIT_PHI;
    (void)mark1;
    ar.reset(mark0);
    return SAIX_OK;
}

// Upper bound of the workspace the driver carves (persistent arrays of every
// level + the largest level's temporaries), see DESIGN.md "DC3 workspace".
static size_t dc3_plan(i64 n, int text_bytes = 4) {
    size_t persistent = 0, temps = 0;
    i64 N = n;
    while (N > 1) {
        SampleLayout L = SampleLayout::of(N);
        i64 m = L.m, k = L.k;
        persistent += (size_t)(3 * m + 8) * 4 + (size_t)N * 4 + 5 * Arena::kAlign;
        i64 sw = os_scratch_words(m) > bs_scratch_words(N / 8 + 2) ? os_scratch_words(m) : bs_scratch_words(N / 8 + 2);
        PsPlan pu = PsPlan::of(m, 4);
        // sort buffers + the largest of the (sequential) bucketed scatters
        size_t ps_u = (size_t)(pu.stage1_items() + pu.stage2_items()) * 8 + (size_t)pu.cursor_words() * 4;
        size_t ps_max = bs_ps_bytes(m) > scatter_u32_bytes(m) ? bs_ps_bytes(m) : scatter_u32_bytes(m);
        ps_max = ps_max > ps_u ? ps_max : ps_u;
        // (+ tie resolution: group heads and run lists next to the sort buffers)
        size_t sort_t = (size_t)m * 24 + (size_t)(sw + scan_tmp_words(m)) * 4 + 4 * Arena::kAlign + ps_max +
                        (size_t)m * 4 + (size_t)(m / 32 + 64) * 24 + 8 * Arena::kAlign;
        i64 words = (2 * m > (1 << 16) ? 2 * m : (1 << 16)) + 1;
        size_t bm_t = (size_t)(2 * words + scan_tmp_words(words)) * 4;
        i64 bw = mod0_bitmap_words(7, m);
        size_t post_t = (size_t)k * 16 + (size_t)k * 32 + (size_t)k * 8 + bs_ps_bytes(k) +
                        (size_t)(sw + merge_split_words(N) + 2 * bw + scan_tmp_words(bw)) * 4;
        // streaming level: RS + (record stage | M0 + partition scratch | M0 + split + pair stage)
        PsPlan pr = PsPlan::of(m, 16, (i64)16 << 11), pm = PsPlan::of(N, 4);
        size_t s1 = (size_t)(pr.stage1_items() + pr.stage2_items()) * 16 + (size_t)pr.cursor_words() * 4;
        size_t s2 = (size_t)k * 16 + (size_t)os_scratch_words(m) * 4;
        size_t s3 = (size_t)k * 16 + (size_t)merge_split_words(N) * 4 +
                    (size_t)(pm.stage1_items() + pm.stage2_items()) * 8 + (size_t)pm.cursor_words() * 4;
        size_t stream_t = (size_t)m * 20 + (s1 > s2 ? (s1 > s3 ? s1 : s3) : (s2 > s3 ? s2 : s3));
        // wide-level finish: RB + (mod-0 bucket sort | merge split + ISA staging)
        size_t wf1 = (size_t)k * 12 + (size_t)bs_scratch_words(N / 8 + 2) * 4 + bs_ps_bytes(k);
        size_t wf2 = (size_t)merge_split_words(N) * 4 + (size_t)(pm.stage1_items() + pm.stage2_items()) * 8 +
                     (size_t)pm.cursor_words() * 4;
        size_t ra_t = (size_t)m * 8 + scatter_u32_bytes(m);
        size_t wf = wf1 > wf2 ? wf1 : wf2;
        wf = wf > ra_t ? wf : ra_t;
        size_t wide_t = sort_t + (size_t)m * 16 + (size_t)k * 20 + wf + 8 * Arena::kAlign;
        size_t t = sort_t > bm_t ? sort_t : bm_t;
        if (!(N == n && text_bytes == 1)) t = t > wide_t ? t : wide_t;  // byte top levels stream
        t = t > post_t ? t : post_t;
        t = t > stream_t ? t : stream_t;
        t += 8 * Arena::kAlign;
        if (t > temps) temps = t;
        N = m;
    }
    return persistent + temps + (1 << 16);
}

}  // namespace saix

using namespace saix;

extern "C" size_t saix_dc3_workspace_bytes(int64_t n, int text_bytes) {
    return dc3_plan(n, text_bytes);
}

extern "C" int saix_dc3(const void *text, int text_bytes, int64_t n, int64_t sigma, uint32_t *sa,
                        uint32_t *isa, void *ws, size_t ws_bytes, saix_dc3_probe *probe, void *stream) {
    return dc3_compute(text, text_bytes, n, sigma, sa, isa, ws, ws_bytes, probe, (cudaStream_t)stream);
}

namespace saix {
int dc3_compute(const void *text, int text_bytes, i64 n, i64 sigma, u32 *sa, u32 *isa, void *ws,
                size_t ws_bytes, saix_dc3_probe *probe, cudaStream_t stream, u32 *phi, bool *phi_done) {
    if (phi_done) *phi_done = false;
    if (n < 0 || n > (int64_t)0xFFFFFFF0LL || (text_bytes != 1 && text_bytes != 4) || sigma < 1 ||
        (n > 0 && (!text || !sa))) {
        set_error("saix_dc3: invalid arguments (n=%lld, text_bytes=%d, sigma=%lld)", (long long)n,
                  text_bytes, (long long)sigma);
        return SAIX_EINVAL;
    }
    if (text_bytes == 1 && sigma > 255) {
        set_error("saix_dc3: sigma %lld does not fit u8 text", (long long)sigma);
        return SAIX_EINVAL;
    }
    if (ws_bytes < dc3_plan(n, text_bytes)) {
        set_error("saix_dc3: workspace %zu < %zu bytes", ws_bytes, dc3_plan(n, text_bytes));
        return SAIX_ENOSPC;
    }
    Arena ar;
    ar.base = (char *)ws;
    ar.cap = ws_bytes;
    Dc3Ctx c{&ar, (cudaStream_t)stream, 0};
    g_trace.clear();
    if (probe) {
        probe->depth = 0;
        probe->n_samples = probe->n_sorted_samples = 0;
        probe->n_sorted_nonsamples = 0;
    }
    if (n == 0) return SAIX_OK;
    if (n == 1) {
        // Dc3Workspace of a single character: pad sample 1 names (0,0,0)
        k_iota_pair<<<1, 32, 0, (cudaStream_t)stream>>>(sa, isa, 1);
        SAIX_LAUNCHED();
        if (probe) {
            u32 h[4] = {1u, 0u, 0u, 0u};
            if (probe->triple_text)
                SAIX_CUDA(cudaMemcpyAsync(probe->triple_text, h, 4, cudaMemcpyHostToDevice, (cudaStream_t)stream));
            if (probe->sample_rank) {
                u32 r[4] = {0u, 1u, 0u, 0u};
                SAIX_CUDA(cudaMemcpyAsync(probe->sample_rank, r, 16, cudaMemcpyHostToDevice, (cudaStream_t)stream));
            }
            if (probe->sorted_nonsamples)
                SAIX_CUDA(cudaMemsetAsync(probe->sorted_nonsamples, 0, 4, (cudaStream_t)stream));
            probe->n_samples = 1;
            probe->n_sorted_nonsamples = 1;
            SAIX_CUDA(cudaStreamSynchronize((cudaStream_t)stream));
        }
        return SAIX_OK;
    }
    int rc = text_bytes == 1
                 ? dc3_level<u8>(c, (const u8 *)text, n, (u64)sigma, sa, isa, probe, 0, phi, phi_done)
                 : dc3_level<u32>(c, (const u32 *)text, n, (u64)sigma, sa, isa, probe, 0);
    if (rc) return rc;
    if (probe) probe->depth = c.max_depth;
    return SAIX_OK;
}
}  // namespace saix

extern "C" size_t saix_dc3_merge_workspace_bytes(int64_t total) {
    return (size_t)merge_split_words(total) * 4 + Arena::kAlign;
}

extern "C" int saix_dc3_merge(const void *text, int text_bytes, int64_t n, const uint32_t *sample_rank,
                              const uint32_t *sorted_samples, int64_t ms, const uint32_t *sorted_nonsamples,
                              int64_t k, uint32_t *sa, void *ws, size_t ws_bytes, void *stream) {
    if (n < 0 || ms < 0 || k < 0 || (text_bytes != 1 && text_bytes != 4) || ms + k > n + 1) {
        set_error("saix_dc3_merge: invalid arguments");
        return SAIX_EINVAL;
    }
    i64 total = ms + k;
    if (total == 0) return SAIX_OK;
    cudaStream_t st = (cudaStream_t)stream;
    if (!ws || ws_bytes < saix_dc3_merge_workspace_bytes(total)) {
        set_error("saix_dc3_merge: workspace too small");
        return SAIX_ENOSPC;
    }
    u32 *split = (u32 *)ws;
    int rc;
    if (text_bytes == 1) {
        MergePos<u8> V{Text<u8>{(const u8 *)text, n}, RankByPos{sample_rank}, sorted_samples, sorted_nonsamples};
        rc = merge_run(V, ms, k, split, sa, nullptr, st);
    } else {
        MergePos<u32> V{Text<u32>{(const u32 *)text, n}, RankByPos{sample_rank}, sorted_samples, sorted_nonsamples};
        rc = merge_run(V, ms, k, split, sa, nullptr, st);
    }
    return rc;
}

extern "C" int saix_dc3_naming(void) { return g_naming; }

extern "C" int saix_dc3_trace(int64_t *out, int max_levels) {
    int n = (int)g_trace.size();
    for (int i = 0; i < n && i < max_levels; i++) {
        out[4 * i + 0] = g_trace[i].n;
        out[4 * i + 1] = g_trace[i].sigma;
        out[4 * i + 2] = g_trace[i].m;
        out[4 * i + 3] = g_trace[i].names;
    }
    return n;
}

extern "C" int saix_dc3_set_window_naming(int on) {
    if (g_window_naming < 0) {
        const char *e = getenv("SAIX_WINDOW_NAMING");
        g_window_naming = (e && e[0] == '0') ? 0 : 1;
    }
    const int old = g_window_naming;
    g_window_naming = on ? 1 : 0;
    return old;
}
