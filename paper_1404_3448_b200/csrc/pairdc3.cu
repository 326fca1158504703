// pairdc3.cu -- batched longest_overlap (overlap.py:110-152 mapped over
// independent pairs, BASELINE config C4) with every pair's whole pipeline on
// chip: one CTA per pair, the pair's generalized text, suffix array and DC3
// rank table live in shared memory from the first residue load to the
// three-int64 answer.  Nothing but the pair's ASCII (in) and its answer (out)
// touches HBM.
//
// Per pair (n = |A| + |B| + 1 <= PD_NMAX, GSA codes: pad 0, separator 1,
// A..T 2..5, N 6 under NPolicy.KEEP -- GeneralizedText.build, overlap.py:83-95
// with encode's ranks shifted by one):
//
//  1. load + encode A, sep, B into T (u8) and validate every residue
//     (sequence.py:144-157; REJECT: the smallest bad offset is reported);
//  2. DC3 sample sort (suffix_index.py:221-271).  The samples -- positions
//     p % 3 != 0 below limit = n+1 if n%3==1 else n (suffix_index.py:
//     143-153), the all-padding sample n included -- are counting-sorted by
//     their first 7 characters (14-bit bucket, a monotone 2-bit map), then
//     each bucket is sorted by exact suffix comparison on T (8 characters per
//     64-bit word).  This replaces the triple naming + recursion: with the
//     whole text on chip, comparing the (rare) samples that share 7
//     characters directly costs less than renaming and recursing, and the
//     order is the same one the recursion returns (sample suffixes are
//     distinct, so their order is unique);
//  3. rank_of[sample] = 1-based rank (suffix_index.py:256-271; rank 0 for
//     positions >= limit);
//  4. non-samples i % 3 == 0 ordered by (T[i], rank_of[i+1]) -- the
//     reference's _sort_nonsamples (suffix_index.py:274-290): the class-1
//     samples in rank order give the successor order, one stable counting
//     pass by T[i] (block scan of per-character counts);
//  5. merge (suffix_index.py:173-218): merge path over the sample run
//     (pad sample dropped) and the non-sample run with the DC3 comparator
//     (char, then rank_of[+1] for mod-1, or char, char, rank_of[+2] for
//     mod-2); outputs are held in registers and written back over the two
//     runs, giving SA in shared memory;
//  6. longest_overlap's two passes (overlap.py:129-152): pass 1 = max LCP
//     over adjacent cross-sequence pairs (word compares on T), pass 2 = runs
//     of lcp >= best as a segmented (head flag, min A, min B) block scan, the
//     answer being the lexicographically smallest (min A, min B) of a run
//     holding both sequences.
//
// Pairs longer than PD_NMAX, and pairs whose sample buckets or comparisons
// exceed the on-chip work bounds (long exact repeats, e.g. poly-A runs), are
// appended to a fallback list; saix_overlap_batch runs those through the
// wave-global DC3 path of overlap.cu.  Both paths are exact, so the split
// only moves time.
#include <algorithm>
#include <mutex>
#include <vector>

#include "common.cuh"

namespace saix {

int overlap_batch_global(const u8 *seqs, const i64 *offs_host, i64 P, int keep_n, i64 *out, i64 *bad, void *ws,
                         size_t ws_bytes, cudaStream_t st);
size_t overlap_batch_global_ws(const i64 *offs_host, i64 P);

namespace pd {

constexpr int THREADS = 512;
constexpr int WARPS = THREADS / 32;
constexpr int NMAX = 20480;            // GSA residues per pair on chip
constexpr int ITEMS = NMAX / THREADS;  // merge outputs / scan items per thread (40)
constexpr int NB = 1 << 14;            // sample buckets: 7 characters x 2 bits
constexpr int TPAD = 64;               // zero bytes after T (word loads past n)
constexpr int MMAX = 2 * ((NMAX + 2) / 3) + 2;
constexpr int KMAX = (NMAX + 2) / 3 + 1;
constexpr int RKMAX = 2 * ((NMAX + 2) / 3 + 1) + 2;  // rank slots of positions 0..n+2
constexpr int SMALL = 32;      // buckets up to this size: one thread, insertion sort
constexpr int MAXBIG = 16;     // larger buckets per pair: whole CTA, rank counting
constexpr u32 WORK_MAX = 1u << 16;  // per-thread word compares in the sample sort
constexpr int LIST_CAP = 64;        // run-joining ranks walked by one thread (else block scan)

__host__ __device__ constexpr int al16(int x) { return (x + 15) & ~15; }
constexpr int OFF_T = 0;
constexpr int OFF_SS = al16(NMAX + TPAD);
constexpr int OFF_S0 = OFF_SS + al16(2 * MMAX);
constexpr int OFF_RK = OFF_S0 + al16(2 * KMAX);
constexpr int QROUND = 16;            // buckets per lane per queue round
constexpr int QCAP = QROUND * 32;     // per-warp queue of small buckets
constexpr int QTOP = QCAP * WARPS;   // queue entries (buckets of >= 2 samples: <= MMAX / 2)
constexpr int OFF_Q = OFF_RK + al16(2 * RKMAX);
constexpr int P2W = NMAX / 32 + 2;    // 2-bit packed text words
constexpr int OFF_P2 = OFF_Q + al16(2 * QCAP * WARPS);
constexpr int OFF_MISC = OFF_P2 + 8 * P2W;
constexpr int BIG_CAP = (OFF_Q - OFF_S0 - 2 * NB) / 2;  // u16 scratch after the counters
constexpr int SMEM = OFF_MISC + 1024;
static_assert(2 * NB <= OFF_Q - OFF_S0, "bucket counters must fit the S0 + RK region");
static_assert(BIG_CAP >= 1024, "big-bucket scratch");
static_assert(QCAP * WARPS >= MMAX / 2, "in-bucket sort queue: every bucket of >= 2 samples");
static_assert(MMAX + KMAX >= NMAX + 1, "SA is written over the sample + non-sample runs");
static_assert(SMEM <= 113 * 1024, "two CTAs per SM");

constexpr int NPHASE = 12;  // phase clocks (SAIX_PD_CLOCKS=1): see PD_MARK uses
struct Misc {
    unsigned long long scan64[2][WARPS + 1];
    u32 scan32[WARPS + 1];
    u32 pair;
    u32 fail;
    u32 nbig;
    u32 nlist;
    u32 big[MAXBIG][2];
    u32 red32[WARPS];  // [0], [1]: the in-bucket sort queue's length / next entry
    unsigned long long red64[WARPS];
    u32 seg[WARPS + 1][3];
    long long t_prev;
    long long acc[NPHASE];
    long long tmax, tsum, acc2[2];
};
static_assert(sizeof(Misc) <= 1024, "misc");

// thread 0's clock since the previous mark, charged to phase k (after a barrier,
// so a phase's time includes waiting for its slowest thread)
#define PD_MARK(k)                                         \
    do {                                                   \
        if (CLK && threadIdx.x == 0) {                     \
            const long long t_ = clock64();                \
            ms.acc[k] += t_ - ms.t_prev;                   \
            ms.t_prev = t_;                                \
        }                                                  \
    } while (0)

// 8 characters at T[off..off+8) (little endian: byte k = T[off + k]): three
// aligned 32-bit shared loads and two byte permutes
__device__ __forceinline__ u64 ld8(const u8 *T, u32 off) {
    const u32 *w = reinterpret_cast<const u32 *>(T + (off & ~3u));
    const u32 a = w[0], b = w[1], c = w[2];
    const u32 sel = 0x3210u + (off & 3u) * 0x1111u;
    return ((u64)__byte_perm(b, c, sel) << 32) | __byte_perm(a, b, sel);
}

// The pair text for suffix comparisons.  Packed mode (no N): the residues
// 2-bit packed, 32 characters per 64-bit word; the separator (position nA)
// and the end (n) are unique, so a comparison runs over at most
// L = min(lim(i), lim(j)) residues, and if those are equal the suffix that
// reaches its special first is smaller (a special, code <= 1, is below every
// residue), on equal distance the one reaching the end (pad 0) is below the
// one reaching the separator (1).  Byte mode (NPolicy.KEEP): 8 codes per step
// on T, where pad 0 < separator 1 < residues makes plain byte order exact.
struct Txt {
    const u8 *T;
    const u64 *P2;
    u32 nA, n;
    bool packed;
    __device__ __forceinline__ u32 step() const { return packed ? 32u : 8u; }
    __device__ __forceinline__ u32 lim(u32 i) const { return i <= nA ? nA - i : n - i; }
    __device__ __forceinline__ u64 ld32(u32 i) const {
        const u32 w = i >> 5, sh = 2u * (i & 31u);
        return (P2[w] >> sh) | ((P2[w + 1] << 1) << (63u - sh));
    }
    // One comparison step of suffixes i != j at offset h.  0: equal so far
    // (continue at h + step()); 1: i < j; 2: i > j.  When decided, *lcp is
    // their longest common prefix.
    // packed step on the 32-character words wi = ld32(i + h), wj = ld32(j + h)
    // (h < L): the first differing character codes come from the words
    __device__ __forceinline__ int cmp_words(u32 i, u32 j, u32 h, u64 wi, u64 wj, u32 &lcp) const {
        const u32 li = lim(i), lj = lim(j), L = min(li, lj);
        const u64 x = wi ^ wj;
        if (!x && h + 32u < L) return 0;
        const u32 b = x ? (u32)(__ffsll((long long)x) - 1) & ~1u : 64u;
        const u32 d = h + (b >> 1);
        if (d < L) {
            lcp = d;
            return ((wi >> b) & 3u) < ((wj >> b) & 3u) ? 1 : 2;
        }
        lcp = L;
        if (li != lj) return li < lj ? 1 : 2;
        return i > nA ? 1 : 2;  // equal distance: the end (pad) is below the separator
    }
    __device__ __forceinline__ int cmp(u32 i, u32 j, u32 h, u32 &lcp) const {
        if (packed) {
            if (h < min(lim(i), lim(j))) return cmp_words(i, j, h, ld32(i + h), ld32(j + h), lcp);
            const u32 li = lim(i), lj = lim(j);
            lcp = min(li, lj);
            if (li != lj) return li < lj ? 1 : 2;
            return i > nA ? 1 : 2;
        }
        const u64 a = ld8(T, i + h), b = ld8(T, j + h);
        if (a == b) return 0;
        const u32 bit = (u32)(__ffsll((long long)(a ^ b)) - 1) & ~7u;
        lcp = h + (bit >> 3);
        return ((a >> bit) & 0xFFu) < ((b >> bit) & 0xFFu) ? 1 : 2;
    }
};

// suffix i < suffix j (i != j); `work` counts 8-character steps.  Distinct
// suffixes differ before the shorter reaches the zero padding.
__device__ __forceinline__ bool suf_less(const u8 *T, u32 i, u32 j, u32 &work) {
    for (u32 h = 0;; h += 8) {
        const u64 a = ld8(T, i + h), b = ld8(T, j + h);
        if (a != b) {
            const int s = (__ffsll((long long)(a ^ b)) - 1) & ~7;
            return ((a >> s) & 0xFFu) < ((b >> s) & 0xFFu);
        }
        work++;
    }
}

// exact LCP of suffixes i != j (bounded by the separator / end: both unique)
__device__ __forceinline__ u32 suf_lcp(const u8 *T, u32 i, u32 j) {
    for (u32 h = 0;; h += 8) {
        const u64 x = ld8(T, i + h) ^ ld8(T, j + h);
        if (x) return h + ((u32)(__ffsll((long long)x) - 1) >> 3);
    }
}

// lcp(i, j) >= need ?
__device__ __forceinline__ bool lcp_at_least(const u8 *T, u32 i, u32 j, u32 need) {
    for (u32 h = 0; h < need; h += 8) {
        const u64 x = ld8(T, i + h) ^ ld8(T, j + h);
        if (x) return h + ((u32)(__ffsll((long long)x) - 1) >> 3) >= need;
    }
    return true;
}

// Bucket of the suffix at s from its first 7 codes, monotone in suffix order:
// A..T -> 0..3; pad / separator -> 0 and every later digit 0; N -> 3 and
// every later digit 3.  (Equal digits with different codes: the smaller code
// is pad/sep, whose zero fill keeps it <=, or the larger is N, whose 3-fill
// keeps it >=.)
__device__ __forceinline__ u32 bucket_of(const u8 *T, u32 s) {
    const u64 w = ld8(T, s);
    const u64 w7 = w & 0x00FFFFFFFFFFFFFFull;
    // fast path (no pad / separator / N among the 7): digit = code - 2, all
    // bytes at once; codes < 128, so byte-wise adds never carry
    const bool ge2 = ((w7 + 0x007E7E7E7E7E7E7Eull) & 0x0080808080808080ull) == 0x0080808080808080ull;
    const bool ge6 = ((w7 + 0x007A7A7A7A7A7A7Aull) & 0x0080808080808080ull) != 0;
    if (ge2 && !ge6) {
        // byte k holds digit k (<= 3); pack with character 0 most significant
        u64 d = w7 - 0x0002020202020202ull;
        const u32 lo = (u32)d, hi = (u32)(d >> 32);
        const u32 r = __byte_perm(lo, 0u, 0x0123);               // bytes 3..0 = c0 c1 c2 c3
        const u32 q = __byte_perm(hi, 0u, 0x4012);               // bytes 2..0 = c4 c5 c6
        const u32 r4 = (r | (r >> 6)) & 0x000F000Fu, r8 = (r4 | (r4 >> 12)) & 0xFFu;  // 8 bits: c0..c3
        const u32 q4 = (q | (q >> 6)) & 0x000F000Fu, q6 = (q4 >> 16 << 4) | (q4 & 0xFu);   // 6 bits: c4..c6
        return (r8 << 6) | q6;
    }
    u32 b = 0, mode = 0;  // 0 normal, 1 zero fill, 2 three fill
#pragma unroll
    for (int k = 0; k < 7; k++) {
        const u32 c = (u32)(w >> (8 * k)) & 0xFFu;
        u32 d;
        if (mode == 1) d = 0;
        else if (mode == 2) d = 3;
        else if (c <= 1) {
            d = 0;
            mode = 1;
        } else if (c >= 6) {
            d = 3;
            mode = 2;
        } else d = c - 2;
        b = (b << 2) | d;
    }
    return b;
}

// rank slot of a sample-class position p (p % 3 != 0)
__device__ __forceinline__ u32 slot(u32 p) { return 2u * (p / 3u) + (p % 3u) - 1u; }

// DC3 merge comparator (suffix_index.py:192-202): sample a < non-sample b ?
__device__ __forceinline__ bool sample_less(const u8 *T, const u16 *RK, u32 a, u32 b) {
    const u32 ca = T[a], cb = T[b];
    if (ca != cb) return ca < cb;
    if (a % 3u == 1u) return RK[slot(a + 1)] < RK[slot(b + 1)];
    const u32 ca1 = T[a + 1], cb1 = T[b + 1];
    if (ca1 != cb1) return ca1 < cb1;
    return RK[slot(a + 2)] < RK[slot(b + 2)];
}

// The same comparator as 32-bit keys (codes < 8, ranks < 2^16):
// K1(x) = T[x] << 16 | R(x+1), K2(x) = T[x] << 24 | T[x+1] << 16 | R(x+2);
// a mod-1 sample compares by K1, a mod-2 sample by K2.
__device__ __forceinline__ u32 key1s(const u8 *T, const u16 *RK, u32 a) {  // a % 3 == 1: slot(a+1) = 2(a/3)+1
    return ((u32)T[a] << 16) | RK[2u * (a / 3u) + 1u];
}
__device__ __forceinline__ u32 key2s(const u8 *T, const u16 *RK, u32 a) {  // a % 3 == 2: slot(a+2) = 2(a/3+1)
    return ((u32)T[a] << 24) | ((u32)T[a + 1] << 16) | RK[2u * (a / 3u) + 2u];
}
__device__ __forceinline__ void key12n(const u8 *T, const u16 *RK, u32 b, u32 &k1, u32 &k2) {  // b % 3 == 0
    const u32 q = 2u * (b / 3u), c0 = T[b], c1 = T[b + 1];
    k1 = (c0 << 16) | RK[q];
    k2 = (c0 << 24) | (c1 << 16) | RK[q + 1];
}

// GSA code of one ASCII residue (rank + 1; 0 = illegal)
__device__ __forceinline__ u32 code_of(u32 c, int keep_n) {
    switch (c) {
        case 'A': return 2;
        case 'C': return 3;
        case 'G': return 4;
        case 'T': return 5;
        case 'N': return keep_n ? 6u : 0u;
        default: return 0;
    }
}

// global loads of the pair's ASCII: streamed batches (the copy engine is
// still writing other parts of the buffer) read at L2 only, so no line with
// not-yet-copied bytes can sit stale in L1 / the non-coherent path
template <bool STREAM>
__device__ __forceinline__ uint4 ld_seq16(const uint4 *p) { return STREAM ? __ldcg(p) : __ldg(p); }
template <bool STREAM>
__device__ __forceinline__ u8 ld_seq1(const u8 *p) { return STREAM ? __ldcg(p) : __ldg(p); }

// T[dst + i] = code(src[i]) for i < len; returns the smallest bad i (or len)
template <bool STREAM>
__device__ __forceinline__ i64 load_codes(const u8 *__restrict__ src, i64 len, u8 *T, u32 dst, int keep_n) {
    i64 bad = len;
    const uintptr_t a0 = (uintptr_t)src;
    const i64 head = (i64)((16 - (a0 & 15)) & 15) < len ? (i64)((16 - (a0 & 15)) & 15) : len;
    for (i64 i = threadIdx.x; i < head; i += THREADS) {
        u32 c = code_of(ld_seq1<STREAM>(src + i), keep_n);
        if (!c) {
            bad = i < bad ? i : bad;
            c = 2;
        }
        T[dst + i] = (u8)c;
    }
    const uint4 *v = reinterpret_cast<const uint4 *>(src + head);
    const i64 nv = (len - head) >> 4;
    for (i64 q = threadIdx.x; q < nv; q += THREADS) {
        const uint4 x = ld_seq16<STREAM>(v + q);
        const u32 w[4] = {x.x, x.y, x.z, x.w};
        const i64 base = head + 16 * q;
        // SWAR: bits 3..1 of A C T G N are 0 1 2 3 7 -- a byte permute maps
        // them to the codes and to the letter each index must be; bytes that
        // are not that letter are illegal (code 2 stands in, as below)
        const u32 codes_lo = 0x04050302u, codes_hi = keep_n ? 0x06000000u : 0u;
        const u32 lets_lo = 0x47544341u, lets_hi = keep_n ? 0x4E000000u : 0u;
#pragma unroll
        for (int k = 0; k < 4; k++) {
            const u32 ix = (w[k] >> 1) & 0x07070707u;
            const u32 sel = (ix & 7u) | ((ix >> 4) & 0x70u) | ((ix >> 8) & 0x700u) | ((ix >> 12) & 0x7000u);
            const u32 want = __byte_perm(lets_lo, lets_hi, sel);
            const u32 ok = __vcmpeq4(w[k], want) & ~__vcmpeq4(want, 0u);
            u32 c = (__byte_perm(codes_lo, codes_hi, sel) & ok) | (0x02020202u & ~ok);
            if (ok != 0xFFFFFFFFu) {
                const i64 at = base + 4 * k + ((__ffs(~ok) - 1) >> 3);
                bad = at < bad ? at : bad;
            }
#pragma unroll
            for (int y = 0; y < 4; y++) T[dst + base + 4 * k + y] = (u8)(c >> (8 * y));
        }
    }
    for (i64 i = head + 16 * nv + threadIdx.x; i < len; i += THREADS) {
        u32 c = code_of(ld_seq1<STREAM>(src + i), keep_n);
        if (!c) {
            bad = i < bad ? i : bad;
            c = 2;
        }
        T[dst + i] = (u8)c;
    }
    return bad;
}

// validation only (pairs that do not fit on chip)
template <bool STREAM>
__device__ __forceinline__ i64 check_codes(const u8 *__restrict__ src, i64 len, int keep_n) {
    i64 bad = len;
    for (i64 i = threadIdx.x; i < len; i += THREADS)
        if (!code_of(ld_seq1<STREAM>(src + i), keep_n) && i < bad) bad = i;
    return bad;
}

template <class V>
__device__ __forceinline__ V warp_incl_add(V v) {
    const int lane = lane_id();
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        V y = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += y;
    }
    return v;
}

// block exclusive sum (all THREADS threads); sh holds WARPS+1 entries
template <class V>
__device__ __forceinline__ V block_exsum(V v, V &total, V *sh) {
    const int w = threadIdx.x >> 5, lane = lane_id();
    V inc = warp_incl_add(v);
    if (lane == 31) sh[w] = inc;
    __syncthreads();
    if (w == 0) {
        V x = lane < WARPS ? sh[lane] : V(0);
        V xi = warp_incl_add(x);
        if (lane < WARPS) sh[lane] = xi - x;
        if (lane == WARPS - 1) sh[WARPS] = xi;
    }
    __syncthreads();
    V ex = sh[w] + inc - v;
    total = sh[WARPS];
    __syncthreads();
    return ex;
}

struct Seg {  // segmented-min state: head flag + min A / min B position
    u32 f, a, b;
};
constexpr u32 kInf = 0xFFFFFFFFu;
__device__ __forceinline__ Seg seg_combine(Seg l, Seg r) {
    if (r.f) return r;
    return Seg{l.f, min(l.a, r.a), min(l.b, r.b)};
}
__device__ __forceinline__ Seg seg_shfl_up(Seg s, int o) {
    return Seg{__shfl_up_sync(0xffffffffu, s.f, o), __shfl_up_sync(0xffffffffu, s.a, o),
               __shfl_up_sync(0xffffffffu, s.b, o)};
}

__device__ __forceinline__ Seg block_seg_exclusive(Seg v, Misc &ms) {
    const int w = threadIdx.x >> 5, lane = lane_id();
    Seg inc = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        Seg y = seg_shfl_up(inc, o);
        if (lane >= o) inc = seg_combine(y, inc);
    }
    if (lane == 31) {
        ms.seg[w][0] = inc.f;
        ms.seg[w][1] = inc.a;
        ms.seg[w][2] = inc.b;
    }
    __syncthreads();
    if (w == 0) {
        Seg x = lane < WARPS ? Seg{ms.seg[lane][0], ms.seg[lane][1], ms.seg[lane][2]} : Seg{0u, kInf, kInf};
        Seg xi = x;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            Seg y = seg_shfl_up(xi, o);
            if (lane >= o) xi = seg_combine(y, xi);
        }
        Seg ex = seg_shfl_up(xi, 1);
        if (lane == 0) ex = Seg{0u, kInf, kInf};
        if (lane < WARPS) {
            ms.seg[lane][0] = ex.f;
            ms.seg[lane][1] = ex.a;
            ms.seg[lane][2] = ex.b;
        }
    }
    __syncthreads();
    Seg prev = seg_shfl_up(inc, 1);
    Seg carry{ms.seg[w][0], ms.seg[w][1], ms.seg[w][2]};
    if (lane > 0) carry = seg_combine(carry, prev);
    __syncthreads();
    return carry;
}

// Streamed batches (saix_overlap_batch_stream): the batch is copied in C
// chunks; bounds[c] = pairs available once chunks 0..c-1 have landed.  Chunk
// sizes ramp up from `first` pairs (one per CTA) by doubling to `per`, and
// mirror that ramp down at the end: the kernel starts after a short copy and
// finishes shortly after the last one.  Returns C (<= kMaxStreamChunks).
constexpr u32 kMaxStreamChunks = 4096 + 64;  // the caller's chunks + both ramps
__host__ __device__ inline int stream_plan(i64 P, i64 per, i64 first, u32 *bounds) {
    i64 up[24];
    int ku = 0;
    i64 sum_up = 0;
    for (i64 s = first; s < per && ku < 24; s *= 2) {
        up[ku++] = s;
        sum_up += s;
    }
    int c = 0;
    i64 done = 0;
    bounds[0] = 0;
    auto push = [&](i64 sz) {
        done = done + sz < P ? done + sz : P;
        bounds[++c] = (u32)done;
    };
    if (2 * sum_up >= P) {  // small batch: uniform chunks
        while (done < P) push(per);
        return c;
    }
    for (int k = 0; k < ku; k++) push(up[k]);
    const i64 mid_end = P - sum_up;
    while (done < mid_end) push(mid_end - done < per ? mid_end - done : per);
    for (int k = ku - 1; k >= 0; k--) push(up[k]);
    return c;
}

__global__ void k_stream_bounds(u32 *bounds, i64 P, i64 per, i64 first) { stream_plan(P, per, first, bounds); }

// STREAM: the batch's ASCII is still arriving (saix_overlap_batch_stream):
// the copy engine publishes chunk c by writing c + 1 to *ready after its
// bytes; a CTA takes pair p only once bounds[ready] > p.
template <bool CLK, bool STREAM>
__global__ void __launch_bounds__(THREADS, 2)
k_pair_dc3(const u8 *__restrict__ seqs, const i64 *__restrict__ offs, i64 P, int keep_n, i64 *__restrict__ out,
           i64 *__restrict__ bad, u32 *__restrict__ next_pair, u32 *__restrict__ nfb, u32 *__restrict__ fb,
           int nmax, unsigned long long *__restrict__ clk, const u32 *ready, const u32 *bounds) {
    extern __shared__ __align__(16) unsigned char smem[];
    u8 *T = smem + OFF_T;
    u16 *SS = reinterpret_cast<u16 *>(smem + OFF_SS);
    u16 *SA = SS;  // written over SS + S0 by the merge
    u16 *S0 = reinterpret_cast<u16 *>(smem + OFF_S0);
    u16 *RK = reinterpret_cast<u16 *>(smem + OFF_RK);
    u32 *CNT = reinterpret_cast<u32 *>(smem + OFF_S0);  // NB u16 counters, two per word
    u16 *BIGS = reinterpret_cast<u16 *>(smem + OFF_S0 + 2 * NB);
    u16 *QW = reinterpret_cast<u16 *>(smem + OFF_Q);
    u64 *P2 = reinterpret_cast<u64 *>(smem + OFF_P2);
    Misc &ms = *reinterpret_cast<Misc *>(smem + OFF_MISC);
    const u32 tid = threadIdx.x;
    // in-bucket sort counters of this warp / thread 0 (SAIX_PD_CLOCKS=1 only)
    unsigned long long clk_steps = 0, clk_wsteps = 0, clk_q = 0;
    if (CLK && tid == 0) {
        ms.t_prev = clock64();
        for (int k = 0; k < NPHASE; k++) ms.acc[k] = 0;
        ms.tmax = ms.tsum = ms.acc2[0] = ms.acc2[1] = 0;
    }

    for (;;) {
        __syncthreads();  // every shared read of the previous pair is done
        if (tid == 0) {
            ms.pair = atomicAdd(next_pair, 1u);
            ms.fail = 0;
            ms.nbig = 0;
            ms.red32[1] = ms.red32[3] = ms.red32[4] = 0;
            if (STREAM && ms.pair < P) {
                for (;;) {
                    u32 c;
                    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(c) : "l"(ready) : "memory");
                    if (bounds[c] > ms.pair) break;
                    __nanosleep(256);
                }
            }
        }
        __syncthreads();
        PD_MARK(11);
        const i64 p = ms.pair;
        if (p >= P) break;
        const i64 a0 = offs[2 * p], b0 = offs[2 * p + 1], b1 = offs[2 * p + 2];
        const i64 la = b0 - a0, lb = b1 - b0;
        if (la == 0 || lb == 0) {  // overlap.py:120-121: (0, 0, 0) before any validation
            if (tid == 0) out[3 * p] = out[3 * p + 1] = out[3 * p + 2] = 0;
            continue;
        }
        const i64 nl = la + lb + 1;
        if (nl > nmax) {  // validate here (bad offsets are relative to this call's seqs), solve elsewhere
            i64 ba = check_codes<STREAM>(seqs + a0, la, keep_n), bb = check_codes<STREAM>(seqs + b0, lb, keep_n);
            i64 mine = ba < la ? a0 + ba : (bb < lb ? b0 + bb : INT64_MAX);
            if (mine != INT64_MAX) atomicMin((unsigned long long *)bad, (unsigned long long)mine);
            if (tid == 0) fb[atomicAdd(nfb, 1u)] = (u32)p;
            continue;
        }
        const u32 n = (u32)nl, nA = (u32)la;

        // ---- 1. text + zeroed counters
        {
            i64 ba = load_codes<STREAM>(seqs + a0, la, T, 0, keep_n);
            i64 bb = load_codes<STREAM>(seqs + b0, lb, T, nA + 1, keep_n);
            i64 mine = ba < la ? a0 + ba : (bb < lb ? b0 + bb : INT64_MAX);
            if (mine != INT64_MAX) atomicMin((unsigned long long *)bad, (unsigned long long)mine);
            if (tid == 0) T[nA] = 1;  // separator (overlap.py:25)
            for (u32 i = tid; i < TPAD; i += THREADS) T[n + i] = 0;
            for (u32 i = tid; i < NB / 2; i += THREADS) CNT[i] = 0;
        }
        __syncthreads();
        PD_MARK(0);

        // ---- 2. sample buckets: sample q <-> position 3(q/2) + 1 + (q&1)
        const u32 limit = (n % 3u == 1u) ? n + 1 : n;
        const u32 qmax = 2u * ((limit + 2u) / 3u);
        const Txt tx{T, P2, nA, n, keep_n == 0};
        if (tx.packed) {  // 2-bit residues, 32 per word (specials: any value, never compared)
            const u32 nw = (n + 31u) / 32u + 1u;
            for (u32 w = tid; w < nw; w += THREADS) {
                const u32 *src = reinterpret_cast<const u32 *>(T + 32u * w);
                u64 acc = 0;
#pragma unroll
                for (int k = 0; k < 8; k++) {
                    const u32 v = ((src[k] | 0x80808080u) - 0x02020202u) & 0x03030303u;
                    const u32 b = (v | (v >> 6) | (v >> 12) | (v >> 18)) & 0xFFu;
                    acc |= (u64)b << (8 * k);
                }
                P2[w] = acc;
            }
        }
        for (u32 q = tid; q < qmax; q += THREADS) {
            const u32 s = 3u * (q >> 1) + 1u + (q & 1u);
            if (s < limit) {
                const u32 b = bucket_of(T, s);
                atomicAdd(&CNT[b >> 1], 1u << (16 * (b & 1)));
            }
        }
        __syncthreads();
        PD_MARK(1);
        // exclusive scan of the 2^14 u16 counts (32 per thread)
        {
            constexpr int W = NB / 2 / THREADS;  // 16 words per thread, moved as 16-byte
            static_assert(W % 4 == 0, "uint4 groups");  // vectors (4x fewer conflicting wavefronts)
            uint4 *C4 = reinterpret_cast<uint4 *>(CNT) + tid * (W / 4);
            u32 loc[W], sum = 0;
#pragma unroll
            for (int k = 0; k < W / 4; k++) {
                const uint4 x = C4[k];
                loc[4 * k] = x.x;
                loc[4 * k + 1] = x.y;
                loc[4 * k + 2] = x.z;
                loc[4 * k + 3] = x.w;
            }
            // the same pass builds the in-bucket sort's queue: buckets of
            // 2..SMALL samples (bit 2k / 2k+1 of wm), counted here and packed
            // above the sample count (m < 2^16), so one block scan yields both
            // offsets; buckets over SMALL (rare) go to the big list as
            // (bucket, size) -- their start is end - size after the scatter
            // Buckets of exactly 2 (w2, most of them) are queued first and
            // sorted by one compare each, outside the lock-step loop.
            u32 w2 = 0, wm = 0, bm = 0;
#pragma unroll
            for (int k = 0; k < W; k++) {
                const u32 c0 = loc[k] & 0xFFFFu, c1 = loc[k] >> 16;
                sum += c0 + c1;
                w2 |= (u32)(c0 == 2u) << (2 * k) | (u32)(c1 == 2u) << (2 * k + 1);
                wm |= (u32)(c0 - 3u <= (u32)SMALL - 3u) << (2 * k) | (u32)(c1 - 3u <= (u32)SMALL - 3u) << (2 * k + 1);
                bm |= (u32)(c0 > (u32)SMALL) << (2 * k) | (u32)(c1 > (u32)SMALL) << (2 * k + 1);
            }
            const u32 b0 = tid * (2 * W);
            while (bm) {
                const u32 b = b0 + (u32)(__ffs(bm) - 1);
                bm &= bm - 1;
                const u32 at = atomicAdd(&ms.nbig, 1u);
                if (at < MAXBIG) {
                    ms.big[at][0] = b;
                    ms.big[at][1] = reinterpret_cast<const u16 *>(CNT)[b];  // still the count
                } else ms.fail = 1;
            }
            // buckets of two fill the queue from the front (offsets from the
            // scan: samples | pairs << 16), longer ones from the back (one
            // shared atomic per thread that has any; their order is free)
            u32 tot;
            u32 run = block_exsum<u32>(sum | ((u32)__popc(w2) << 16), tot, ms.scan32);
            u32 qat2 = run >> 16;
            run &= 0xFFFFu;
            if (tid == 0) ms.red32[2] = tot >> 16;  // [0, n2): buckets of two
            u32 qat = 0;
            if (wm) qat = (u32)QTOP - atomicAdd(&ms.red32[3], (u32)__popc(wm)) - (u32)__popc(wm);
#pragma unroll
            for (int k = 0; k < W; k++) {
                const u32 lo = run, hi = run + (loc[k] & 0xFFFFu);
                run = hi + (loc[k] >> 16);
                loc[k] = lo | (hi << 16);
            }
            while (w2) {
                QW[qat2++] = (u16)(b0 + (u32)(__ffs(w2) - 1));
                w2 &= w2 - 1;
            }
            while (wm) {
                QW[qat++] = (u16)(b0 + (u32)(__ffs(wm) - 1));
                wm &= wm - 1;
            }
#pragma unroll
            for (int k = 0; k < W / 4; k++) C4[k] = make_uint4(loc[4 * k], loc[4 * k + 1], loc[4 * k + 2], loc[4 * k + 3]);
        }
        __syncthreads();
        PD_MARK(2);
        for (u32 q = tid; q < qmax; q += THREADS) {
            const u32 s = 3u * (q >> 1) + 1u + (q & 1u);
            if (s < limit) {
                const u32 b = bucket_of(T, s), sh = 16 * (b & 1);
                const u32 at = (atomicAdd(&CNT[b >> 1], 1u << sh) >> sh) & 0xFFFFu;
                SS[at] = (u16)s;
            }
        }
        __syncthreads();
        PD_MARK(3);
        const u32 m = (CNT[NB / 2 - 1] >> 16);  // end of the last bucket = number of samples

        // ---- in-bucket exact sort (counters now hold bucket ends)
        {
            const long long t_in = CLK ? clock64() : 0;
            u32 work = 0;
            const u16 *C16 = reinterpret_cast<const u16 *>(CNT);
            // Insertion sort of every bucket of 2..SMALL samples, one word compare
            // per step.  The bucket scan queued those buckets (in bucket order) in
            // one CTA-wide queue; a warp's lanes pull buckets from it as they
            // finish, so the lanes run in lock step with balanced work (a per-lane
            // loop over its own buckets serialises the lanes).
            u16 *Q = QW;
            // [0, n2): buckets of two; [q0, QTOP): buckets of 3..SMALL
            const u32 n2 = ms.red32[2], q0 = (u32)QTOP - ms.red32[3], qn = (u32)QTOP;
            const u32 lane = lane_id(), lt = lanemask_lt();
            if (CLK && tid == 0) clk_q += clock64() - t_in;
            u32 nsteps = 0, nwsteps = 0;
            // queue entries are claimed 32 at a time per warp (one atomic on the
            // shared counter per 32 buckets, not one per step); [cnext, cend) is
            // the warp's claimed, unassigned remainder (warp-uniform)
            constexpr u32 QCLAIM = 32;
            u32 t0 = 0;
            if (lane == 0) t0 = q0 + atomicAdd(&ms.red32[1], 2 * QCLAIM);
            t0 = __shfl_sync(0xffffffffu, t0, 0);
            u32 cnext = t0 + 32, cend = t0 + 2 * QCLAIM;
            u32 start = 0, end = 0, i = 0, j = 0, x = 0, h = 0;
            bool live = t0 + lane < qn;
            if (live) {
                const u32 b = Q[t0 + lane];
                start = b ? C16[b - 1] : 0u;
                end = C16[b];
                i = j = start + 1;
                x = SS[i];
            }
            while (__any_sync(0xffffffffu, live)) {
                bool done = false;
                if (CLK) {
                    nsteps += live;
                    nwsteps++;
                }
                if (live) {
                    const u32 y = SS[j - 1];
                    u32 l_;
                    const int c = tx.cmp(x, y, h, l_);
                    if (c == 0) {
                        h += tx.step();
                        if (++work > WORK_MAX) {
                            ms.fail = 1;
                            live = false;
                        }
                    } else {
                        const bool less = c == 1;
                        h = 0;
                        if (less) {
                            SS[j] = (u16)y;
                            j--;
                        }
                        if (!less || j == start) {
                            SS[j] = (u16)x;
                            if (++i < end) {
                                x = SS[i];
                                j = i;
                            } else {
                                done = true;
                            }
                        }
                    }
                }
                // lanes that finished a bucket claim the next queued ones
                const u32 dm = __ballot_sync(0xffffffffu, done);
                if (dm) {
                    const u32 need = __popc(dm), avail = cend - cnext;
                    u32 nb = 0;
                    if (need > avail) {  // warp-uniform
                        if (lane == 0) nb = q0 + atomicAdd(&ms.red32[1], QCLAIM);
                        nb = __shfl_sync(0xffffffffu, nb, 0);
                    }
                    if (done) {
                        const u32 rk = __popc(dm & lt);
                        const u32 t = rk < avail ? cnext + rk : nb + (rk - avail);
                        live = t < qn;
                        if (live) {
                            const u32 b = Q[t];
                            start = b ? C16[b - 1] : 0u;
                            end = C16[b];
                            i = j = start + 1;
                            x = SS[i];
                        }
                    }
                    if (need > avail) {
                        cnext = nb + (need - avail);
                        cend = nb + QCLAIM;
                    } else {
                        cnext += need;
                    }
                }
            }
            // buckets of two, one compare (of as many words as it takes) each:
            // warps take 32 at a time as they leave the lock-step loop, so the
            // early finishers absorb them and the phase ends balanced
            for (;;) {
                u32 base = 0;
                if (lane == 0) base = atomicAdd(&ms.red32[4], 32u);
                base = __shfl_sync(0xffffffffu, base, 0);
                if (base >= n2) break;
                const u32 t = base + lane;
                if (t < n2) {
                    const u32 b = Q[t];
                    const u32 st = b ? C16[b - 1] : 0u;
                    const u32 y = SS[st], x = SS[st + 1];
                    u32 hh = 0, l_;
                    int c;
                    while ((c = tx.cmp(x, y, hh, l_)) == 0) {
                        hh += tx.step();
                        if (++work > WORK_MAX) {
                            ms.fail = 1;
                            break;
                        }
                    }
                    if (c == 1) {
                        SS[st] = (u16)x;
                        SS[st + 1] = (u16)y;
                    }
                }
            }
            if (CLK) {
                clk_steps += __reduce_add_sync(0xffffffffu, nsteps);
                clk_wsteps += nwsteps;
                atomicMax((unsigned long long *)&ms.tmax, (unsigned long long)(clock64() - t_in));
                atomicAdd((unsigned long long *)&ms.tsum, (unsigned long long)(clock64() - t_in));
            }
        }
        __syncthreads();
        PD_MARK(4);
        if (CLK && tid == 0) {
            ms.acc2[0] += ms.tmax;
            ms.acc2[1] += ms.tsum / THREADS;
            ms.tmax = 0;
            ms.tsum = 0;
        }
        // big buckets (rare): rank counting over the whole CTA, through scratch
        {
            const u32 nbig = ms.nbig < MAXBIG ? ms.nbig : MAXBIG;
            for (u32 g = 0; g < nbig && !ms.fail; g++) {
                const u32 sz = ms.big[g][1], st = reinterpret_cast<const u16 *>(CNT)[ms.big[g][0]] - sz;
                if (sz > (u32)BIG_CAP) {
                    ms.fail = 1;  // uniform: every thread reads the same sz
                    break;
                }
                u32 work = 0;
                for (u32 i = tid; i < sz; i += THREADS) {
                    const u32 x = SS[st + i];
                    u32 r = 0;
                    for (u32 j = 0; j < sz && work <= 8 * WORK_MAX; j++)
                        if (j != i && suf_less(T, SS[st + j], x, work)) r++;
                    if (work > 8 * WORK_MAX) ms.fail = 1;
                    else BIGS[r] = (u16)x;
                }
                __syncthreads();
                for (u32 i = tid; i < sz; i += THREADS) SS[st + i] = BIGS[i];
                __syncthreads();
            }
        }
        __syncthreads();
        PD_MARK(5);
        if (ms.fail) {
            if (tid == 0) fb[atomicAdd(nfb, 1u)] = (u32)p;
            continue;
        }

        // ---- 3. rank_of (1-based; 0 for positions >= limit): zeroed here, filled
        //         in the non-sample counting pass below
        const u32 rkn = 2u * ((n + 2u) / 3u + 1u) + 2u;
        for (u32 i = tid; i < (rkn + 1) / 2; i += THREADS) reinterpret_cast<u32 *>(RK)[i] = 0;
        __syncthreads();
        PD_MARK(6);

        // ---- 4. non-samples: class-1 samples in rank order -> i = s-1,
        //         stable by T[i] (codes 1..6; 16-bit lanes, codes 1-4 / 5-6)
        {
            const u32 per = (m + THREADS - 1) / THREADS;
            const u32 r0 = tid * per, r1 = min(m, r0 + per);
            unsigned long long c0 = 0, c1 = 0;
            // the rank table is filled in the same pass (ranks and the
            // non-sample counts both read only the sorted samples)
            for (u32 r = r0; r < r1; r++) {
                const u32 s = SS[r];
                RK[slot(s)] = (u16)(r + 1);
                if (s % 3u == 1u) {
                    const u32 c = T[s - 1];
                    if (c <= 4) c0 += 1ull << (16 * (c - 1));
                    else c1 += 1ull << (16 * (c - 5));
                }
            }
            unsigned long long t0, t1;
            unsigned long long e0 = block_exsum<unsigned long long>(c0, t0, ms.scan64[0]);
            unsigned long long e1 = block_exsum<unsigned long long>(c1, t1, ms.scan64[1]);
            u32 base[7];
            u32 acc = 0;
#pragma unroll
            for (int c = 1; c <= 6; c++) {
                base[c] = acc;
                acc += (u32)(((c <= 4 ? t0 : t1) >> (16 * (c <= 4 ? c - 1 : c - 5))) & 0xFFFFu);
            }
            // this thread's cursors, packed like the counts (16-bit lanes: codes
            // 1-4 in pb0, 5-6 in pb1; every cursor < n < 2^16), so placing a
            // non-sample is one shift + add instead of a select over six
            unsigned long long pb0 = 0, pb1 = 0;
#pragma unroll
            for (int c = 1; c <= 6; c++) {
                const u32 v = base[c] + (u32)(((c <= 4 ? e0 : e1) >> (16 * (c <= 4 ? c - 1 : c - 5))) & 0xFFFFu);
                if (c <= 4) pb0 |= (unsigned long long)v << (16 * (c - 1));
                else pb1 |= (unsigned long long)v << (16 * (c - 5));
            }
            for (u32 r = r0; r < r1; r++) {
                const u32 s = SS[r];
                if (s % 3u == 1u) {
                    const u32 c = T[s - 1];
                    u32 at;
                    if (c <= 4) {
                        const u32 sh = 16u * (c - 1u);
                        at = (u32)(pb0 >> sh) & 0xFFFFu;
                        pb0 += 1ull << sh;
                    } else {
                        const u32 sh = 16u * (c - 5u);
                        at = (u32)(pb1 >> sh) & 0xFFFFu;
                        pb1 += 1ull << sh;
                    }
                    S0[at] = (u16)(s - 1);
                }
            }
        }
        __syncthreads();
        PD_MARK(7);

        // ---- 5. merge path: samples (pad sample dropped) with non-samples
        {
            const u32 pad = (n % 3u == 1u) ? 1u : 0u;
            const u16 *A = SS + pad;
            const u32 ma = m - pad, mb = (n + 2u) / 3u;
            const u32 d0 = tid * ITEMS;
            u32 outw[ITEMS / 2];
            if (d0 < n) {
                u32 lo = d0 > mb ? d0 - mb : 0u, hi = d0 < ma ? d0 : ma;
                while (lo < hi) {  // number of samples among the first d0 outputs
                    const u32 mid = (lo + hi) >> 1;
                    if (sample_less(T, RK, A[mid], S0[d0 - mid - 1])) lo = mid + 1;
                    else hi = mid;
                }
                // the comparator's keys of the two run heads, recomputed only
                // when a head advances: sample a -> its own key (K1 for mod 1,
                // K2 for mod 2); non-sample b -> both K1(b) and K2(b).  One
                // branch-free head update per output (either side).
                u32 ia = lo, ib = d0 - lo;
                u32 ha = 0, hb = 0, ka = 0, kb1 = 0, kb2 = 0;
                bool a1 = true;
                if (ia < ma) {
                    ha = A[ia];
                    a1 = ha % 3u == 1u;
                    ka = a1 ? key1s(T, RK, ha) : key2s(T, RK, ha);
                }
                if (ib < mb) {
                    hb = S0[ib];
                    key12n(T, RK, hb, kb1, kb2);
                }
#pragma unroll
                for (int q = 0; q < ITEMS; q++) {
                    u32 v = 0;
                    if (d0 + q < n) {
                        const bool ta = ib >= mb || (ia < ma && (a1 ? ka < kb1 : ka < kb2));
                        v = ta ? ha : hb;
                        ia += ta;
                        ib += !ta;
                        const bool more = ta ? ia < ma : ib < mb;
                        const u32 p = more ? (ta ? A[ia] : S0[ib]) : 0u;
                        const u32 q3 = p / 3u, pm = p - 3u * q3;
                        const u32 o1 = ta ? (pm == 1u ? 1u : 2u) : 0u, o2 = ta ? o1 : 1u;
                        const u32 c0 = T[p], c1 = T[p + 1];
                        const u32 k1 = (c0 << 16) | RK[2u * q3 + o1];
                        const u32 k2 = (c0 << 24) | (c1 << 16) | RK[2u * q3 + o2];
                        if (ta) {
                            ha = p;
                            a1 = pm == 1u;
                            ka = a1 ? k1 : k2;
                        } else {
                            hb = p;
                            kb1 = k1;
                            kb2 = k2;
                        }
                    }
                    if (q & 1) outw[q >> 1] |= v << 16;
                    else outw[q >> 1] = v;
                }
            }
            __syncthreads();
            if (d0 < n) {  // 16-byte stores (a thread's 40 outputs start 80 bytes apart:
                           // conflict-free at this width); zeros past n stay inside SS + S0
                static_assert(ITEMS % 8 == 0 && ITEMS * THREADS <= MMAX + KMAX, "whole 8-output groups");
#pragma unroll
                for (int g = 0; g < ITEMS / 8; g++)
                    if (d0 + 8 * g < n)
                        reinterpret_cast<uint4 *>(SA + d0)[g] =
                            make_uint4(outw[4 * g], outw[4 * g + 1], outw[4 * g + 2], outw[4 * g + 3]);
            }
        }
        __syncthreads();
        PD_MARK(8);

        // ---- 6a. lcp of every adjacent pair (saturated to a byte, in the
        //          rank table's place) and best = max over cross-sequence pairs
        u8 *LC = reinterpret_cast<u8 *>(RK);
        const u32 r0 = tid * ITEMS;
        u32 mx = 0;
        if (tx.packed) {
            // 2-bit text: one 32-character word compare decides almost every
            // pair; the word of rank r's suffix is reused as rank r+1's
            // predecessor word
            // SA read 8 ranks per 16-byte load, LC written 8 per 8-byte store
            // (a thread's 40 ranks start 80 / 40 bytes apart: conflict-free at
            // these widths, 4-way / 2-way for single ranks)
            if (r0 < n) {
                u32 prev = r0 ? SA[r0 - 1] : 0u;
                u64 wp = r0 ? tx.ld32(prev) : 0ull;
                // the predecessor's limit and side (0: A, 1: B, 2: the
                // separator) carry over from the previous rank; a pair is
                // cross-sequence iff the sides sum to 1
                u32 lp = tx.lim(prev), sp = prev < nA ? 0u : (prev == nA ? 2u : 1u);
                const u32 cnt = min((u32)ITEMS, n - r0);
                for (u32 q0 = 0; q0 < cnt; q0 += 8) {
                    const uint4 sv4 = reinterpret_cast<const uint4 *>(SA + r0)[q0 >> 3];  // inside SS + S0
                    const u32 svw[4] = {sv4.x, sv4.y, sv4.z, sv4.w};
                    u64 lcw = 0;
#pragma unroll
                    for (int k = 0; k < 8; k++) {
                        if (q0 + k < cnt) {
                            const u32 cur = (svw[k >> 1] >> (16 * (k & 1))) & 0xFFFFu;
                            const u64 wc = tx.ld32(cur);
                            const u32 lc = tx.lim(cur), sc = cur < nA ? 0u : (cur == nA ? 2u : 1u);
                            u32 l = 0;
                            if (r0 + q0 + k) {
                                const u32 L = min(lp, lc);
                                u64 x = wp ^ wc;
                                u32 h = 0;
                                while (!x && h + 32u < L) {
                                    h += 32u;
                                    x = tx.ld32(prev + h) ^ tx.ld32(cur + h);
                                }
                                l = x ? min(L, h + ((u32)(__ffsll((long long)x) - 1) >> 1)) : L;
                                if (sp + sc == 1u) mx = max(mx, l);
                            }
                            lcw |= (u64)min(l, 255u) << (8 * k);
                            prev = cur;
                            wp = wc;
                            lp = lc;
                            sp = sc;
                        }
                    }
                    reinterpret_cast<u64 *>(LC + r0)[q0 >> 3] = lcw;  // bytes past n: inside the RK region
                }
            }
#pragma unroll
            for (int o = 16; o; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
            if (lane_id() == 0) ms.red32[tid >> 5] = mx;
            __syncthreads();
            PD_MARK(9);
            mx = 0;
#pragma unroll
            for (int w = 0; w < WARPS; w++) mx = max(mx, ms.red32[w]);
        } else {
            // one 8-character word compare per step, lanes in lock step (see
            // the in-bucket sort); rank 0 has no predecessor (lcp 0)
            u32 q = 0, h = 0, prev = 0, cur = 0;
            bool live = r0 < n;
            if (live) {
                cur = SA[r0];
                prev = r0 ? SA[r0 - 1] : cur;
            }
            while (__any_sync(0xffffffffu, live)) {
                if (live) {
                    u32 l = 0;
                    const int c = (r0 + q == 0) ? 1 : tx.cmp(prev, cur, h, l);
                    if (c == 0) {
                        h += tx.step();
                    } else {
                        const bool cross = prev != nA && cur != nA && ((prev < nA) != (cur < nA));
                        if (cross) mx = max(mx, l);
                        LC[r0 + q] = (u8)min(l, 255u);
                        h = 0;
                        if (++q < (u32)ITEMS && r0 + q < n) {
                            prev = cur;
                            cur = SA[r0 + q];
                        } else {
                            live = false;
                        }
                    }
                }
            }
#pragma unroll
            for (int o = 16; o; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
            if (lane_id() == 0) ms.red32[tid >> 5] = mx;
            __syncthreads();
            PD_MARK(9);
            mx = 0;
#pragma unroll
            for (int w = 0; w < WARPS; w++) mx = max(mx, ms.red32[w]);
        }
        const u32 best = mx;
        if (best == 0) {
            if (tid == 0) out[3 * p] = out[3 * p + 1] = out[3 * p + 2] = 0;
            continue;
        }
        // ---- 6b. runs of lcp >= best; smallest (min A, min B) of a run with both sides.
        //          A rank r joins the run of r - 1 iff lcp(r-1, r) >= best: such
        //          ranks are few (the planted copies, the odd best-length match),
        //          so they are listed (in the free queue region) and one thread
        //          walks the runs; a long list (repetitive pairs) takes the
        //          segmented block scan below.
        const u32 bcap = min(best, 255u);
        {
            u16 *LST = QW;
            if (tid == 0) ms.nlist = 0;
            __syncthreads();
            // 8 lcp bytes per load (conflict-free at the 40-byte thread stride);
            // bytes >= bcap found four at a time (__vcmpgeu4)
            const u32 bc4 = bcap * 0x01010101u;
            for (u32 q0 = 0; q0 < (u32)ITEMS && r0 + q0 < n; q0 += 8) {
                const u64 w = reinterpret_cast<const u64 *>(LC + r0)[q0 >> 3];
                u64 hit = ((u64)__vcmpgeu4((u32)(w >> 32), bc4) << 32) | __vcmpgeu4((u32)w, bc4);
                while (hit) {
                    const u32 k = (u32)(__ffsll((long long)hit) - 1) >> 3;
                    hit &= ~(0xFFull << (8 * k));
                    const u32 r = r0 + q0 + k;
                    if (r == 0 || r >= n) continue;
                    if (best > 255u && !lcp_at_least(T, SA[r - 1], SA[r], best)) continue;  // saturated entry
                    const u32 at = atomicAdd(&ms.nlist, 1u);
                    if (at < (u32)LIST_CAP) LST[at] = (u16)r;
                }
            }
            __syncthreads();
            const u32 nl = ms.nlist;
            if (nl <= (u32)LIST_CAP) {
                if (tid == 0) {
                    for (u32 a = 1; a < nl; a++) {  // insertion sort (tiny list)
                        const u16 v = LST[a];
                        u32 b = a;
                        for (; b > 0 && LST[b - 1] > v; b--) LST[b] = LST[b - 1];
                        LST[b] = v;
                    }
                    unsigned long long win = ~0ull;
                    for (u32 a = 0; a < nl;) {
                        u32 e = a;  // run = ranks LST[a]-1 .. LST[e] (consecutive list entries)
                        while (e + 1 < nl && LST[e + 1] == LST[e] + 1u) e++;
                        u32 ma = kInf, mb = kInf;
                        for (u32 r = LST[a] - 1u; r <= (u32)LST[e]; r++) {
                            const u32 x = SA[r];
                            if (x < nA) ma = min(ma, x);
                            else if (x > nA) mb = min(mb, x);
                        }
                        if (ma != kInf && mb != kInf) win = min(win, ((unsigned long long)ma << 32) | mb);
                        a = e + 1;
                    }
                    out[3 * p] = best;
                    out[3 * p + 1] = win == ~0ull ? 0 : (i64)(win >> 32);
                    out[3 * p + 2] = win == ~0ull ? 0 : (i64)(win & 0xFFFFFFFFull) - (i64)nA - 1;
                }
                PD_MARK(10);
                continue;
            }
        }
        {
            unsigned long long head = 0;  // bit q: element r0+q starts a run; bit ITEMS: element r0+ITEMS
            for (u32 q = 0; q <= ITEMS && r0 + q < n; q++) {
                const u32 r = r0 + q, l = LC[r];
                bool h = (r == 0) || l < bcap;
                if (!h && best > 255u) h = !lcp_at_least(T, SA[r - 1], SA[r], best);  // saturated entry
                if (h) head |= 1ull << q;
            }
            if (r0 + ITEMS >= n) head |= 1ull << (n > r0 ? n - r0 : 0);  // end of the array closes a run
            Seg agg{0u, kInf, kInf};
            for (u32 q = 0; q < ITEMS && r0 + q < n; q++) {
                const u32 x = SA[r0 + q];
                agg = seg_combine(agg, Seg{(u32)((head >> q) & 1ull), x < nA ? x : kInf, x > nA ? x : kInf});
            }
            Seg run = block_seg_exclusive(agg, ms);
            unsigned long long win = ~0ull;
            for (u32 q = 0; q < ITEMS && r0 + q < n; q++) {
                const u32 x = SA[r0 + q];
                run = seg_combine(run, Seg{(u32)((head >> q) & 1ull), x < nA ? x : kInf, x > nA ? x : kInf});
                if (((head >> (q + 1)) & 1ull) && run.a != kInf && run.b != kInf)
                    win = min(win, ((unsigned long long)run.a << 32) | run.b);
            }
#pragma unroll
            for (int o = 16; o; o >>= 1) win = min(win, __shfl_xor_sync(0xffffffffu, win, o));
            if (lane_id() == 0) ms.red64[tid >> 5] = win;
            __syncthreads();
            PD_MARK(10);
            if (tid == 0) {
#pragma unroll
                for (int w = 1; w < WARPS; w++) win = min(win, ms.red64[w]);
                out[3 * p] = best;
                out[3 * p + 1] = (i64)(win >> 32);
                out[3 * p + 2] = (i64)(win & 0xFFFFFFFFull) - (i64)nA - 1;
            }
        }
    }
    if (CLK && tid == 0) {
        for (int k = 0; k < NPHASE; k++) atomicAdd(clk + k, (unsigned long long)ms.acc[k]);
        atomicAdd(clk + NPHASE, (unsigned long long)ms.acc2[0]);
        atomicAdd(clk + NPHASE + 1, (unsigned long long)ms.acc2[1]);
        atomicAdd(clk + NPHASE + 4, clk_q);
    }
    if (CLK && lane_id() == 0) {
        atomicAdd(clk + NPHASE + 2, clk_steps);
        atomicAdd(clk + NPHASE + 3, clk_wsteps);
    }
}

__global__ void k_fb_scatter(const u32 *__restrict__ list, i64 cnt, const i64 *__restrict__ sub, i64 *__restrict__ out) {
    for (i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x; i < cnt; i += (i64)gridDim.x * blockDim.x) {
        const i64 p = list[i];
        out[3 * p] = sub[3 * i];
        out[3 * p + 1] = sub[3 * i + 1];
        out[3 * p + 2] = sub[3 * i + 2];
    }
}

__global__ void k_pd_init(i64 *__restrict__ out3, i64 *__restrict__ bad, u32 *__restrict__ ctr) {
    out3[0] = out3[1] = out3[2] = 0;
    *bad = INT64_MAX;
    ctr[0] = ctr[1] = ctr[2] = 0;
}

}  // namespace pd

// Fallback capacity: the wave-global path re-runs the listed pairs in waves
// of at most kFbResidues residues (or one pair, if a pair is longer).
constexpr i64 kFbResidues = (i64)1 << 24;

struct PairsWs {
    i64 *offs;     // device copy of the caller's offsets
    u32 *ctr;      // [0] next pair, [1] fallback count
    u32 *fb;       // fallback pair list
    u32 *bounds;   // streamed chunk plan (pd::stream_plan)
    unsigned long long *clk;  // phase clocks (SAIX_PD_CLOCKS=1)
    i64 *dummy_bad;
    u8 *fseqs;     // compacted fallback residues
    i64 *fout;     // fallback results
    void *gws;     // wave-global workspace
    size_t gws_bytes;
    i64 cap;       // residues per fallback wave
};

static i64 fb_capacity(const i64 *offs, i64 P) {
    i64 cap = 0, total = 0;
    for (i64 p = 0; p < P; p++) {
        i64 la = offs[2 * p + 1] - offs[2 * p], lb = offs[2 * p + 2] - offs[2 * p + 1];
        i64 len = (la && lb) ? la + lb : 0;
        total += len;
        if (len > cap) cap = len;
    }
    if (cap < kFbResidues) cap = kFbResidues;
    if (cap > total) cap = total;
    return cap;
}

// worst-case wave-global workspace for a fallback wave of <= cap residues
// over <= pmax pairs; depends on (cap, pmax) only, so it is planned once per
// shape (the probe layout costs ~1 ms of host time at C4 size, which would
// otherwise sit in front of every call's first copy)
static size_t fb_global_ws(i64 cap, i64 pmax) {
    if (cap <= 0) return 0;
    static std::mutex mu;
    static std::vector<std::pair<std::pair<i64, i64>, size_t>> memo;
    {
        std::lock_guard<std::mutex> g(mu);
        for (auto &e : memo)
            if (e.first.first == cap && e.first.second == pmax) return e.second;
    }
    std::vector<i64> probe(2 * pmax + 1);
    for (i64 q = 0; q <= 2 * pmax; q++) probe[q] = q * (cap / (2 * pmax > 0 ? 2 * pmax : 1));
    size_t bytes = overlap_batch_global_ws(probe.data(), pmax);
    // a wave with fewer, longer pairs needs at most the single-pair workspace
    i64 one[3] = {0, cap / 2, cap};
    const size_t s1 = overlap_batch_global_ws(one, 1);
    if (s1 > bytes) bytes = s1;
    std::lock_guard<std::mutex> g(mu);
    if (memo.size() >= 16) memo.erase(memo.begin());
    memo.push_back({{cap, pmax}, bytes});
    return bytes;
}

static size_t pairs_ws(Arena &ar, const i64 *offs, i64 P, PairsWs *w) {
    PairsWs t;
    t.offs = ar.alloc<i64>(2 * P + 1);
    t.ctr = ar.alloc<u32>(4);
    t.fb = ar.alloc<u32>(P);
    t.bounds = ar.alloc<u32>(pd::kMaxStreamChunks + 1);
    t.clk = ar.alloc<unsigned long long>(pd::NPHASE + 5);
    t.dummy_bad = ar.alloc<i64>(1);
    t.cap = fb_capacity(offs, P);
    t.fseqs = ar.alloc<u8>(t.cap + 16);
    i64 pmax = t.cap / 2 + 1;  // pairs per fallback wave (each non-empty pair has >= 2 residues)
    if (pmax > P) pmax = P;
    t.fout = ar.alloc<i64>(3 * pmax + 3);
    t.gws_bytes = fb_global_ws(t.cap, pmax);
    t.gws = ar.alloc<char>((i64)t.gws_bytes);
    if (w) *w = t;
    return ar.peak;
}

}  // namespace saix

using namespace saix;

// Largest pair (GSA residues) the on-chip kernel takes; 0 sends every pair to
// the wave-global path (A/B runs and tests of the fallback).
static std::atomic<int> g_onchip_nmax{pd::NMAX};

static thread_local long long g_last_fallbacks = 0;
static unsigned long long g_phase_clk[pd::NPHASE + 5];

static bool clocks_on() {
    static const bool on = [] {
        const char *e = getenv("SAIX_PD_CLOCKS");
        return e && e[0] == '1';
    }();
    return on;
}

// Per-phase SM cycles (summed over CTAs) of the last call when SAIX_PD_CLOCKS=1:
// 0 load, 1 bucket counts, 2 scan, 3 scatter, 4 in-bucket sort, 5 big buckets,
// 6 ranks, 7 non-samples, 8 merge, 9 LCP pass 1, 10 runs pass 2, 11 pair fetch.
extern "C" int saix_overlap_batch_phase_clocks(int64_t *out, int max) {
    int k = 0;
    for (; k < max && k < pd::NPHASE + 5; k++) out[k] = (int64_t)g_phase_clk[k];
    return k;
}

extern "C" int64_t saix_overlap_batch_last_fallbacks(void) { return g_last_fallbacks; }

namespace saix {
int pd_onchip_enabled() { return g_onchip_nmax.load() != 0; }
}  // namespace saix

extern "C" int saix_overlap_batch_set_onchip(int on) {
    return g_onchip_nmax.exchange(on ? pd::NMAX : 0) != 0;
}

extern "C" size_t saix_overlap_batch_workspace_bytes(const int64_t *offs_host, int64_t npairs) {
    if (npairs < 0 || (npairs > 0 && !offs_host)) return 0;
    for (i64 p = 0; p < 2 * npairs; p++)
        if (offs_host[p + 1] < offs_host[p]) return 0;
    Arena ar;
    return pairs_ws(ar, offs_host, npairs, nullptr) + Arena::kAlign;
}

extern "C" int saix_overlap_batch(const uint8_t *seqs, const int64_t *offs_host, int64_t npairs, int keep_n,
                                  int64_t *out, int64_t *bad, void *ws, size_t ws_bytes, void *stream) {
    return saix_overlap_batch_dev(seqs, offs_host, nullptr, npairs, keep_n, out, bad, ws, ws_bytes, stream);
}

static int overlap_batch_run(const uint8_t *seqs, const int64_t *offs_host, const int64_t *offs_dev, int64_t npairs,
                             int keep_n, int64_t *out, int64_t *bad, void *ws, size_t ws_bytes, void *stream,
                             const uint8_t *host_seqs, int nchunks, void *copy_stream);

extern "C" int saix_overlap_batch_dev(const uint8_t *seqs, const int64_t *offs_host, const int64_t *offs_dev,
                                      int64_t npairs, int keep_n, int64_t *out, int64_t *bad, void *ws,
                                      size_t ws_bytes, void *stream) {
    return overlap_batch_run(seqs, offs_host, offs_dev, npairs, keep_n, out, bad, ws, ws_bytes, stream, nullptr, 0,
                             nullptr);
}

// chunk counts 1, 2, ... as pinned host words: the flag copies behind each
// chunk's bytes read from here (constant, so calls in flight never race)
static const u32 *ready_values() {
    using pd::kMaxStreamChunks;
    static u32 *vals = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        if (cudaHostAlloc(&vals, (kMaxStreamChunks + 1) * sizeof(u32), cudaHostAllocPortable) != cudaSuccess) {
            vals = nullptr;
            return;
        }
        for (u32 k = 0; k <= kMaxStreamChunks; k++) vals[k] = k;
    });
    return vals;
}

extern "C" int saix_overlap_batch_stream(const uint8_t *seqs_dev, const uint8_t *seqs_host, const int64_t *offs_host,
                                         const int64_t *offs_dev, int64_t npairs, int nchunks, int keep_n,
                                         int64_t *out, int64_t *bad, void *ws, size_t ws_bytes, void *stream,
                                         void *copy_stream) {
    if (!seqs_host || nchunks < 1 || nchunks > 4096 || !copy_stream || copy_stream == stream) {
        set_error("saix_overlap_batch_stream: invalid arguments");
        return SAIX_EINVAL;
    }
    // the kernel waits on the copies: the copy stream must not be ordered
    // behind it by the legacy default stream's implicit synchronisation
    unsigned flags = 0;
    SAIX_CUDA(cudaStreamGetFlags((cudaStream_t)copy_stream, &flags));
    if (!(flags & cudaStreamNonBlocking)) {
        set_error("saix_overlap_batch_stream: copy_stream must be created with cudaStreamNonBlocking");
        return SAIX_EINVAL;
    }
    return overlap_batch_run(seqs_dev, offs_host, offs_dev, npairs, keep_n, out, bad, ws, ws_bytes, stream,
                             seqs_host, nchunks, copy_stream);
}

static int overlap_batch_run(const uint8_t *seqs, const int64_t *offs_host, const int64_t *offs_dev, int64_t npairs,
                             int keep_n, int64_t *out, int64_t *bad, void *ws, size_t ws_bytes, void *stream,
                             const uint8_t *host_seqs, int nchunks, void *copy_stream) {
    if (npairs < 0 || (npairs > 0 && (!offs_host || !out)) || !bad) {
        set_error("saix_overlap_batch: invalid arguments");
        return SAIX_EINVAL;
    }
    for (i64 p = 0; p < 2 * npairs; p++)
        if (offs_host[p + 1] < offs_host[p]) {
            set_error("saix_overlap_batch: offsets must be non-decreasing");
            return SAIX_EINVAL;
        }
    cudaStream_t st = (cudaStream_t)stream;
    const i64 P = npairs;
    Arena ar{(char *)ws, ws_bytes};
    PairsWs w;
    pairs_ws(ar, offs_host, P, &w);
    SAIX_ARENA_OK(ar);
    g_last_fallbacks = 0;
    pd::k_pd_init<<<1, 1, 0, st>>>(out, bad, w.ctr);  // out[0..2] zero, bad = INT64_MAX
    SAIX_LAUNCHED();
    if (P == 0) return SAIX_OK;
    // offsets: the caller's device copy, or uploaded here (a pageable H2D copy
    // queues behind any bulk H2D already in flight on the copy engine)
    const i64 *doffs = offs_dev;
    if (!doffs) {
        SAIX_CUDA(cudaMemcpyAsync(w.offs, offs_host, (size_t)(2 * P + 1) * 8, cudaMemcpyHostToDevice, st));
        doffs = w.offs;
    }
    {
        static DeviceFlags attr;
        if (attr.need()) {
            SAIX_CUDA(cudaFuncSetAttribute(pd::k_pair_dc3<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           pd::SMEM));
            SAIX_CUDA(cudaFuncSetAttribute(pd::k_pair_dc3<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           pd::SMEM));
            SAIX_CUDA(cudaFuncSetAttribute(pd::k_pair_dc3<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           pd::SMEM));
            attr.set();
        }
        // C4 algorithmic bytes: 4,791,288 B per 20,001-residue pair (DC3 model + LCP + scan)
        Prof prof_("pairs.dc3_onchip", 239.56 * (double)(offs_host[2 * P] - offs_host[0]), st);
        const i64 grid = P < 2 * kNumSMs ? P : 2 * kNumSMs;
        if (host_seqs) {
            // one launch over the whole batch while the copy engine streams it in:
            // chunk c's bytes, then the count c + 1 into ctr[2] (the kernel's gate)
            const u32 *vals = ready_values();
            if (!vals) {
                set_error("saix_overlap_batch_stream: pinned flag buffer");
                return SAIX_ECUDA;
            }
            cudaStream_t cs = (cudaStream_t)copy_stream;
            const i64 per = (P + nchunks - 1) / nchunks, first = grid;
            std::vector<u32> hb(pd::kMaxStreamChunks + 1);
            const int C = pd::stream_plan(P, per, first, hb.data());
            pd::k_stream_bounds<<<1, 1, 0, st>>>(w.bounds, P, per, first);  // the same plan, for the gate
            SAIX_LAUNCHED();
            cudaEvent_t e0, e1;
            SAIX_CUDA(cudaEventCreateWithFlags(&e0, cudaEventDisableTiming));
            SAIX_CUDA(cudaEventCreateWithFlags(&e1, cudaEventDisableTiming));
            SAIX_CUDA(cudaEventRecord(e0, st));  // ready = 0 and earlier readers of the buffer are done
            SAIX_CUDA(cudaStreamWaitEvent(cs, e0, 0));
            pd::k_pair_dc3<false, true><<<(unsigned)grid, pd::THREADS, pd::SMEM, st>>>(
                seqs, doffs, P, keep_n, out, bad, w.ctr, w.ctr + 1, w.fb, g_onchip_nmax.load(), nullptr, w.ctr + 2,
                w.bounds);
            SAIX_LAUNCHED();
            for (int c = 0; c < C; c++) {
                const i64 a = hb[c], b = hb[c + 1];
                const i64 lo = offs_host[2 * a], hi = offs_host[2 * b];
                if (hi > lo)
                    SAIX_CUDA(cudaMemcpyAsync((void *)(seqs + lo), host_seqs + lo, (size_t)(hi - lo),
                                              cudaMemcpyHostToDevice, cs));
                SAIX_CUDA(cudaMemcpyAsync(w.ctr + 2, vals + c + 1, 4, cudaMemcpyHostToDevice, cs));
            }
            SAIX_CUDA(cudaEventRecord(e1, cs));
            SAIX_CUDA(cudaStreamWaitEvent(st, e1, 0));  // later work on st sees the whole batch
            SAIX_CUDA(cudaEventDestroy(e0));
            SAIX_CUDA(cudaEventDestroy(e1));
        } else if (clocks_on()) {
            SAIX_CUDA(cudaMemsetAsync(w.clk, 0, sizeof(unsigned long long) * (pd::NPHASE + 5), st));
            pd::k_pair_dc3<true, false><<<(unsigned)grid, pd::THREADS, pd::SMEM, st>>>(
                seqs, doffs, P, keep_n, out, bad, w.ctr, w.ctr + 1, w.fb, g_onchip_nmax.load(), w.clk, nullptr, nullptr);
        } else {
            pd::k_pair_dc3<false, false><<<(unsigned)grid, pd::THREADS, pd::SMEM, st>>>(
                seqs, doffs, P, keep_n, out, bad, w.ctr, w.ctr + 1, w.fb, g_onchip_nmax.load(), nullptr, nullptr, nullptr);
        }
    }
    SAIX_LAUNCHED();
    u32 nfb = 0;
    SAIX_CUDA(cudaMemcpyAsync(&nfb, w.ctr + 1, sizeof(u32), cudaMemcpyDeviceToHost, st));
    if (clocks_on())
        SAIX_CUDA(cudaMemcpyAsync(g_phase_clk, w.clk, sizeof(g_phase_clk), cudaMemcpyDeviceToHost, st));
    SAIX_CUDA(cudaStreamSynchronize(st));
    g_last_fallbacks = nfb;
    if (nfb == 0) return SAIX_OK;
    // fallback pairs: compact their residues and run the wave-global path
    std::vector<u32> list(nfb);
    SAIX_CUDA(cudaMemcpyAsync(list.data(), w.fb, (size_t)nfb * 4, cudaMemcpyDeviceToHost, st));
    SAIX_CUDA(cudaStreamSynchronize(st));
    std::sort(list.begin(), list.end());
    u32 *dlist = w.fb;
    SAIX_CUDA(cudaMemcpyAsync(dlist, list.data(), (size_t)nfb * 4, cudaMemcpyHostToDevice, st));
    for (size_t i = 0; i < list.size();) {
        std::vector<i64> sub{0};
        size_t j = i;
        i64 used = 0;
        while (j < list.size()) {
            const i64 p = list[j];
            const i64 a0 = offs_host[2 * p], b0 = offs_host[2 * p + 1], b1 = offs_host[2 * p + 2];
            if (j > i && used + (b1 - a0) > w.cap) break;
            SAIX_CUDA(cudaMemcpyAsync(w.fseqs + used, seqs + a0, (size_t)(b1 - a0), cudaMemcpyDeviceToDevice, st));
            sub.push_back(used + (b0 - a0));
            used += b1 - a0;
            sub.push_back(used);
            j++;
        }
        SAIX_TRY(overlap_batch_global(w.fseqs, sub.data(), (i64)(j - i), keep_n, w.fout, w.dummy_bad, w.gws,
                                      w.gws_bytes, st));
        pd::k_fb_scatter<<<grid_for((i64)(j - i), 256), 256, 0, st>>>(dlist + i, (i64)(j - i), w.fout, out);
        SAIX_LAUNCHED();
        i = j;
    }
    return SAIX_OK;
}
