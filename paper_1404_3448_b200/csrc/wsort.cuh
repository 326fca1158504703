// wsort.cuh -- level-0 window naming for DNA texts (ranks 1..4, or the
// generalized text's residues 2..5 around one separator; N < 2^29): an MSD
// sort of the samples' 21-character windows in streaming passes.  It stands
// in for _name_triples + the recursion of _sort_samples (reference
// suffix_index.py:221-271) on level 0 and yields the same sample order; the
// separator handling follows GeneralizedText.build (overlap.py:83-95).
//
// The generic window sort (bsort.cuh over WindowSrc) builds 63-bit keys
// twice from unaligned global words, moves 16 B staging records through two
// HBM round trips and re-reads the sorted output to order 2^24 tiny buckets.
// Here the text is staged per tile in shared memory as 2-bit packed words
// (a 21-character window is three funnel shifts) and every sample becomes
// ONE 8-byte record that carries the rest of its key:
//
//   rec = chars 5..21 (34 bits) | flag (1) | low (29)
//
// flag = 1 for a full window (low = 2^29-1-pos), 0 for a window that stops
// early -- it reaches the end or the separator (at most 41 of them; digits
// from the stop on are 0 and low = distance << 1 | kind, see ws_rec).
// Sorting records as u64 orders equal 0-filled windows "nearer stop first,
// the end before the separator", which is the suffix order, so stopped
// windows stay unique names (the property DC3's padding triples give).
//
//   P1 k_ws_count   text tiles -> 2^16 fine bins (first 8 chars) in 16-bit
//                   shared-memory counters, one flush per CTA
//   (scan)          fine offsets: bucket f occupies [off[f], off[f+1]) in
//                   both staging arrays and in the sorted order
//   P2a k_ws_part1  text tiles -> records bucketed by the first 4 chars
//                   (256 coarse regions; runs of ~32 records per tile)
//   P2b k_ws_part2  each coarse region -> 256 fine buckets (chars 5..8)
//   P3  k_ws_sort   persistent CTAs, one unit of 2^G fine buckets at a time
//                   (bulk-copy prefetch of the next): counting split into
//                   4096 sub-buckets in shared memory, rank by counting inside
//                   the ~0.7-record sub-buckets, then in the same pass: the
//                   sorted sample indices (= SAc), their first two
//                   characters (CH, for the compact records), distinct-name
//                   count, tied runs for resolve_ties, and ISAc[s] = rank
//                   through pass A of the bucketed scatter (pscatter.cuh).
// Reference: suffix_index.py:221-253 (_name_triples), 256-271 (_sort_samples).
#pragma once

#include "pscatter.cuh"
#include "scan.cuh"

namespace saix {

constexpr int WS_TP = 12288;              // text positions per tile (multiple of 48)
constexpr int WS_TS = WS_TP / 3 * 2;      // samples per tile
constexpr int WS_WORDS = WS_TP / 16 + 2;  // packed words per tile (+ 32 halo characters)
constexpr int WS_FINE = 1 << 16;          // fine buckets: 8 leading characters
constexpr int WS_COARSE = 256;            // coarse regions: 4 leading characters
constexpr int WS_POS_BITS = 29;
constexpr u64 WS_POS_MASK = (1ull << WS_POS_BITS) - 1;
constexpr int WS_PT = 512;                // P2 threads
constexpr int WS_PI = 16;                 // P2 items per thread
constexpr int WS_PTILE = WS_PT * WS_PI;   // 8192 records
constexpr int WS_PI2 = 8;                 // P2b items per thread (3 CTAs per SM)
constexpr int WS_PTILE2 = WS_PT * WS_PI2; // 4096 records
constexpr int WS_ST = 512;                // P3 threads
constexpr int WS_CAP_MIN = 1024;
constexpr int WS_CAP_MAX = 10240;         // largest fine bucket P3 takes (shared memory <= 227 KB)
constexpr int WS_MAX_RUN = 4096;          // longest tied run handed to resolve_ties

// The text's alphabet: residues lo..lo+3 are the 2-bit digits 0..3; with
// sep >= 0, position sep holds the one rank below them (the generalized
// text's separator, overlap.py:25) and, like the end, stops every window
// that reaches it (its digits from there on are 0, the flag says "stopped").
struct WsAlpha {
    u32 lo;   // 1: DNA ranks 1..4; 2: generalized text (separator 1, residues 2..5)
    i64 sep;  // position of the unique separator, or -1
};

// 16 ranks -> one 32-bit word of 2-bit digits, first at the top (saturating:
// the separator's rank lo-1 packs as digit 0; its windows are masked anyway)
__device__ __forceinline__ u32 ws_pack4(u32 x, u32 lo4) {
    const u32 r = __byte_perm(__vsubus4(x, lo4), 0, 0x0123) & 0x03030303u;
    const u32 pp = r | (r >> 6);
    return ((pp >> 12) & 0xF0u) | (pp & 0xFu);
}
__device__ __forceinline__ u32 ws_pack16(uint4 v, u32 lo4) {
    return (ws_pack4(v.x, lo4) << 24) | (ws_pack4(v.y, lo4) << 16) | (ws_pack4(v.z, lo4) << 8) | ws_pack4(v.w, lo4);
}

// stage positions [p0, p0 + WS_TP + 32) as packed words; past the end reads
// as digit 0 (the flag tells end windows apart)
__device__ __forceinline__ void ws_stage(const u8 *__restrict__ t, i64 N, i64 p0, u32 *__restrict__ W,
                                         int nthreads, u32 lo) {
    const u32 lo4 = lo * 0x01010101u;
    for (int w = threadIdx.x; w < WS_WORDS; w += nthreads) {
        const i64 q = p0 + 16 * (i64)w;
        uint4 v;
        if (q + 16 <= N) {
            v = __ldg(reinterpret_cast<const uint4 *>(t + q));
        } else {
            u32 x[4];
#pragma unroll
            for (int k = 0; k < 4; k++) {
                u32 word = 0;
#pragma unroll
                for (int b = 0; b < 4; b++) {
                    const i64 at = q + 4 * k + b;
                    word |= (at < N ? (u32)t[at] : lo) << (8 * b);
                }
                x[k] = word;
            }
            v = make_uint4(x[0], x[1], x[2], x[3]);
        }
        W[w] = ws_pack16(v, lo4);
    }
}

// 21-character window at tile offset o: 42 bits, first character on top
__device__ __forceinline__ u64 ws_key(const u32 *__restrict__ W, int o) {
    const int w = o >> 4, sh = 2 * (o & 15);
    const u32 w0 = W[w], w1 = W[w + 1], w2 = W[w + 2];
    const u32 a = __funnelshift_l(w1, w0, sh);
    const u32 b = __funnelshift_l(w2, w1, sh);
    return ((u64)a << 10) | (b >> 22);
}

// local sample q of a tile: position, validity
__device__ __forceinline__ int ws_off(int q) { return 3 * (q >> 1) + 1 + (q & 1); }
__device__ __forceinline__ bool ws_valid(i64 p, const SampleLayout &L) { return p < L.n || (p == L.n && L.pad); }
// A window that reaches the separator keeps only its characters before it.
template <bool SEP>
__device__ __forceinline__ u64 ws_mask_sep(u64 key, i64 p, const WsAlpha &A) {
    if (SEP && A.sep >= p && A.sep < p + 21) {
        const int keep = (int)(A.sep - p);  // characters before the separator
        key &= ~((1ull << (42 - 2 * keep)) - 1);
    }
    return key;
}
// Low 29 bits: full window -> 2^29-1-pos (any order among equal names);
// stopped window -> (distance to its stop) << 1 | stop kind (end 0,
// separator 1): equal 0-filled keys order by the nearer stop, the end
// before the separator -- the suffix order (pad 0 < separator < residues),
// and the position follows from (distance, kind).
template <bool SEP>
__device__ __forceinline__ u64 ws_rec(u64 key, i64 p, i64 N, const WsAlpha &A) {
    u64 low;
    u64 flag = 0;
    if (SEP && A.sep >= p && A.sep < p + 21) low = ((u64)(A.sep - p) << 1) | 1ull;
    else if (p + 21 > N) low = (u64)(N - p) << 1;
    else {
        flag = 1;
        low = WS_POS_MASK - (u64)p;
    }
    return ((key & ((1ull << 34) - 1)) << 30) | (flag << 29) | low;
}
template <bool SEP>
__device__ __forceinline__ i64 ws_pos(u64 rec, i64 N, const WsAlpha &A) {
    const u64 low = rec & WS_POS_MASK;
    if ((rec >> 29) & 1) return (i64)(WS_POS_MASK - low);
    return (SEP && (low & 1)) ? A.sep - (i64)(low >> 1) : N - (i64)(low >> 1);
}
// equal names: same 21 characters and both full windows
__device__ __forceinline__ bool ws_same(u64 a, u64 b) { return ((a ^ b) >> 29) == 0 && ((a >> 29) & 1); }

// ---------------------------------------------------------------- P1
// raw text tile [p0, p0 + WS_TP + 32) -> packed words; bytes past N read as lo
__device__ __forceinline__ void ws_pack_tile(const u8 *__restrict__ raw, i64 N, i64 p0, u32 *__restrict__ W,
                                             int nthreads, u32 lo) {
    const u32 lo4 = lo * 0x01010101u;
    for (int w = threadIdx.x; w < WS_WORDS; w += nthreads) {
        const i64 q = p0 + 16 * (i64)w;
        uint4 v;
        if (q + 16 <= N) {
            v = reinterpret_cast<const uint4 *>(raw)[w];
        } else {
            u32 x[4];
#pragma unroll
            for (int k = 0; k < 4; k++) {
                u32 word = 0;
#pragma unroll
                for (int b = 0; b < 4; b++) {
                    const i64 at = q + 4 * k + b;
                    word |= (at < N ? (u32)raw[16 * w + 4 * k + b] : lo) << (8 * b);
                }
                x[k] = word;
            }
            v = make_uint4(x[0], x[1], x[2], x[3]);
        }
        W[w] = ws_pack16(v, lo4);
    }
}
constexpr int WS_RAW = (WS_WORDS * 16 + 15) & ~15;  // raw tile bytes (16-aligned)

// P1: persistent CTAs; the next text tile arrives by a bulk copy (TMA)
// while the current one is counted
template <bool SEP>
__global__ void __launch_bounds__(1024, 1)
k_ws_count(const u8 *__restrict__ t, SampleLayout L, WsAlpha A, i64 ntiles, u32 *__restrict__ hist,
           u32 *__restrict__ overflow) {
    // WS_FINE 16-bit counters, two per word, then 4096 u32 counters of the
    // first 6 characters: a fine counter can only wrap inside a CTA whose
    // 6-character counter passed 65535, so the adds need no return value
    // (fire-and-forget shared reductions) and the wrap check is one pass at
    // the end (false positives only send skewed texts to the generic sort);
    // then two raw text tiles
    extern __shared__ __align__(16) u32 ws_h16[];
    u32 *ws_c6 = ws_h16 + WS_FINE / 2;
    u8 *raw0 = reinterpret_cast<u8 *>(ws_c6 + 4096);
    __shared__ u32 W[WS_WORDS];
    __shared__ __align__(8) u64 bar;
    for (int i = threadIdx.x; i < WS_FINE / 2 + 4096; i += 1024) ws_h16[i] = 0;
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        fence_async_smem();
    }
    __syncthreads();
    const i64 N = L.n;
    auto issue = [&](i64 tile, int slot) {  // one thread: the tile's whole 16-byte words inside the text
        const i64 p0 = tile * WS_TP;
        i64 end = p0 + WS_RAW < N ? p0 + WS_RAW : N;
        const u32 bytes = end > p0 ? (u32)((end - p0) & ~(i64)15) : 0u;
        mbar_expect_tx(&bar, bytes);
        if (bytes) bulk_g2s(raw0 + slot * WS_RAW, t + p0, bytes, &bar);
    };
    bool ovf = false;
    u32 parity = 0;
    int slot = 0;
    i64 tile = blockIdx.x;
    if (threadIdx.x == 0 && tile < ntiles) issue(tile, 0);
    for (; tile < ntiles; tile += gridDim.x) {
        const i64 p0 = tile * WS_TP;
        u8 *raw = raw0 + slot * WS_RAW;
        mbar_wait(&bar, parity);
        parity ^= 1;
        // bytes the bulk copy did not cover (the text's last < 16) come from global
        const i64 covered = p0 + (((p0 + WS_RAW < N ? p0 + WS_RAW : N) - p0) & ~(i64)15);
        if (covered < N && covered < p0 + WS_RAW)
            for (i64 a = covered + threadIdx.x; a < N && a < p0 + WS_RAW; a += 1024)
                raw[a - p0] = t[a];
        __syncthreads();
        ws_pack_tile(raw, N, p0, W, 1024, A.lo);
        __syncthreads();  // raw[slot] consumed: the next tile may land in the other slot
        if (threadIdx.x == 0 && tile + gridDim.x < ntiles) {
            fence_async_smem();
            issue(tile + gridDim.x, slot ^ 1);
        }
        slot ^= 1;
#pragma unroll 4
        for (int q = threadIdx.x; q < WS_TS; q += 1024) {
            const int o = ws_off(q);
            if (!ws_valid(p0 + o, L)) continue;
            const u32 f = (u32)(ws_mask_sep<SEP>(ws_key(W, o), p0 + o, A) >> 26);
            atomicAdd(&ws_h16[f >> 1], 1u << (16 * (f & 1)));
            atomicAdd(&ws_c6[f >> 4], 1u);
        }
        __syncthreads();  // W is rewritten by the next tile
    }
    __syncthreads();
    for (int i = threadIdx.x; i < 4096; i += 1024) ovf |= ws_c6[i] > 0xFFFFu;
    for (int i = threadIdx.x; i < WS_FINE / 2; i += 1024) {
        const u32 v = ws_h16[i];
        if (v & 0xFFFFu) atomicAdd(&hist[2 * i], v & 0xFFFFu);
        if (v >> 16) atomicAdd(&hist[2 * i + 1], v >> 16);
    }
    if (ovf) atomicMax(overflow, 1u);
}
constexpr int WS_COUNT_SMEM = WS_FINE * 2 + 16384 + 2 * WS_RAW;

// fine offsets (exclusive), staging cursors and the largest bucket
struct WsHistIn {
    const u32 *hist;
    __device__ u32 operator()(i64 i) const { return hist[i]; }
};
struct WsOffOut {
    u32 *off, *cur_fine, *cur_coarse, *maxb;
    __device__ void operator()(i64 i, u32 excl, u32 v) const {
        off[i] = excl;
        cur_fine[i] = excl;
        if ((i & (WS_COARSE - 1)) == 0) cur_coarse[i / WS_COARSE] = excl;
        const u32 mx = __reduce_max_sync(__activemask(), v);
        if (lane_id() == __ffs(__activemask()) - 1 && mx) atomicMax(maxb, mx);
    }
};

// P2b tile table: coarse region c owns tiles [tstart[c], tstart[c+1])
__global__ void __launch_bounds__(WS_COARSE) k_ws_tiles(const u32 *__restrict__ off, i64 m, u32 *__restrict__ tstart) {
    __shared__ u32 sh_warp[WS_COARSE / 32 + 1];
    const int c = threadIdx.x;
    const i64 lo = off[c * WS_COARSE];
    const i64 hi = c + 1 < WS_COARSE ? (i64)off[(c + 1) * WS_COARSE] : m;
    const u32 nt = (u32)ceil_div(hi - lo, (i64)WS_PTILE2);
    u32 excl;
    const u32 tot = block_exclusive_scan<WS_COARSE>(nt, excl, sh_warp);
    tstart[c] = excl;
    if (c == 0) tstart[WS_COARSE] = tot;
}

// largest P3 unit (2^G consecutive fine buckets)
__global__ void k_ws_unit_max(const u32 *__restrict__ off, i64 m, int G, u32 *__restrict__ out) {
    const u32 units = WS_FINE >> G;
    u32 mx = 0;
    for (u32 u = blockIdx.x * blockDim.x + threadIdx.x; u < units; u += gridDim.x * blockDim.x) {
        const i64 lo = off[u << G], hi = u + 1 < units ? (i64)off[(u + 1) << G] : m;
        mx = (u32)(hi - lo) > mx ? (u32)(hi - lo) : mx;
    }
    for (int o = 16; o; o >>= 1) {
        const u32 y = __shfl_xor_sync(0xffffffffu, mx, o);
        mx = y > mx ? y : mx;
    }
    if (lane_id() == 0 && mx) atomicMax(out, mx);
}

// Block-level bucketed write of WS_PT*PI records into runs reserved on
// absolute cursors: item r goes to bucket bk[r] (< 256), cursor cur[bk].
template <int PI>
__device__ __forceinline__ void ws_block_emit(const u64 (&rec)[PI], const u8 (&bk)[PI], const bool (&ok)[PI],
                                              u32 *__restrict__ cur, u64 *__restrict__ out, u64 *__restrict__ sh_rec,
                                              u8 *__restrict__ sh_bk, u32 *__restrict__ sh_cnt, u32 *__restrict__ sh_start,
                                              u32 *__restrict__ sh_base) {
    __shared__ u32 sh_warp[WS_PT / 32 + 1];
    if (threadIdx.x < 256) sh_cnt[threadIdx.x] = 0;
    __syncthreads();
    u32 slot[PI];
#pragma unroll
    for (int r = 0; r < PI; r++)
        if (ok[r]) slot[r] = atomicAdd(&sh_cnt[bk[r]], 1u);
    __syncthreads();
    const u32 c = threadIdx.x < 256 ? sh_cnt[threadIdx.x] : 0u;
    u32 excl;
    const u32 tot = block_exclusive_scan<WS_PT>(c, excl, sh_warp);
    // the run reservation's round trip overlaps the staging loop
    const u32 res = (threadIdx.x < 256 && c) ? atomicAdd(&cur[threadIdx.x], c) : 0u;
    if (threadIdx.x < 256) sh_start[threadIdx.x] = excl;
    __syncthreads();
#pragma unroll
    for (int r = 0; r < PI; r++)
        if (ok[r]) {
            const u32 at = sh_start[bk[r]] + slot[r];
            sh_rec[at] = rec[r];
            sh_bk[at] = bk[r];
        }
    if (threadIdx.x < 256) sh_base[threadIdx.x] = res;
    __syncthreads();
    for (u32 x = threadIdx.x; x < tot; x += WS_PT) {
        const u32 b = sh_bk[x];
        __stcs(out + sh_base[b] + (x - sh_start[b]), sh_rec[x]);
    }
}
constexpr size_t WS_P2_SMEM = (size_t)WS_PTILE * 9 + 3 * 256 * 4;
constexpr size_t WS_P2B_SMEM = (size_t)WS_PTILE2 * 9 + 3 * 256 * 4;

// ---------------------------------------------------------------- P2a
template <bool SEP>
__global__ void __launch_bounds__(WS_PT, 2)
k_ws_part1(const u8 *__restrict__ t, SampleLayout L, WsAlpha A, u32 *__restrict__ cur_coarse,
           u64 *__restrict__ stageA) {
    extern __shared__ __align__(16) unsigned char ws_smem[];
    u64 *sh_rec = reinterpret_cast<u64 *>(ws_smem);
    u8 *sh_bk = ws_smem + (size_t)WS_PTILE * 8;
    u32 *sh_cnt = reinterpret_cast<u32 *>(sh_bk + WS_PTILE), *sh_start = sh_cnt + 256, *sh_base = sh_start + 256;
    __shared__ u32 W[WS_WORDS];
    const i64 p0 = (i64)blockIdx.x * WS_TP;
    ws_stage(t, L.n, p0, W, WS_PT, A.lo);
    __syncthreads();
    u64 rec[WS_PI];
    u8 bk[WS_PI];
    bool ok[WS_PI];
#pragma unroll
    for (int r = 0; r < WS_PI; r++) {
        const int o = ws_off(r * WS_PT + threadIdx.x);
        const i64 p = p0 + o;
        ok[r] = ws_valid(p, L);
        const u64 key = ws_mask_sep<SEP>(ws_key(W, o), p, A);
        rec[r] = ws_rec<SEP>(key, p, L.n, A);
        bk[r] = (u8)(key >> 34);
    }
    ws_block_emit(rec, bk, ok, cur_coarse, stageA, sh_rec, sh_bk, sh_cnt, sh_start, sh_base);
}

// ---------------------------------------------------------------- P2b
__global__ void __launch_bounds__(WS_PT, 3)
k_ws_part2(const u64 *__restrict__ stageA, const u32 *__restrict__ off, const u32 *__restrict__ tstart, i64 m,
           u32 *__restrict__ cur_fine, u64 *__restrict__ stageB) {
    extern __shared__ __align__(16) unsigned char ws_smem[];
    u64 *sh_rec = reinterpret_cast<u64 *>(ws_smem);
    u8 *sh_bk = ws_smem + (size_t)WS_PTILE2 * 8;
    u32 *sh_cnt = reinterpret_cast<u32 *>(sh_bk + WS_PTILE2), *sh_start = sh_cnt + 256, *sh_base = sh_start + 256;
    const u32 b = blockIdx.x;
    if (b >= tstart[WS_COARSE]) return;
    int c = 0;  // largest region with tstart[c] <= b
#pragma unroll
    for (int s = 128; s; s >>= 1)
        if (tstart[c + s] <= b) c += s;
    const i64 lo = off[c * WS_COARSE] + (i64)(b - tstart[c]) * WS_PTILE2;
    const i64 hi_r = c + 1 < WS_COARSE ? (i64)off[(c + 1) * WS_COARSE] : m;
    const i64 hi = lo + WS_PTILE2 < hi_r ? lo + WS_PTILE2 : hi_r;
    u64 rec[WS_PI2];
    u8 bk[WS_PI2];
    bool ok[WS_PI2];
#pragma unroll
    for (int r = 0; r < WS_PI2; r++) {
        const i64 x = lo + r * WS_PT + threadIdx.x;
        ok[r] = x < hi;
        rec[r] = ok[r] ? __ldcs(stageA + x) : 0ull;
    }
#pragma unroll
    for (int r = 0; r < WS_PI2; r++) bk[r] = (u8)(rec[r] >> 56);
    ws_block_emit(rec, bk, ok, cur_fine + c * WS_COARSE, stageB, sh_rec, sh_bk, sh_cnt, sh_start, sh_base);
}

// ---------------------------------------------------------------- P3
// Persistent: CTA b sorts fine buckets b, b + grid, ...  The next bucket's
// records arrive by a bulk copy (TMA, cp.async.bulk) into IN while the
// current one is ranked and written.  Per bucket (L records, all sharing
// characters 1..8):
//   split   IN -> S by the next 12 bits (4096 sub-buckets, ~0.7 records
//           each on random text) with shared-memory atomics
//   rank    every record counts, inside its sub-bucket, the smaller records
//           (its rank), the smaller records of the same name (0: it heads
//           its name) and the records of its name (the tied run's length);
//           the sample index lands at its rank in R (u32)
//   emit    R streamed out as the sorted order; (sample, rank) pairs bucketed
//           in shared memory and written as runs = pass A of the ISA scatter
// Equal names share characters 1..14, hence a sub-bucket: no comparison
// crosses one.  Sub-buckets over WS_BIG_SUB records (low-complexity text)
// set the overflow flag and the caller takes the generic window sort.
// scal (resolve_ties layout): [2] tied runs, [4] overflow, [5] distinct names;
// [8] a sub-bucket over WS_BIG_SUB
constexpr int WS_BIG_SUB = 256;
// A work unit of P3 is a group of 2^G consecutive fine buckets (G = 0 at
// C3-size levels; small levels group buckets so a unit still holds ~3 k
// records).  Its 4096 sub-buckets are record bits SHIFT+11 .. SHIFT: the
// group's own low G bits of characters 5..8 (bits 63..56), then the next
// bits -- records of a unit share bits 63..SHIFT+12, so sub-bucket order is
// suffix order and the unit's sorted order is consecutive ranks.
template <int G>
struct WsSub {
    static constexpr int SUBS = 4096;
    static constexpr int SHIFT = 44 + G;
    static constexpr int HI = SHIFT - 32;        // u32 compare window: bits SHIFT-1 .. HI
    static constexpr int NAME = 29 - HI;         // name bits (.. flag) inside that window
    static constexpr u32 UNITS = WS_FINE >> G;
    __device__ __forceinline__ static u32 of(u64 r) { return (u32)(r >> SHIFT) & (SUBS - 1); }
};

template <int G, bool SEP>
__global__ void __launch_bounds__(WS_ST, 3)
k_ws_sort(const u64 *__restrict__ stageB, const u32 *__restrict__ off, i64 m, i64 m1, int capA,
          u32 *__restrict__ sorted, PsPlan plan, uint2 *__restrict__ stage1, u32 *__restrict__ rs,
          u32 *__restrict__ rl, u32 cap_runs, u32 *__restrict__ scal, u8 *__restrict__ ch, i64 N, WsAlpha A) {
    extern __shared__ __align__(16) unsigned char ws_smem[];
    u64 *IN = reinterpret_cast<u64 *>(ws_smem);
    u64 *S = IN + capA + 2;
    u32 *R = reinterpret_cast<u32 *>(S + capA);
    using Sb = WsSub<G>;
    constexpr int SUBS = Sb::SUBS;
    u32 *scnt = R + capA;  // SUBS 16-bit counters, two per word
    u32 *e_cnt = scnt + SUBS / 2, *e_base = e_cnt + plan.a.buckets;
    u8 *CHS = reinterpret_cast<u8 *>(e_base + plan.a.buckets);  // (c0 | c1 << 4) per rank
    __shared__ __align__(8) u64 bar;
    __shared__ u32 sh_d;
    const int tid = threadIdx.x;
    const int nq = (int)plan.a.buckets;
    if (tid == 0) {
        mbar_init(&bar, 1);
        sh_d = 0;
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        fence_async_smem();
    }
    __syncthreads();
    auto span = [&](u32 f, i64 &lo, int &L) {
        lo = off[f << G];
        L = (int)((f + 1 < Sb::UNITS ? (i64)off[(f + 1) << G] : m) - lo);
    };
    auto issue = [&](i64 lo, int L) {  // one thread: the bucket's 16 B-aligned cover
        const i64 a0 = lo & ~(i64)1, a1 = (lo + L + 1) & ~(i64)1;
        const u32 bytes = (u32)((a1 - a0) * 8);
        mbar_expect_tx(&bar, bytes);
        bulk_g2s(IN, stageB + a0, bytes, &bar);
    };
    u32 f = blockIdx.x, parity = 0, d = 0;  // f: unit (group of 2^G fine buckets)
    i64 lo = 0;
    int L = 0;
    if (f < Sb::UNITS) span(f, lo, L);
    if (tid == 0 && f < Sb::UNITS && L > 0) issue(lo, L);
    for (; f < Sb::UNITS; f += gridDim.x) {
        const u32 fn = f + gridDim.x;
        i64 lo_n = 0;
        int L_n = 0;
        if (fn < Sb::UNITS) span(fn, lo_n, L_n);
        if (L > 0) {
            for (int i = tid; i < SUBS / 2; i += WS_ST) scnt[i] = 0;
            for (int i = tid; i < nq; i += WS_ST) e_cnt[i] = 0;
            mbar_wait(&bar, parity);
            parity ^= 1;
            const u64 *in = IN + (lo & 1);
            __syncthreads();
            for (int x = tid; x < L; x += WS_ST) {
                const u32 k = Sb::of(in[x]);
                atomicAdd(&scnt[k >> 1], 1u << (16 * (k & 1)));
            }
            __syncthreads();
            {  // exclusive scan of the sub-bucket counts (16-bit pairs)
                constexpr int WORDS = SUBS / 2;
                constexpr int PER = WORDS >= WS_ST ? WORDS / WS_ST : 1;
                const bool own = tid * PER < WORDS;
                __shared__ u32 sh_warp[WS_ST / 32 + 1];
                u32 v[PER], sum = 0;
#pragma unroll
                for (int k = 0; k < PER; k++) {
                    v[k] = own ? scnt[tid * PER + k] : 0u;
                    sum += (v[k] & 0xFFFFu) + (v[k] >> 16);
                }
                u32 excl;
                block_exclusive_scan<WS_ST>(sum, excl, sh_warp);
#pragma unroll
                for (int k = 0; k < PER; k++) {
                    const u32 a = excl, b = excl + (v[k] & 0xFFFFu);
                    if (own) scnt[tid * PER + k] = a | (b << 16);
                    excl = b + (v[k] >> 16);
                }
            }
            __syncthreads();
            for (int x = tid; x < L; x += WS_ST) {
                const u64 r = in[x];
                const u32 k = Sb::of(r), sh = 16 * (k & 1);
                S[(atomicAdd(&scnt[k >> 1], 1u << sh) >> sh) & 0xFFFFu] = r;
            }
            __syncthreads();  // IN is free: the next bucket streams in behind the rest
            if (tid == 0 && L_n > 0) {
                fence_async_smem();
                issue(lo_n, L_n);
            }
            // scnt[k] = end of sub-bucket k
            for (int i = tid; i < L; i += WS_ST) {
                const u64 v = S[i];
                const u32 k = Sb::of(v);
                const u32 wk = scnt[k >> 1];
                const int e = (int)((k & 1) ? wk >> 16 : wk & 0xFFFFu);
                const int s0 = (k & 1) ? (int)(wk & 0xFFFFu) : (k ? (int)(scnt[(k >> 1) - 1] >> 16) : 0);
                int lt = 0, same_lt = 0, same = 0;
                if (e - s0 > WS_BIG_SUB) {
                    // the caller discards this pass; keep R a permutation
                    atomicMax(&scal[8], 1u);
                    lt = i - s0;
                } else if (e - s0 > 1) {
                    // a sub-bucket shares bits 63..44, so 32-bit compares decide:
                    // hi = bits 43..12 (characters 15..21, flag, top of pos'),
                    // lo only on equal hi; same name = equal bits 43..29 and v a
                    // full window (flag bit 29)
                    const u32 vhi = (u32)(v >> Sb::HI), vlo = (u32)v;
                    const u32 vname = (vhi >> Sb::NAME) & 1u ? vhi >> Sb::NAME : 0xFFFFFFFFu;
                    for (int j = s0; j < e; j++) {
                        const u64 o = S[j];
                        const u32 ohi = (u32)(o >> Sb::HI), olo = (u32)o;
                        const bool less = ohi < vhi || (ohi == vhi && olo < vlo);
                        const bool eq = (ohi >> Sb::NAME) == vname;
                        lt += less;
                        same_lt += less && eq;
                        same += eq;
                    }
                }
                const int rank = s0 + lt;
                if (same_lt == 0) {
                    d++;
                    if (same > 1) {
                        const u32 at = atomicAdd(&scal[2], 1u);
                        if (at < cap_runs) {
                            rs[at] = (u32)(lo + rank);
                            rl[at] = (u32)same;
                        } else {
                            atomicMax(&scal[4], 1u);
                        }
                    }
                }
                const u32 p = (u32)ws_pos<SEP>(v, N, A);
                const u32 sidx = (p % 3u == 1u) ? p / 3u : (u32)m1 + p / 3u;
                R[rank] = sidx;
                if (ch) {  // the first two characters (ranks; 0 past the end) from the bucket's digits
                    const u32 fb = f << G;  // its characters 1..2 (G <= 12)
                    const u32 c0 = (i64)p >= N ? 0u : (SEP && (i64)p == A.sep) ? A.lo - 1u : ((fb >> 14) & 3u) + A.lo;
                    const u32 c1 = (i64)p + 1 >= N   ? 0u
                                   : (SEP && (i64)p + 1 == A.sep) ? A.lo - 1u
                                                                   : ((fb >> 12) & 3u) + A.lo;
                    CHS[rank] = (u8)(c0 | (c1 << 4));
                }
                atomicAdd(&e_cnt[sidx >> plan.a.shift], 1u);
            }
            __syncthreads();
            // run reservation per coarse ISA bucket: one atomic per bucket, all in
            // flight at once; their results are consumed only after the staging
            // loop, so the round trip overlaps it (nq <= WS_ST)
            u32 base_q = 0, start_q = 0;
            {
                __shared__ u32 sh_w[WS_ST / 32 + 1];
                const u32 c = tid < nq ? e_cnt[tid] : 0u;
                if (c) base_q = atomicAdd(&plan.a.cursor[tid], c);
                block_exclusive_scan<WS_ST>(c, start_q, sh_w);
                if (tid < nq) e_cnt[tid] = start_q;
            }
            __syncthreads();
            uint2 *E = reinterpret_cast<uint2 *>(S);  // S is free: emit staging
            for (int x = tid; x < L; x += WS_ST) {
                const u32 sidx = R[x];
                __stcs(sorted + lo + x, sidx);
                if (ch) ch[lo + x] = CHS[x];
                E[atomicAdd(&e_cnt[sidx >> plan.a.shift], 1u)] = make_uint2(sidx, (u32)(lo + x));
            }
            if (tid < nq) e_base[tid] = base_q - start_q;
            __syncthreads();
            // e_base[q] = q's run in its staging region minus its local start
            for (int x = tid; x < L; x += WS_ST) {
                const uint2 it = E[x];
                const u32 q = it.x >> plan.a.shift;
                st_stream(stage1 + ((i64)q << plan.a.shift) + (u32)(e_base[q] + (u32)x), it);
            }
            __syncthreads();
        } else if (tid == 0 && L_n > 0) {  // empty bucket: nothing in flight, IN is free
            fence_async_smem();
            issue(lo_n, L_n);
        }
        lo = lo_n;
        L = L_n;
    }
    for (int o = 16; o; o >>= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
    if (lane_id() == 0 && d) atomicAdd(&sh_d, d);
    __syncthreads();
    if (tid == 0 && sh_d) atomicAdd(&scal[5], sh_d);
}
inline size_t ws_sort_smem(int capA, const PsPlan &plan, int subs) {
    return (size_t)(2 * capA + 2) * 8 + (size_t)capA * 4 + (size_t)subs * 2 + 8 * (size_t)plan.a.buckets +
           (size_t)capA;
}

}  // namespace saix
