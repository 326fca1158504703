// rmq.cu -- sparse-table RMQ (rmq.py:30-58 SparseTable, 254-259) on sm_100a.
//
// Entries pack (value - bias, index) into one integer so that a plain
// unsigned min is the reference's leftmost-argmin rule (`v[l] <= v[r] ? l :
// r`, rmq.py:48-58): equal values tie-break on the smaller index.  When the
// pack fits 32 bits (LCP arrays: <= 6 value bits + 26 index bits at 2^26) the
// table is half the bytes of a u64 table; INDEX mode keeps u32 indices and
// gathers values for value ranges too wide to pack.
//
// Level k (window 2^k) has n - 2^k + 1 entries at offset
// off(k) = k (n + 1) - (2^k - 1).
#include "common.cuh"

namespace saix {

__host__ __device__ inline i64 level_off(i64 n, int k) { return (i64)k * (n + 1) - (((i64)1 << k) - 1); }

template <typename V>
struct Vals {
    const V *v;
    __device__ __forceinline__ i64 operator()(i64 i) const { return (i64)v[i]; }
};

template <typename E, typename V>
__global__ void k_sparse_level0(Vals<V> val, i64 n, i64 bias, int ib, E *__restrict__ out) {
    for (i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x)
        out[i] = ((E)((u64)val(i) - (u64)bias) << ib) | (E)i;
}

template <typename E>
__global__ void k_sparse_level(const E *__restrict__ prev, i64 len, i64 half, E *__restrict__ out) {
    for (i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x; i < len; i += (i64)gridDim.x * blockDim.x) {
        E a = prev[i], b = prev[i + half];
        out[i] = a <= b ? a : b;
    }
}

template <typename V>
__global__ void k_sparse_idx_level(Vals<V> val, const u32 *__restrict__ prev, i64 len, i64 half,
                                   u32 *__restrict__ out, int level0) {
    for (i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x; i < len; i += (i64)gridDim.x * blockDim.x) {
        if (level0) {
            out[i] = (u32)i;
        } else {
            u32 l = prev[i], r = prev[i + half];
            out[i] = val(l) <= val(r) ? l : r;
        }
    }
}

__device__ __forceinline__ int floor_log2(u64 x) { return 63 - __clzll((long long)x); }

// ------------------------------------------------------------ blocked mode
// SAIX_SPARSE_BLOCKED (values spanning <= 254 after the bias, e.g. LCP
// arrays): an RMQ whose structures sit in L2 instead of a 6.7-13 GB table of
// random HBM probes.  Blocks of 32 values, superblocks of 32 blocks (1024
// values).  One table buffer holds
//   vals8  n bytes: v - bias (0xFF past the end; 16 B slack)        64 MB at 2^26
//   bpre   per block: leftmost min of [superblock start, block end]
//   bsuf   per block: leftmost min of [block start, superblock end]
//          both (v << 16 | offset in the superblock), u32          2 x 8 MB
//   bmin   per block: (v << 8 | offset in the block), u16           4 MB
//   stab   sparse table over superblock minima, (v << sbits | sb)    4 MB
// A query [i, j] takes the leftmost minimum of: i's block scanned from i,
// bsuf of the next block, stab over the superblocks strictly between, bpre
// of the block before j's, j's block scanned up to j -- one 32 B sector of
// vals8 per end plus four small L2 probes (same-superblock ranges scan bmin).
// Candidates are combined as (value << 32 | position) keys, so equal values
// keep the leftmost position (rmq.py:48-58).
constexpr int BLK_SHIFT = 5, SB_SHIFT = 10;
constexpr i64 BLK = (i64)1 << BLK_SHIFT, SBK = (i64)1 << SB_SHIFT;
constexpr int BPS = (int)(SBK / BLK);  // blocks per superblock (32 = one warp)
struct BlkLayout {
    i64 n, nb, ns, n8, o_pre, o_suf, o_min, o_stab;
    int sbits, slevels;
    int pb;  // > 0: stab entries are (v << pb | position of the leftmost min), else (v << sbits | superblock)
    __host__ __device__ static BlkLayout of(i64 n) {
        BlkLayout L;
        L.n = n;
        L.ns = (n + SBK - 1) >> SB_SHIFT;
        L.nb = L.ns * BPS;  // whole superblocks (blocks past the end hold 0xFF)
        L.n8 = L.nb * BLK + 16;
        L.o_pre = L.n8;
        L.o_suf = L.o_pre + 4 * L.nb;
        L.o_min = L.o_suf + 4 * L.nb;
        L.o_stab = L.o_min + ((2 * L.nb + 15) & ~(i64)15);
        L.sbits = 0;
        while (((i64)1 << L.sbits) < L.ns) L.sbits++;
        L.slevels = 0;
        while (L.slevels < 40 && ((i64)1 << L.slevels) <= L.ns) L.slevels++;
        L.pb = 0;
        return L;
    }
    __host__ __device__ i64 bytes() const { return o_stab + 4 * level_off(ns, slevels); }
};

// one warp per superblock, lane l = block l: vals8, bmin, bpre / bsuf (warp
// min-scans), stab level 0
template <typename V>
__global__ void k_blk_pack(Vals<V> val, BlkLayout L, i64 bias, u8 *__restrict__ tab) {
    u32 *bpre = reinterpret_cast<u32 *>(tab + L.o_pre), *bsuf = reinterpret_cast<u32 *>(tab + L.o_suf);
    u16 *bmin = reinterpret_cast<u16 *>(tab + L.o_min);
    u32 *stab = reinterpret_cast<u32 *>(tab + L.o_stab);
    const int lane = lane_id();
    const i64 warps = ((i64)gridDim.x * blockDim.x) >> 5;
    for (i64 sb = ((i64)blockIdx.x * blockDim.x + threadIdx.x) >> 5; sb < L.ns; sb += warps) {
        const i64 b = sb * BPS + lane, p0 = b << BLK_SHIFT;
        u32 w[8];
        u32 best = 0xFFFFu;  // (v << 8 | offset in block)
        u32 raw[32];  // u32 values: the block's 128 bytes as 8 vector loads, all in flight
        const bool vec = sizeof(V) == 4 && p0 + 32 <= L.n;
        if (vec) {
            const uint4 *src = reinterpret_cast<const uint4 *>(val.v + p0);
#pragma unroll
            for (int q = 0; q < 8; q++) {
                const uint4 t = __ldcs(src + q);
                raw[4 * q] = t.x;
                raw[4 * q + 1] = t.y;
                raw[4 * q + 2] = t.z;
                raw[4 * q + 3] = t.w;
            }
        }
#pragma unroll
        for (int q = 0; q < 8; q++) {
            u32 word = 0;
#pragma unroll
            for (int y = 0; y < 4; y++) {
                const i64 p = p0 + 4 * q + y;
                const u32 x = vec ? raw[4 * q + y] - (u32)bias
                                  : (p < L.n ? (u32)((u64)val(p) - (u64)bias) : 0xFFu);
                word |= x << (8 * y);
                const u32 key = (x << 8) | (u32)(4 * q + y);
                best = key < best ? key : best;
            }
            w[q] = word;
        }
        uint4 *dst = reinterpret_cast<uint4 *>(tab + p0);
        dst[0] = make_uint4(w[0], w[1], w[2], w[3]);
        dst[1] = make_uint4(w[4], w[5], w[6], w[7]);
        bmin[b] = (u16)best;
        // (v << 16 | offset in superblock): min-scans over the warp's blocks
        const u32 own = ((best >> 8) << 16) | (u32)(lane * BLK + (best & 0xFF));
        u32 pre = own, suf = own;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const u32 a = __shfl_up_sync(0xffffffffu, pre, o);
            const u32 c = __shfl_down_sync(0xffffffffu, suf, o);
            if (lane >= o) pre = a < pre ? a : pre;
            if (lane + o < 32) suf = c < suf ? c : suf;
        }
        bpre[b] = pre;
        bsuf[b] = suf;
        if (lane == 0)
            stab[sb] = L.pb ? ((suf >> 16) << L.pb) | (u32)((sb << SB_SHIFT) + (suf & 0xFFFFu))
                            : ((suf >> 16) << L.sbits) | (u32)sb;
    }
    if (blockIdx.x == 0 && threadIdx.x < 16) tab[L.n8 - 16 + threadIdx.x] = 0xFF;
}

// leftmost minimum of v8[a..b] inside one 32-value block, (v << 32 | position)
__device__ __forceinline__ u64 blk_scan(const u8 *__restrict__ v8, i64 a, i64 b) {
    const i64 c0 = a & ~(BLK - 1);
    const uint4 q0 = __ldg(reinterpret_cast<const uint4 *>(v8 + c0));
    const uint4 q1 = __ldg(reinterpret_cast<const uint4 *>(v8 + c0 + 16));
    u32 w[8] = {q0.x, q0.y, q0.z, q0.w, q1.x, q1.y, q1.z, q1.w};
    const int lo = (int)(a - c0), hi = (int)(b - c0);
    u32 m = 0xFFFFFFFFu;
#pragma unroll
    for (int k = 0; k < 8; k++) {
        // bytes outside [lo, hi] -> 0xFF (never a value: values are <= 254)
        const int s = 4 * k;
        u32 keep = 0xFFFFFFFFu;
        if (s < lo) keep &= lo - s >= 4 ? 0u : (0xFFFFFFFFu << (8 * (lo - s)));
        if (s + 3 > hi) keep &= hi - s < 0 ? 0u : (0xFFFFFFFFu >> (8 * (3 - (hi - s))));
        w[k] |= ~keep;
        m = __vminu4(m, w[k]);
    }
    m = __vminu4(m, m >> 16);
    m = __vminu4(m, m >> 8) & 0xFFu;
    const u32 pat = m * 0x01010101u;
    int pos = 31;
#pragma unroll
    for (int k = 7; k >= 0; k--) {
        const u32 e = __vcmpeq4(w[k], pat);
        if (e) pos = 4 * k + ((__ffs(e) - 1) >> 3);
    }
    return ((u64)m << 32) | (u64)(c0 + pos);
}

__device__ __forceinline__ void blocked_query(const u8 *__restrict__ tab, i64 n, i64 bias, int pb, i64 i, i64 j,
                                              i64 &idx, i64 &val) {
    const BlkLayout L = BlkLayout::of(n);
    const u32 *bpre = reinterpret_cast<const u32 *>(tab + L.o_pre), *bsuf = reinterpret_cast<const u32 *>(tab + L.o_suf);
    const u16 *bmin = reinterpret_cast<const u16 *>(tab + L.o_min);
    const u32 *stab = reinterpret_cast<const u32 *>(tab + L.o_stab);
    const i64 bi = i >> BLK_SHIFT, bj = j >> BLK_SHIFT;
    u64 best;
    if (bi == bj) {
        best = blk_scan(tab, i, j);
    } else {
        best = blk_scan(tab, i, ((bi + 1) << BLK_SHIFT) - 1);
        const i64 si = i >> SB_SHIFT, sj = j >> SB_SHIFT;
        auto cand = [&](u32 e, i64 sb) {  // (v << 16 | offset in superblock sb)
            const u64 key = ((u64)(e >> 16) << 32) | (u64)((sb << SB_SHIFT) + (e & 0xFFFFu));
            best = key < best ? key : best;
        };
        if (si == sj) {
            for (i64 b = bi + 1; b < bj; b++) {  // rare: range inside one superblock
                const u32 e = __ldg(bmin + b);
                const u64 key = ((u64)(e >> 8) << 32) | (u64)((b << BLK_SHIFT) + (e & 0xFF));
                best = key < best ? key : best;
            }
        } else {
            if (bi + 1 < (si + 1) * BPS) cand(__ldg(bsuf + bi + 1), si);
            if (si + 1 <= sj - 1) {
                const i64 lo = si + 1, hi = sj - 1;
                const int k = floor_log2((u64)(hi - lo + 1));
                const u32 *lv = stab + level_off(L.ns, k);
                const u32 a = __ldg(lv + lo), b = __ldg(lv + hi - ((i64)1 << k) + 1);
                const u32 mn = a <= b ? a : b;
                if (pb) {  // the entry holds the position itself (one probe fewer)
                    const u64 key = ((u64)(mn >> pb) << 32) | (u64)(mn & ((1u << pb) - 1));
                    best = key < best ? key : best;
                } else {
                    const i64 sb = (i64)(mn & ((1u << L.sbits) - 1));
                    cand(((mn >> L.sbits) << 16) | (__ldg(bsuf + sb * BPS) & 0xFFFFu), sb);
                }
            }
            if (bj - 1 >= sj * BPS) cand(__ldg(bpre + bj - 1), sj);
        }
        const u64 r = blk_scan(tab, bj << BLK_SHIFT, j);
        best = r < best ? r : best;
    }
    idx = (i64)(best & 0xFFFFFFFFull);
    val = (i64)(best >> 32) + bias;
}

// One query: leftmost argmin index of [i, j] and its value.
template <typename E>
__device__ __forceinline__ void packed_query(const E *__restrict__ tab, i64 n, i64 bias, int ib, i64 i, i64 j,
                                             i64 &idx, i64 &val) {
    int k = floor_log2((u64)(j - i + 1));
    const E *lv = tab + level_off(n, k);
    E a = lv[i], b = lv[j - ((i64)1 << k) + 1];
    E mn = a <= b ? a : b;
    idx = (i64)(mn & (((E)1 << ib) - 1));
    val = (i64)((u64)(mn >> ib) + (u64)bias);
}

template <typename V>
__device__ __forceinline__ void index_query(const u32 *__restrict__ tab, Vals<V> val, i64 n, i64 i, i64 j,
                                            i64 &idx, i64 &v) {
    int k = floor_log2((u64)(j - i + 1));
    const u32 *lv = tab + level_off(n, k);
    u32 a = lv[i], b = lv[j - ((i64)1 << k) + 1];
    i64 va = val(a), vb = val(b);
    if (va <= vb) { idx = a; v = va; }
    else { idx = b; v = vb; }
}

struct PlanDev {
    i64 n, bias;
    int mode, ib, vb;
};
// blocked mode: superblock-table entries carry positions when they fit
__host__ __device__ inline int blk_pos_bits(int value_bits, int index_bits) {
    return value_bits + index_bits <= 32 ? (index_bits > 0 ? index_bits : 1) : 0;
}

template <typename V>
__device__ __forceinline__ void any_query(const PlanDev &P, const void *tab, Vals<V> val, i64 i, i64 j,
                                          i64 &idx, i64 &v) {
    if (P.mode == SAIX_SPARSE_BLOCKED)
        blocked_query((const u8 *)tab, P.n, P.bias, blk_pos_bits(P.vb, P.ib), i, j, idx, v);
    else if (P.mode == SAIX_SPARSE_PACK32) packed_query<u32>((const u32 *)tab, P.n, P.bias, P.ib, i, j, idx, v);
    else if (P.mode == SAIX_SPARSE_PACK64) packed_query<u64>((const u64 *)tab, P.n, P.bias, P.ib, i, j, idx, v);
    else index_query<V>((const u32 *)tab, val, P.n, i, j, idx, v);
}

template <typename V>
__global__ void k_sparse_query(PlanDev P, const void *tab, Vals<V> val, const i64 *__restrict__ qi,
                               const i64 *__restrict__ qj, i64 q, i64 *__restrict__ out_idx,
                               i64 *__restrict__ out_val, int32_t *err) {
    for (i64 t = (i64)blockIdx.x * blockDim.x + threadIdx.x; t < q; t += (i64)gridDim.x * blockDim.x) {
        i64 i = qi[t], j = qj[t];
        if (i < 0 || i >= P.n || j < 0 || j >= P.n) {
            *err = 1;
            continue;
        }
        if (i > j) { i64 x = i; i = j; j = x; }
        i64 idx, v;
        any_query<V>(P, tab, val, i, j, idx, v);
        if (out_idx) out_idx[t] = idx;
        if (out_val) out_val[t] = v;
    }
}

// lcp_query (overlap.py:58-69)
template <typename V>
__global__ void k_lcp_query(PlanDev P, const void *tab, Vals<V> val, const u32 *__restrict__ isa,
                            const i64 *__restrict__ qi, const i64 *__restrict__ qj, i64 q,
                            i64 *__restrict__ out, int32_t *err) {
    for (i64 t = (i64)blockIdx.x * blockDim.x + threadIdx.x; t < q; t += (i64)gridDim.x * blockDim.x) {
        i64 i = qi[t], j = qj[t];
        if (i < 0 || i >= P.n || j < 0 || j >= P.n) {
            *err = 1;
            continue;
        }
        if (i == j) {
            out[t] = P.n - i;
            continue;
        }
        i64 ri = isa[i], rj = isa[j];
        i64 lo = ri < rj ? ri : rj, hi = ri < rj ? rj : ri;
        i64 idx, v;
        any_query<V>(P, tab, val, lo + 1, hi, idx, v);
        out[t] = v;
    }
}

static PlanDev dev_plan(const saix_sparse_plan *p) {
    return PlanDev{p->n, p->value_bias, p->mode, p->index_bits, p->value_bits};
}

__global__ void k_minmax_init(i64 *out2) {
    out2[0] = INT64_MAX;
    out2[1] = INT64_MIN;
}

template <typename V>
__global__ void k_minmax(Vals<V> val, i64 n, i64 *out2) {
    i64 lo = INT64_MAX, hi = INT64_MIN;
    for (i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x) {
        i64 x = val(i);
        lo = x < lo ? x : lo;
        hi = x > hi ? x : hi;
    }
    for (int o = 16; o; o >>= 1) {
        i64 a = __shfl_xor_sync(0xffffffffu, lo, o), b = __shfl_xor_sync(0xffffffffu, hi, o);
        lo = a < lo ? a : lo;
        hi = b > hi ? b : hi;
    }
    if (lane_id() == 0) {
        atomicMin((long long *)&out2[0], (long long)lo);
        atomicMax((long long *)&out2[1], (long long)hi);
    }
}

// u8 / u32 device arrays -> int64 (the reference API's host array dtype),
// four items per thread with 128-bit stores
template <typename V>
__global__ void k_widen_i64(const V *__restrict__ src, i64 n, i64 *__restrict__ dst) {
    for (i64 i = 4 * ((i64)blockIdx.x * blockDim.x + threadIdx.x); i < n; i += 4 * (i64)gridDim.x * blockDim.x) {
        if (i + 4 <= n && ((reinterpret_cast<uintptr_t>(dst + i) & 15) == 0)) {
            i64 a = (i64)src[i], b = (i64)src[i + 1], c = (i64)src[i + 2], d = (i64)src[i + 3];
            __stcs(reinterpret_cast<longlong2 *>(dst + i), make_longlong2(a, b));
            __stcs(reinterpret_cast<longlong2 *>(dst + i + 2), make_longlong2(c, d));
        } else {
            for (i64 k = i; k < n && k < i + 4; k++) dst[k] = (i64)src[k];
        }
    }
}

}  // namespace saix

using namespace saix;

extern "C" int saix_widen_i64(const void *src, int src_bytes, int64_t n, int64_t *dst, void *stream) {
    if (n < 0 || (n > 0 && (!src || !dst)) || (src_bytes != 1 && src_bytes != 4)) {
        set_error("saix_widen_i64: invalid arguments");
        return SAIX_EINVAL;
    }
    if (n == 0) return SAIX_OK;
    cudaStream_t st = (cudaStream_t)stream;
    int g = grid_for(ceil_div(n, 4), 256);
    if (src_bytes == 1) k_widen_i64<u8><<<g, 256, 0, st>>>((const u8 *)src, n, dst);
    else k_widen_i64<u32><<<g, 256, 0, st>>>((const u32 *)src, n, dst);
    SAIX_LAUNCHED();
    return SAIX_OK;
}

extern "C" int saix_minmax(const void *values, int value_bytes, int64_t n, int64_t *out2, void *stream) {
    if (!values || !out2 || n <= 0 || (value_bytes != 1 && value_bytes != 4 && value_bytes != 8)) {
        set_error("saix_minmax: invalid arguments");
        return SAIX_EINVAL;
    }
    cudaStream_t st = (cudaStream_t)stream;
    k_minmax_init<<<1, 1, 0, st>>>(out2);
    int g = grid_for(n, 256, kNumSMs * 8);
    if (value_bytes == 1) k_minmax<u8><<<g, 256, 0, st>>>(Vals<u8>{(const u8 *)values}, n, out2);
    else if (value_bytes == 4) k_minmax<u32><<<g, 256, 0, st>>>(Vals<u32>{(const u32 *)values}, n, out2);
    else k_minmax<i64><<<g, 256, 0, st>>>(Vals<i64>{(const i64 *)values}, n, out2);
    SAIX_LAUNCHED();
    return SAIX_OK;
}

extern "C" int saix_sparse_plan_make(int64_t n, int64_t vmin, int64_t vmax, saix_sparse_plan *plan) {
    if (!plan || n <= 0 || vmin > vmax || n > ((int64_t)1 << 32) - 1) {
        set_error("cannot build a sparse table over an empty array");
        return SAIX_EINVAL;
    }
    plan->n = n;
    plan->value_bias = vmin;
    int levels = 0;
    while (levels < 63 && ((int64_t)1 << levels) <= n) levels++;
    plan->levels = levels < 1 ? 1 : levels;
    plan->index_bits = bits_for((u64)(n - 1));
    u64 range = (u64)vmax - (u64)vmin;  // exact: |vmax - vmin| < 2^64
    plan->value_bits = bits_for(range);
    int total = plan->value_bits + plan->index_bits;
    if (total <= 32) plan->mode = SAIX_SPARSE_PACK32;
    else if (total <= 64) plan->mode = SAIX_SPARSE_PACK64;
    else plan->mode = SAIX_SPARSE_INDEX;
    int esz = plan->mode == SAIX_SPARSE_PACK64 ? 8 : 4;
    plan->table_bytes = level_off(n, plan->levels) * esz;
    return SAIX_OK;
}

extern "C" int saix_sparse_plan_blocked(int64_t n, int64_t vmin, int64_t vmax, saix_sparse_plan *plan) {
    SAIX_TRY(saix_sparse_plan_make(n, vmin, vmax, plan));
    if ((u64)vmax - (u64)vmin > 254 || n > ((int64_t)1 << 32) - 1) return SAIX_OK;  // keeps the full table
    plan->mode = SAIX_SPARSE_BLOCKED;
    plan->table_bytes = BlkLayout::of(n).bytes();
    return SAIX_OK;
}

extern "C" int saix_sparse_build(const saix_sparse_plan *plan, const void *values, int value_bytes, void *table,
                                 void *stream) {
    if (!plan || !values || !table || (value_bytes != 4 && value_bytes != 8)) {
        set_error("saix_sparse_build: invalid arguments");
        return SAIX_EINVAL;
    }
    cudaStream_t st = (cudaStream_t)stream;
    if (plan->mode == SAIX_SPARSE_BLOCKED) {
        BlkLayout B = BlkLayout::of(plan->n);
        B.pb = blk_pos_bits(plan->value_bits, plan->index_bits);
        u8 *tab = (u8 *)table;
        u32 *bt = reinterpret_cast<u32 *>(tab + B.o_stab);
        {
            Prof prof_("rmq.block_pack", (double)(value_bytes + 1) * B.n + 10.0 * B.nb + 4.0 * B.ns, st);
            const int g = grid_for(B.ns * 32, 256);
            if (value_bytes == 4)
                k_blk_pack<u32><<<g, 256, 0, st>>>(Vals<u32>{(const u32 *)values}, B, plan->value_bias, tab);
            else
                k_blk_pack<i64><<<g, 256, 0, st>>>(Vals<i64>{(const i64 *)values}, B, plan->value_bias, tab);
            SAIX_LAUNCHED();
        }
        Prof prof_("rmq.block_levels", 12.0 * (double)level_off(B.ns, B.slevels), st);
        for (int k = 1; k < B.slevels; k++) {
            const i64 len = B.ns - ((i64)1 << k) + 1;
            k_sparse_level<u32><<<grid_for(len, 256), 256, 0, st>>>(bt + level_off(B.ns, k - 1), len,
                                                                    (i64)1 << (k - 1), bt + level_off(B.ns, k));
            SAIX_LAUNCHED();
        }
        return SAIX_OK;
    }
    i64 n = plan->n;
    int ib = plan->index_bits;
    for (int k = 0; k < plan->levels; k++) {
        i64 len = n - ((i64)1 << k) + 1;
        i64 half = k ? ((i64)1 << (k - 1)) : 0;
        int g = grid_for(len, 256);
        int esz = plan->mode == SAIX_SPARSE_PACK64 ? 8 : 4;
        Prof prof_(k == 0 ? "rmq.level0" : "rmq.level", k == 0 ? (double)(value_bytes + esz) * n : 3.0 * esz * len, st);
        if (plan->mode == SAIX_SPARSE_PACK32 || plan->mode == SAIX_SPARSE_PACK64) {
            bool p32 = plan->mode == SAIX_SPARSE_PACK32;
            if (k == 0) {
                if (p32 && value_bytes == 4)
                    k_sparse_level0<u32, u32><<<g, 256, 0, st>>>(Vals<u32>{(const u32 *)values}, n, plan->value_bias, ib, (u32 *)table);
                else if (p32)
                    k_sparse_level0<u32, i64><<<g, 256, 0, st>>>(Vals<i64>{(const i64 *)values}, n, plan->value_bias, ib, (u32 *)table);
                else if (value_bytes == 4)
                    k_sparse_level0<u64, u32><<<g, 256, 0, st>>>(Vals<u32>{(const u32 *)values}, n, plan->value_bias, ib, (u64 *)table);
                else
                    k_sparse_level0<u64, i64><<<g, 256, 0, st>>>(Vals<i64>{(const i64 *)values}, n, plan->value_bias, ib, (u64 *)table);
            } else if (p32) {
                const u32 *t = (const u32 *)table;
                k_sparse_level<u32><<<g, 256, 0, st>>>(t + level_off(n, k - 1), len, half, (u32 *)table + level_off(n, k));
            } else {
                const u64 *t = (const u64 *)table;
                k_sparse_level<u64><<<g, 256, 0, st>>>(t + level_off(n, k - 1), len, half, (u64 *)table + level_off(n, k));
            }
        } else {
            u32 *t = (u32 *)table;
            const u32 *prev = k ? t + level_off(n, k - 1) : nullptr;
            if (value_bytes == 4)
                k_sparse_idx_level<u32><<<g, 256, 0, st>>>(Vals<u32>{(const u32 *)values}, prev, len, half, t + level_off(n, k), k == 0);
            else
                k_sparse_idx_level<i64><<<g, 256, 0, st>>>(Vals<i64>{(const i64 *)values}, prev, len, half, t + level_off(n, k), k == 0);
        }
        SAIX_LAUNCHED();
    }
    return SAIX_OK;
}

extern "C" int saix_sparse_query(const saix_sparse_plan *plan, const void *table, const void *values, int value_bytes,
                                 const int64_t *qi, const int64_t *qj, int64_t q, int64_t *out_index,
                                 int64_t *out_value, int32_t *err, void *stream) {
    if (!plan || !table || q < 0 || (q > 0 && (!qi || !qj || !err)) ||
        (plan->mode == SAIX_SPARSE_INDEX && (!values || (value_bytes != 4 && value_bytes != 8)))) {
        set_error("saix_sparse_query: invalid arguments");
        return SAIX_EINVAL;
    }
    if (q == 0) return SAIX_OK;
    cudaStream_t st = (cudaStream_t)stream;
    int g = grid_for(q, 256);
    PlanDev P = dev_plan(plan);
    // SURVEY.md 8(d) algorithmic bytes, every layout: 2 x int64 in, int64 out,
    // two random table probes at one 32 B sector each = 88 B per query (the
    // blocked layout's ~6 probes are sector-granular too: its 88 MB working
    // set is past the random-access L2 knee, ~97 B/query of DRAM measured)
    Prof prof_("rmq.query", 88.0 * q, st);
    if (value_bytes == 4)
        k_sparse_query<u32><<<g, 256, 0, st>>>(P, table, Vals<u32>{(const u32 *)values}, qi, qj, q, out_index, out_value, err);
    else
        k_sparse_query<i64><<<g, 256, 0, st>>>(P, table, Vals<i64>{(const i64 *)values}, qi, qj, q, out_index, out_value, err);
    SAIX_LAUNCHED();
    return SAIX_OK;
}

extern "C" int saix_lcp_query(const saix_sparse_plan *plan, const void *table, const void *lcp, int lcp_bytes,
                              const uint32_t *isa, const int64_t *qi, const int64_t *qj, int64_t q, int64_t *out,
                              int32_t *err, void *stream) {
    if (!plan || !table || !isa || q < 0 || (q > 0 && (!qi || !qj || !out || !err)) ||
        (plan->mode == SAIX_SPARSE_INDEX && (!lcp || (lcp_bytes != 4 && lcp_bytes != 8)))) {
        set_error("saix_lcp_query: invalid arguments");
        return SAIX_EINVAL;
    }
    if (q == 0) return SAIX_OK;
    cudaStream_t st = (cudaStream_t)stream;
    int g = grid_for(q, 256);
    PlanDev P = dev_plan(plan);
    Prof prof_("rmq.lcp_query", 152.0 * q, st);
    if (lcp_bytes == 8)
        k_lcp_query<i64><<<g, 256, 0, st>>>(P, table, Vals<i64>{(const i64 *)lcp}, isa, qi, qj, q, out, err);
    else
        k_lcp_query<u32><<<g, 256, 0, st>>>(P, table, Vals<u32>{(const u32 *)lcp}, isa, qi, qj, q, out, err);
    SAIX_LAUNCHED();
    return SAIX_OK;
}
