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
    int mode, ib;
};

template <typename V>
__device__ __forceinline__ void any_query(const PlanDev &P, const void *tab, Vals<V> val, i64 i, i64 j,
                                          i64 &idx, i64 &v) {
    if (P.mode == SAIX_SPARSE_PACK32) packed_query<u32>((const u32 *)tab, P.n, P.bias, P.ib, i, j, idx, v);
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

static PlanDev dev_plan(const saix_sparse_plan *p) { return PlanDev{p->n, p->value_bias, p->mode, p->index_bits}; }

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

extern "C" int saix_sparse_build(const saix_sparse_plan *plan, const void *values, int value_bytes, void *table,
                                 void *stream) {
    if (!plan || !values || !table || (value_bytes != 4 && value_bytes != 8)) {
        set_error("saix_sparse_build: invalid arguments");
        return SAIX_EINVAL;
    }
    cudaStream_t st = (cudaStream_t)stream;
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
    // 2 x int64 in, int64 out, two random table probes at one 32 B sector each
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
