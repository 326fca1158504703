// psort.cu -- the reference's "parallel sort" engine primitives on sm_100a
// (parallel_sort.py:110-293): exclusive_scan, split_by_bit, radix_sort /
// chunked_sort.  The reference models a GPU split kernel in numpy (doubling
// scan, stable 1-bit split, LSD over digits, chunk-then-merge); here they are
// the device scan and the onesweep LSD radix sort of this library, with the
// same results (a stable ascending sort of keys alone is unique, so digit
// width, chunk size and worker count cannot change the output).
#include "onesweep.cuh"

namespace saix {

// ------------------------------------------------------------ i64 scan

constexpr int PS64_THREADS = 256, PS64_ITEMS = 8, PS64_TILE = PS64_THREADS * PS64_ITEMS;

__device__ __forceinline__ i64 warp_incl_i64(i64 v) {
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        i64 y = __shfl_up_sync(0xffffffffu, v, o);
        if (lane_id() >= o) v += y;
    }
    return v;
}
// block exclusive scan of one i64 per thread; returns the block total
__device__ __forceinline__ i64 block_excl_i64(i64 v, i64 &excl) {
    __shared__ i64 sw[PS64_THREADS / 32 + 1];
    int w = threadIdx.x >> 5;
    i64 inc = warp_incl_i64(v);
    if (lane_id() == 31) sw[w] = inc;
    __syncthreads();
    if (w == 0) {
        i64 x = lane_id() < PS64_THREADS / 32 ? sw[lane_id()] : 0;
        i64 xi = warp_incl_i64(x);
        if (lane_id() < PS64_THREADS / 32) sw[lane_id()] = xi - x;
        if (lane_id() == PS64_THREADS / 32 - 1) sw[PS64_THREADS / 32] = xi;
    }
    __syncthreads();
    excl = sw[w] + inc - v;
    i64 tot = sw[PS64_THREADS / 32];
    __syncthreads();
    return tot;
}

// In: __device__ i64 operator()(i64 i) const
template <class In>
__global__ void __launch_bounds__(PS64_THREADS) k_scan64_reduce(In in, i64 n, i64 *__restrict__ sums) {
    i64 base = (i64)blockIdx.x * PS64_TILE + (i64)threadIdx.x * PS64_ITEMS;
    i64 s = 0;
#pragma unroll
    for (int q = 0; q < PS64_ITEMS; q++)
        if (base + q < n) s += in(base + q);
    i64 excl;
    i64 tot = block_excl_i64(s, excl);
    if (threadIdx.x == 0) sums[blockIdx.x] = tot;
}
static __global__ void __launch_bounds__(PS64_THREADS) k_scan64_sums(i64 *sums, i64 nb) {
    i64 carry = 0;
    for (i64 c = 0; c < nb; c += PS64_THREADS) {
        i64 i = c + threadIdx.x;
        i64 v = i < nb ? sums[i] : 0;
        i64 excl;
        i64 tot = block_excl_i64(v, excl);
        if (i < nb) sums[i] = carry + excl;
        carry += tot;
    }
}
// Out: __device__ void operator()(i64 i, i64 excl, i64 v) const
template <class In, class Out>
__global__ void __launch_bounds__(PS64_THREADS) k_scan64_apply(In in, Out out, i64 n, const i64 *__restrict__ sums) {
    i64 base = (i64)blockIdx.x * PS64_TILE + (i64)threadIdx.x * PS64_ITEMS;
    i64 v[PS64_ITEMS], s = 0;
#pragma unroll
    for (int q = 0; q < PS64_ITEMS; q++) {
        v[q] = base + q < n ? in(base + q) : 0;
        s += v[q];
    }
    i64 excl;
    block_excl_i64(s, excl);
    excl += sums[blockIdx.x];
#pragma unroll
    for (int q = 0; q < PS64_ITEMS; q++) {
        if (base + q < n) out(base + q, excl, v[q]);
        excl += v[q];
    }
}
inline i64 scan64_tmp_words(i64 n) { return ceil_div(n > 0 ? n : 1, PS64_TILE) + 1; }

template <class In, class Out>
static int scan64(In in, Out out, i64 n, i64 *tmp, cudaStream_t st) {
    if (n <= 0) return SAIX_OK;
    i64 nb = ceil_div(n, PS64_TILE);
    k_scan64_reduce<In><<<(unsigned)nb, PS64_THREADS, 0, st>>>(in, n, tmp);
    SAIX_LAUNCHED();
    k_scan64_sums<<<1, PS64_THREADS, 0, st>>>(tmp, nb);
    SAIX_LAUNCHED();
    k_scan64_apply<In, Out><<<(unsigned)nb, PS64_THREADS, 0, st>>>(in, out, n, tmp);
    SAIX_LAUNCHED();
    return SAIX_OK;
}

struct ArrIn64 {
    const i64 *a;
    __device__ i64 operator()(i64 i) const { return a[i]; }
};
struct ExclOut64 {
    i64 *o;
    __device__ void operator()(i64 i, i64 excl, i64) const { o[i] = excl; }
};

// ------------------------------------------------------------ split_by_bit

struct ZeroFlagIn {
    const i64 *keys;
    int bit;
    __device__ i64 operator()(i64 i) const { return ((keys[i] >> bit) & 1) ^ 1; }
};
// scanned[i] = exclusive count of zero bits; the last lane also leaves the total
struct SplitScanOut {
    const i64 *keys;
    int bit;
    i64 n;
    i64 *bits, *zero_flags, *scanned, *zero_total;
    __device__ void operator()(i64 i, i64 excl, i64 zf) const {
        if (bits) bits[i] = zf ^ 1;
        if (zero_flags) zero_flags[i] = zf;
        scanned[i] = excl;
        if (i == n - 1) *zero_total = excl + zf;
    }
};
__global__ void k_split_dest(const i64 *__restrict__ keys, i64 n, int bit, const i64 *__restrict__ scanned,
                             const i64 *__restrict__ zero_total, i64 *__restrict__ dest, i64 *__restrict__ out) {
    const i64 zt = *zero_total;
    for (i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x) {
        i64 k = keys[i];
        i64 d = ((k >> bit) & 1) ? i - scanned[i] + zt : scanned[i];
        if (dest) dest[i] = d;
        out[d] = k;
    }
}

// ------------------------------------------------------------ radix sort

struct KeySrc64 {
    const u64 *k;
    __device__ __forceinline__ bool get(i64 i, u64 &key, u32 &v) const {
        key = k[i];
        v = 0;
        return true;
    }
};

}  // namespace saix

using namespace saix;

extern "C" size_t saix_psort_workspace_bytes(int64_t n) {
    Arena ar;
    ar.alloc<i64>(scan64_tmp_words(n));
    ar.alloc<i64>(2);
    ar.alloc<u64>(n);
    ar.alloc<u64>(n);
    ar.alloc<u32>(n);
    ar.alloc<u32>(n);
    ar.alloc<u32>(os_scratch_words(n));
    return ar.peak + Arena::kAlign;
}

extern "C" int saix_exclusive_scan_i64(const int64_t *in, int64_t n, int64_t *out, void *ws, size_t ws_bytes,
                                       void *stream) {
    if (n < 0 || (n > 0 && (!in || !out))) {
        set_error("saix_exclusive_scan_i64: invalid arguments");
        return SAIX_EINVAL;
    }
    if (n == 0) return SAIX_OK;
    Arena ar{(char *)ws, ws_bytes};
    i64 *tmp = ar.alloc<i64>(scan64_tmp_words(n));
    SAIX_ARENA_OK(ar);
    Prof prof_("psort.scan", 16.0 * n, (cudaStream_t)stream);
    return scan64(ArrIn64{in}, ExclOut64{out}, n, tmp, (cudaStream_t)stream);
}

extern "C" int saix_split_by_bit(const int64_t *keys, int64_t n, int bit, int64_t *out, int64_t *bits,
                                 int64_t *zero_flags, int64_t *scanned, int64_t *dest, int64_t *zero_total, void *ws,
                                 size_t ws_bytes, void *stream) {
    if (n < 0 || bit < 0 || bit > 63 || !zero_total || (n > 0 && (!keys || !out || !scanned))) {
        set_error("saix_split_by_bit: invalid arguments");
        return SAIX_EINVAL;
    }
    cudaStream_t st = (cudaStream_t)stream;
    SAIX_CUDA(cudaMemsetAsync(zero_total, 0, sizeof(int64_t), st));
    if (n == 0) return SAIX_OK;
    Arena ar{(char *)ws, ws_bytes};
    i64 *tmp = ar.alloc<i64>(scan64_tmp_words(n));
    SAIX_ARENA_OK(ar);
    Prof prof_("psort.split", 48.0 * n, st);
    SAIX_TRY(scan64(ZeroFlagIn{keys, bit}, SplitScanOut{keys, bit, n, bits, zero_flags, scanned, zero_total}, n, tmp,
                    st));
    k_split_dest<<<grid_for(n, 256), 256, 0, st>>>(keys, n, bit, scanned, zero_total, dest, out);
    SAIX_LAUNCHED();
    return SAIX_OK;
}

extern "C" int saix_radix_sort_i64(const int64_t *keys, int64_t n, int total_bits, int64_t *out, void *ws,
                                   size_t ws_bytes, void *stream) {
    if (n < 0 || total_bits < 1 || total_bits > 63 || (n > 0 && (!keys || !out))) {
        set_error("saix_radix_sort_i64: invalid arguments");
        return SAIX_EINVAL;
    }
    if (n >= ((i64)1 << 30)) {
        set_error("saix_radix_sort_i64: n=%lld too large for one call", (long long)n);
        return SAIX_EINVAL;
    }
    cudaStream_t st = (cudaStream_t)stream;
    if (n == 0) return SAIX_OK;
    if (ws_bytes < saix_psort_workspace_bytes(n)) {
        set_error("saix_radix_sort_i64: workspace too small");
        return SAIX_ENOSPC;
    }
    Arena ar{(char *)ws, ws_bytes};
    ar.alloc<i64>(scan64_tmp_words(n));
    ar.alloc<i64>(2);
    u64 *k0 = ar.alloc<u64>(n), *k1 = ar.alloc<u64>(n);
    u32 *v0 = ar.alloc<u32>(n), *v1 = ar.alloc<u32>(n);
    u32 *scratch = ar.alloc<u32>(os_scratch_words(n));
    SAIX_ARENA_OK(ar);
    int passes = (total_bits + OS_BITS - 1) / OS_BITS;
    u64 *rk = nullptr;
    u32 *rv = nullptr;
    KeySrc64 src{reinterpret_cast<const u64 *>(keys)};
    SAIX_TRY(onesweep_sort<u64>(src, n, src, n, n, 0, passes, k0, v0, k1, v1, scratch, rk, rv, nullptr, st,
                                "psort.radix"));
    SAIX_CUDA(cudaMemcpyAsync(out, rk, (size_t)n * 8, cudaMemcpyDeviceToDevice, st));
    return SAIX_OK;
}
