// bsort.cuh -- MSD bucket sort for large-alphabet keys.
//
// Deep DC3 levels sort items whose leading key component ranges over a large
// alphabet (level-2 names of DNA: ~2^18): LSD radix needs 7 passes of 8 bits
// there, while an MSD split on the leading component leaves buckets of a few
// dozen items.  Three streaming passes plus small in-shared-memory sorts:
//   count    histogram of bucket ids (global atomics: buckets are many)
//   scan     exclusive bucket starts
//   scatter  item -> its bucket's next slot (atomic cursor; order inside a
//            bucket is arbitrary and fixed by the segment sort)
//   segsort  warp-per-bucket bitonic sort in shared memory (<= 256 items),
//            CTA-per-bucket bitonic (<= 4096); larger buckets are reported
//            so the caller can fall back to a full LSD sort.
// Sources: struct { __device__ void get(i64 i, u32 &bucket, u64 &key, u32 &val) const; }
// with the bucket a monotone function of the key (e.g. its top component);
// the result is sorted by key (ties in any order).
#pragma once

#include "scan.cuh"

namespace saix {

constexpr int BS_SMALL = 256;   // warp-per-bucket limit
constexpr int BS_LARGE = 4096;  // CTA-per-bucket limit

template <class Src>
__global__ void k_bs_count(Src src, i64 n, u32 *__restrict__ cnt) {
    for (i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x) {
        u32 b;
        u64 k;
        u32 v;
        src.get(i, b, k, v);
        atomicAdd(&cnt[b], 1u);
    }
}

struct BsCntIn {
    const u32 *cnt;
    __device__ u32 operator()(i64 i) const { return cnt[i]; }
};
// bucket starts + cursor copy; buckets beyond BS_SMALL are listed for the
// CTA-per-bucket pass and the largest size is recorded
struct BsStartOut {
    const u32 *cnt;
    u32 *start, *cursor, *big_list, *big_count, *max_size;
    __device__ void operator()(i64 i, u32 excl, u32 v) const {
        start[i] = excl;
        cursor[i] = excl;
        if (v > BS_SMALL) {
            big_list[atomicAdd(big_count, 1u)] = (u32)i;
            atomicMax(max_size, v);
        }
    }
};

template <class Src>
__global__ void k_bs_scatter(Src src, i64 n, u32 *__restrict__ cursor, u64 *__restrict__ keys,
                             u32 *__restrict__ vals) {
    for (i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x) {
        u32 b;
        u64 k;
        u32 v;
        src.get(i, b, k, v);
        u32 at = atomicAdd(&cursor[b], 1u);
        keys[at] = k;
        vals[at] = v;
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

constexpr int BS_WARPS = 8;

// one warp per bucket of <= BS_SMALL items
__global__ void __launch_bounds__(32 * BS_WARPS)
k_bs_small(const u32 *__restrict__ start, const u32 *__restrict__ cnt, i64 nb, u64 *__restrict__ keys,
           u32 *__restrict__ vals) {
    __shared__ u64 sk[BS_WARPS][BS_SMALL];
    __shared__ u32 sv[BS_WARPS][BS_SMALL];
    int w = threadIdx.x >> 5, lane = lane_id();
    for (i64 b = (i64)blockIdx.x * BS_WARPS + w; b < nb; b += (i64)gridDim.x * BS_WARPS) {
        u32 len = cnt[b];
        if (len <= 1 || len > BS_SMALL) continue;
        u32 s0 = start[b];
        for (u32 x = lane; x < len; x += 32) {
            sk[w][x] = keys[s0 + x];
            sv[w][x] = vals[s0 + x];
        }
        __syncwarp();
        bitonic_smem(sk[w], sv[w], (int)len, lane, 32, true);
        for (u32 x = lane; x < len; x += 32) {
            keys[s0 + x] = sk[w][x];
            vals[s0 + x] = sv[w][x];
        }
        __syncwarp();
    }
}

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

// scratch words: cnt, start, cursor (nb each), big list (nb), 3 scalars, scan tmp
inline i64 bs_scratch_words(i64 nb) { return 4 * (nb + 1) + 8 + scan_tmp_words(nb) + 64; }

// Returns false (after the count pass only) when some bucket exceeds
// BS_LARGE; the caller then sorts with onesweep instead.  One host sync.
template <class Src>
int bucket_sort(Src src, i64 n, i64 nb, u64 *keys, u32 *vals, u32 *scratch, bool &ok, cudaStream_t st,
                const char *prof = "bsort") {
    ok = true;
    if (n <= 0) return SAIX_OK;
    Prof prof_(prof, 24.0 * n + 16.0 * nb, st);
    u32 *cnt = scratch, *start = cnt + (nb + 1), *cursor = start + (nb + 1), *list = cursor + (nb + 1);
    u32 *scal = list + (nb + 1);  // [0] big count, [1] max size
    u32 *tmp = scal + 8;
    SAIX_CUDA(cudaMemsetAsync(cnt, 0, (size_t)(nb + 1) * 4, st));
    SAIX_CUDA(cudaMemsetAsync(scal, 0, 8 * 4, st));
    int g = grid_for(n, 256);
    k_bs_count<Src><<<g, 256, 0, st>>>(src, n, cnt);
    SAIX_LAUNCHED();
    SAIX_TRY(scan_transform(BsCntIn{cnt}, BsStartOut{cnt, start, cursor, list, scal, scal + 1}, nb, tmp, nullptr, st,
                            "bsort.scan", 16.0 * nb));
    u32 h[2];
    SAIX_CUDA(cudaMemcpyAsync(h, scal, 8, cudaMemcpyDeviceToHost, st));
    SAIX_CUDA(cudaStreamSynchronize(st));
    if (h[1] > (u32)BS_LARGE) {
        ok = false;
        return SAIX_OK;
    }
    k_bs_scatter<Src><<<g, 256, 0, st>>>(src, n, cursor, keys, vals);
    SAIX_LAUNCHED();
    k_bs_small<<<grid_for(nb, 32 * BS_WARPS, kNumSMs * 64), 32 * BS_WARPS, 0, st>>>(start, cnt, nb, keys, vals);
    SAIX_LAUNCHED();
    if (h[0]) {
        static bool attr = false;
        size_t smem = (size_t)BS_LARGE * 12;
        if (!attr) {
            SAIX_CUDA(cudaFuncSetAttribute(k_bs_large, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            attr = true;
        }
        k_bs_large<<<h[0] < 4 * kNumSMs ? h[0] : 4 * kNumSMs, 256, smem, st>>>(start, cnt, list, scal, keys, vals);
        SAIX_LAUNCHED();
    }
    return SAIX_OK;
}

}  // namespace saix
