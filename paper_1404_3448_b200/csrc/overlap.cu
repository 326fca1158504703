// overlap.cu -- encode / generalized text and the longest-overlap scan
// (overlap.py:72-152) on sm_100a, plus the end-to-end pair pipeline.
//
// Scan, two streaming passes over the GSA's (sa, lcp):
//   pass 1  best = max lcp[i] over adjacent pairs whose suffixes start on
//           opposite sides of the separator (overlap.py:129-136); block max +
//           one atomicMax per CTA.
//   pass 2  runs = maximal SA intervals with lcp >= best; per run min A-pos /
//           min B-pos (overlap.py:138-152) as a segmented min-scan
//           (reduce -> scan tile carries -> apply).  Every A position lies in
//           exactly one run, so the reference's lexicographic (minA, minB)
//           choice is a u64 atomicMin of (minA << 32 | minB) at run ends.
#include <vector>

#include "lcp_direct.cuh"
#include "lsd.cuh"
#include "onesweep.cuh"
#include "scan.cuh"

namespace saix {

// ------------------------------------------------------------ encode

__device__ __forceinline__ u32 rank_of_ascii(u32 c, int keep_n) {
    // encode LUT (sequence.py:144-150): A1 C2 G3 T4, N5 under NPolicy.KEEP
    switch (c) {
        case 'A': return 1;
        case 'C': return 2;
        case 'G': return 3;
        case 'T': return 4;
        case 'N': return keep_n ? 5u : 0u;
        default: return 0;
    }
}

__device__ __forceinline__ u32 encode_at(const u8 *__restrict__ a, i64 na, const u8 *__restrict__ b, i64 i,
                                          int keep_n, int shift, i64 &local_bad) {
    u32 r;
    if (i < na) r = rank_of_ascii(a[i], keep_n);
    else if (i == na) return 1u;  // separator rank (overlap.py:25)
    else r = rank_of_ascii(b[i - na - 1], keep_n);
    if (r == 0) {
        if (i < local_bad) local_bad = i;
        r = 1;
    }
    return r + shift;
}

// Sixteen output ranks per thread, stored as one 16-byte word (out must be
// 16-byte aligned; the ABI entry points check and fall back to bytes).
__global__ void k_encode_gsa(const u8 *__restrict__ a, i64 na, const u8 *__restrict__ b, i64 nb, int keep_n,
                             int shift, u8 *__restrict__ out, i64 *__restrict__ bad, int words) {
    i64 n = na + nb + (b ? 1 : 0);
    i64 local_bad = INT64_MAX;
    i64 stride = (i64)gridDim.x * blockDim.x;
    if (words) {
        // 16 output ranks per thread, stored as one 16-byte word (out 16-byte
        // aligned); runs that lie inside A or inside B skip the side test
        uint4 *out16 = reinterpret_cast<uint4 *>(out);
        i64 nv = n / 16;
        for (i64 v = (i64)blockIdx.x * blockDim.x + threadIdx.x; v < nv; v += stride) {
            const i64 p0 = 16 * v;
            u32 w[4] = {0, 0, 0, 0};
            if (p0 + 16 <= na) {
#pragma unroll
                for (int j = 0; j < 16; j++) {
                    u32 r = rank_of_ascii(a[p0 + j], keep_n);
                    if (r == 0) {
                        if (p0 + j < local_bad) local_bad = p0 + j;
                        r = 1;
                    }
                    w[j >> 2] |= (r + shift) << (8 * (j & 3));
                }
            } else if (p0 > na) {
                const u8 *bb = b + (p0 - na - 1);
#pragma unroll
                for (int j = 0; j < 16; j++) {
                    u32 r = rank_of_ascii(bb[j], keep_n);
                    if (r == 0) {
                        if (p0 + j < local_bad) local_bad = p0 + j;
                        r = 1;
                    }
                    w[j >> 2] |= (r + shift) << (8 * (j & 3));
                }
            } else {
#pragma unroll
                for (int j = 0; j < 16; j++) w[j >> 2] |= encode_at(a, na, b, p0 + j, keep_n, shift, local_bad) << (8 * (j & 3));
            }
            out16[v] = make_uint4(w[0], w[1], w[2], w[3]);
        }
        for (i64 i = 16 * nv + (i64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
            out[i] = (u8)encode_at(a, na, b, i, keep_n, shift, local_bad);
    } else {
        for (i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
            out[i] = (u8)encode_at(a, na, b, i, keep_n, shift, local_bad);
    }
    if (local_bad != INT64_MAX) atomicMin((unsigned long long *)bad, (unsigned long long)local_bad);
}

// ------------------------------------------------------------ pass 1

constexpr int OV_THREADS = 256;
constexpr int OV_ITEMS = 16;
constexpr int OV_TILE = OV_THREADS * OV_ITEMS;

__device__ __forceinline__ int side_of(u32 p, u32 boundary) { return p < boundary ? 0 : (p > boundary ? 1 : -1); }

__global__ void __launch_bounds__(OV_THREADS)
k_cross_max(const u32 *__restrict__ sa, const u32 *__restrict__ lcp, i64 n, u32 boundary, u32 *best) {
    u32 mx = 0;
    for (i64 i = 1 + (i64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x) {
        int a = side_of(sa[i - 1], boundary), b = side_of(sa[i], boundary);
        if (a >= 0 && b >= 0 && a != b) mx = max(mx, lcp[i]);
    }
    for (int o = 16; o; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    __shared__ u32 sh[OV_THREADS / 32];
    if (lane_id() == 0) sh[threadIdx.x >> 5] = mx;
    __syncthreads();
    if (threadIdx.x < 32) {
        mx = threadIdx.x < OV_THREADS / 32 ? sh[threadIdx.x] : 0;
        for (int o = 16; o; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        if (threadIdx.x == 0 && mx) atomicMax(best, mx);
    }
}

// ------------------------------------------------------------ pass 2

struct Seg {  // segmented-min state: head flag + min A / min B position
    u32 f, a, b;
};
__device__ __forceinline__ Seg seg_combine(Seg l, Seg r) {
    if (r.f) return r;
    return Seg{l.f, min(l.a, r.a), min(l.b, r.b)};
}
__device__ __forceinline__ Seg seg_shfl_up(Seg s, int o) {
    return Seg{__shfl_up_sync(0xffffffffu, s.f, o), __shfl_up_sync(0xffffffffu, s.a, o),
               __shfl_up_sync(0xffffffffu, s.b, o)};
}
constexpr u32 kInf = 0xFFFFFFFFu;

__device__ __forceinline__ Seg seg_elem(u32 p, u32 l, i64 i, u32 best, u32 boundary) {
    Seg s;
    s.f = (i == 0 || l < best) ? 1u : 0u;
    s.a = p < boundary ? p : kInf;
    s.b = p > boundary ? p : kInf;
    return s;
}

// Block-wide exclusive segmented scan of per-thread aggregates; returns the
// carry-in for this thread and the block aggregate.
__device__ Seg block_seg_exclusive(Seg v, Seg &block_total) {
    __shared__ Seg sh[OV_THREADS / 32 + 1];
    int w = threadIdx.x >> 5, lane = lane_id();
    Seg inc = v;
    for (int o = 1; o < 32; o <<= 1) {
        Seg y = seg_shfl_up(inc, o);
        if (lane >= o) inc = seg_combine(y, inc);
    }
    if (lane == 31) sh[w] = inc;
    __syncthreads();
    if (w == 0) {
        Seg x = lane < OV_THREADS / 32 ? sh[lane] : Seg{0u, kInf, kInf};
        Seg xi = x;
        for (int o = 1; o < 32; o <<= 1) {
            Seg y = seg_shfl_up(xi, o);
            if (lane >= o) xi = seg_combine(y, xi);
        }
        Seg ex = seg_shfl_up(xi, 1);
        if (lane == 0) ex = Seg{0u, kInf, kInf};
        if (lane < OV_THREADS / 32) sh[lane] = ex;
        if (lane == OV_THREADS / 32 - 1) sh[OV_THREADS / 32] = xi;
    }
    __syncthreads();
    Seg prev = seg_shfl_up(inc, 1);
    Seg carry = sh[w];
    if (lane > 0) carry = seg_combine(carry, prev);
    block_total = sh[OV_THREADS / 32];
    __syncthreads();
    return carry;
}

__device__ __forceinline__ void load_tile(const u32 *__restrict__ sa, const u32 *__restrict__ lcp, i64 n, i64 base,
                                          u32 *sh_sa, u32 *sh_l) {
    for (int x = threadIdx.x; x < OV_TILE; x += OV_THREADS) {
        i64 i = base + x;
        sh_sa[x + (x >> 5)] = i < n ? sa[i] : 0u;  // never read past n
        sh_l[x + (x >> 5)] = i < n ? lcp[i] : 0u;
    }
}

__global__ void __launch_bounds__(OV_THREADS)
k_runs_reduce(const u32 *__restrict__ sa, const u32 *__restrict__ lcp, i64 n, const u32 *__restrict__ best_p,
              u32 boundary, Seg *__restrict__ tile_agg, u32 *__restrict__ tile_join) {
    __shared__ u32 sh_sa[OV_TILE + OV_TILE / 32], sh_l[OV_TILE + OV_TILE / 32];
    u32 best = *best_p;
    i64 base = (i64)blockIdx.x * OV_TILE;
    if (best == 0) {
        if (threadIdx.x == 0) tile_agg[blockIdx.x] = Seg{0u, kInf, kInf};
        return;
    }
    // Most tiles hold no adjacent pair with lcp >= best: every element is
    // then a singleton run (one side only, never a candidate) and only the
    // last element can open a run into the next tile.  Such tiles read the
    // LCP tile and one SA entry.
    int join = 0;
    for (int x = threadIdx.x; x < OV_TILE; x += OV_THREADS) {
        i64 i = base + x;
        u32 l = i < n ? __ldcs(lcp + i) : 0u;
        sh_l[x + (x >> 5)] = l;
        join |= (i > 0 && i < n && l >= best);
    }
    join = __syncthreads_or(join);
    if (!join) {
        if (threadIdx.x == 0) {
            i64 last = (base + OV_TILE < n ? base + OV_TILE : n) - 1;
            u32 p = sa[last];
            tile_agg[blockIdx.x] = Seg{1u, p < boundary ? p : kInf, p > boundary ? p : kInf};
            tile_join[blockIdx.x] = 0;
        }
        return;
    }
    if (threadIdx.x == 0) tile_join[blockIdx.x] = 1;
    for (int x = threadIdx.x; x < OV_TILE; x += OV_THREADS) {
        i64 i = base + x;
        sh_sa[x + (x >> 5)] = i < n ? sa[i] : 0u;
    }
    __syncthreads();
    Seg acc{0u, kInf, kInf};
    for (int r = 0; r < OV_ITEMS; r++) {
        int x = threadIdx.x * OV_ITEMS + r;
        i64 i = base + x;
        if (i >= n) break;
        acc = seg_combine(acc, seg_elem(sh_sa[x + (x >> 5)], sh_l[x + (x >> 5)], i, best, boundary));
    }
    Seg tot;
    block_seg_exclusive(acc, tot);
    if (threadIdx.x == 0) tile_agg[blockIdx.x] = tot;
}

// Single CTA: exclusive segmented scan of tile aggregates (tile carries).
__global__ void __launch_bounds__(OV_THREADS) k_runs_carry(Seg *__restrict__ agg, i64 ntiles) {
    Seg carry{0u, kInf, kInf};
    for (i64 c = 0; c < ntiles; c += OV_THREADS) {
        i64 t = c + threadIdx.x;
        Seg v = t < ntiles ? agg[t] : Seg{0u, kInf, kInf};
        Seg tot;
        Seg ex = block_seg_exclusive(v, tot);
        if (t < ntiles) agg[t] = seg_combine(carry, ex);
        carry = seg_combine(carry, tot);
    }
}

__global__ void __launch_bounds__(OV_THREADS)
k_runs_apply(const u32 *__restrict__ sa, const u32 *__restrict__ lcp, i64 n, const u32 *__restrict__ best_p,
             u32 boundary, const Seg *__restrict__ tile_carry, const u32 *__restrict__ tile_join,
             unsigned long long *__restrict__ winner) {
    __shared__ u32 sh_sa[OV_TILE + OV_TILE / 32], sh_l[OV_TILE + OV_TILE / 32];
    u32 best = *best_p;
    if (best == 0 || !tile_join[blockIdx.x]) return;  // no join: no candidate run ends here
    i64 base = (i64)blockIdx.x * OV_TILE;
    load_tile(sa, lcp, n, base, sh_sa, sh_l);
    __syncthreads();
    Seg acc{0u, kInf, kInf};
    for (int r = 0; r < OV_ITEMS; r++) {
        int x = threadIdx.x * OV_ITEMS + r;
        i64 i = base + x;
        if (i >= n) break;
        acc = seg_combine(acc, seg_elem(sh_sa[x + (x >> 5)], sh_l[x + (x >> 5)], i, best, boundary));
    }
    Seg tot;
    Seg carry = seg_combine(tile_carry[blockIdx.x], block_seg_exclusive(acc, tot));
    Seg run = carry;
    for (int r = 0; r < OV_ITEMS; r++) {
        int x = threadIdx.x * OV_ITEMS + r;
        i64 i = base + x;
        if (i >= n) break;
        run = seg_combine(run, seg_elem(sh_sa[x + (x >> 5)], sh_l[x + (x >> 5)], i, best, boundary));
        bool end;
        if (i + 1 >= n) end = true;
        else if (x + 1 < OV_TILE) end = sh_l[(x + 1) + ((x + 1) >> 5)] < best;
        else end = lcp[i + 1] < best;
        if (end && run.a != kInf && run.b != kInf)
            atomicMin(winner, ((unsigned long long)run.a << 32) | run.b);
    }
}

__global__ void k_pipeline_init(i64 *__restrict__ out3, i64 *__restrict__ bad) {
    out3[0] = out3[1] = out3[2] = 0;
    *bad = INT64_MAX;
}

__global__ void k_overlap_finish(const u32 *__restrict__ best_p, const unsigned long long *__restrict__ winner,
                                 u32 boundary, i64 *__restrict__ out3) {
    u32 best = *best_p;
    unsigned long long w = *winner;
    if (best == 0 || w == ~0ull) {
        out3[0] = out3[1] = out3[2] = 0;
    } else {
        out3[0] = best;
        out3[1] = (i64)(w >> 32);
        out3[2] = (i64)(w & 0xFFFFFFFFull) - (i64)boundary - 1;
    }
}

struct OverlapWs {
    u32 *best;
    unsigned long long *winner;
    Seg *agg;
    u32 *join;
};

static OverlapWs carve_overlap(Arena &ar, i64 n) {
    OverlapWs w;
    w.best = ar.alloc<u32>(2);
    w.winner = ar.alloc<unsigned long long>(1);
    w.agg = ar.alloc<Seg>(ceil_div(n > 0 ? n : 1, OV_TILE) + 1);
    w.join = ar.alloc<u32>(ceil_div(n > 0 ? n : 1, OV_TILE) + 1);
    return w;
}

// best_ready: *w.best already holds the cross-adjacent maximum (the pipeline
// computes it inside the LCP permute kernel).
static int overlap_scan(const u32 *sa, const u32 *lcp, i64 n, i64 boundary, i64 *out3, OverlapWs w,
                        cudaStream_t st, bool best_ready = false) {
    SAIX_CUDA(cudaMemsetAsync(w.winner, 0xFF, sizeof(unsigned long long), st));
    i64 ntiles = ceil_div(n, OV_TILE);
    int g = grid_for(n, OV_THREADS, kNumSMs * 8);
    if (!best_ready) {
        SAIX_CUDA(cudaMemsetAsync(w.best, 0, sizeof(u32), st));
        Prof prof_("overlap.cross_max", 8.0 * n, st);
        k_cross_max<<<g, OV_THREADS, 0, st>>>(sa, lcp, n, (u32)boundary, w.best);
    }
    SAIX_LAUNCHED();
    {
        // the run scan must read every LCP entry; SA only where runs join
        Prof prof_("overlap.runs", 4.0 * n, st);
        k_runs_reduce<<<(unsigned)ntiles, OV_THREADS, 0, st>>>(sa, lcp, n, w.best, (u32)boundary, w.agg, w.join);
        k_runs_carry<<<1, OV_THREADS, 0, st>>>(w.agg, ntiles);
        k_runs_apply<<<(unsigned)ntiles, OV_THREADS, 0, st>>>(sa, lcp, n, w.best, (u32)boundary, w.agg, w.join,
                                                              w.winner);
    }
    SAIX_LAUNCHED();
    k_overlap_finish<<<1, 1, 0, st>>>(w.best, w.winner, (u32)boundary, out3);
    SAIX_LAUNCHED();
    return SAIX_OK;
}

}  // namespace saix

using namespace saix;

extern "C" int saix_encode_gsa(const uint8_t *a_ascii, int64_t na, const uint8_t *b_ascii, int64_t nb, int keep_n,
                               uint8_t *gsa, int64_t *bad_pos, void *stream) {
    if (na < 0 || nb < 0 || !gsa || !bad_pos || (na && !a_ascii) || (nb && !b_ascii)) {
        set_error("saix_encode_gsa: invalid arguments");
        return SAIX_EINVAL;
    }
    cudaStream_t st = (cudaStream_t)stream;
    i64 n = na + nb + 1;
    Prof prof_("encode.gsa", 2.0 * n, st);
    int words = ((uintptr_t)gsa & 15) == 0;
    k_encode_gsa<<<grid_for(words ? n / 16 + 1 : n, 256), 256, 0, st>>>(a_ascii, na, b_ascii ? b_ascii : a_ascii,
                                                                       nb, keep_n, 1, gsa, bad_pos, words);
    SAIX_LAUNCHED();
    return SAIX_OK;
}

extern "C" int saix_encode(const uint8_t *ascii, int64_t n, int keep_n, uint8_t *ranks, int64_t *bad_pos,
                           void *stream) {
    if (n < 0 || (n && (!ascii || !ranks)) || !bad_pos) {
        set_error("saix_encode: invalid arguments");
        return SAIX_EINVAL;
    }
    if (n == 0) return SAIX_OK;
    cudaStream_t st = (cudaStream_t)stream;
    int words = ((uintptr_t)ranks & 15) == 0;
    k_encode_gsa<<<grid_for(words ? n / 16 + 1 : n, 256), 256, 0, st>>>(ascii, n, nullptr, 0, keep_n, 0, ranks,
                                                                       bad_pos, words);
    SAIX_LAUNCHED();
    return SAIX_OK;
}

extern "C" size_t saix_overlap_workspace_bytes(int64_t n) {
    Arena ar;
    carve_overlap(ar, n);
    return ar.peak + Arena::kAlign;
}

extern "C" int saix_overlap_scan(const uint32_t *sa, const uint32_t *lcp, int64_t n, int64_t boundary, int64_t *out3,
                                 void *ws, size_t ws_bytes, void *stream) {
    if (n < 0 || !out3 || (n > 0 && (!sa || !lcp)) || boundary < 0 || boundary >= (n > 0 ? n : 1)) {
        set_error("saix_overlap_scan: invalid arguments");
        return SAIX_EINVAL;
    }
    Arena ar{(char *)ws, ws_bytes};
    OverlapWs w = carve_overlap(ar, n);
    SAIX_ARENA_OK(ar);
    return overlap_scan(sa, lcp, n, boundary, out3, w, (cudaStream_t)stream);
}

// ------------------------------------------------------------ pipeline

namespace saix {
struct PairWs {
    u8 *gsa;
    u32 *sa, *isa, *lcp, *phi;
    OverlapWs ov;
    void *rest;
    size_t rest_bytes;
};
static size_t pair_ws(Arena &ar, i64 n, PairWs *w) {
    PairWs t;
    t.gsa = ar.alloc<u8>(n + 8);
    t.sa = ar.alloc<u32>(n);
    t.isa = ar.alloc<u32>(n);
    t.lcp = ar.alloc<u32>(n);
    t.phi = ar.alloc<u32>(n);
    t.ov = carve_overlap(ar, n);
    size_t need = saix_dc3_workspace_bytes(n, 1);
    size_t l = saix_lcp_workspace_bytes(n);
    if (l > need) need = l;
    t.rest = ar.alloc<char>((i64)need);
    t.rest_bytes = need;
    if (w) *w = t;
    return ar.peak;
}
}  // namespace saix

// Pairs of up to pd::NMAX generalized-text residues run through the on-chip
// pair kernel (pairdc3.cu) as a batch of one: A and B copied back to back
// into the workspace, then saix_overlap_batch_dev.  One launch instead of the
// multi-pass DC3 pipeline; pd_onchip_enabled() off (the batch A/B knob) keeps
// the pipeline.
constexpr i64 kOnchipResidues = 20480;  // pd::NMAX
namespace saix {
int pd_onchip_enabled();  // pairdc3.cu
}

static size_t small_pair_ws(i64 na, i64 nb) {
    const int64_t offs[3] = {0, na, na + nb};
    return (size_t)((na + nb + 15) & ~15ll) + saix_overlap_batch_workspace_bytes(offs, 1);
}

__global__ void k_small_bad(i64 *__restrict__ bad, i64 na) {
    // batch offsets put B right after A; the pipeline reports GSA positions
    if (*bad != INT64_MAX && *bad >= na) *bad += 1;
}

extern "C" size_t saix_longest_overlap_workspace_bytes(int64_t na, int64_t nb) {
    Arena ar;
    size_t bytes = pair_ws(ar, na + nb + 1, nullptr) + Arena::kAlign;
    if (na > 0 && nb > 0 && na + nb + 1 <= kOnchipResidues) {
        const size_t sm = small_pair_ws(na, nb) + Arena::kAlign;
        if (sm > bytes) bytes = sm;
    }
    return bytes;
}

extern "C" int saix_longest_overlap(const uint8_t *a_ascii, int64_t na, const uint8_t *b_ascii, int64_t nb,
                                    int keep_n, int64_t *out3, int64_t *bad_pos, void *ws, size_t ws_bytes,
                                    void *stream) {
    if (na < 0 || nb < 0 || !out3 || !bad_pos) {
        set_error("saix_longest_overlap: invalid arguments");
        return SAIX_EINVAL;
    }
    cudaStream_t st = (cudaStream_t)stream;
    k_pipeline_init<<<1, 1, 0, st>>>(out3, bad_pos);
    SAIX_LAUNCHED();
    // overlap.py:120-121: empty input returns before encoding (no validation)
    if (na == 0 || nb == 0) return SAIX_OK;
    i64 n = na + nb + 1;
    if (n <= kOnchipResidues && pd_onchip_enabled()) {
        char *base = (char *)(((uintptr_t)ws + 15) & ~(uintptr_t)15);
        const size_t skip = (size_t)(base - (char *)ws), cat = (size_t)((na + nb + 15) & ~15ll);
        if (!ws || ws_bytes < skip + cat) {
            set_error("saix_longest_overlap: workspace too small");
            return SAIX_EINVAL;
        }
        uint8_t *seqs = (uint8_t *)base;
        SAIX_CUDA(cudaMemcpyAsync(seqs, a_ascii, (size_t)na, cudaMemcpyDeviceToDevice, st));
        SAIX_CUDA(cudaMemcpyAsync(seqs + na, b_ascii, (size_t)nb, cudaMemcpyDeviceToDevice, st));
        const int64_t offs[3] = {0, na, na + nb};
        SAIX_TRY(saix_overlap_batch_dev(seqs, offs, nullptr, 1, keep_n, out3, bad_pos, base + cat,
                                        ws_bytes - skip - cat, stream));
        k_small_bad<<<1, 1, 0, st>>>(bad_pos, na);
        SAIX_LAUNCHED();
        return SAIX_OK;
    }
    Arena ar{(char *)ws, ws_bytes};
    PairWs w;
    pair_ws(ar, n, &w);
    SAIX_ARENA_OK(ar);
    SAIX_TRY(saix_encode_gsa(a_ascii, na, b_ascii, nb, keep_n, w.gsa, bad_pos, stream));
    int sigma = (keep_n ? 5 : 4) + 1;  // max(sigma_A, sigma_B) + 1 (overlap.py:88)
    // the pipeline never needs the top-level ISA (LCP compares SA neighbours)
    SAIX_TRY(dc3_compute(w.gsa, 1, n, sigma, w.sa, nullptr, w.rest, w.rest_bytes, nullptr, st));
    SAIX_CUDA(cudaMemsetAsync(w.ov.best, 0, sizeof(u32), st));
    // direct word-compare LCP on the 2-bit packed GSA (separator at na);
    // N residues (keep_n) fall back to the byte compare / Kasai
    SAIX_TRY(lcp_compute(w.gsa, 1, n, w.sa, w.lcp, w.rest, w.rest_bytes, st, na, w.ov.best, w.phi, false, sigma, na));
    return overlap_scan(w.sa, w.lcp, n, na, out3, w.ov, st, true);
}

// ============================================================ batched pairs
//
// A wave of P pairs becomes ONE generalized text
//     X = (A_0+2) 2 (B_0+2) 1 | (A_1+2) 2 (B_1+2) 1 | ...
// with the in-pair separator at rank 2 and a terminator 1 below every other
// symbol.  Two suffixes of the same pair compare exactly as in the pair's own
// generalized text (overlap.py:83-95, padding 0): the first one to reach its
// terminator is smaller, and no match can run past a terminator.  So:
//   DC3(X)  ->  stable partition of SA(X) by pair id  (each pair's suffixes
//   in their own order; pair p's block is [xoff[p], xoff[p+1]) with the
//   terminator suffix first)  ->  Phi within each block  ->  PLCP walk over
//   X  ->  one CTA per pair: LCP permute + both overlap passes on chip.

namespace saix {

__device__ __forceinline__ u32 pair_of(const i64 *__restrict__ xoff, i64 P, i64 stride, i64 g) {
    if (stride > 0) return (u32)g / (u32)stride;  // waves hold < 2^30 residues: 32-bit division
    i64 lo = 0, hi = P - 1;  // largest p with xoff[p] <= g
    while (lo < hi) {
        i64 mid = (lo + hi + 1) >> 1;
        if (xoff[mid] <= g) lo = mid;
        else hi = mid - 1;
    }
    return (u32)lo;
}

__global__ void k_batch_build_x(const u8 *__restrict__ seqs, const i64 *__restrict__ offs,
                                const i64 *__restrict__ xoff, i64 P, int keep_n, u8 *__restrict__ X,
                                i64 *__restrict__ bad) {
    i64 local_bad = INT64_MAX;
    for (i64 p = blockIdx.x; p < P; p += gridDim.x) {
        i64 x0 = xoff[p], len = xoff[p + 1] - x0;
        if (len == 0) continue;  // empty side: (0, 0, 0) without validation
        i64 a0 = offs[2 * p], la = offs[2 * p + 1] - a0, b0 = offs[2 * p + 1];
        for (i64 i = threadIdx.x; i < len; i += blockDim.x) {
            u32 r;
            i64 src = -1;
            if (i < la) src = a0 + i;
            else if (i > la && i < len - 1) src = b0 + (i - la - 1);
            if (src >= 0) {
                r = rank_of_ascii(seqs[src], keep_n);
                if (r == 0) {
                    if (src < local_bad) local_bad = src;
                    r = 1;
                }
                r += 2;
            } else {
                r = (i == la) ? 2u : 1u;  // in-pair separator / terminator
            }
            X[x0 + i] = (u8)r;
        }
    }
    if (local_bad != INT64_MAX) atomicMin((unsigned long long *)bad, (unsigned long long)local_bad);
}

struct PairKey {
    const i64 *xoff;
    i64 P, stride;
    U32Div dv;  // fixed-length pairs: v / stride by multiply-high
    __device__ __forceinline__ u32 operator()(u32 v) const {
        return stride > 0 ? dv.div(v) : pair_of(xoff, P, stride, v);
    }
};

struct PairSrc {
    const u32 *sa;
    const i64 *xoff;
    i64 P, stride;
    __device__ __forceinline__ bool get(i64 i, u32 &k, u32 &v) const {
        v = __ldcs(sa + i);
        k = pair_of(xoff, P, stride, v);
        return true;
    }
};

// Phi within each pair block: the terminator entry and the block's first
// real suffix have no predecessor.
__global__ void k_batch_phi(const u32 *__restrict__ sap, i64 nx, const i64 *__restrict__ xoff, i64 P, i64 stride,
                            u32 *__restrict__ phi) {
    for (i64 r = (i64)blockIdx.x * blockDim.x + threadIdx.x; r < nx; r += (i64)gridDim.x * blockDim.x) {
        u32 g = sap[r];
        i64 x0 = xoff[pair_of(xoff, P, stride, (i64)r)];
        phi[g] = (r <= x0 + 1) ? 0xFFFFFFFFu : sap[r - 1];
    }
}

// Direct LCP inside each pair block of the partitioned SA: lcp[r] of the
// adjacent suffixes sap[r-1], sap[r] (same pair) by word compares on the
// 2-bit packed wave text.  The pair's separator xs and terminator xt are
// unique inside the pair, so a match stops at the nearer of them for either
// suffix (the packed codes of those two symbols are never trusted).
struct PairClamp {
    const i64 *xoff, *offs;
    i64 P, stride;
    __device__ __forceinline__ u32 lim(u32 g, u32 i, u32 j) const {
        i64 x0 = xoff[g];
        i64 xs = x0 + (offs[2 * g + 1] - offs[2 * g]), xt = xoff[g + 1] - 1;
        i64 li = (i <= xs ? xs : xt) - (i64)i, lj = (j <= xs ? xs : xt) - (i64)j;
        return (u32)(li < lj ? li : lj);
    }
};

template <class Txt>
__global__ void k_batch_lcp(Txt tx, const u32 *__restrict__ sap, i64 nx, PairClamp pc, u32 *__restrict__ lcp,
                            u32 *__restrict__ ncap, u32 *__restrict__ list, u32 list_cap) {
    for (i64 r = (i64)blockIdx.x * blockDim.x + threadIdx.x; r < nx; r += (i64)gridDim.x * blockDim.x) {
        u32 g = pair_of(pc.xoff, pc.P, pc.stride, r);
        u32 h = 0;
        if (r > pc.xoff[g] + 1) {  // the terminator entry and the first real suffix have no predecessor
            u32 i = sap[r - 1], j = __ldcs(sap + r);
            u32 lim = pc.lim(g, i, j);
            u32 stop = lim < LCP_CAP ? lim : LCP_CAP;
            h = tx.match(i, j, 0, stop);
            if (h == LCP_CAP && lim > LCP_CAP) {
                u32 at = atomicAdd(ncap, 1u);
                if (at < list_cap) list[at] = (u32)r;
            }
        }
        __stcs(lcp + r, h);
    }
}

// packed-text variant with LD_ILP pairs per thread in flight (see lcp.cu)
constexpr int BL_ILP = 4;
__global__ void __launch_bounds__(256)
k_batch_lcp_p2(Pack2Text tx, const u32 *__restrict__ sap, i64 nx, PairClamp pc, U32Div dv, u32 *__restrict__ lcp,
               u32 *__restrict__ ncap, u32 *__restrict__ list, u32 list_cap) {
    const i64 step = (i64)gridDim.x * 256 * BL_ILP;
    for (i64 base = (i64)blockIdx.x * 256 * BL_ILP; base < nx; base += step) {
        u32 iv[BL_ILP], jv[BL_ILP], gv[BL_ILP];
        u64 wi[BL_ILP], wj[BL_ILP];
#pragma unroll
        for (int q = 0; q < BL_ILP; q++) {
            i64 r = base + q * 256 + threadIdx.x;
            gv[q] = 0xFFFFFFFFu;
            jv[q] = iv[q] = 0u;
            if (r < nx) {
                u32 g = pc.stride > 0 ? dv.div((u32)r) : pair_of(pc.xoff, pc.P, pc.stride, r);
                if (r > pc.xoff[g] + 1) {  // the terminator entry and the first real suffix have no predecessor
                    gv[q] = g;
                    jv[q] = __ldcs(sap + r);
                    iv[q] = sap[r - 1];
                }
            }
        }
#pragma unroll
        for (int q = 0; q < BL_ILP; q++) {
            wi[q] = load2(tx.W, iv[q]);
            wj[q] = load2(tx.W, jv[q]);
        }
#pragma unroll
        for (int q = 0; q < BL_ILP; q++) {
            i64 r = base + q * 256 + threadIdx.x;
            if (r >= nx) continue;
            u32 h = 0;
            if (gv[q] != 0xFFFFFFFFu) {
                u32 i = iv[q], j = jv[q];
                u32 lim = pc.lim(gv[q], i, j);
                u32 stop = lim < LCP_CAP ? lim : LCP_CAP;
                u64 d = wi[q] ^ wj[q];
                if (d) h = min((u32)(__ffsll((long long)d) - 1) >> 1, stop);
                else h = tx.match(i, j, 32u < stop ? 32u : stop, stop);
                if (h == LCP_CAP && lim > LCP_CAP) {
                    u32 at = atomicAdd(ncap, 1u);
                    if (at < list_cap) list[at] = (u32)r;
                }
            }
            __stcs(lcp + r, h);
        }
    }
}

template <class Txt>
__global__ void k_batch_lcp_extend(Txt tx, const u32 *__restrict__ sap, PairClamp pc, u32 *__restrict__ lcp,
                                   const u32 *__restrict__ ncap, const u32 *__restrict__ list) {
    const u32 cnt = *ncap;
    const int lane = lane_id();
    for (u32 e = ((i64)blockIdx.x * blockDim.x + threadIdx.x) >> 5; e < cnt; e += ((i64)gridDim.x * blockDim.x) >> 5) {
        u32 r = list[e];
        u32 i = sap[r - 1], j = sap[r];
        u32 lim = pc.lim(pair_of(pc.xoff, pc.P, pc.stride, r), i, j);
        u32 h = LCP_CAP;
        while (h < lim) {
            u32 lo = h + 32u * lane;
            u32 hi = min(lo + 32u, lim);
            u32 got = lo < lim ? tx.match(i, j, lo, hi) : lo;
            u32 short_ = __ballot_sync(0xffffffffu, lo < lim && got < hi);
            if (short_) {
                h = __shfl_sync(0xffffffffu, got, __ffs(short_) - 1);
                break;
            }
            h = min(h + 32u * 32u, lim);
        }
        if (lane == 0) lcp[r] = h;
    }
}

constexpr int BO_ITEMS = 16;
__global__ void __launch_bounds__(OV_THREADS)
k_batch_overlap(const u32 *__restrict__ sap, const u32 *__restrict__ plcp, const i64 *__restrict__ xoff,
                const i64 *__restrict__ offs, i64 P, i64 *__restrict__ out, int by_rank) {
    __shared__ u32 sh_red[OV_THREADS / 32];
    __shared__ unsigned long long sh_win[OV_THREADS / 32];
    for (i64 p = blockIdx.x; p < P; p += gridDim.x) {
        i64 x0 = xoff[p], x1 = xoff[p + 1];
        if (x1 == x0) {
            if (threadIdx.x == 0) out[3 * p] = out[3 * p + 1] = out[3 * p + 2] = 0;
            continue;
        }
        const u32 la = (u32)(offs[2 * p + 1] - offs[2 * p]);
        const i64 s0 = x0 + 1;  // first real suffix (the terminator sorts first)
        // pass 1: best cross-sequence adjacent LCP (overlap.py:129-136)
        u32 mx = 0;
        for (i64 r = s0 + 1 + threadIdx.x; r < x1; r += OV_THREADS) {
            u32 ga = (u32)(sap[r - 1] - x0), gb = (u32)(sap[r] - x0);
            bool cross = ga != la && gb != la && ((ga < la) != (gb < la));
            if (cross) mx = max(mx, plcp[by_rank ? (u32)r : sap[r]]);
        }
        for (int o = 16; o; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        if (lane_id() == 0) sh_red[threadIdx.x >> 5] = mx;
        __syncthreads();
        u32 best = 0;
        for (int w = 0; w < OV_THREADS / 32; w++) best = max(best, sh_red[w]);
        __syncthreads();
        if (best == 0) {
            if (threadIdx.x == 0) out[3 * p] = out[3 * p + 1] = out[3 * p + 2] = 0;
            continue;
        }
        // pass 2: runs of lcp >= best, per-run min A / B position (138-152):
        // each thread folds BO_ITEMS consecutive elements, one block scan of
        // the per-thread aggregates per chunk, then the same elements again
        // with the carry-in to close runs
        Seg carry{0u, kInf, kInf};
        unsigned long long win = ~0ull;
        for (i64 c = s0; c < x1; c += (i64)OV_THREADS * BO_ITEMS) {
            const i64 r0 = c + (i64)threadIdx.x * BO_ITEMS;
            u32 lv[BO_ITEMS + 1], gv[BO_ITEMS];
#pragma unroll
            for (int q = 0; q <= BO_ITEMS; q++) {
                i64 r = r0 + q;
                lv[q] = r < x1 ? (r == s0 ? 0u : plcp[by_rank ? (u32)r : sap[r]]) : 0u;
                if (q < BO_ITEMS) gv[q] = r < x1 ? sap[r] - (u32)x0 : 0u;
            }
            Seg agg{0u, kInf, kInf};
#pragma unroll
            for (int q = 0; q < BO_ITEMS; q++) {
                i64 r = r0 + q;
                if (r >= x1) break;
                Seg e{(r == s0 || lv[q] < best) ? 1u : 0u, gv[q] < la ? gv[q] : kInf, gv[q] > la ? gv[q] : kInf};
                agg = seg_combine(agg, e);
            }
            Seg tot;
            Seg run = seg_combine(carry, block_seg_exclusive(agg, tot));
#pragma unroll
            for (int q = 0; q < BO_ITEMS; q++) {
                i64 r = r0 + q;
                if (r >= x1) break;
                Seg e{(r == s0 || lv[q] < best) ? 1u : 0u, gv[q] < la ? gv[q] : kInf, gv[q] > la ? gv[q] : kInf};
                run = seg_combine(run, e);
                bool end = (r + 1 >= x1) || lv[q + 1] < best;
                if (end && run.a != kInf && run.b != kInf) win = min(win, ((unsigned long long)run.a << 32) | run.b);
            }
            carry = seg_combine(carry, tot);
        }
        for (int o = 16; o; o >>= 1) win = min(win, __shfl_xor_sync(0xffffffffu, win, o));
        if (lane_id() == 0) sh_win[threadIdx.x >> 5] = win;
        __syncthreads();
        if (threadIdx.x == 0) {
            for (int w = 1; w < OV_THREADS / 32; w++) win = min(win, sh_win[w]);
            out[3 * p] = best;
            out[3 * p + 1] = (i64)(win >> 32);
            out[3 * p + 2] = (i64)(win & 0xFFFFFFFFull) - (i64)la - 1;
        }
        __syncthreads();
    }
}

// One warp per pair: pass 1 (best cross-sequence adjacent LCP) and pass 2
// (runs of lcp >= best, per-run min A / B, overlap.py:129-152) as lane-strided
// streams over the pair block; pass 2 folds 16 consecutive elements per lane
// and closes runs with a warp segmented scan per 512-element chunk.  Many
// pairs in flight per SM hide the latency the CTA-per-pair form exposed.
constexpr int BW_ITEMS = 16;
__global__ void __launch_bounds__(256)
k_batch_overlap_warp(const u32 *__restrict__ sap, const u32 *__restrict__ lcp, const i64 *__restrict__ xoff,
                     const i64 *__restrict__ offs, i64 P, i64 *__restrict__ out) {
    const int lane = lane_id();
    const i64 warps = ((i64)gridDim.x * blockDim.x) >> 5;
    for (i64 p = ((i64)blockIdx.x * blockDim.x + threadIdx.x) >> 5; p < P; p += warps) {
        const i64 x0 = xoff[p], x1 = xoff[p + 1];
        if (x1 == x0) {
            if (lane == 0) out[3 * p] = out[3 * p + 1] = out[3 * p + 2] = 0;
            continue;
        }
        const u32 la = (u32)(offs[2 * p + 1] - offs[2 * p]);
        const i64 s0 = x0 + 1;  // first real suffix (the terminator sorts first)
        u32 mx = 0;
        for (i64 c = s0; c < x1; c += 32 * BW_ITEMS) {  // 16 consecutive pairs per lane, loads in flight together
            const i64 r0 = c + (i64)lane * BW_ITEMS;
            u32 gv[BW_ITEMS + 1], lv[BW_ITEMS];
#pragma unroll
            for (int q = 0; q <= BW_ITEMS; q++) {
                i64 r = r0 + q - 1;
                gv[q] = (r >= s0 && r < x1) ? __ldg(sap + r) - (u32)x0 : la;
                if (q < BW_ITEMS) lv[q] = r + 1 < x1 ? __ldg(lcp + r + 1) : 0u;
            }
#pragma unroll
            for (int q = 0; q < BW_ITEMS; q++) {
                u32 ga = gv[q], gb = gv[q + 1];  // suffixes r0+q-1, r0+q
                bool cross = ga != la && gb != la && ((ga < la) != (gb < la));
                if (cross && lv[q] > mx) mx = lv[q];
            }
        }
        for (int o = 16; o; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        const u32 best = mx;
        if (best == 0) {
            if (lane == 0) out[3 * p] = out[3 * p + 1] = out[3 * p + 2] = 0;
            continue;
        }
        Seg carry{0u, kInf, kInf};
        unsigned long long win = ~0ull;
        for (i64 c = s0; c < x1; c += 32 * BW_ITEMS) {
            const i64 r0 = c + (i64)lane * BW_ITEMS;
            u32 lv[BW_ITEMS + 1], gv[BW_ITEMS];
#pragma unroll
            for (int q = 0; q <= BW_ITEMS; q++) {
                i64 r = r0 + q;
                lv[q] = r < x1 ? (r == s0 ? 0u : __ldg(lcp + r)) : 0u;
                if (q < BW_ITEMS) gv[q] = r < x1 ? __ldg(sap + r) - (u32)x0 : 0u;
            }
            Seg agg{0u, kInf, kInf};
#pragma unroll
            for (int q = 0; q < BW_ITEMS; q++) {
                if (r0 + q >= x1) break;
                Seg e{(r0 + q == s0 || lv[q] < best) ? 1u : 0u, gv[q] < la ? gv[q] : kInf, gv[q] > la ? gv[q] : kInf};
                agg = seg_combine(agg, e);
            }
            // warp exclusive segmented scan of the lane aggregates
            Seg inc = agg;
            for (int o = 1; o < 32; o <<= 1) {
                Seg y = seg_shfl_up(inc, o);
                if (lane >= o) inc = seg_combine(y, inc);
            }
            Seg ex = seg_shfl_up(inc, 1);
            if (lane == 0) ex = Seg{0u, kInf, kInf};
            Seg run = seg_combine(carry, ex);
#pragma unroll
            for (int q = 0; q < BW_ITEMS; q++) {
                i64 r = r0 + q;
                if (r >= x1) break;
                Seg e{(r == s0 || lv[q] < best) ? 1u : 0u, gv[q] < la ? gv[q] : kInf, gv[q] > la ? gv[q] : kInf};
                run = seg_combine(run, e);
                bool end = (r + 1 >= x1) || lv[q + 1] < best;
                if (end && run.a != kInf && run.b != kInf) win = min(win, ((unsigned long long)run.a << 32) | run.b);
            }
            Seg tot{__shfl_sync(0xffffffffu, inc.f, 31), __shfl_sync(0xffffffffu, inc.a, 31),
                    __shfl_sync(0xffffffffu, inc.b, 31)};
            carry = seg_combine(carry, tot);
        }
        for (int o = 16; o; o >>= 1) win = min(win, __shfl_xor_sync(0xffffffffu, win, o));
        if (lane == 0) {
            out[3 * p] = best;
            out[3 * p + 1] = (i64)(win >> 32);
            out[3 * p + 2] = (i64)(win & 0xFFFFFFFFull) - (i64)la - 1;
        }
    }
}

struct BatchLayout {
    i64 P, nx, stride;
    std::vector<i64> xoff;
};

static int batch_layout(const i64 *offs, i64 P, BatchLayout &b) {
    b.P = P;
    b.xoff.assign((size_t)P + 1, 0);
    i64 common = -1;
    bool fixed = true;
    for (i64 p = 0; p < P; p++) {
        i64 la = offs[2 * p + 1] - offs[2 * p], lb = offs[2 * p + 2] - offs[2 * p + 1];
        if (la < 0 || lb < 0) {
            set_error("saix_overlap_batch: offsets must be non-decreasing");
            return SAIX_EINVAL;
        }
        i64 len = (la && lb) ? la + lb + 2 : 0;
        if (common < 0) common = len;
        if (len != common) fixed = false;
        b.xoff[p + 1] = b.xoff[p] + len;
    }
    b.nx = b.xoff[P];
    b.stride = (fixed && common > 0) ? common : 0;
    if (b.nx >= ((i64)1 << 30)) {
        set_error("saix_overlap_batch: %lld residues in one call; split into waves < 2^30", (long long)b.nx);
        return SAIX_EINVAL;
    }
    return SAIX_OK;
}

struct BatchWs {
    u8 *X;
    u32 *sa;
    i64 *xoff, *offs;
    void *dc3;
    size_t dc3_bytes;
    u32 *k0, *v0, *k1, *v1, *scratch;
    void *plcp_ws;
    size_t plcp_bytes;
    u64 *W2;
    u32 *ncap, *list;
};

static size_t batch_ws(Arena &ar, i64 P, i64 nx, BatchWs *w) {
    BatchWs t;
    t.X = ar.alloc<u8>(nx + 8);
    t.sa = ar.alloc<u32>(nx);
    t.xoff = ar.alloc<i64>(P + 1);
    t.offs = ar.alloc<i64>(2 * P + 1);
    size_t mark = ar.mark();
    t.dc3_bytes = saix_dc3_workspace_bytes(nx, 1);
    t.dc3 = ar.alloc<char>((i64)t.dc3_bytes);
    size_t peak_dc3 = ar.mark();
    ar.reset(mark);
    t.k0 = ar.alloc<u32>(nx);
    t.v0 = ar.alloc<u32>(nx);
    t.k1 = ar.alloc<u32>(nx);
    t.v1 = ar.alloc<u32>(nx);
    t.scratch = ar.alloc<u32>(lsd_scratch_words(nx) > os_scratch_words(nx) ? lsd_scratch_words(nx) : os_scratch_words(nx));
    t.plcp_bytes = plcp_workspace_bytes(nx);
    t.plcp_ws = ar.alloc<char>((i64)t.plcp_bytes);
    t.W2 = ar.alloc<u64>(pack2_words(nx));
    t.ncap = ar.alloc<u32>(2);
    t.list = ar.alloc<u32>(lcp_list_cap(nx));
    if (ar.mark() < peak_dc3) ar.reset(peak_dc3);
    if (w) *w = t;
    return ar.peak;
}

}  // namespace saix

namespace saix {

// The wave-global batched path: all pairs of a call share one generalized
// text (< 2^30 residues).  saix_overlap_batch (pairdc3.cu) runs every pair
// that fits on chip in its own CTA and sends the rest here.
size_t overlap_batch_global_ws(const i64 *offs_host, i64 npairs) {
    BatchLayout b;
    if (npairs < 0 || (npairs > 0 && !offs_host) || batch_layout(offs_host, npairs, b)) return 0;
    Arena ar;
    return batch_ws(ar, npairs, b.nx, nullptr) + Arena::kAlign;
}

int overlap_batch_global(const u8 *seqs, const i64 *offs_host, i64 npairs, int keep_n, i64 *out, i64 *bad,
                         void *ws, size_t ws_bytes, cudaStream_t st) {
    if (npairs < 0 || (npairs > 0 && (!offs_host || !out)) || !bad) {
        set_error("saix_overlap_batch: invalid arguments");
        return SAIX_EINVAL;
    }
    k_pipeline_init<<<1, 1, 0, st>>>(out, bad);  // out[0..2] zero, bad = INT64_MAX
    SAIX_LAUNCHED();
    if (npairs == 0) return SAIX_OK;
    BatchLayout b;
    SAIX_TRY(batch_layout(offs_host, npairs, b));
    Arena ar{(char *)ws, ws_bytes};
    BatchWs w;
    batch_ws(ar, npairs, b.nx, &w);
    SAIX_ARENA_OK(ar);
    i64 P = npairs, nx = b.nx;
    SAIX_CUDA(cudaMemcpyAsync(w.xoff, b.xoff.data(), (size_t)(P + 1) * 8, cudaMemcpyHostToDevice, st));
    SAIX_CUDA(cudaMemcpyAsync(w.offs, offs_host, (size_t)(2 * P + 1) * 8, cudaMemcpyHostToDevice, st));
    {
        Prof prof_("batch.build_x", 2.0 * nx, st);
        k_batch_build_x<<<(unsigned)(P < 65535 ? P : 65535), 256, 0, st>>>(seqs, w.offs, w.xoff, P, keep_n, w.X, bad);
    }
    SAIX_LAUNCHED();
    if (nx == 0) {
        k_batch_overlap<<<1, OV_THREADS, 0, st>>>(nullptr, nullptr, w.xoff, w.offs, P, out, 0);
        SAIX_LAUNCHED();
        return SAIX_OK;
    }
    int sigma = keep_n ? 7 : 6;  // terminator 1, separator 2, residues 3..6 (N 7)
    {
        const int prev = dc3_window_naming_override(0);
        const int rc = dc3_compute(w.X, 1, nx, sigma, w.sa, nullptr, w.dc3, w.dc3_bytes, nullptr, st);
        dc3_window_naming_override(prev);
        SAIX_TRY(rc);
    }
    // stable partition by pair id: each pair's suffixes keep their order
    u32 *sap = nullptr;
    int pbits = P > 1 ? bits_for((u64)(P - 1)) : 0;
    SAIX_TRY(lsd_partition(PairKey{w.xoff, P, b.stride, U32Div::of(b.stride > 0 ? (u32)b.stride : 1u)}, w.sa,
                           w.v0, nx, pbits, w.scratch, sap, st,
                           "batch.partition"));
    // LCP inside each pair block: direct word compares (2-bit packed wave
    // text: residues 3..6; N residues -> byte compares), capped entries
    // extended by one warp each; highly repetitive pairs -> Phi / PLCP walk
    u32 *lcp = sap == w.sa ? w.v0 : w.sa;  // SA(X) is no longer needed
    PairClamp pc{w.xoff, w.offs, P, b.stride};
    bool pack = !keep_n;
    u32 lc = (u32)lcp_list_cap(nx);
    SAIX_CUDA(cudaMemsetAsync(w.ncap, 0, sizeof(u32), st));
    if (pack) {
        i64 nw = pack2_words(nx);
        {
            Prof prof_("lcp.pack2", (double)nx + 8.0 * nw, st);
            k_pack2<<<grid_for(nw, 256), 256, 0, st>>>(w.X, nx, 3u, w.W2, nw);
        }
        SAIX_LAUNCHED();
    }
    {
        Prof prof_("batch.lcp", 12.0 * nx + nx / 2.0, st);
        if (pack)
            k_batch_lcp_p2<<<grid_for(ceil_div(nx, BL_ILP), 256), 256, 0, st>>>(
                Pack2Text{w.W2}, sap, nx, pc, U32Div::of(b.stride > 0 ? (u32)b.stride : 1u), lcp, w.ncap, w.list, lc);
        else k_batch_lcp<ByteText><<<grid_for(nx, 256), 256, 0, st>>>(ByteText{w.X, nx}, sap, nx, pc, lcp, w.ncap,
                                                                     w.list, lc);
    }
    SAIX_LAUNCHED();
    u32 hc = 0;
    SAIX_CUDA(cudaMemcpyAsync(&hc, w.ncap, sizeof(u32), cudaMemcpyDeviceToHost, st));
    SAIX_CUDA(cudaStreamSynchronize(st));
    int by_rank = 1;
    if (hc > 0 && hc <= lc) {
        Prof prof_("batch.lcp_extend", 0.0, st);
        int ge = grid_for((i64)hc * 32, 256);
        if (pack) k_batch_lcp_extend<Pack2Text><<<ge, 256, 0, st>>>(Pack2Text{w.W2}, sap, pc, lcp, w.ncap, w.list);
        else k_batch_lcp_extend<ByteText><<<ge, 256, 0, st>>>(ByteText{w.X, nx}, sap, pc, lcp, w.ncap, w.list);
        SAIX_LAUNCHED();
    } else if (hc > lc) {
        u32 *phi = lcp;
        {
            Prof prof_("batch.phi", 12.0 * nx, st);
            k_batch_phi<<<grid_for(nx, 256), 256, 0, st>>>(sap, nx, w.xoff, P, b.stride, phi);
        }
        SAIX_LAUNCHED();
        SAIX_TRY(plcp_from_phi(w.X, nx, phi, w.plcp_ws, w.plcp_bytes, st));
        by_rank = 0;
    }
    {
        Prof prof_("batch.overlap", 8.0 * nx, st);
        if (by_rank)
            k_batch_overlap_warp<<<grid_for(P * 32, 256), 256, 0, st>>>(sap, lcp, w.xoff, w.offs, P, out);
        else
            k_batch_overlap<<<(unsigned)(P < 65535 ? P : 65535), OV_THREADS, 0, st>>>(sap, lcp, w.xoff, w.offs, P,
                                                                                       out, by_rank);
    }
    SAIX_LAUNCHED();
    return SAIX_OK;
}

}  // namespace saix
