// cartesian.cu -- the reference's Cartesian-tree RMQ pipeline on the device
// (rmq.py:61-251): build_cartesian, euler_tour, PlusMinusOneRmq, CartesianRmq.
//
// Tree.  The stack construction (rmq.py:91-117: pop while top > v[i]) gives
// the min-heap tree whose leftmost minimum is the ancestor.  Its parent links
// follow from two nearest-value searches: L(i) = previous j with v[j] <= v[i]
// and R(i) = next j with v[j] < v[i]; parent(i) = R(i) if it exists and
// (no L(i) or v[R] >= v[L]), else L(i).  Subtree of v = (L(v), R(v)), so
// a_v = L+1, b_v = R-1.  Both searches run as
//   1. a 2048-element tile in shared memory: each thread walks its 8-element
//      segment with the chain rule (j <- L(j) skips only larger values), then
//      unresolved elements chain across earlier segments of the tile;
//   2. elements still unresolved find the nearest earlier (later) tile whose
//      minimum qualifies by binary lifting over a sparse table of tile minima,
//      then the position inside it by binary search over the tile's suffix
//      (prefix) minima.
// Tour.  With in-order = index order, the tour (node on entry and after each
// child, rmq.py:120-152) has closed forms: depth(v) = #{u: a_u <= v} -
// #{u: b_u < v} - 1 (nested intervals), preorder(v) = a_v + #{u: a_u <= v} -
// (v+1), first_visit(v) = 2 preorder(v) - depth(v), and v is re-emitted at
// first + 2(v - a_v) (after a left child) and + 2(b_v - v) (after a right
// child).  Two histograms and two scans, no pointer chasing.
// ±1 RMQ.  Block minima / leftmost argmin / step-pattern codes per block
// (padded with ascents as in rmq.py:180-186), a presence bitmap of the codes,
// one b x b in-block table per code (rmq.py:199-213), and batched queries
// (rmq.py:219-236, then the LCA map of rmq.py:247-251).
#include "scan.cuh"

namespace saix {

constexpr int CT_THREADS = 256;
constexpr int CT_SEG = 8;
constexpr int CT_TILE = CT_THREADS * CT_SEG;  // 2048
constexpr int CT_NONE = -1;
constexpr int CT_OPEN = -2;  // not resolved inside the tile

template <typename V>
struct CtVals {
    const V *v;
    __device__ __forceinline__ V operator()(i64 i) const { return v[i]; }
};

template <typename V>
__device__ __forceinline__ V ct_min(V a, V b) { return b < a ? b : a; }

// Tile pass: in-tile L / R (CT_OPEN where the answer lies outside the tile),
// the tile's prefix / suffix minima and its minimum.
template <typename V>
__global__ void __launch_bounds__(CT_THREADS)
k_ct_tile(const V *__restrict__ val, i64 n, int *__restrict__ Lo, int *__restrict__ Ro, V *__restrict__ pmin,
          V *__restrict__ smin, V *__restrict__ tmin) {
    // one pad slot per 32 (4-byte V) / 16 (8-byte V) elements: a warp's
    // threads walk their 8-element segments in lockstep without bank conflicts
    constexpr int PSH = sizeof(V) == 4 ? 5 : 4;
    __shared__ V sv_[CT_TILE + (CT_TILE >> PSH)];
    __shared__ short sl_[CT_TILE + (CT_TILE >> 4)], sr_[CT_TILE + (CT_TILE >> 4)];
    __shared__ V wred[2][CT_THREADS / 32];
    auto sv = [&](int k) -> V & { return sv_[k + (k >> PSH)]; };
    auto sl = [&](int k) -> short & { return sl_[k + (k >> 4)]; };
    auto sr = [&](int k) -> short & { return sr_[k + (k >> 4)]; };
    const i64 t0 = (i64)blockIdx.x * CT_TILE;
    const int cnt = n - t0 < CT_TILE ? (int)(n - t0) : CT_TILE;
    for (int k = threadIdx.x; k < cnt; k += CT_THREADS) sv(k) = val[t0 + k];
    __syncthreads();
    const int s0 = threadIdx.x * CT_SEG;
    const int s1 = s0 + CT_SEG < cnt ? s0 + CT_SEG : cnt;
    // phase a: inside the segment
    for (int i = s0; i < s1; i++) {
        int j = i - 1;
        const V x = sv(i);
        while (j >= s0 && sv(j) > x) j = sl(j) >= 0 ? sl(j) : s0 - 1;
        sl(i) = (short)(j >= s0 ? j : CT_OPEN);
    }
    for (int i = s1 - 1; i >= s0; i--) {
        int j = i + 1;
        const V x = sv(i);
        while (j < s1 && sv(j) >= x) j = sr(j) >= 0 ? sr(j) : s1;
        sr(i) = (short)(j < s1 ? j : CT_OPEN);
    }
    __syncthreads();
    // phase b: elements whose answer lies in another segment.  A sparse
    // table over the 256 segment minima (smem) finds the nearest qualifying
    // segment by binary lifting; the element inside it by a <= 8-step walk.
    constexpr int NSEG = CT_THREADS, SLV = 9;  // 2^8 = 256 segments
    __shared__ V segt[SLV][NSEG];
    {
        V m0 = s0 < s1 ? sv(s0) : V(0);
        for (int i = s0 + 1; i < s1; i++) m0 = ct_min(m0, sv(i));
        segt[0][threadIdx.x] = m0;
    }
    const int nseg = (cnt + CT_SEG - 1) / CT_SEG;
    __syncthreads();
    for (int k = 1; k < SLV; k++) {
        const int h = 1 << (k - 1);
        const int u = threadIdx.x;
        if (u < nseg) segt[k][u] = u + h < nseg ? ct_min(segt[k - 1][u], segt[k - 1][u + h]) : segt[k - 1][u];
        __syncthreads();
    }
    const int myseg = threadIdx.x;
    int Lr[CT_SEG], Rr[CT_SEG];
#pragma unroll
    for (int q = 0; q < CT_SEG; q++) {
        const int i = s0 + q;
        Lr[q] = Rr[q] = CT_OPEN;
        if (i >= s1) continue;
        const V x = sv(i);
        int j = sl(i);
        if (j == CT_OPEN) {
            int pos = myseg;  // segments [pos, myseg) all have min > x
            for (int k = SLV - 1; k >= 0; k--) {
                const int w = 1 << k;
                if (pos - w >= 0 && segt[k][pos - w] > x) pos -= w;
            }
            if (pos >= 1) {
                j = pos * CT_SEG - 1;  // last element of segment pos-1, walked left by phase-a links
                while (sv(j) > x) j = sl(j);
            } else {
                j = CT_OPEN;
            }
        }
        Lr[q] = j;
        j = sr(i);
        if (j == CT_OPEN) {
            int pos = myseg + 1;  // segments (myseg, pos) all have min >= x
            for (int k = SLV - 1; k >= 0; k--) {
                const int w = 1 << k;
                if (pos + w <= nseg && segt[k][pos] >= x) pos += w;
            }
            if (pos < nseg) {
                j = pos * CT_SEG;  // first element of segment pos, walked right by phase-a links
                while (sv(j) >= x) j = sr(j);
            } else {
                j = CT_OPEN;
            }
        }
        Rr[q] = j;
    }
    // prefix / suffix minima of the tile (sequential in the segment, then a
    // warp + block combine)
    V pre[CT_SEG], suf[CT_SEG];
    V run = s0 < s1 ? sv(s0) : V(0);
#pragma unroll
    for (int q = 0; q < CT_SEG; q++) {
        if (s0 + q < s1) run = ct_min(run, sv(s0 + q));
        pre[q] = run;
    }
    V run2 = s1 > s0 ? sv(s1 - 1) : V(0);
#pragma unroll
    for (int q = CT_SEG - 1; q >= 0; q--) {
        if (s0 + q < s1) run2 = ct_min(run2, sv(s0 + q));
        suf[q] = run2;
    }
    const bool has = s0 < s1;
    // exclusive prefix-min over threads (carry from the left), suffix-min from the right
    const int lane = lane_id(), w = threadIdx.x >> 5;
    V segmin = run;  // min of my segment (== pre[last])
    bool inc_has = has;
    V inc = segmin;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        V y = __shfl_up_sync(0xffffffffu, inc, o);
        bool yh = __shfl_up_sync(0xffffffffu, inc_has, o);
        if (lane >= o && yh) {
            inc = inc_has ? ct_min(inc, y) : y;
            inc_has = true;
        }
    }
    V incs = segmin;
    bool incs_has = has;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        V y = __shfl_down_sync(0xffffffffu, incs, o);
        bool yh = __shfl_down_sync(0xffffffffu, incs_has, o);
        if (lane + o < 32 && yh) {
            incs = incs_has ? ct_min(incs, y) : y;
            incs_has = true;
        }
    }
    __shared__ bool whas[2][CT_THREADS / 32];
    if (lane == 31) {
        wred[0][w] = inc;
        whas[0][w] = inc_has;
    }
    if (lane == 0) {
        wred[1][w] = incs;
        whas[1][w] = incs_has;
    }
    __syncthreads();
    // carry-in from the left: earlier warps' totals + earlier lanes
    bool cl_has = false, cr_has = false;
    V cl = V(0), cr = V(0);
    for (int u = 0; u < w; u++)
        if (whas[0][u]) {
            cl = cl_has ? ct_min(cl, wred[0][u]) : wred[0][u];
            cl_has = true;
        }
    {
        V y = __shfl_up_sync(0xffffffffu, inc, 1);
        bool yh = __shfl_up_sync(0xffffffffu, inc_has, 1);
        if (lane >= 1 && yh) {
            cl = cl_has ? ct_min(cl, y) : y;
            cl_has = true;
        }
    }
    for (int u = w + 1; u < CT_THREADS / 32; u++)
        if (whas[1][u]) {
            cr = cr_has ? ct_min(cr, wred[1][u]) : wred[1][u];
            cr_has = true;
        }
    {
        V y = __shfl_down_sync(0xffffffffu, incs, 1);
        bool yh = __shfl_down_sync(0xffffffffu, incs_has, 1);
        if (lane + 1 < 32 && yh) {
            cr = cr_has ? ct_min(cr, y) : y;
            cr_has = true;
        }
    }
#pragma unroll
    for (int q = 0; q < CT_SEG; q++) {
        const int i = s0 + q;
        if (i >= s1) continue;
        const i64 g = t0 + i;
        Lo[g] = Lr[q] == CT_OPEN ? CT_OPEN : (int)(t0 + Lr[q]);
        Ro[g] = Rr[q] == CT_OPEN ? CT_OPEN : (int)(t0 + Rr[q]);
        pmin[g] = cl_has ? ct_min(cl, pre[q]) : pre[q];
        smin[g] = cr_has ? ct_min(cr, suf[q]) : suf[q];
    }
    if (threadIdx.x == 0) {
        V m = sv(0);
        for (int u = 0; u < CT_THREADS / 32; u++)
            if (whas[0][u]) m = ct_min(m, wred[0][u]);
        tmin[blockIdx.x] = m;
    }
}

// level k of the tile-minimum sparse table: st[k][t] = min(tmin[t .. t + 2^k - 1])
template <typename V>
__global__ void k_ct_tmin_level(V *__restrict__ st, i64 T, int k) {
    const V *prev = st + (i64)(k - 1) * T;
    V *cur = st + (i64)k * T;
    const i64 h = (i64)1 << (k - 1);
    for (i64 t = (i64)blockIdx.x * blockDim.x + threadIdx.x; t < T; t += (i64)gridDim.x * blockDim.x)
        cur[t] = t + h < T ? ct_min(prev[t], prev[t + h]) : prev[t];
}

// Elements whose L / R lie outside their tile.
template <typename V>
__global__ void k_ct_resolve(const V *__restrict__ val, i64 n, const V *__restrict__ st, i64 T, int levels,
                             const V *__restrict__ pmin, const V *__restrict__ smin, int *__restrict__ Lo,
                             int *__restrict__ Ro) {
    for (i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x) {
        const bool lo = Lo[i] == CT_OPEN, ro = Ro[i] == CT_OPEN;
        if (!lo && !ro) continue;
        const V x = val[i];
        const i64 t = i / CT_TILE;
        if (lo) {
            // nearest tile t' < t with tmin[t'] <= x
            i64 pos = t;  // exclusive end
            for (int k = levels - 1; k >= 0; k--) {
                const i64 w = (i64)1 << k;
                if (pos - w >= 0 && st[(i64)k * T + pos - w] > x) pos -= w;
            }
            int res = CT_NONE;
            if (pos >= 1) {
                const i64 tt = pos - 1;  // last position j in tile tt with smin[j] <= x
                i64 a = tt * CT_TILE, b = a + CT_TILE - 1;
                while (a < b) {
                    const i64 mid = (a + b + 1) >> 1;
                    if (smin[mid] <= x) a = mid;
                    else b = mid - 1;
                }
                res = (int)a;
            }
            Lo[i] = res;
        }
        if (ro) {
            // nearest tile t' > t with tmin[t'] < x
            i64 pos = t + 1;
            for (int k = levels - 1; k >= 0; k--) {
                const i64 w = (i64)1 << k;
                if (pos + w <= T && st[(i64)k * T + pos] >= x) pos += w;
            }
            int res = CT_NONE;
            if (pos < T) {
                i64 a = pos * CT_TILE, b = a + CT_TILE - 1 < n - 1 ? a + CT_TILE - 1 : n - 1;
                while (a < b) {  // first j with pmin[j] < x
                    const i64 mid = (a + b) >> 1;
                    if (pmin[mid] < x) b = mid;
                    else a = mid + 1;
                }
                res = (int)a;
            }
            Ro[i] = res;
        }
    }
}

// parent / children / subtree bounds; histograms of a_v and b_v
template <typename V>
__global__ void k_ct_link(const V *__restrict__ val, i64 n, const int *__restrict__ Lo, const int *__restrict__ Ro,
                          int *__restrict__ parent, int *__restrict__ left, int *__restrict__ right,
                          u32 *__restrict__ cnt_a, u32 *__restrict__ cnt_b, i64 *__restrict__ root) {
    for (i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x) {
        const int l = Lo[i], r = Ro[i];
        int p;
        if (r >= 0 && (l < 0 || val[r] >= val[l])) p = r;
        else p = l;
        parent[i] = p;
        if (p < 0) *root = i;
        else if (i < p) left[p] = (int)i;
        else right[p] = (int)i;
        const i64 a = l + 1, b = r >= 0 ? r - 1 : n - 1;
        atomicAdd(cnt_a + a, 1u);
        atomicAdd(cnt_b + b, 1u);
    }
}

struct CtCountIn {
    const u32 *c;
    __device__ u32 operator()(i64 i) const { return c[i]; }
};
struct CtInclOut {  // inclusive scan in place
    u32 *o;
    __device__ void operator()(i64 i, u32 excl, u32 v) const { o[i] = excl + v; }
};
struct CtExclOut {
    u32 *o;
    __device__ void operator()(i64 i, u32 excl, u32) const { o[i] = excl; }
};

__global__ void k_ct_tour(i64 n, const int *__restrict__ Lo, const int *__restrict__ Ro, const u32 *__restrict__ Ca,
                          const u32 *__restrict__ Cb, int *__restrict__ nodes, int *__restrict__ depths,
                          int *__restrict__ first) {
    for (i64 v = (i64)blockIdx.x * blockDim.x + threadIdx.x; v < n; v += (i64)gridDim.x * blockDim.x) {
        const i64 a = (i64)Lo[v] + 1, b = Ro[v] >= 0 ? (i64)Ro[v] - 1 : n - 1;
        const i64 depth = (i64)Ca[v] - (i64)Cb[v] - 1;
        const i64 pre = a + (i64)Ca[v] - (v + 1);
        i64 f = 2 * pre - depth;
        first[v] = (int)f;
        nodes[f] = (int)v;
        depths[f] = (int)depth;
        if (v > a) {
            f += 2 * (v - a);
            nodes[f] = (int)v;
            depths[f] = (int)depth;
        }
        if (b > v) {
            f += 2 * (b - v);
            nodes[f] = (int)v;
            depths[f] = (int)depth;
        }
    }
}

// ------------------------------------------------------------ ±1 RMQ

// per block: leftmost argmin and min over the padded block, step code; flags
// a non-unit step
__global__ void k_pm1_blocks(const int *__restrict__ d, i64 m, int b, i64 nblocks, int *__restrict__ bargmin,
                             int *__restrict__ bmin, int *__restrict__ types, u8 *__restrict__ present,
                             int *__restrict__ bad) {
    for (i64 k = (i64)blockIdx.x * blockDim.x + threadIdx.x; k < nblocks; k += (i64)gridDim.x * blockDim.x) {
        const i64 lo = k * b;
        const int last = d[m - 1];
        int best = 0, bestv = d[lo], prev = d[lo];
        u32 code = 0;
        for (int q = 1; q < b; q++) {
            const i64 i = lo + q;
            const int x = i < m ? d[i] : last + 1 + (int)(i - m);
            const int step = x - prev;
            if (i < m && step != 1 && step != -1) *bad = 1;
            if (step < 0) code |= 1u << (q - 1);
            if (x < bestv) {
                bestv = x;
                best = q;
            }
            prev = x;
        }
        if (k + 1 < nblocks) {  // the step into the next block
            const int nx = d[lo + b];
            if (nx - prev != 1 && nx - prev != -1) *bad = 1;
        }
        bargmin[k] = best;
        bmin[k] = bestv;
        types[k] = (int)code;
        if (!present[code]) present[code] = 1;  // plain racing stores of the same value
    }
}

// in-block answer tables of every present code: tab[code][i][j] (u8)
__global__ void k_pm1_tables(int b, u32 ncodes, const u8 *__restrict__ present, u8 *__restrict__ tab) {
    for (i64 x = (i64)blockIdx.x * blockDim.x + threadIdx.x; x < (i64)ncodes * b; x += (i64)gridDim.x * blockDim.x) {
        const u32 code = (u32)(x / b);
        const int i = (int)(x % b);
        if (!present[code]) continue;
        int walk[32];
        walk[0] = 0;
        for (int k = 0; k + 1 < b; k++) walk[k + 1] = walk[k] + (((code >> k) & 1u) ? -1 : 1);
        u8 *row = tab + ((i64)code * b + i) * b;
        int best = i;
        for (int j = 0; j < b; j++) {
            if (j < i) {
                row[j] = 0;
                continue;
            }
            if (walk[j] < walk[best]) best = j;
            row[j] = (u8)best;
        }
    }
}

// queries, part 1 (rmq.py:219-236): in-block candidates and the block range
// between them (answered by the block-minimum sparse table, then part 2).
// first != nullptr maps (i, j) to tour positions first the LCA way (rmq.py:247-250).
__global__ void k_pm1_query_a(int b, const int *__restrict__ types, const u8 *__restrict__ tab,
                              const int *__restrict__ first, const i64 *__restrict__ qi, const i64 *__restrict__ qj,
                              i64 q, i64 *__restrict__ mid_lo, i64 *__restrict__ mid_hi, int *__restrict__ cand) {
    for (i64 t = (i64)blockIdx.x * blockDim.x + threadIdx.x; t < q; t += (i64)gridDim.x * blockDim.x) {
        i64 i = qi[t], j = qj[t];
        if (first) {
            i = first[i];
            j = first[j];
        }
        if (i > j) {
            const i64 x = i;
            i = j;
            j = x;
        }
        const i64 bi = i / b, bj = j / b;
        const int li = (int)(i - bi * b), lj = (int)(j - bj * b);
        int best, right = -1;
        i64 lo = 0, hi = 0, has_mid = 0;
        if (bi == bj) {
            best = (int)(bi * b + tab[((i64)types[bi] * b + li) * b + lj]);
        } else {
            best = (int)(bi * b + tab[((i64)types[bi] * b + li) * b + (b - 1)]);
            right = (int)(bj * b + tab[((i64)types[bj] * b + 0) * b + lj]);
            if (bi + 1 <= bj - 1) {
                lo = bi + 1;
                hi = bj - 1;
                has_mid = 1;
            }
        }
        mid_lo[t] = lo;  // (0, 0) when there is no middle range: always a valid sparse query
        mid_hi[t] = hi;
        cand[3 * t] = best;
        cand[3 * t + 1] = right;
        cand[3 * t + 2] = (int)has_mid;
    }
}

// part 2: combine in positional order so ties resolve leftmost
__global__ void k_pm1_query_b(const int *__restrict__ d, int b, const int *__restrict__ bargmin,
                              const i64 *__restrict__ mid_blk,
                              const int *__restrict__ cand, const int *__restrict__ nodes, i64 q,
                              i64 *__restrict__ out) {
    for (i64 t = (i64)blockIdx.x * blockDim.x + threadIdx.x; t < q; t += (i64)gridDim.x * blockDim.x) {
        int best = cand[3 * t];
        if (cand[3 * t + 2]) {
            const i64 mb = mid_blk[t];
            const int mid = (int)(mb * b + bargmin[mb]);
            if (d[mid] < d[best]) best = mid;
        }
        const int right = cand[3 * t + 1];
        if (right >= 0 && d[right] < d[best]) best = right;
        out[t] = nodes ? nodes[best] : best;
    }
}

}  // namespace saix

using namespace saix;

extern "C" size_t saix_cartesian_workspace_bytes(int64_t n) {
    Arena ar;
    const i64 T = ceil_div(n > 0 ? n : 1, CT_TILE);
    int levels = 1;
    while (((i64)1 << levels) <= T) levels++;
    ar.alloc<int>(n);            // L
    ar.alloc<int>(n);            // R
    ar.alloc<i64>(n);            // pmin (widest V)
    ar.alloc<i64>(n);            // smin
    ar.alloc<i64>(T * levels);   // tile-min sparse table
    ar.alloc<u32>(n + 1);        // cnt_a
    ar.alloc<u32>(n + 1);        // cnt_b
    ar.alloc<u32>(scan_tmp_words(n + 1));
    ar.alloc<i64>(2);
    return ar.peak + Arena::kAlign;
}

template <typename V>
static int cartesian_run(const V *val, i64 n, int *parent, int *left, int *right, int *nodes, int *depths,
                         int *first, int64_t *root_host, void *ws, size_t ws_bytes, cudaStream_t st) {
    Arena ar{(char *)ws, ws_bytes};
    const i64 T = ceil_div(n, CT_TILE);
    int levels = 1;
    while (((i64)1 << levels) <= T) levels++;
    int *Lo = ar.alloc<int>(n), *Ro = ar.alloc<int>(n);
    V *pmin = reinterpret_cast<V *>(ar.alloc<i64>(n)), *smin = reinterpret_cast<V *>(ar.alloc<i64>(n));
    V *stab = reinterpret_cast<V *>(ar.alloc<i64>(T * levels));
    u32 *ca = ar.alloc<u32>(n + 1), *cb = ar.alloc<u32>(n + 1);
    u32 *tmp = ar.alloc<u32>(scan_tmp_words(n + 1));
    i64 *root = ar.alloc<i64>(2);
    SAIX_ARENA_OK(ar);
    {
        Prof prof_("cartesian.nearest", (double)n * (sizeof(V) * 4 + 8), st);
        k_ct_tile<V><<<(unsigned)T, CT_THREADS, 0, st>>>(val, n, Lo, Ro, pmin, smin, stab);
        SAIX_LAUNCHED();
        for (int k = 1; k < levels; k++) {
            k_ct_tmin_level<V><<<grid_for(T, 256), 256, 0, st>>>(stab, T, k);
            SAIX_LAUNCHED();
        }
        k_ct_resolve<V><<<grid_for(n, 256), 256, 0, st>>>(val, n, stab, T, levels, pmin, smin, Lo, Ro);
        SAIX_LAUNCHED();
    }
    {
        Prof prof_("cartesian.link", (double)n * 32, st);
        SAIX_CUDA(cudaMemsetAsync(left, 0xFF, (size_t)n * 4, st));
        SAIX_CUDA(cudaMemsetAsync(right, 0xFF, (size_t)n * 4, st));
        SAIX_CUDA(cudaMemsetAsync(ca, 0, (size_t)(n + 1) * 4, st));
        SAIX_CUDA(cudaMemsetAsync(cb, 0, (size_t)(n + 1) * 4, st));
        k_ct_link<V><<<grid_for(n, 256), 256, 0, st>>>(val, n, Lo, Ro, parent, left, right, ca, cb, root);
        SAIX_LAUNCHED();
    }
    SAIX_TRY(scan_transform(CtCountIn{ca}, CtInclOut{ca}, n, tmp, nullptr, st, "cartesian.scan", 8.0 * n));
    SAIX_TRY(scan_transform(CtCountIn{cb}, CtExclOut{cb}, n, tmp, nullptr, st, "cartesian.scan", 8.0 * n));
    {
        Prof prof_("cartesian.tour", (double)n * 36, st);
        k_ct_tour<<<grid_for(n, 256), 256, 0, st>>>(n, Lo, Ro, ca, cb, nodes, depths, first);
        SAIX_LAUNCHED();
    }
    SAIX_CUDA(cudaMemcpyAsync(root_host, root, 8, cudaMemcpyDeviceToHost, st));
    SAIX_CUDA(cudaStreamSynchronize(st));
    return SAIX_OK;
}

extern "C" int saix_cartesian_build(const void *values, int value_bytes, int64_t n, int32_t *parent, int32_t *left,
                                    int32_t *right, int32_t *tour_nodes, int32_t *tour_depths, int32_t *first_visit,
                                    int64_t *root_host, void *ws, size_t ws_bytes, void *stream) {
    if (n <= 0) {
        set_error("cannot build a Cartesian tree over an empty array");
        return SAIX_EINVAL;
    }
    if (!values || !parent || !left || !right || !tour_nodes || !tour_depths || !first_visit || !root_host ||
        (value_bytes != 4 && value_bytes != 8) || n >= ((i64)1 << 30)) {
        set_error("saix_cartesian_build: invalid arguments");
        return SAIX_EINVAL;
    }
    if (ws_bytes < saix_cartesian_workspace_bytes(n)) {
        set_error("saix_cartesian_build: workspace too small");
        return SAIX_ENOSPC;
    }
    cudaStream_t st = (cudaStream_t)stream;
    if (value_bytes == 4)
        return cartesian_run<u32>((const u32 *)values, n, parent, left, right, tour_nodes, tour_depths, first_visit,
                                  root_host, ws, ws_bytes, st);
    return cartesian_run<i64>((const i64 *)values, n, parent, left, right, tour_nodes, tour_depths, first_visit,
                              root_host, ws, ws_bytes, st);
}

// PlusMinusOneRmq.__init__ (rmq.py:167-197) minus the block sparse table
// (built by the caller with saix_sparse_build over bmin): block size b,
// nblocks = ceil(m / b); per block leftmost argmin / min / code; the present
// codes' in-block tables (tab: (2^(b-1)) x b x b bytes); *bad_host = 1 if
// some adjacent depths differ by other than 1.
extern "C" int saix_pm1_build(const int32_t *depths, int64_t m, int b, int32_t *bargmin, int32_t *bmin,
                              int32_t *types, uint8_t *present, uint8_t *tab, int32_t *bad_host, void *stream) {
    if (!depths || m <= 0 || b < 1 || b > 16 || !bargmin || !bmin || !types || !present || !tab || !bad_host) {
        set_error("saix_pm1_build: invalid arguments");
        return SAIX_EINVAL;
    }
    cudaStream_t st = (cudaStream_t)stream;
    const i64 nblocks = ceil_div(m, b);
    const u32 ncodes = 1u << (b - 1);
    int *bad = reinterpret_cast<int *>(present + ((ncodes + 3) & ~3u));  // caller sized present + 4 bytes
    SAIX_CUDA(cudaMemsetAsync(present, 0, (size_t)((ncodes + 3) & ~3u) + 4, st));
    {
        Prof prof_("pm1.blocks", (double)m * 4 + nblocks * 12.0, st);
        k_pm1_blocks<<<grid_for(nblocks, 256), 256, 0, st>>>(depths, m, b, nblocks, bargmin, bmin, types, present,
                                                             bad);
        SAIX_LAUNCHED();
        k_pm1_tables<<<grid_for((i64)ncodes * b, 256), 256, 0, st>>>(b, ncodes, present, tab);
        SAIX_LAUNCHED();
    }
    SAIX_CUDA(cudaMemcpyAsync(bad_host, bad, 4, cudaMemcpyDeviceToHost, st));
    SAIX_CUDA(cudaStreamSynchronize(st));
    return SAIX_OK;
}

extern "C" int saix_pm1_query_begin(int b, const int32_t *types, const uint8_t *tab, const int32_t *first,
                                    const int64_t *qi, const int64_t *qj, int64_t q, int64_t *mid_lo,
                                    int64_t *mid_hi, int32_t *cand, void *stream) {
    if (b < 1 || !types || !tab || q < 0 || (q > 0 && (!qi || !qj || !mid_lo || !mid_hi || !cand))) {
        set_error("saix_pm1_query_begin: invalid arguments");
        return SAIX_EINVAL;
    }
    if (q == 0) return SAIX_OK;
    cudaStream_t st = (cudaStream_t)stream;
    k_pm1_query_a<<<grid_for(q, 256), 256, 0, st>>>(b, types, tab, first, qi, qj, q, mid_lo, mid_hi, cand);
    SAIX_LAUNCHED();
    return SAIX_OK;
}

extern "C" int saix_pm1_query_end(const int32_t *depths, int b, const int32_t *bargmin, const int64_t *mid_blk,
                                  const int32_t *cand, const int32_t *nodes, int64_t q, int64_t *out, void *stream) {
    if (!depths || b < 1 || !bargmin || q < 0 || (q > 0 && (!mid_blk || !cand || !out))) {
        set_error("saix_pm1_query_end: invalid arguments");
        return SAIX_EINVAL;
    }
    if (q == 0) return SAIX_OK;
    cudaStream_t st = (cudaStream_t)stream;
    k_pm1_query_b<<<grid_for(q, 256), 256, 0, st>>>(depths, b, bargmin, mid_blk, cand, nodes, q, out);
    SAIX_LAUNCHED();
    return SAIX_OK;
}
