// common.cuh -- error plumbing, workspace carving and small device helpers
// shared by every kernel file of libsaix_b200.so (sm_100a only).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <cstdio>
#include <string>

#include "../../include/saix_b200.h"

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ < 1000)
#error "libsaix_b200 targets sm_100a (B200) only"
#endif

namespace saix {

using u8 = uint8_t;
using u16 = uint16_t;
using u32 = uint32_t;
using u64 = uint64_t;
using i64 = int64_t;

constexpr int kNumSMs = 148;  // B200: 2 dies x 74 SMs

// Below this many items a permutation's random 4-12 B writes stay in L2 and
// beat the three streaming passes of the bucketed scatter (pscatter.cuh).
constexpr i64 kDirectScatterItems = (i64)1 << 23;

// ---------------------------------------------------------------- errors

void set_error(const char *fmt, ...);

#define SAIX_CUDA(call)                                                        \
    do {                                                                       \
        cudaError_t e_ = (call);                                               \
        if (e_ != cudaSuccess) {                                               \
            ::saix::set_error("%s:%d %s: %s", __FILE__, __LINE__, #call,       \
                              cudaGetErrorString(e_));                         \
            return SAIX_ECUDA;                                                 \
        }                                                                      \
    } while (0)

#define SAIX_LAUNCHED()                                                        \
    do {                                                                       \
        cudaError_t e_ = cudaGetLastError();                                   \
        if (e_ != cudaSuccess) {                                               \
            ::saix::set_error("%s:%d kernel launch: %s", __FILE__, __LINE__,   \
                              cudaGetErrorString(e_));                         \
            return SAIX_ECUDA;                                                 \
        }                                                                      \
    } while (0)

#define SAIX_TRY(expr)                                                         \
    do {                                                                       \
        int rc_ = (expr);                                                      \
        if (rc_ != SAIX_OK) return rc_;                                        \
    } while (0)

// Per-device "done" bits for one-time kernel attributes
// (cudaFuncSetAttribute applies per device context): need() is true until
// set() ran on the current device.  Two host threads may both run the
// (idempotent) attribute call; the bits themselves are atomic.
struct DeviceFlags {
    std::atomic<unsigned long long> bits{0};
    static unsigned long long bit() {
        int d = 0;
        if (cudaGetDevice(&d) != cudaSuccess) d = 0;
        return 1ull << (d & 63);
    }
    bool need() const { return (bits.load(std::memory_order_acquire) & bit()) == 0; }
    void set() { bits.fetch_or(bit(), std::memory_order_release); }
};

// ------------------------------------------------------------- profiling

// Optional per-kernel CUDA-event timing (saix_prof_enable): each Prof scope
// brackets one launch on its stream and carries the launch's algorithmic
// bytes so bench.py can report achieved GB/s.
bool prof_on();
void prof_mark(const char *name, double bytes, cudaStream_t st, bool begin);

struct Prof {
    bool on;
    const char *name;
    double bytes;
    cudaStream_t st;
    Prof(const char *n, double b, cudaStream_t s) : on(prof_on()), name(n), bytes(b), st(s) {
        if (on) prof_mark(name, bytes, st, true);
    }
    ~Prof() {
        if (on) prof_mark(name, bytes, st, false);
    }
};

// ------------------------------------------------------------- workspace

// Bump allocator over the caller's workspace.  With base == nullptr it only
// measures (used by the *_workspace_bytes planners).
struct Arena {
    char *base = nullptr;
    size_t cap = 0;
    size_t off = 0;
    size_t peak = 0;
    bool overflow = false;

    static constexpr size_t kAlign = 256;

    template <typename T>
    T *alloc(i64 count) {
        size_t bytes = (size_t)(count > 0 ? count : 1) * sizeof(T);
        off = (off + kAlign - 1) & ~(kAlign - 1);
        size_t at = off;
        off += bytes;
        if (off > peak) peak = off;
        if (base == nullptr) return nullptr;
        if (off > cap) {
            overflow = true;
            return nullptr;
        }
        return reinterpret_cast<T *>(base + at);
    }
    size_t mark() const { return off; }
    void reset(size_t m) { off = m; }
};

#define SAIX_ARENA_OK(arena)                                                   \
    do {                                                                       \
        if ((arena).overflow) {                                                \
            ::saix::set_error("workspace too small (%zu bytes needed)",        \
                              (arena).peak);                                   \
            return SAIX_ENOSPC;                                                \
        }                                                                      \
    } while (0)

// --------------------------------------------------------------- helpers

__host__ __device__ inline i64 ceil_div(i64 a, i64 b) { return (a + b - 1) / b; }

inline int grid_for(i64 n, int threads, int max_blocks = kNumSMs * 32) {
    i64 b = ceil_div(n > 0 ? n : 1, threads);
    return (int)(b < max_blocks ? b : max_blocks);
}

__device__ __forceinline__ u32 lanemask_lt() {
    u32 m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }

// ------------------------------------------- bulk copies (TMA) + mbarriers
// One-dimensional cp.async.bulk global -> shared completing on an mbarrier
// (sm_90+ async proxy; on sm_100a the copy engine behind UBLKCP).  src/dst
// 16-byte aligned, bytes a multiple of 16.
__device__ __forceinline__ u32 smem_u32(const void *p) { return (u32)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(u64 *bar, u32 count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
// make the barrier init (and prior generic-proxy smem writes) visible to the async proxy
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void mbar_expect_tx(u64 *bar, u32 bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, u32 bytes, u64 *bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void mbar_wait(u64 *bar, u32 parity) {
    asm volatile(
        "{\n .reg .pred p;\n"
        "WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

// Peer mask of lanes holding the same 8-bit digit: eight ballots + ANDs
// (cheaper than __match_any_sync on sm_100).  Lanes with d == OS_RADIX (no
// item) differ from every valid digit in bit 8 via the `valid` ballot.
__device__ __forceinline__ u32 digit_peers(u32 d) {
    u32 peers = __ballot_sync(0xffffffffu, d < 256u);
    if (d >= 256u) peers = ~peers;
#pragma unroll
    for (int b = 0; b < 8; b++) {
        u32 m = __ballot_sync(0xffffffffu, (d >> b) & 1u);
        peers &= ((d >> b) & 1u) ? m : ~m;
    }
    return peers;
}

// u32 division by a runtime-constant divisor d >= 1 (Granlund-Montgomery,
// exact for every 32-bit dividend): q = (t + ((x - t) >> 1)) >> (l - 1),
// t = umulhi(m, x), l = ceil(log2 d), m = floor(2^32 (2^l - d) / d) + 1.
struct U32Div {
    u32 m = 0, d = 1;
    int l = 0;
    static U32Div of(u32 d) {
        U32Div r;
        r.d = d;
        int l = 0;
        while (((u64)1 << l) < d) l++;
        r.l = l;
        r.m = (u32)((((u64)1 << 32) * (((u64)1 << l) - d)) / d + 1);
        return r;
    }
    __device__ __forceinline__ u32 div(u32 x) const {
        if (l == 0) return x;
        u32 t = __umulhi(m, x);
        return (t + ((x - t) >> 1)) >> (l - 1);
    }
};

// digit_peers for digits in [0, mask] (mask = 2^w - 1), 256 = no item:
// w + 1 ballots instead of 9
__device__ __forceinline__ u32 digit_peers_w(u32 d, u32 mask) {
    u32 peers = __ballot_sync(0xffffffffu, d < 256u);
    if (d >= 256u) peers = ~peers;
    for (u32 b = 0; (1u << b) <= mask; b++) {
        u32 m = __ballot_sync(0xffffffffu, (d >> b) & 1u);
        peers &= ((d >> b) & 1u) ? m : ~m;
    }
    return peers;
}

inline int bits_for(u64 v) {  // bit width of v (>= 1), like int.bit_length()
    int b = 1;
    while (b < 64 && (v >> b)) b++;
    return b;
}

// LCP (lcp.cu) with the pipeline option of folding longest_overlap's pass 1
// (max LCP over cross-sequence adjacent pairs, separator at `boundary`) into
// the final permute kernel; boundary < 0 disables it.
// phi_in (nullable): caller storage for Phi/PLCP; phi_ready says it already
// holds Phi (Phi[sa[r]] = sa[r-1]).
// sigma / sep (alphabet bound, unique separator position; -1 = unknown /
// none) select the direct word-compare LCP when the text allows it.
int lcp_compute(const void *text, int text_bytes, i64 n, const u32 *sa, u32 *lcp, void *ws, size_t ws_bytes,
                cudaStream_t st, i64 boundary, u32 *best, u32 *phi_in = nullptr, bool phi_ready = false,
                i64 sigma = -1, i64 sep = -1);

// PLCP (in place over Phi) for u8 text -- the batched-pairs path.
size_t plcp_workspace_bytes(i64 n);
int plcp_from_phi(const u8 *text, i64 n, u32 *phi_plcp, void *ws, size_t ws_bytes, cudaStream_t st);

// DC3 (dc3.cu); isa may be null when the caller does not need the ranks.
// phi (nullable): when the top level runs the streaming path without an ISA
// request, Phi[sa[r]] = sa[r-1] (0xFFFFFFFF at r = 0) is produced by the
// merge and *phi_done is set.
int dc3_compute(const void *text, int text_bytes, i64 n, i64 sigma, u32 *sa, u32 *isa, void *ws,
                size_t ws_bytes, saix_dc3_probe *probe, cudaStream_t stream, u32 *phi = nullptr,
                bool *phi_done = nullptr);
// Per-thread override of the level-0 window naming (-1: the global setting);
// returns the previous override.  The batched-pairs path turns it off: its
// planted pair overlaps leave long tied runs that the recursion handles better.
int dc3_window_naming_override(int v);

// L2 eviction-priority hints (sm_80+ createpolicy / L2::cache_hint): random
// gather targets that should stay on chip are loaded / stored evict_last,
// while streaming arrays use the .cs (evict-first) variants.
__device__ __forceinline__ u64 l2_evict_last() {
    u64 p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint4 ldg_last(const uint4 *a, u64 pol) {
    uint4 r;
    asm volatile("ld.global.nc.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(a), "l"(pol));
    return r;
}
__device__ __forceinline__ u32 ldg_last(const u32 *a, u64 pol) {
    u32 r;
    asm volatile("ld.global.nc.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(r) : "l"(a), "l"(pol));
    return r;
}
__device__ __forceinline__ u32 ld_last(const u32 *a, u64 pol) {  // coherent (buffer written earlier)
    u32 r;
    asm volatile("ld.global.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(r) : "l"(a), "l"(pol));
    return r;
}
__device__ __forceinline__ void st_last(u32 *a, u32 v, u64 pol) {
    asm volatile("st.global.L2::cache_hint.u32 [%0], %1, %2;" ::"l"(a), "r"(v), "l"(pol) : "memory");
}

// DC3 sample layout (suffix_index.py:149-153): mod-1 positions 1,4,... and
// mod-2 positions 2,5,... below limit = n+1 if n%3==1 else n.
struct SampleLayout {
    i64 n, m1, m2, m, k;  // k = number of mod-0 positions = ceil(n/3)
    bool pad;             // padding sample n present (n % 3 == 1)
    __host__ __device__ static SampleLayout of(i64 n) {
        SampleLayout s;
        s.n = n;
        i64 limit = (n % 3 == 1) ? n + 1 : n;
        s.m1 = limit > 1 ? (limit + 1) / 3 : 0;
        s.m2 = limit > 2 ? limit / 3 : 0;
        s.m = s.m1 + s.m2;
        s.k = (n + 2) / 3;
        s.pad = (n % 3 == 1);
        return s;
    }
    __host__ __device__ i64 pos(i64 s) const { return s < m1 ? 3 * s + 1 : 3 * (s - m1) + 2; }
};

}  // namespace saix
