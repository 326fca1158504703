// store.cu -- ".saix" index files (index_store.py:1-134) packed and checked on
// the device.
//
// CRC-32 (zlib's polynomial and conventions -- the reference's zlib.crc32) as
// one streaming pass: a persistent grid, each CTA walking a contiguous range
// of 16 KB blocks (512 threads x 32 bytes).  A block is staged in shared
// memory (padded so every thread's 32-byte segment is read conflict-free), each thread runs the
// byte-table CRC over its segment (the 256-entry table is replicated once per
// bank, so all 32 lanes look up in one wavefront) and folds it into a
// per-thread accumulator with acc = acc * x^(8*16K) + raw (a constant GF(2)
// multiply done with four byte tables).  At the end of its range each thread
// shifts its accumulator to the block end (x^(8*32*(511-t))), the CTA XORs
// them, shifts the result to the end of the message and XORs it into the
// answer with one atomic; CTA 0 adds zlib's init term
// (0xFFFFFFFF * x^(8L) + 0xFFFFFFFF).  CRC is linear, so the order in which
// CTAs arrive does not matter.  The message's partial last block is staged
// right-aligned behind zeros (leading zeros leave a raw CRC unchanged).
//
// save: the block producer IS the file packer -- each thread builds its
// 16-byte output chunks straight from the device text / SA / LCP (u32 ->
// little-endian u64), stores them to the file image and into the CRC stage,
// so the image is written once and never re-read (26n bytes of traffic).
// load: the CRC pass over the image, then one decode pass (u64 -> u32, text
// bytes) and the ISA by the bucketed scatter for large n.
#include "pscatter.cuh"

namespace saix {

constexpr u32 kCrcPoly = 0xEDB88320u;  // reflected 0x04C11DB7
constexpr int SC_THREADS = 512;
constexpr int SC_SEG = 32;                            // bytes per thread per block
constexpr int SC_BLOCK = SC_THREADS * SC_SEG;         // 16 KB
constexpr int SC_PSEG = SC_SEG + 16;                  // padded smem stride per segment
constexpr int SC_STAGE = SC_THREADS * SC_PSEG;        // 20 KB
constexpr int SC_TAB_WORDS = 256 * 32;                // byte table x 32 bank copies
constexpr size_t SC_SMEM = (size_t)SC_TAB_WORDS * 4 + 1024 * 4 + SC_STAGE + 64 * 4 + 32 * 4;
constexpr i64 kHeader = 8 + 4 * 8;                    // magic, version, flags, n, sigma

__host__ __device__ __forceinline__ u32 crc_table_entry(u32 b) {
    u32 c = b;
#pragma unroll
    for (int k = 0; k < 8; k++) c = (c & 1) ? (c >> 1) ^ kCrcPoly : c >> 1;
    return c;
}

// a * b mod P in zlib's reflected representation (bit 31 = x^0)
__host__ __device__ __forceinline__ u32 multmodp(u32 a, u32 b) {
    u32 p = 0;
    for (u32 m = 1u << 31; m; m >>= 1) {
        if (a & m) {
            p ^= b;
            if ((a & (m - 1)) == 0) break;
        }
        b = (b & 1) ? (b >> 1) ^ kCrcPoly : b >> 1;
    }
    return p;
}
// x^(8 * len) mod P, x2n[k] = x^(2^k) mod P
__host__ __device__ __forceinline__ u32 x8nmodp(u64 len, const u32 *x2n) {
    u32 p = 1u << 31;
    int k = 3;
    while (len) {
        if (len & 1) p = multmodp(x2n[k & 63], p);
        len >>= 1;
        k++;
    }
    return p;
}

struct CrcConsts {
    u32 x2n[64];
    u32 seg_shift[SC_THREADS];  // x^(8 * SEG * (T-1-t)): segment end -> block end
    u32 blk;                    // x^(8 * SC_BLOCK)
    u32 init;                   // zlib's init / final-xor term for this length
};

static CrcConsts crc_consts(i64 L) {
    CrcConsts c;
    u32 p = 1u << 30;  // x^1
    for (int k = 0; k < 64; k++) {
        c.x2n[k] = p;
        p = multmodp(p, p);
    }
    for (int t = 0; t < SC_THREADS; t++) c.seg_shift[t] = x8nmodp((u64)SC_SEG * (SC_THREADS - 1 - t), c.x2n);
    c.blk = x8nmodp(SC_BLOCK, c.x2n);
    c.init = multmodp(x8nmodp((u64)L, c.x2n), 0xFFFFFFFFu) ^ 0xFFFFFFFFu;
    return c;
}

// tab: this lane's column (32-bit shared address) of the bank-replicated
// table; entry i sits 128 * i bytes further
__device__ __forceinline__ u32 crc_word(u32 c, u32 w, u32 tab) {
    c ^= w;
#pragma unroll
    for (int b = 0; b < 4; b++) {
        u32 t;
        asm volatile("ld.shared.u32 %0, [%1];" : "=r"(t) : "r"(tab + (__byte_perm(c, 0, 0x4440) << 7)));
        c = t ^ (c >> 8);
    }
    return c;
}

// Src: __device__ uint4 chunk(i64 o) (o % 16 == 0, [o, o+16) inside the
// message) and __device__ u8 byte(i64 o); both may also emit what they read.
template <class Src>
__global__ void __launch_bounds__(SC_THREADS, 3)
k_crc_stream(Src src, i64 L, i64 per_cta, const __grid_constant__ CrcConsts C, u32 *__restrict__ crc_out) {
    extern __shared__ __align__(16) unsigned char sc_smem[];
    u32 *tab = reinterpret_cast<u32 *>(sc_smem);
    u32 *mul = tab + SC_TAB_WORDS;
    unsigned char *stage = reinterpret_cast<unsigned char *>(mul + 1024);
    u32 *x2n = reinterpret_cast<u32 *>(stage + SC_STAGE);
    u32 *red = x2n + 64;
    const int t = threadIdx.x, lane = t & 31;
    {
        const int e = t & 255, half = t >> 8;  // two threads per entry, 16 copies each
        const u32 v = crc_table_entry((u32)e);
#pragma unroll 8
        for (int l = 0; l < 16; l++) tab[e * 32 + ((l + 16 * half + lane) & 31)] = v;
#pragma unroll
        for (int k = 0; k < 2; k++) mul[(2 * half + k) * 256 + e] = multmodp((u32)e << (8 * (2 * half + k)), C.blk);
        if (t < 64) x2n[t] = C.x2n[t];
    }
    __syncthreads();
    const u32 mytab = (u32)__cvta_generic_to_shared(tab + lane);
    const i64 J = ceil_div(L, SC_BLOCK);
    const i64 jb0 = (i64)blockIdx.x * per_cta;
    const i64 jb1 = jb0 + per_cta < J ? jb0 + per_cta : J;
    u32 acc = 0;
    // chunks of the next full block are fetched before the current block's
    // CRC runs, so loads stay in flight through the compute phase
    constexpr int NCH = SC_SEG / 16;
    uint4 nxt[NCH];
    auto fetch = [&](i64 jb) {
        if (jb < jb1 && (jb + 1) * SC_BLOCK <= L) {
#pragma unroll
            for (int k = 0; k < NCH; k++) nxt[k] = src.chunk(jb * SC_BLOCK + 16 * t + (SC_THREADS * 16) * k);
        }
    };
    fetch(jb0);
    for (i64 jb = jb0; jb < jb1; jb++) {
        const i64 b0 = jb * SC_BLOCK;
        const i64 r = L - b0 < SC_BLOCK ? L - b0 : SC_BLOCK;
        if (r == SC_BLOCK) {
#pragma unroll
            for (int k = 0; k < NCH; k++) {
                const int pos = 16 * t + (SC_THREADS * 16) * k;
                *reinterpret_cast<uint4 *>(stage + pos + (pos >> 5) * 16) = nxt[k];
            }
        } else {
            const i64 D = SC_BLOCK - r;  // right-aligned behind D zeros
            for (int vp = t; vp < SC_BLOCK; vp += SC_THREADS) {
                const i64 p = vp - D;
                stage[vp + (vp >> 5) * 16] = p >= 0 ? src.byte(b0 + p) : (u8)0;
            }
        }
        __syncthreads();
        fetch(jb + 1);
        const uint4 *sp = reinterpret_cast<const uint4 *>(stage + t * SC_PSEG);
        u32 raw = 0;
#pragma unroll
        for (int q = 0; q < SC_SEG / 16; q++) {
            uint4 v = sp[q];
            raw = crc_word(raw, v.x, mytab);
            raw = crc_word(raw, v.y, mytab);
            raw = crc_word(raw, v.z, mytab);
            raw = crc_word(raw, v.w, mytab);
        }
        if (r == SC_BLOCK)
            acc = mul[acc & 0xFFu] ^ mul[256 + ((acc >> 8) & 0xFFu)] ^ mul[512 + ((acc >> 16) & 0xFFu)] ^
                  mul[768 + (acc >> 24)] ^ raw;
        else
            acc = multmodp(x8nmodp((u64)r, x2n), acc) ^ raw;
        __syncthreads();
    }
    if (jb0 >= jb1) return;
    u32 v = multmodp(C.seg_shift[t], acc);
#pragma unroll
    for (int o = 16; o; o >>= 1) v ^= __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) red[t >> 5] = v;
    __syncthreads();
    if (t == 0) {
        u32 tot = 0;
        for (int w = 0; w < SC_THREADS / 32; w++) tot ^= red[w];
        const i64 end = jb1 * SC_BLOCK < L ? jb1 * SC_BLOCK : L;
        tot = multmodp(x8nmodp((u64)(L - end), x2n), tot);
        if (blockIdx.x == 0) tot ^= C.init;
        atomicXor(crc_out, tot);
    }
}

struct BufSrc {
    const u8 *p;
    bool aligned;
    __device__ __forceinline__ uint4 chunk(i64 o) const {
        if (aligned) return __ldcs(reinterpret_cast<const uint4 *>(p + o));
        u32 w[4];
#pragma unroll
        for (int k = 0; k < 4; k++)
            w[k] = (u32)p[o + 4 * k] | (u32)p[o + 4 * k + 1] << 8 | (u32)p[o + 4 * k + 2] << 16 |
                   (u32)p[o + 4 * k + 3] << 24;
        return make_uint4(w[0], w[1], w[2], w[3]);
    }
    __device__ __forceinline__ u8 byte(i64 o) const { return p[o]; }
};

struct Header {
    u64 w[5];
};

// The file image, produced chunk by chunk from the device arrays and stored
// to `out` as it is produced.
struct PackSrc {
    const u8 *text;
    const u32 *sa, *lcp;
    i64 n;
    u8 *out;
    bool text_aligned;
    Header hdr;

    __device__ __forceinline__ u8 byte_at(i64 p) const {
        if (p < kHeader) {
            u64 w = hdr.w[0];
#pragma unroll
            for (int k = 1; k < 5; k++) w = (p >> 3) == k ? hdr.w[k] : w;  // no local-memory indexing
            return (u8)(w >> (8 * (p & 7)));
        }
        p -= kHeader;
        if (p < n) return text[p];
        p -= n;
        const u32 *a = sa;
        if (p >= 8 * n) {
            p -= 8 * n;
            a = lcp;
        }
        return (p & 7) < 4 ? (u8)(a[p >> 3] >> (8 * (p & 7))) : (u8)0;
    }
    // bytes [q, q+16) of the little-endian u64 image of a (zero-extended u32)
    static __device__ __forceinline__ uint4 entries(const u32 *a, i64 q) {
        const i64 e = q >> 3;
        const int s = (int)(q & 7);
        u64 w0 = a[e], w1 = a[e + 1], lo, hi;
        if (s == 0) {
            lo = w0;
            hi = w1;
        } else {
            u64 w2 = a[e + 2];
            lo = (w0 >> (8 * s)) | (w1 << (64 - 8 * s));
            hi = (w1 >> (8 * s)) | (w2 << (64 - 8 * s));
        }
        return make_uint4((u32)lo, (u32)(lo >> 32), (u32)hi, (u32)(hi >> 32));
    }
    __device__ __forceinline__ uint4 chunk(i64 o) const {
        const i64 ts = kHeader, ss = ts + n, ls = ss + 8 * n, le = ls + 8 * n;
        uint4 r;
        if (o >= ts && o + 16 <= ss && text_aligned) {
            // o % 16 == 0 and kHeader % 16 == 8: the text slice is 8-byte aligned
            const uint2 *q = reinterpret_cast<const uint2 *>(text + (o - ts));
            uint2 a = q[0], b = q[1];
            r = make_uint4(a.x, a.y, b.x, b.y);
        } else if (o >= ss && o + 16 <= ls) {
            r = entries(sa, o - ss);
        } else if (o >= ls && o + 16 <= le) {
            r = entries(lcp, o - ls);
        } else {
            u32 w[4];
#pragma unroll
            for (int k = 0; k < 4; k++)
                w[k] = (u32)byte_at(o + 4 * k) | (u32)byte_at(o + 4 * k + 1) << 8 |
                       (u32)byte_at(o + 4 * k + 2) << 16 | (u32)byte_at(o + 4 * k + 3) << 24;
            r = make_uint4(w[0], w[1], w[2], w[3]);
        }
        __stcs(reinterpret_cast<uint4 *>(out + o), r);
        return r;
    }
    __device__ __forceinline__ u8 byte(i64 o) const {
        u8 b = byte_at(o);
        out[o] = b;
        return b;
    }
};

template <class Src>
static int crc_stream(const Src &src, i64 L, u32 *crc, cudaStream_t st, const char *prof, double bytes) {
    SAIX_CUDA(cudaMemsetAsync(crc, 0, 4, st));
    if (L <= 0) return SAIX_OK;  // zlib.crc32(b"") == 0
    static DeviceFlags attr;
    static std::atomic<int> per_sm_cached{1};
    if (attr.need()) {
        int per_sm = 0;
        SAIX_CUDA(cudaFuncSetAttribute(k_crc_stream<Src>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SC_SMEM));
        SAIX_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_crc_stream<Src>, SC_THREADS, SC_SMEM));
        per_sm_cached.store(per_sm < 1 ? 1 : per_sm);  // same on every B200
        attr.set();
    }
    const int per_sm = per_sm_cached.load();
    const i64 J = ceil_div(L, SC_BLOCK);
    i64 grid = (i64)kNumSMs * per_sm;
    if (grid > J) grid = J;
    const i64 per = ceil_div(J, grid);
    grid = ceil_div(J, per);
    CrcConsts C = crc_consts(L);
    Prof prof_(prof, bytes, st);
    k_crc_stream<Src><<<(unsigned)grid, SC_THREADS, SC_SMEM, st>>>(src, L, per, C, crc);
    SAIX_LAUNCHED();
    return SAIX_OK;
}

__global__ void k_put_crc(const u32 *__restrict__ crc, u8 *__restrict__ at) {
    if (threadIdx.x < 8) at[threadIdx.x] = threadIdx.x < 4 ? (u8)(*crc >> (8 * threadIdx.x)) : (u8)0;
}

// u64 little-endian entry k of a section starting at byte `base` of blob
__device__ __forceinline__ u64 load_entry(const u8 *__restrict__ blob, i64 base, i64 k) {
    const i64 at = base + 8 * k;
    const int s = (int)(at & 7);
    const u64 *a = reinterpret_cast<const u64 *>(blob + (at - s));
    if (s == 0) return __ldcs(a);
    return (__ldcs(a) >> (8 * s)) | (__ldcs(a + 1) << (64 - 8 * s));
}

__global__ void k_unpack_index(const u8 *__restrict__ blob, i64 n, u8 *__restrict__ text, u32 *__restrict__ sa,
                               u32 *__restrict__ lcp, u32 *__restrict__ bad) {
    const i64 ss = kHeader + n, ls = ss + 8 * n;
    u32 nbad = 0;
    for (i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x) {
        u64 a = load_entry(blob, ss, i), b = load_entry(blob, ls, i);
        text[i] = blob[kHeader + i];
        const bool oob = a >= (u64)n;  // never scatter out of range (a crafted file)
        // sa >= n: the reference's rank[sa] = arange(n) raises IndexError.  Any
        // lcp value loads there; the device keeps u32 LCPs, so only values
        // >= 2^32 (impossible for n < 2^32, i.e. a crafted file) are refused.
        nbad |= (oob ? 1u : 0u) | ((b >> 32) ? 2u : 0u);
        sa[i] = oob ? 0u : (u32)a;
        lcp[i] = (u32)b;
    }
    nbad = __reduce_or_sync(0xffffffffu, nbad);
    if (nbad && lane_id() == 0) atomicOr(bad, nbad);
}

}  // namespace saix

using namespace saix;

extern "C" size_t saix_crc32_workspace_bytes(int64_t) { return 256; }

extern "C" int saix_crc32(const void *data, int64_t nbytes, uint32_t *crc_out, void *ws, size_t ws_bytes,
                          void *stream) {
    (void)ws;
    if (nbytes < 0 || !crc_out || (nbytes > 0 && !data) || ws_bytes < saix_crc32_workspace_bytes(nbytes)) {
        set_error("saix_crc32: invalid arguments");
        return SAIX_EINVAL;
    }
    BufSrc src{(const u8 *)data, ((uintptr_t)data & 15) == 0};
    return crc_stream(src, nbytes, crc_out, (cudaStream_t)stream, "store.crc32", (double)nbytes);
}

extern "C" int64_t saix_index_bytes(int64_t n) { return kHeader + 17 * n + 8; }

extern "C" int saix_index_pack(const uint8_t *text, const uint32_t *sa, const uint32_t *lcp, int64_t n,
                               int64_t sigma, int64_t flags, uint8_t *out, void *ws, size_t ws_bytes, void *stream) {
    if (n < 0 || !out || !ws || (n > 0 && (!text || !sa || !lcp)) || sigma < 0 || sigma > 255) {
        set_error("saix_index_pack: invalid arguments");
        return SAIX_EINVAL;
    }
    if (((uintptr_t)out & 15) != 0) {
        set_error("saix_index_pack: out must be 16-byte aligned");
        return SAIX_EINVAL;
    }
    if (ws_bytes < saix_crc32_workspace_bytes(0)) {
        set_error("saix_index_pack: workspace too small");
        return SAIX_ENOSPC;
    }
    cudaStream_t st = (cudaStream_t)stream;
    PackSrc src;
    src.text = text;
    src.sa = sa;
    src.lcp = lcp;
    src.n = n;
    src.out = out;
    src.text_aligned = ((uintptr_t)text & 7) == 0;
    const char magic[8] = {'S', 'A', 'I', 'X', '1', 0, 0, 0};
    memcpy(&src.hdr.w[0], magic, 8);
    src.hdr.w[1] = 1;  // version
    src.hdr.w[2] = (u64)flags;
    src.hdr.w[3] = (u64)n;
    src.hdr.w[4] = (u64)sigma;
    const i64 payload = kHeader + 17 * n;
    u32 *crc = (u32 *)ws;
    SAIX_TRY(crc_stream(src, payload, crc, st, "store.pack_crc", 9.0 * n + 17.0 * n));
    k_put_crc<<<1, 32, 0, st>>>(crc, out + payload);
    SAIX_LAUNCHED();
    return SAIX_OK;
}

extern "C" size_t saix_index_unpack_workspace_bytes(int64_t n) {
    return 256 + (n >= kDirectScatterItems ? scatter_u32_bytes(n) : 0) + Arena::kAlign;
}

// Verifies the CRC of a device file image whose header (magic, version,
// length) the caller has checked; unpacks text, SA, LCP (u32) and the ISA.
extern "C" int saix_index_unpack(const uint8_t *blob, int64_t n, uint8_t *text, uint32_t *sa, uint32_t *lcp,
                                 uint32_t *isa, void *ws, size_t ws_bytes, void *stream) {
    if (n < 0 || !blob || !ws || (n > 0 && (!text || !sa || !lcp || !isa))) {
        set_error("saix_index_unpack: invalid arguments");
        return SAIX_EINVAL;
    }
    if (n >= ((i64)1 << 32) - 4) {
        set_error("saix_index_unpack: n=%lld too large", (long long)n);
        return SAIX_EINVAL;
    }
    if (ws_bytes < saix_index_unpack_workspace_bytes(n)) {
        set_error("saix_index_unpack: workspace too small");
        return SAIX_ENOSPC;
    }
    cudaStream_t st = (cudaStream_t)stream;
    Arena ar{(char *)ws, ws_bytes};
    u32 *flags = ar.alloc<u32>(4);  // crc, bad
    SAIX_ARENA_OK(ar);
    const i64 payload = kHeader + 17 * n;
    SAIX_CUDA(cudaMemsetAsync(flags, 0, 16, st));
    BufSrc src{blob, ((uintptr_t)blob & 15) == 0};
    SAIX_TRY(crc_stream(src, payload, flags, st, "store.crc32", (double)payload));
    if (n > 0) {
        {
            Prof prof_("store.unpack", 17.0 * n + 9.0 * n, st);
            k_unpack_index<<<grid_for(n, 256), 256, 0, st>>>(blob, n, text, sa, lcp, flags + 1);
            SAIX_LAUNCHED();
        }
        SAIX_TRY(scatter_u32(ar, sa, nullptr, n, n, isa, st, "store.isa"));
    }
    u32 host[2];
    u8 stored[8];
    SAIX_CUDA(cudaMemcpyAsync(host, flags, 8, cudaMemcpyDeviceToHost, st));
    SAIX_CUDA(cudaMemcpyAsync(stored, blob + payload, 8, cudaMemcpyDeviceToHost, st));
    SAIX_CUDA(cudaStreamSynchronize(st));
    u64 want = 0;
    for (int k = 0; k < 8; k++) want |= (u64)stored[k] << (8 * k);
    if ((u64)host[0] != want) {
        set_error("checksum mismatch; file is corrupt");
        return SAIX_EINVAL;
    }
    if (host[1] & 1u) {
        set_error("index entries out of range");
        return SAIX_EINVAL;
    }
    if (host[1] & 2u) {
        set_error("lcp entries beyond 2^32-1 do not fit the device's u32 LCP layout");
        return SAIX_EINVAL;
    }
    return SAIX_OK;
}
