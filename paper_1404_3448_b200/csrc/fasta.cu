// fasta.cu -- FASTA ingest on the device (sequence.py:77-125 parse_fasta,
// 144-157 encode): line splitting, whitespace stripping, header / sequence
// classification, residue upper-casing + validation, record concatenation,
// and (optionally) the rank encoding, over the raw file bytes in HBM.
//
// Semantics are the reference's for a `str` source (io.StringIO: lines end
// at '\n' only): every line is str.strip()-ed (Python's ASCII whitespace:
// \t \n \v \f \r \x1c-\x1f and space); blank lines are skipped; a line
// starting with '>' opens a record whose header is the rest of the line,
// stripped again (empty -> "empty FASTA header"); any other line before the
// first header is "sequence data before any '>' header"; sequence lines are
// upper-cased and every byte must be in the policy's alphabet.  The first
// error in file order wins, as in the reference's sequential loop: every
// error is keyed by its byte position and reduced with atomicMin.
//
// Passes (B input bytes, L lines):
//   1. newline count per 16 KB tile (SWAR byte compare), tile scan, then the
//      '\n' positions emitted in order                            ~2B reads
//   2. thread per line: strip, classify; three line scans give each
//      sequence line its output offset, each header its record index and
//      header-text offset                                           ~40L bytes
//   3. warp per line: copy + upper + validate (+ encode) residues; headers
//      copied to a compact text buffer; record starts written        ~2B
// The workspace carries the line tables from saix_fasta_scan to
// saix_fasta_emit.
#include "scan.cuh"

namespace saix {

constexpr int FA_THREADS = 256;
constexpr int FA_BYTES = 64;                         // per thread
constexpr int FA_TILE = FA_THREADS * FA_BYTES;       // 16 KB

__device__ __forceinline__ bool fa_ws(u32 c) {       // Python str.isspace() on ASCII
    return c == 32 || (c >= 9 && c <= 13) || (c >= 28 && c <= 31);
}
__device__ __forceinline__ u32 fa_upper(u32 c) { return (c >= 'a' && c <= 'z') ? c - 32 : c; }
// rank of an upper-cased residue, 0 if not in the alphabet
// (branch-free: u in 0x40..0x5F indexes a 3-bit-per-entry table by u & 31;
// A=1 C=3 G=7 N=14 T=20)
__device__ __forceinline__ u32 fa_rank(u32 u, int keep_n) {
    const u64 tab = (1ull << 3) | (2ull << 9) | (3ull << 21) | (4ull << 60) | (keep_n ? (5ull << 42) : 0ull);
    return (u & 0xE0u) == 0x40u ? (u32)((tab >> (3 * (u & 31u))) & 7u) : 0u;
}

// '\n' count of the 64 bytes of thread t of tile `tile`
__device__ __forceinline__ u32 fa_count(const u8 *__restrict__ d, i64 B, i64 base, bool vec) {
    u32 c = 0;
    if (vec && base + FA_BYTES <= B) {
        const uint4 *p = reinterpret_cast<const uint4 *>(d + base);
#pragma unroll
        for (int q = 0; q < FA_BYTES / 16; q++) {
            uint4 v = __ldg(p + q);
            c += __popc(__vcmpeq4(v.x, 0x0A0A0A0Au)) + __popc(__vcmpeq4(v.y, 0x0A0A0A0Au)) +
                 __popc(__vcmpeq4(v.z, 0x0A0A0A0Au)) + __popc(__vcmpeq4(v.w, 0x0A0A0A0Au));
        }
        return c >> 3;
    }
    for (i64 i = base; i < B && i < base + FA_BYTES; i++) c += d[i] == '\n';
    return c;
}

__global__ void __launch_bounds__(FA_THREADS) k_fa_nl_count(const u8 *__restrict__ d, i64 B, bool vec,
                                                            u32 *__restrict__ tile_cnt) {
    __shared__ u32 sh_warp[FA_THREADS / 32 + 1];
    const i64 base = (i64)blockIdx.x * FA_TILE + (i64)threadIdx.x * FA_BYTES;
    u32 c = fa_count(d, B, base, vec);
    u32 excl;
    u32 tot = block_exclusive_scan<FA_THREADS>(c, excl, sh_warp);
    if (threadIdx.x == 0) tile_cnt[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(FA_THREADS) k_fa_nl_emit(const u8 *__restrict__ d, i64 B, bool vec,
                                                           const u32 *__restrict__ tile_off, u32 *__restrict__ nl) {
    __shared__ u32 sh_warp[FA_THREADS / 32 + 1];
    const i64 base = (i64)blockIdx.x * FA_TILE + (i64)threadIdx.x * FA_BYTES;
    const bool full = vec && base + FA_BYTES <= B;
    u32 m[FA_BYTES / 4];  // per word: 0xFF in each '\n' byte
    u32 c = 0;
    if (full) {
        const uint4 *p = reinterpret_cast<const uint4 *>(d + base);
#pragma unroll
        for (int q = 0; q < FA_BYTES / 16; q++) {
            uint4 v = __ldg(p + q);
            m[4 * q] = __vcmpeq4(v.x, 0x0A0A0A0Au);
            m[4 * q + 1] = __vcmpeq4(v.y, 0x0A0A0A0Au);
            m[4 * q + 2] = __vcmpeq4(v.z, 0x0A0A0A0Au);
            m[4 * q + 3] = __vcmpeq4(v.w, 0x0A0A0A0Au);
        }
#pragma unroll
        for (int k = 0; k < FA_BYTES / 4; k++) c += __popc(m[k]);
        c >>= 3;
    } else {
        c = fa_count(d, B, base, false);
    }
    u32 excl;
    block_exclusive_scan<FA_THREADS>(c, excl, sh_warp);
    if (!c) return;
    u32 o = tile_off[blockIdx.x] + excl;
    if (full) {
#pragma unroll
        for (int k = 0; k < FA_BYTES / 4; k++) {
            u32 x = m[k] & 0x80808080u;
            while (x) {
                const int b = (__ffs(x) - 1) >> 3;
                nl[o++] = (u32)(base + 4 * k + b);
                x &= x - 1;
            }
        }
    } else {
        for (i64 i = base; i < B && i < base + FA_BYTES; i++)
            if (d[i] == '\n') nl[o++] = (u32)i;
    }
}

enum : u8 { FA_BLANK = 0, FA_HEADER = 1, FA_SEQ = 2 };

struct FaLines {
    u32 *start;   // sequence: first residue byte; header: first byte of the stripped header text
    u32 *len;     // residue count / header text length
    u8 *kind;
    u32 *seq_off;  // exclusive scan of residue counts
    u32 *hdr_idx;  // exclusive scan of header flags
    u32 *hdr_off;  // exclusive scan of header text lengths
};

__global__ void k_fa_classify(const u8 *__restrict__ d, i64 B, const u32 *__restrict__ nl, i64 nnl, i64 L,
                              FaLines ln, unsigned long long *__restrict__ err) {
    for (i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x; i < L; i += (i64)gridDim.x * blockDim.x) {
        i64 s = i ? (i64)nl[i - 1] + 1 : 0;
        i64 e = i < nnl ? (i64)nl[i] : B;
        while (s < e && fa_ws(d[s])) s++;
        while (e > s && fa_ws(d[e - 1])) e--;
        u8 kind = FA_BLANK;
        u32 st = (u32)s, len = 0;
        if (s < e) {
            if (d[s] == '>') {
                kind = FA_HEADER;
                i64 h = s + 1;
                while (h < e && fa_ws(d[h])) h++;
                st = (u32)h;
                len = (u32)(e - h);
                if (len == 0) atomicMin(err, (unsigned long long)s);  // empty FASTA header
            } else {
                kind = FA_SEQ;
                len = (u32)(e - s);
            }
        }
        ln.start[i] = st;
        ln.len[i] = len;
        ln.kind[i] = kind;
    }
}

struct FaSeqLenIn {
    const u8 *kind;
    const u32 *len;
    __device__ u32 operator()(i64 i) const { return kind[i] == FA_SEQ ? len[i] : 0u; }
};
struct FaHdrFlagIn {
    const u8 *kind;
    __device__ u32 operator()(i64 i) const { return kind[i] == FA_HEADER; }
};
struct FaHdrLenIn {
    const u8 *kind;
    const u32 *len;
    __device__ u32 operator()(i64 i) const { return kind[i] == FA_HEADER ? len[i] : 0u; }
};
struct FaStoreOut {
    u32 *out;
    __device__ void operator()(i64 i, u32 excl, u32) const { out[i] = excl; }
};
// header index scan; a sequence line with no header before it is an error
struct FaHdrIdxOut {
    u32 *out;
    u32 *hdr_line;  // line index of header k
    const u8 *kind;
    const u32 *start;
    unsigned long long *err;
    __device__ void operator()(i64 i, u32 excl, u32 v) const {
        out[i] = excl;
        if (v) hdr_line[excl] = (u32)i;
        if (excl == 0 && kind[i] == FA_SEQ) atomicMin(err, (unsigned long long)start[i]);
    }
};

// warp per header: record start and header text (sequence lines are
// k_fa_emit_seq's)
__global__ void k_fa_emit_hdr(const u8 *__restrict__ d, i64 R, const u32 *__restrict__ hdr_line, FaLines ln,
                              u32 *__restrict__ rec_start, u8 *__restrict__ hdr, u32 *__restrict__ hdr_off) {
    const int lane = lane_id();
    const i64 w0 = ((i64)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const i64 nw = ((i64)gridDim.x * blockDim.x) >> 5;
    for (i64 k = w0; k < R; k += nw) {
        const u32 i = hdr_line[k];
        const u32 s = ln.start[i], len = ln.len[i], o = ln.hdr_off[i];
        if (lane == 0) {
            rec_start[k] = ln.seq_off[i];
            hdr_off[k] = o;
        }
        for (u32 j = lane; j < len; j += 32) hdr[o + j] = d[s + j];
    }
}

// Sequence lines, FA_LINES per CTA: the batch's input bytes (contiguous in
// the file) are staged in shared memory with 16-byte loads, each warp
// transforms its lines smem -> smem, and the batch's output (contiguous in
// the residue buffer) leaves with 16-byte stores.  Batches whose input span
// exceeds the stage fall back to warp-per-line global copies.
constexpr int FA_LINES = 128;
constexpr int FA_STAGE = 16384;

__device__ __forceinline__ void fa_line_bytes(const u8 *src, u32 len, u8 *dst, int keep_n, int as_ranks, u32 s,
                                              unsigned long long *err) {
    const int lane = lane_id();
    for (u32 j0 = 0; j0 < len; j0 += 32) {
        const u32 j = j0 + lane;
        u32 r = 1;
        if (j < len) {
            const u32 u = fa_upper(src[j]);
            r = fa_rank(u, keep_n);
            dst[j] = as_ranks ? (u8)r : (u8)u;
        }
        const unsigned bad = __ballot_sync(0xffffffffu, r == 0);
        if (bad) {
            if (lane == 0) atomicMin(err, (unsigned long long)(s + j0 + __ffs(bad) - 1));
            break;
        }
    }
}

__global__ void __launch_bounds__(256) k_fa_emit_seq(const u8 *__restrict__ d, i64 B, const u32 *__restrict__ nl,
                                                     i64 nnl, i64 L, FaLines ln, int keep_n, int as_ranks,
                                                     u8 *__restrict__ res, unsigned long long *__restrict__ err) {
    __shared__ __align__(16) u8 sin_buf[FA_STAGE + 48];  // 16 bytes of front slack for the funnel reads
    __shared__ __align__(16) u8 sout[FA_STAGE + 32];
    __shared__ u32 s_start[FA_LINES], s_len[FA_LINES], s_off[FA_LINES];
    u8 *sin = sin_buf + 16;
    const i64 l0 = (i64)blockIdx.x * FA_LINES;
    const i64 l1 = l0 + FA_LINES < L ? l0 + FA_LINES : L;
    const int nlines = (int)(l1 - l0);
    // the batch's line table (sequence lines only; others get len 0)
    if (threadIdx.x < nlines) {
        const i64 i = l0 + threadIdx.x;
        const bool seq = ln.kind[i] == FA_SEQ;
        s_start[threadIdx.x] = ln.start[i];
        s_len[threadIdx.x] = seq ? ln.len[i] : 0u;
        s_off[threadIdx.x] = ln.seq_off[i];
    }
    const i64 in_lo = l0 ? (i64)nl[l0 - 1] + 1 : 0;
    const i64 in_hi = (l1 - 1 < nnl) ? (i64)nl[l1 - 1] + 1 : B;
    const i64 a_lo = in_lo & ~(i64)15;
    const int warp = threadIdx.x >> 5;
    const bool staged = in_hi - a_lo <= FA_STAGE;
    if (staged) {
        const bool vec = ((reinterpret_cast<uintptr_t>(d) & 15) == 0);
        for (i64 q = a_lo + 16 * (i64)threadIdx.x; q < in_hi; q += 16 * 256) {
            if (vec && q + 16 <= B) {
                *reinterpret_cast<uint4 *>(sin + (q - a_lo)) = __ldg(reinterpret_cast<const uint4 *>(d + q));
            } else {
                for (int k = 0; k < 16 && q + k < B; k++) sin[q - a_lo + k] = d[q + k];
            }
        }
    }
    __syncthreads();
    const i64 out_lo = s_off[0];
    const i64 out_hi = (i64)s_off[nlines - 1] + s_len[nlines - 1];
    if (!staged) {  // long lines: direct
        for (int k = warp; k < nlines; k += 8)
            if (s_len[k])
                fa_line_bytes(d + s_start[k], s_len[k], res + s_off[k], keep_n, as_ranks, s_start[k], err);
        return;
    }
    // sout byte x <-> res byte out_lo - sh + x, with sh = (res + out_lo) % 16,
    // so the store loop is 16-byte aligned on both sides
    const int sh = (int)((reinterpret_cast<uintptr_t>(res) + out_lo) & 15);
    for (int k = warp; k < nlines; k += 8)
        if (s_len[k])
            fa_line_bytes(sin + (s_start[k] - a_lo), s_len[k], sout + sh + (s_off[k] - out_lo), keep_n, as_ranks,
                          s_start[k], err);
    __syncthreads();
    const i64 n = out_hi - out_lo;
    u8 *g = res + out_lo - sh;  // 16-byte aligned
    const i64 blocks = (sh + n + 15) >> 4;
    for (i64 v = threadIdx.x; v < blocks; v += 256) {
        const i64 x0 = 16 * v;
        if (x0 >= sh && x0 + 16 <= sh + n) {
            *reinterpret_cast<uint4 *>(g + x0) = *reinterpret_cast<const uint4 *>(sout + x0);
        } else {
            for (int k = 0; k < 16; k++)
                if (x0 + k >= sh && x0 + k < sh + n) g[x0 + k] = sout[x0 + k];
        }
    }
}

// the line holding byte `pos` (binary search over the newline positions)
__global__ void k_fa_err_info(const unsigned long long *__restrict__ err, const u32 *__restrict__ nl, i64 nnl,
                              FaLines ln, i64 *__restrict__ info) {
    const unsigned long long pos = *err;
    if (pos == ~0ull) {
        info[0] = -1;
        return;
    }
    i64 lo = 0, hi = nnl;  // first newline >= pos
    while (lo < hi) {
        i64 mid = (lo + hi) >> 1;
        if ((unsigned long long)nl[mid] < pos) lo = mid + 1;
        else hi = mid;
    }
    info[0] = (i64)pos;
    info[1] = lo;                // 0-based line index
    info[2] = ln.kind[lo];
    info[3] = ln.start[lo];
    info[4] = ln.hdr_idx[lo];    // headers before this line
}

struct FaWs {
    u32 *tile;                   // tile counts / offsets
    u32 *nl;
    u32 *hdr_line;
    FaLines ln;
    u32 *tmp;                    // scan scratch
    u32 *totals;                 // [0] newlines, [1] residues, [2] records, [3] header bytes
    unsigned long long *err;
    i64 *info;
};

static bool fa_layout(Arena &ar, i64 B, i64 L, FaWs &w) {
    const i64 tiles = ceil_div(B > 0 ? B : 1, FA_TILE);
    w.tile = ar.alloc<u32>(tiles + 1);
    w.nl = ar.alloc<u32>(L + 1);
    w.hdr_line = ar.alloc<u32>(L + 1);
    w.ln.start = ar.alloc<u32>(L + 1);
    w.ln.len = ar.alloc<u32>(L + 1);
    w.ln.seq_off = ar.alloc<u32>(L + 1);
    w.ln.hdr_idx = ar.alloc<u32>(L + 1);
    w.ln.hdr_off = ar.alloc<u32>(L + 1);
    w.ln.kind = ar.alloc<u8>(L + 1);
    w.tmp = ar.alloc<u32>(scan_tmp_words(L > tiles ? L : tiles));
    w.totals = ar.alloc<u32>(8);
    w.err = ar.alloc<unsigned long long>(1);
    w.info = ar.alloc<i64>(8);
    return !ar.overflow;
}

}  // namespace saix

using namespace saix;

extern "C" size_t saix_fasta_workspace_bytes(int64_t nbytes, int64_t lines) {
    Arena ar;
    FaWs w;
    fa_layout(ar, nbytes, lines, w);
    return ar.peak + Arena::kAlign;
}

extern "C" int saix_fasta_lines(const uint8_t *data, int64_t nbytes, int64_t *lines_host, void *ws, size_t ws_bytes,
                                void *stream) {
    if (nbytes < 0 || !lines_host || (nbytes > 0 && !data) || nbytes >= ((int64_t)1 << 32) - 1) {
        set_error("saix_fasta_lines: invalid arguments (inputs must be < 4 GiB)");
        return SAIX_EINVAL;
    }
    *lines_host = 0;
    if (nbytes == 0) return SAIX_OK;
    const i64 tiles = ceil_div(nbytes, FA_TILE);
    if (ws_bytes < (size_t)(tiles + 8) * 4 + 2 * Arena::kAlign) {
        set_error("saix_fasta_lines: workspace too small");
        return SAIX_ENOSPC;
    }
    cudaStream_t st = (cudaStream_t)stream;
    Arena ar{(char *)ws, ws_bytes};
    u32 *tile = ar.alloc<u32>(tiles);
    u32 *tot = ar.alloc<u32>(4);
    SAIX_ARENA_OK(ar);
    const bool vec = ((uintptr_t)data & 15) == 0;
    {
        Prof prof_("fasta.lines", (double)nbytes, st);
        k_fa_nl_count<<<(unsigned)tiles, FA_THREADS, 0, st>>>(data, nbytes, vec, tile);
        SAIX_LAUNCHED();
        k_scan_block_sums<<<1, 1024, 0, st>>>(tile, tiles, tot);
        SAIX_LAUNCHED();
    }
    u32 h[1];
    u8 last;
    SAIX_CUDA(cudaMemcpyAsync(h, tot, 4, cudaMemcpyDeviceToHost, st));
    SAIX_CUDA(cudaMemcpyAsync(&last, data + nbytes - 1, 1, cudaMemcpyDeviceToHost, st));
    SAIX_CUDA(cudaStreamSynchronize(st));
    *lines_host = (i64)h[0] + (last != '\n');
    return SAIX_OK;
}

// Pass 1 + 2: line table, scans and the line-level errors.  counts_host:
// [0] residues, [1] records, [2] header-text bytes, [3] error byte position
// so far (-1 if none).  `lines` must be what saix_fasta_lines returned.
extern "C" int saix_fasta_scan(const uint8_t *data, int64_t nbytes, int64_t lines, int64_t *counts_host, void *ws,
                               size_t ws_bytes, void *stream) {
    if (nbytes < 0 || lines < 0 || !counts_host || (nbytes > 0 && !data) || nbytes >= ((int64_t)1 << 32) - 1) {
        set_error("saix_fasta_scan: invalid arguments");
        return SAIX_EINVAL;
    }
    cudaStream_t st = (cudaStream_t)stream;
    Arena ar{(char *)ws, ws_bytes};
    FaWs w;
    if (!fa_layout(ar, nbytes, lines, w)) {
        set_error("saix_fasta_scan: workspace too small");
        return SAIX_ENOSPC;
    }
    SAIX_CUDA(cudaMemsetAsync(w.totals, 0, 32, st));
    SAIX_CUDA(cudaMemsetAsync(w.err, 0xFF, 8, st));
    if (nbytes > 0) {
        const i64 tiles = ceil_div(nbytes, FA_TILE);
        const bool vec = ((uintptr_t)data & 15) == 0;
        u32 nnl = 0;
        {
            Prof prof_("fasta.newlines", 2.0 * nbytes + 4.0 * lines, st);
            k_fa_nl_count<<<(unsigned)tiles, FA_THREADS, 0, st>>>(data, nbytes, vec, w.tile);
            SAIX_LAUNCHED();
            k_scan_block_sums<<<1, 1024, 0, st>>>(w.tile, tiles, w.totals);
            SAIX_LAUNCHED();
            k_fa_nl_emit<<<(unsigned)tiles, FA_THREADS, 0, st>>>(data, nbytes, vec, w.tile, w.nl);
            SAIX_LAUNCHED();
            SAIX_CUDA(cudaMemcpyAsync(&nnl, w.totals, 4, cudaMemcpyDeviceToHost, st));
            SAIX_CUDA(cudaStreamSynchronize(st));
        }
        if ((i64)nnl > lines || lines > (i64)nnl + 1) {
            set_error("saix_fasta_scan: line count does not match the data");
            return SAIX_EINVAL;
        }
        {
            Prof prof_("fasta.classify", 17.0 * lines, st);
            k_fa_classify<<<grid_for(lines, 256), 256, 0, st>>>(data, nbytes, w.nl, nnl, lines, w.ln, w.err);
            SAIX_LAUNCHED();
        }
        SAIX_TRY(scan_transform(FaSeqLenIn{w.ln.kind, w.ln.len}, FaStoreOut{w.ln.seq_off}, lines, w.tmp,
                                w.totals + 1, st, "fasta.line_scans", 9.0 * lines));
        SAIX_TRY(scan_transform(FaHdrFlagIn{w.ln.kind},
                                FaHdrIdxOut{w.ln.hdr_idx, w.hdr_line, w.ln.kind, w.ln.start, w.err}, lines, w.tmp, w.totals + 2,
                                st, "fasta.line_scans", 5.0 * lines));
        SAIX_TRY(scan_transform(FaHdrLenIn{w.ln.kind, w.ln.len}, FaStoreOut{w.ln.hdr_off}, lines, w.tmp,
                                w.totals + 3, st, "fasta.line_scans", 9.0 * lines));
    }
    u32 h[4];
    unsigned long long e;
    SAIX_CUDA(cudaMemcpyAsync(h, w.totals, 16, cudaMemcpyDeviceToHost, st));
    SAIX_CUDA(cudaMemcpyAsync(&e, w.err, 8, cudaMemcpyDeviceToHost, st));
    SAIX_CUDA(cudaStreamSynchronize(st));
    counts_host[0] = h[1];
    counts_host[1] = h[2];
    counts_host[2] = h[3];
    counts_host[3] = e == ~0ull ? -1 : (i64)e;
    return SAIX_OK;
}

// Pass 3: residues (as_ranks: A1 C2 G3 T4 [N5], else upper-cased ASCII) into
// res (counts[0] bytes), record starts into rec_start (records + 1 u32),
// header texts into hdr (counts[2] bytes) with hdr_off (records + 1 u32).
// err_host[0..4]: -1, or the first error's byte position, its 0-based line,
// the line kind (1 header, 2 sequence), the line's first byte, and the number
// of headers before the line.
extern "C" int saix_fasta_emit(const uint8_t *data, int64_t nbytes, int64_t lines, int keep_n, int as_ranks,
                               uint8_t *res, uint32_t *rec_start, uint8_t *hdr, uint32_t *hdr_off,
                               int64_t *err_host, void *ws, size_t ws_bytes, void *stream) {
    if (nbytes < 0 || lines < 0 || !err_host || !rec_start || !hdr_off || (nbytes > 0 && !data)) {
        set_error("saix_fasta_emit: invalid arguments");
        return SAIX_EINVAL;
    }
    cudaStream_t st = (cudaStream_t)stream;
    Arena ar{(char *)ws, ws_bytes};
    FaWs w;
    if (!fa_layout(ar, nbytes, lines, w)) {
        set_error("saix_fasta_emit: workspace too small");
        return SAIX_ENOSPC;
    }
    u32 h[4];
    SAIX_CUDA(cudaMemcpyAsync(h, w.totals, 16, cudaMemcpyDeviceToHost, st));
    SAIX_CUDA(cudaStreamSynchronize(st));
    if (lines > 0) {
        Prof prof_("fasta.emit", 2.0 * (double)nbytes + 17.0 * lines, st);
        k_fa_emit_seq<<<(unsigned)ceil_div(lines, FA_LINES), 256, 0, st>>>(data, nbytes, w.nl, (i64)h[0], lines,
                                                                          w.ln, keep_n, as_ranks, res, w.err);
        SAIX_LAUNCHED();
    }
    if (h[2]) {
        Prof prof_("fasta.headers", 2.0 * h[3] + 24.0 * h[2], st);
        k_fa_emit_hdr<<<grid_for((i64)h[2] * 32, 256), 256, 0, st>>>(data, h[2], w.hdr_line, w.ln, rec_start, hdr,
                                                                    hdr_off);
        SAIX_LAUNCHED();
    }
    // closing offsets
    SAIX_CUDA(cudaMemcpyAsync(rec_start + h[2], &h[1], 4, cudaMemcpyHostToDevice, st));
    SAIX_CUDA(cudaMemcpyAsync(hdr_off + h[2], &h[3], 4, cudaMemcpyHostToDevice, st));
    k_fa_err_info<<<1, 1, 0, st>>>(w.err, w.nl, (i64)h[0], w.ln, w.info);
    SAIX_LAUNCHED();
    SAIX_CUDA(cudaMemcpyAsync(err_host, w.info, 5 * 8, cudaMemcpyDeviceToHost, st));
    SAIX_CUDA(cudaStreamSynchronize(st));
    return SAIX_OK;
}
