/*
 * saix_b200.h -- C ABI of libsaix_b200.so, the sm_100a implementation of the
 * reference `saix` longest-overlap hot path (DC3 suffix array -> LCP ->
 * sparse-table RMQ -> cross-sequence overlap scan).
 *
 * Conventions
 *   - All array pointers are DEVICE pointers unless the name ends in `_host`.
 *   - Every call is stream-ordered on `stream` (a cudaStream_t passed as
 *     void*; NULL = legacy default stream) and performs no hidden device
 *     allocation: scratch comes from the caller's `ws` of at least the size
 *     the matching *_workspace_bytes() returns.
 *   - Return 0 on success or a negative SAIX_E* code; saix_last_error()
 *     returns a thread-local message for the last failure on this thread.
 *   - Positions, ranks and LCP values are uint32 on the device (n < 2^32-4);
 *     the Python layer widens them to the reference's int64 arrays.
 *
 * Each entry point names the reference interface it replaces
 * (paths relative to the reference checkout, pkg/src/saix/...).
 */
#ifndef SAIX_B200_H
#define SAIX_B200_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define SAIX_API __attribute__((visibility("default")))
#else
#define SAIX_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define SAIX_OK 0
#define SAIX_EINVAL (-22)   /* bad argument: reference ValueError            */
#define SAIX_ERANGE (-34)   /* index out of range: reference IndexError      */
#define SAIX_ENOSPC (-28)   /* workspace smaller than *_workspace_bytes()     */
#define SAIX_ECUDA (-100)   /* CUDA runtime error (message has the details)   */
#define SAIX_ESEQ (-101)    /* illegal residue: reference SequenceError       */
#define SAIX_ENCCL (-102)   /* NCCL unavailable or failed (message: details)  */

SAIX_API const char *saix_last_error(void);
SAIX_API int saix_abi_version(void);

/* Per-kernel CUDA-event timing for measurement tools (bench.py): when
 * enabled every instrumented launch is bracketed by events on its stream and
 * tagged with its algorithmic bytes (DESIGN.md roofline model).
 * saix_prof_enable(on) clears the log; saix_prof_collect() synchronizes the
 * events, aggregates by kernel name into `out` and returns the entry count. */
typedef struct saix_prof_entry {
    char name[64];
    int64_t launches;
    double total_ms;
    double bytes;
} saix_prof_entry;

SAIX_API void saix_prof_enable(int on);
SAIX_API int saix_prof_collect(saix_prof_entry *out, int max_entries);

/* ---------------------------------------------------------------- encode */

/* encode (sequence.py:144-157) fused with GeneralizedText.build
 * (overlap.py:83-95): ASCII A and B -> u8 GSA ranks encode(A)+1 ++ [1] ++
 * encode(B)+1, n = na+nb+1.  keep_n selects NPolicy.KEEP (N -> rank 5).
 * *bad_pos (device int64, caller sets INT64_MAX) receives the smallest GSA
 * offset of an illegal residue (offset na+1+i for B[i]). */
SAIX_API int saix_encode_gsa(const uint8_t *a_ascii, int64_t na, const uint8_t *b_ascii,
                    int64_t nb, int keep_n, uint8_t *gsa, int64_t *bad_pos,
                    void *stream);

/* encode (sequence.py:144-157) alone: ASCII -> u8 ranks (A1 C2 G3 T4 [N5]). */
SAIX_API int saix_encode(const uint8_t *ascii, int64_t n, int keep_n, uint8_t *ranks,
                int64_t *bad_pos, void *stream);

/* ------------------------------------------------------------------- DC3 */

/* Level-0 introspection (Dc3Workspace, suffix_index.py:119-140,414-449).
 * Device arrays may be NULL individually; sizes: triple_text m,
 * sample_rank n+3 (1-based ranks by position), sorted_samples m,
 * sorted_nonsamples ceil(n/3).  The scalar outputs are written by the call. */
typedef struct saix_dc3_probe {
    uint32_t *triple_text;
    uint32_t *sample_rank;
    uint32_t *sorted_samples;
    uint32_t *sorted_nonsamples;
    int64_t n_samples;            /* m (incl. the padding sample)           */
    int64_t n_sorted_samples;     /* real samples (< n)                      */
    int64_t n_sorted_nonsamples;  /* k = ceil(n/3)                           */
    int32_t depth;                /* recursion levels below the top          */
    int32_t reserved;
} saix_dc3_probe;

SAIX_API size_t saix_dc3_workspace_bytes(int64_t n, int text_bytes);

/* build_sa_dc3 (suffix_index.py:395-399) + SuffixArray.from_order (96-101).
 * text: n ranks in 1..sigma (0 never appears), text_bytes = 1 (u8) or 4 (u32).
 * sa, isa: n entries each (isa = the reference's 0-based `rank`; may be NULL
 * only if not needed).  probe may be NULL. */
SAIX_API int saix_dc3(const void *text, int text_bytes, int64_t n, int64_t sigma,
             uint32_t *sa, uint32_t *isa, void *ws, size_t ws_bytes,
             saix_dc3_probe *probe, void *stream);

SAIX_API size_t saix_dc3_merge_workspace_bytes(int64_t total);

/* merge_sample_nonsample (suffix_index.py:452-457, _merge 362-378): step 3
 * alone.  sample_rank: n+3 by position; sorted_samples (ms entries) and
 * sorted_nonsamples (k entries) as in the probe; sa gets ms+k entries. */
SAIX_API int saix_dc3_merge(const void *text, int text_bytes, int64_t n,
                   const uint32_t *sample_rank, const uint32_t *sorted_samples,
                   int64_t ms, const uint32_t *sorted_nonsamples, int64_t k,
                   uint32_t *sa, void *ws, size_t ws_bytes, void *stream);

/* Level trace of the last saix_dc3 call on this host thread: per recursion
 * level (top first) {N, sigma, samples m, distinct triple names}; returns
 * the number of levels (at most max_levels are written to out[4*i..]). */
SAIX_API int saix_dc3_trace(int64_t *out, int max_levels);

/* Level-0 naming path of the last byte-text DC3 level 0 on this host thread:
 * 0 triple naming (+ recursion), 1 generic 21-character window sort, 2 the
 * DNA window sort (ranks 1..4: MSD record sort, csrc/wsort.cuh).  Test and
 * A/B aid; the SA / ISA are the same on every path. */
SAIX_API int saix_dc3_naming(void);

/* Level-0 window naming (byte texts, sigma <= 7): samples named by their
 * 21-character windows, ties ordered by prefix doubling, no recursion below
 * level 0 (same SA / ISA).  on = 0 runs the reference recursion instead.
 * Returns the previous setting (default on; env SAIX_WINDOW_NAMING=0). */
SAIX_API int saix_dc3_set_window_naming(int on);

/* ------------------------------------------------- parallel sort engine */
/* The reference's split-kernel engine (parallel_sort.py:110-293) on the
 * device scan and radix sort. Keys are int64 (nonnegative for the sort). */

SAIX_API size_t saix_psort_workspace_bytes(int64_t n);

/* exclusive_scan (parallel_sort.py:110-131): out[0] = 0, out[i] = sum(in[<i]). */
SAIX_API int saix_exclusive_scan_i64(const int64_t *in, int64_t n, int64_t *out,
             void *ws, size_t ws_bytes, void *stream);

/* split_by_bit (parallel_sort.py:150-163): stable zero-then-one partition by
 * bit `bit`; bits, zero_flags, dest nullable; scanned = exclusive scan of the
 * zero flags; *zero_total (device) = number of zero bits. */
SAIX_API int saix_split_by_bit(const int64_t *keys, int64_t n, int bit, int64_t *out,
             int64_t *bits, int64_t *zero_flags, int64_t *scanned, int64_t *dest,
             int64_t *zero_total, void *ws, size_t ws_bytes, void *stream);

/* radix_sort / chunked_sort (parallel_sort.py:195-254): ascending stable sort
 * of nonnegative keys < 2^total_bits (the caller checks the width). */
SAIX_API int saix_radix_sort_i64(const int64_t *keys, int64_t n, int total_bits,
             int64_t *out, void *ws, size_t ws_bytes, void *stream);

/* ------------------------------------------------------------------- LCP */

SAIX_API size_t saix_lcp_workspace_bytes(int64_t n);

/* build_lcp (suffix_index.py:479-506): lcp[r] = |lcp(suffix sa[r-1],
 * suffix sa[r])|, lcp[0] = 0. */
SAIX_API int saix_lcp(const void *text, int text_bytes, int64_t n, const uint32_t *sa,
             const uint32_t *isa, uint32_t *lcp, void *ws, size_t ws_bytes,
             void *stream);

/* build_lcp with the alphabet known (suffix_index.py:479-506, same output):
 * sigma = largest rank (<= 0: unknown), separator = position of a unique
 * separator rank 1 (generalized text, overlap.py:83-95) or -1.  Byte texts
 * with <= 4 residue ranks (plus the separator) are compared 32 characters per
 * word on a 2-bit packed copy; u8 text must be 16-byte aligned. */
SAIX_API int saix_lcp_sigma(const void *text, int text_bytes, int64_t n, int64_t sigma,
             int64_t separator, const uint32_t *sa, uint32_t *lcp, void *ws,
             size_t ws_bytes, void *stream);

/* ------------------------------------------------------------------- RMQ */

#define SAIX_SPARSE_PACK32 0  /* entry = (value-bias) << ibits | index, u32 */
#define SAIX_SPARSE_PACK64 1  /* same packing in u64                        */
#define SAIX_SPARSE_INDEX 2   /* entry = u32 index; values gathered (int64) */
#define SAIX_SPARSE_BLOCKED 3 /* u8 values + 256-value blocks + sparse table
                                 over block minima (L2-resident; queries scan
                                 the two end blocks); values span <= 254    */

typedef struct saix_sparse_plan {
    int64_t n;
    int64_t value_bias;    /* subtracted before packing (min value)        */
    int64_t table_bytes;   /* bytes the table needs                        */
    int32_t levels;        /* SparseTable levels (rmq.py:38-47)            */
    int32_t mode;          /* SAIX_SPARSE_*                                */
    int32_t index_bits;
    int32_t value_bits;
} saix_sparse_plan;

/* min and max of n device values (value_bytes 4 = u32, 8 = int64) into
 * out2 (device int64[2]); lets a sparse table over a device array (e.g. an
 * LCP array) be planned without copying it to the host. */
SAIX_API int saix_minmax(const void *values, int value_bytes, int64_t n, int64_t *out2, void *stream);

/* dst[i] = (int64)src[i] for a u8 (src_bytes 1) or u32 (4) device array: the
 * reference API's int64 host arrays are widened on the device before the
 * download. */
SAIX_API int saix_widen_i64(const void *src, int src_bytes, int64_t n, int64_t *dst, void *stream);

/* Choose the table layout for n values in [vmin, vmax]. */
SAIX_API int saix_sparse_plan_make(int64_t n, int64_t vmin, int64_t vmax,
                          saix_sparse_plan *plan);

/* The query-optimised layout for the same SparseTable: SAIX_SPARSE_BLOCKED
 * when vmax - vmin <= 254 (LCP arrays), else exactly saix_sparse_plan_make.
 * Same answers (leftmost argmin); the per-level reference layout
 * (SparseTable.table) then needs a saix_sparse_plan_make table. */
SAIX_API int saix_sparse_plan_blocked(int64_t n, int64_t vmin, int64_t vmax,
                          saix_sparse_plan *plan);

/* SparseTable.__init__ (rmq.py:33-50).  values: n entries of
 * value_bytes = 4 (u32, e.g. a device LCP array) or 8 (int64). */
SAIX_API int saix_sparse_build(const saix_sparse_plan *plan, const void *values,
                      int value_bytes, void *table, void *stream);

/* SparseTable.query / query_sparse (rmq.py:52-58, 254-259), batched:
 * out_index[t] = leftmost argmin of values[min(i,j)..max(i,j)].
 * out_value (nullable) receives values[out_index].  Out-of-range pairs set
 * *err (device int32, caller zeroes) to 1 (reference: IndexError). */
SAIX_API int saix_sparse_query(const saix_sparse_plan *plan, const void *table,
                      const void *values, int value_bytes, const int64_t *qi,
                      const int64_t *qj, int64_t q, int64_t *out_index,
                      int64_t *out_value, int32_t *err, void *stream);

/* lcp_query (overlap.py:58-69), batched over an engine whose sparse table
 * was built over its LCP array: i == j -> n - i, otherwise
 * lcp[argmin(lcp[lo+1..hi])] with lo/hi the sorted ranks isa[i], isa[j]. */
SAIX_API int saix_lcp_query(const saix_sparse_plan *plan, const void *table,
                   const void *lcp, int lcp_bytes, const uint32_t *isa,
                   const int64_t *qi, const int64_t *qj, int64_t q,
                   int64_t *out, int32_t *err, void *stream);

/* ------------------------------------------------------- multi-GPU (8e) */
/* Batched pairs shard across ranks (one process per GPU); the per-pair
 * results are the only exchange.  NCCL is bound at run time (libnccl.so.2,
 * shared with the process's NCCL if already loaded).  The 128-byte id from
 * rank 0 reaches the other ranks through the caller's bootstrap (e.g. a
 * torch.distributed broadcast), then every rank calls saix_comm_init with
 * its own device.  Collectives are stream-ordered on `stream`.
 * Reference: overlap.py:110-152 (the per-pair call being sharded). */
SAIX_API int saix_comm_unique_id(uint8_t *out128);
SAIX_API int saix_comm_init(void **comm, int nranks, const uint8_t *id128, int rank, int device);
SAIX_API int saix_comm_destroy(void *comm);
/* recv (device, nranks * count int64) = every rank's send (count int64), in
 * rank order: the padded per-shard result blocks */
SAIX_API int saix_comm_allgather_i64(void *comm, const int64_t *send, int64_t count, int64_t *recv, void *stream);
/* recv = elementwise MIN over ranks (the first illegal residue of the job) */
SAIX_API int saix_comm_allreduce_min_i64(void *comm, const int64_t *send, int64_t *recv, int64_t count,
                                         void *stream);

/* --------------------------------------------------------------- overlap */

SAIX_API size_t saix_overlap_workspace_bytes(int64_t n);

/* The scan half of longest_overlap (overlap.py:128-152) over a generalized
 * suffix array of n = |A|+|B|+1 with the separator at `boundary` = |A|:
 * out3 (device int64[3]) = {length, pos_a, pos_b}, (0,0,0) when no
 * cross-sequence pair shares a prefix. */
SAIX_API int saix_overlap_scan(const uint32_t *sa, const uint32_t *lcp, int64_t n,
                      int64_t boundary, int64_t *out3, void *ws, size_t ws_bytes,
                      void *stream);

SAIX_API size_t saix_longest_overlap_workspace_bytes(int64_t na, int64_t nb);

/* longest_overlap (overlap.py:110-152) end to end on the device: encode +
 * GSA + DC3 + LCP + scan.  a_ascii/b_ascii are device buffers; out3 and
 * bad_pos are device int64 (bad_pos set to INT64_MAX by the callee; else the
 * first illegal residue's generalized-text position, B's residue k at
 * na + 1 + k).  Pairs with na + 1 + nb <= 20480 run through the on-chip pair
 * kernel as a batch of one (saix_overlap_batch_dev; same results), unless
 * saix_overlap_batch_set_onchip(0). */
SAIX_API int saix_longest_overlap(const uint8_t *a_ascii, int64_t na,
                         const uint8_t *b_ascii, int64_t nb, int keep_n,
                         int64_t *out3, int64_t *bad_pos, void *ws,
                         size_t ws_bytes, void *stream);

/* ------------------------------------------------------- batched pairs */

/* Batched longest_overlap over P independent pairs (BASELINE config C4):
 * equals [longest_overlap(A_p, B_p) for p] (overlap.py:110-152, the
 * reference's per-pair entry point mapped over the batch).
 * seqs: device ASCII of all pairs; offs_host: HOST int64[2P+1], pair p is
 * A = seqs[offs[2p], offs[2p+1]), B = seqs[offs[2p+1], offs[2p+2]).
 * out: device int64[3P] (length, pos_a, pos_b per pair); *bad (device int64)
 * receives the smallest seqs offset of an illegal residue (INT64_MAX if
 * none; pairs with an empty side are not validated, like the reference).
 * Every pair with |A|+|B|+1 <= 20480 runs its whole DC3 + LCP + overlap scan
 * in one CTA's shared memory (csrc/pairdc3.cu); longer pairs and pairs over
 * the on-chip work bounds go through the wave-global DC3 (one generalized
 * text per wave of <= 2^24 residues).  No limit on the call's total size.
 * The call synchronizes the stream once (the fallback count). */
SAIX_API size_t saix_overlap_batch_workspace_bytes(const int64_t *offs_host, int64_t npairs);
SAIX_API int saix_overlap_batch(const uint8_t *seqs, const int64_t *offs_host, int64_t npairs,
                                int keep_n, int64_t *out, int64_t *bad, void *ws,
                                size_t ws_bytes, void *stream);
/* The same with the offsets also resident on the device (offs_dev, equal to
 * offs_host): no H2D inside the call, so it can run while bulk host-to-device
 * copies are in flight on the copy engine (chunked e2e pipelines). */
SAIX_API int saix_overlap_batch_dev(const uint8_t *seqs, const int64_t *offs_host,
                                    const int64_t *offs_dev, int64_t npairs, int keep_n,
                                    int64_t *out, int64_t *bad, void *ws, size_t ws_bytes,
                                    void *stream);

/* saix_overlap_batch over a batch still on the host: one kernel launch over
 * all pairs while the copy engine streams seqs_host (pinned) into seqs_dev on
 * copy_stream (cudaStreamNonBlocking, != stream) in nchunks chunks, each
 * followed by a 4-byte count the kernel's CTAs wait on before taking a pair
 * of that chunk -- the H2D overlaps the pairs without a launch per chunk.
 * Results and errors as saix_overlap_batch_dev; the caller keeps seqs_host
 * alive and unmodified until the call returns (it synchronises stream). */
SAIX_API int saix_overlap_batch_stream(const uint8_t *seqs_dev, const uint8_t *seqs_host,
                                       const int64_t *offs_host, const int64_t *offs_dev, int64_t npairs,
                                       int nchunks, int keep_n, int64_t *out, int64_t *bad, void *ws,
                                       size_t ws_bytes, void *stream, void *copy_stream);
/* 0: route every pair through the wave-global path (A/B and tests); returns
 * the previous setting. */
SAIX_API int saix_overlap_batch_set_onchip(int on);
/* Pairs of this thread's last saix_overlap_batch call that took the
 * wave-global path. */
SAIX_API int64_t saix_overlap_batch_last_fallbacks(void);
/* Diagnostics: per-phase SM cycles of the last call with SAIX_PD_CLOCKS=1. */
SAIX_API int saix_overlap_batch_phase_clocks(int64_t *out, int max_phases);

/* ------------------------------------------------ Cartesian tree / ±1 RMQ */
/* build_cartesian + euler_tour (rmq.py:91-152) on the device: parent, left,
 * right (-1 = none), the 2n-1 tour nodes / depths and first_visit (int32),
 * *root_host = the leftmost minimum.  values: n entries of value_bytes 4
 * (u32) or 8 (int64), n < 2^30. */
SAIX_API size_t saix_cartesian_workspace_bytes(int64_t n);
SAIX_API int saix_cartesian_build(const void *values, int value_bytes, int64_t n, int32_t *parent,
             int32_t *left, int32_t *right, int32_t *tour_nodes, int32_t *tour_depths,
             int32_t *first_visit, int64_t *root_host, void *ws, size_t ws_bytes, void *stream);

/* PlusMinusOneRmq.__init__ (rmq.py:167-197) minus the block-minimum sparse
 * table (built with saix_sparse_build over bmin): block size b (1..16),
 * nblocks = ceil(m/b) leftmost argmins / minima / step codes, the in-block
 * tables tab[code][i][j] (u8, 2^(b-1) codes) of the codes present; present
 * (one flag byte per code) holds round_up(2^(b-1), 4) + 4 bytes; *bad_host =
 * 1 on a non-unit step. */
SAIX_API int saix_pm1_build(const int32_t *depths, int64_t m, int b, int32_t *bargmin, int32_t *bmin,
             int32_t *types, uint8_t *present, uint8_t *tab, int32_t *bad_host, void *stream);

/* PlusMinusOneRmq.query / CartesianRmq.query (rmq.py:219-251), batched in two
 * halves around a saix_sparse_query over the block minima:
 * begin -> (mid_lo, mid_hi) block ranges ((0, 0) when unused) and three ints
 * per query in cand (left candidate, right candidate or -1, has-middle);
 * saix_sparse_query(mid_lo, mid_hi) -> mid_blk; end -> out[t] (tour
 * position, or the node when `nodes` is given; `first` maps array positions
 * to tour positions). */
SAIX_API int saix_pm1_query_begin(int b, const int32_t *types, const uint8_t *tab, const int32_t *first,
             const int64_t *qi, const int64_t *qj, int64_t q, int64_t *mid_lo, int64_t *mid_hi,
             int32_t *cand, void *stream);
SAIX_API int saix_pm1_query_end(const int32_t *depths, int b, const int32_t *bargmin,
             const int64_t *mid_blk, const int32_t *cand, const int32_t *nodes, int64_t q,
             int64_t *out, void *stream);

/* ------------------------------------------------------------ FASTA ingest */
/* parse_fasta (sequence.py:77-125) + encode (sequence.py:144-157) over raw
 * FASTA bytes in device memory (inputs < 4 GiB), with the reference's
 * semantics for a str source: lines end at '\n', each line str.strip()-ed,
 * blank lines skipped, '>' lines open records (header stripped again),
 * sequence lines upper-cased and validated against ACGT (+N when keep_n).
 * Three calls: saix_fasta_lines (line count, sizes the workspace),
 * saix_fasta_scan (line table + counts; the workspace carries it), and
 * saix_fasta_emit (residues, record starts, header texts, first error). */
SAIX_API int saix_fasta_lines(const uint8_t *data, int64_t nbytes, int64_t *lines_host, void *ws,
             size_t ws_bytes, void *stream);
SAIX_API size_t saix_fasta_workspace_bytes(int64_t nbytes, int64_t lines);
SAIX_API int saix_fasta_scan(const uint8_t *data, int64_t nbytes, int64_t lines, int64_t *counts_host,
             void *ws, size_t ws_bytes, void *stream);
SAIX_API int saix_fasta_emit(const uint8_t *data, int64_t nbytes, int64_t lines, int keep_n, int as_ranks,
             uint8_t *res, uint32_t *rec_start, uint8_t *hdr, uint32_t *hdr_off, int64_t *err_host,
             void *ws, size_t ws_bytes, void *stream);

/* ------------------------------------------------------ .saix index files */
/* save_index / load_index (index_store.py:65-134) fed from device buffers.
 * Layout (index_store.py:1-14): "SAIX1\0\0\0", u64 version=1, flags, n,
 * sigma; text (n rank bytes); sa (n x u64); lcp (n x u64); u64 zlib crc32 of
 * everything above. All integers little-endian. */

SAIX_API size_t saix_crc32_workspace_bytes(int64_t nbytes);

/* zlib.crc32(data[0:nbytes]) of a device buffer into *crc_out (device). */
SAIX_API int saix_crc32(const void *data, int64_t nbytes, uint32_t *crc_out,
             void *ws, size_t ws_bytes, void *stream);

/* Size of a .saix file for n positions: 40 + 17n + 8. */
SAIX_API int64_t saix_index_bytes(int64_t n);

/* Writes the whole file image (saix_index_bytes(n) bytes) into device `out`
 * (16-byte aligned) from device text ranks / SA / LCP (sigma <= 255; ws >=
 * saix_crc32_workspace_bytes(0)); the CRC is computed as the image is written. */
SAIX_API int saix_index_pack(const uint8_t *text, const uint32_t *sa, const uint32_t *lcp,
             int64_t n, int64_t sigma, int64_t flags, uint8_t *out,
             void *ws, size_t ws_bytes, void *stream);

/* Verifies the CRC of a device file image whose header (magic, version,
 * length) the caller has checked; then unpacks text, sa, lcp and the ISA
 * (isa[sa[i]] = i). SAIX_EINVAL with "checksum mismatch" on a bad CRC, or
 * "out of range" if an SA/LCP entry does not fit. */
SAIX_API size_t saix_index_unpack_workspace_bytes(int64_t n);
SAIX_API int saix_index_unpack(const uint8_t *blob, int64_t n, uint8_t *text, uint32_t *sa,
             uint32_t *lcp, uint32_t *isa, void *ws, size_t ws_bytes, void *stream);

#ifdef __cplusplus
}
#endif

#endif /* SAIX_B200_H */
