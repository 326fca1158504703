"""paper_1404_3448_b200 -- B200-native (sm_100a) longest-overlap hot path of
arXiv 1404.3448, drop-in for the reference ``saix`` package's suffix-array /
LCP / RMQ / longest-overlap entry points (saix/__init__.py:9-46).

Compute runs in libsaix_b200.so (hand-written CUDA, C ABI in
include/saix_b200.h); PyTorch provides device memory and streams only.
"""

from .fasta import FastaIngest, ingest_fasta
from .index_store import (BadMagicError, ChecksumError, IndexFileError, TruncatedFileError,
                          UnsupportedVersionError, load_index, save_index)
from .overlap import (GeneralizedText, LcpQueryEngine, OverlapBatch, OverlapPipeline, OverlapResult,
                      lcp_query, lcp_query_batch, longest_overlap, longest_overlap_batch,
                      overlap_report, pack_pairs, parse_overlap_record)
from .parallel_sort import (ChunkPlan, SortConfig, SplitState, chunked_sort, exclusive_scan,
                            parallel_build_sa, plan_chunks, radix_sort, split_by_bit)
from .rmq import (CartesianRmq, CartesianTree, EulerTour, PlusMinusOneRmq, SparseTable, build_cartesian,
                  build_pm1, build_sparse, euler_tour, query_pm1, query_sparse, query_sparse_batch, rmq_via_lca)
from .sequence import (DnaSequence, NPolicy, RankedText, SequenceError, decode, encode,
                       gen_random, parse_fasta, write_fasta)
from .suffix_index import (Dc3Workspace, LcpArray, SuffixArray, build_lcp, build_sa_dc3,
                           build_sa_oracle, merge_sample_nonsample, prepare_dc3_workspace,
                           sample_ranks)

__version__ = "0.1.0"

__all__ = [
    "BadMagicError", "ChecksumError", "IndexFileError", "TruncatedFileError", "UnsupportedVersionError",
    "load_index", "save_index", "FastaIngest", "ingest_fasta",
    "CartesianRmq", "CartesianTree", "EulerTour", "PlusMinusOneRmq", "build_cartesian", "build_pm1",
    "euler_tour", "query_pm1", "rmq_via_lca",
    "ChunkPlan", "SortConfig", "SplitState", "chunked_sort", "exclusive_scan", "parallel_build_sa",
    "plan_chunks", "radix_sort", "split_by_bit",
    "Dc3Workspace", "DnaSequence", "GeneralizedText", "LcpArray", "LcpQueryEngine",
    "NPolicy", "OverlapBatch", "OverlapPipeline", "OverlapResult", "RankedText", "SequenceError",
    "SparseTable", "SuffixArray", "build_lcp", "build_sa_dc3", "build_sa_oracle",
    "build_sparse", "decode", "encode", "gen_random", "lcp_query", "lcp_query_batch",
    "longest_overlap", "longest_overlap_batch", "merge_sample_nonsample", "pack_pairs", "overlap_report", "parse_fasta",
    "parse_overlap_record", "prepare_dc3_workspace", "query_sparse", "query_sparse_batch",
    "sample_ranks", "write_fasta",
]
