"""One small pass over every kernel family, checked against the C oracle --
the workload compute-sanitizer (memcheck / racecheck / synccheck) runs in
tools/gpu_check.sh `sanitize`.

    SAIX_WS_MIN_M=4096 compute-sanitizer --tool racecheck python tools/sanitize_run.py

SAIX_WS_MIN_M lowers the DNA window sort's sample threshold so its kernels
(csrc/wsort.cuh) run on a text small enough for racecheck."""
import io
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import oracle  # noqa: E402
import paper_1404_3448_b200 as sx  # noqa: E402
from paper_1404_3448_b200 import _lib  # noqa: E402
from paper_1404_3448_b200.sequence import RankedText, encode, gen_random  # noqa: E402
from paper_1404_3448_b200.workloads import c4_pairs  # noqa: E402


def step(name, ok):
    print(f"{name:28s} {'ok' if ok else 'MISMATCH'}", flush=True)
    if not ok:
        raise SystemExit(f"sanitize_run: {name} differs from the oracle")


def main():
    n = int(os.environ.get("SAIX_SAN_N", "30000"))
    # end-to-end pair (encode GSA, DC3, direct LCP, overlap scan)
    a, b = gen_random(n // 2, 1), gen_random(n // 2, 2)
    r = sx.longest_overlap(a, b)
    step("longest_overlap", (r.length, r.pos_a, r.pos_b) == oracle.longest_overlap(a.residues, b.residues))
    # DC3 on DNA (window naming: wsort when SAIX_WS_MIN_M allows) + LCP
    t = encode(gen_random(n, 3))
    ix = sx.build_sa_dc3(t)
    sa, rank = oracle.dc3(t.ranks, 4)
    step(f"build_sa_dc3 (naming {_lib.dc3_naming()})", np.array_equal(ix.sa, sa))
    lcp = sx.build_lcp(t, ix).lcp
    step("build_lcp", np.array_equal(lcp, oracle.lcp(t.ranks, sa, rank)))
    # recursion path (repetitive text) and a wide alphabet
    rep = np.tile(np.array([1, 2, 3, 4, 4, 2, 1], np.uint8), n // 7 + 1)[:n].copy()
    rep[n // 2] = 3
    ix = sx.build_sa_dc3(RankedText(ranks=rep.astype(np.int64), sigma=4))
    step("build_sa_dc3 (recursion)", np.array_equal(ix.sa, oracle.dc3(rep, 4)[0]))
    wide = np.random.default_rng(5).integers(1, 1 << 20, n)
    ix = sx.build_sa_dc3(RankedText(ranks=wide, sigma=1 << 20))
    step("build_sa_dc3 (wide)", np.array_equal(ix.sa, oracle.dc3(wide, 1 << 20)[0]))
    # sparse table + batched queries
    st = sx.SparseTable(lcp)
    qi = np.random.default_rng(7).integers(0, n, 20000)
    qj = np.random.default_rng(8).integers(0, n, 20000)
    step("query_sparse_batch", np.array_equal(sx.query_sparse_batch(st, qi, qj),
                                              oracle.argmin_blocked(lcp, qi, qj)))
    # batched pairs (on-chip pair DC3)
    seqs, offs = c4_pairs(0, 24)
    ob = sx.OverlapBatch(seqs, offs)
    ob.run_device()
    step("OverlapBatch", np.array_equal(ob.results(), oracle.overlap_batch(seqs, offs)))
    # the same kernel gated on a streamed host batch (ramped chunk plan: 1000
    # short pairs in 2 chunks -> 296 + 408 + 296 pairs)
    import torch
    rng = np.random.default_rng(5)
    lens = rng.integers(20, 200, 2000)
    sseqs = np.frombuffer(b"ACGT", np.uint8)[rng.integers(0, 4, int(lens.sum()))]
    soffs = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    sb = sx.OverlapBatch(sseqs, soffs)
    sb.run_from_host(torch.from_numpy(sseqs.copy()).pin_memory(), stream_chunks=2)
    step("OverlapBatch (streamed)", np.array_equal(sb.results(), oracle.overlap_batch(sseqs, soffs)))
    # parallel-sort engine
    keys = np.random.default_rng(9).integers(0, 1 << 31, 50000)
    step("radix_sort", np.array_equal(sx.radix_sort(keys), np.sort(keys, kind="stable")))
    # .saix round trip
    eng = sx.LcpQueryEngine.build(t)
    buf = io.BytesIO()
    sx.save_index(eng, buf)
    back = sx.load_index(io.BytesIO(buf.getvalue()))
    step("save/load_index", np.array_equal(back.sa.sa, eng.sa.sa))
    # FASTA ingest
    fa = b">x\nACGT" + b"ACGTTGCA" * 300 + b"\n>y\nGGCCAATT\n"
    got = sx.ingest_fasta(fa)
    step("ingest_fasta", got is not None)
    # Cartesian / +-1 RMQ
    vals = np.random.default_rng(11).integers(0, 50, 5000)
    cr = sx.CartesianRmq(vals)
    qa = np.random.default_rng(12).integers(0, 5000, 200)
    qb = np.random.default_rng(13).integers(0, 5000, 200)
    want = oracle.argmin_blocked(vals, qa, qb)
    step("CartesianRmq", all(cr.query(int(x), int(y)) == int(w) for x, y, w in zip(qa, qb, want)))
    print("sanitize_run: all steps match", flush=True)


if __name__ == "__main__":
    main()
