"""Generate golden vectors by running the REFERENCE saix package itself.

Run in the dev container (the reference exists only there):

    cd /tmp && PYTHONDONTWRITEBYTECODE=1 NUMBA_CACHE_DIR=/tmp/numba_cache \
        python /root/repo/tests/golden/make_golden.py

It imports the reference from /root/reference/pkg/src (read-only; numba's
cache is redirected to /tmp so nothing is written into the reference tree) and
writes tests/golden/reference_vectors.npz.  The tests pin the C oracle
(oracle/) against these vectors and the CUDA path against both.
"""

from __future__ import annotations

import hashlib
import os
import random
import sys

import numpy as np

REF = "/root/reference/pkg/src"
OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "reference_vectors.npz")

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
sys.dont_write_bytecode = True
sys.path.insert(0, REF)

import saix  # noqa: E402
from saix import rmq, suffix_index as si  # noqa: E402
from saix.overlap import LcpQueryEngine, lcp_query, longest_overlap  # noqa: E402
from saix.sequence import DnaSequence, RankedText, encode, gen_random  # noqa: E402


def random_dna(rng: random.Random, n: int) -> str:
    return "".join(rng.choice("ACGT") for _ in range(n))


def pack(chunks, dtype):
    offs = np.zeros(len(chunks) + 1, np.int64)
    offs[1:] = np.cumsum([len(c) for c in chunks])
    flat = np.concatenate([np.asarray(c, dtype) for c in chunks]) if chunks else np.zeros(0, dtype)
    return flat, offs


def sha(arr) -> str:
    return hashlib.sha256(np.ascontiguousarray(arr, np.int64).tobytes()).hexdigest()


def main():
    out = {}

    # --- DC3 / LCP / level-0 probes over seeded random DNA + edge cases ----
    rng = random.Random(1404_3448)
    texts = ["", "A", "AC", "ATTGCTAC", "AAAA", "A" * 17, "A" * 200, "ACGT" * 64,
             "ACGTACG", "TTTTTTTTTT" * 7 + "A"]
    for _ in range(220):
        texts.append(random_dna(rng, rng.randrange(0, 2000)))
    for n in (1000, 3000, 9999):                      # gen_random (PCG64) inputs
        texts.append(gen_random(n, n + 7).residues)
    ranks, sa, rank, lcp, depth = [], [], [], [], []
    tt, srank, ssamp, snon = [], [], [], []
    for s in texts:
        t = encode(DnaSequence("t", s))
        ix = si.build_sa_dc3(t)
        ranks.append(t.ranks)
        sa.append(ix.sa)
        rank.append(ix.rank)
        lcp.append(si.build_lcp(t, ix).lcp)
        ws = si.prepare_dc3_workspace(t)
        depth.append(ws.depth)
        tt.append(ws.triple_text)
        srank.append(ws.sample_rank)
        ssamp.append(ws.sorted_samples)
        snon.append(ws.sorted_nonsamples)
    out["dna_ranks"], out["dna_offs"] = pack(ranks, np.uint8)
    out["dna_sa"], _ = pack(sa, np.int32)
    out["dna_rank"], _ = pack(rank, np.int32)
    out["dna_lcp"], _ = pack(lcp, np.int32)
    out["dna_depth"] = np.asarray(depth, np.int32)
    out["dna_triple_text"], out["dna_triple_offs"] = pack(tt, np.int32)
    out["dna_sample_rank"], out["dna_sample_rank_offs"] = pack(srank, np.int32)
    out["dna_sorted_samples"], out["dna_sorted_samples_offs"] = pack(ssamp, np.int32)
    out["dna_sorted_nonsamples"], out["dna_sorted_nonsamples_offs"] = pack(snon, np.int32)

    # --- wide alphabets (test_suffix_index.py:84-105 style) -----------------
    wr = np.random.default_rng(3)
    wide, wide_sa, wide_sigma = [], [], []
    for _ in range(40):
        n = int(wr.integers(2, 400))
        sigma = int(wr.choice([7, 300, 70000, 2 ** 22]))
        r = wr.integers(1, sigma + 1, size=n)
        t = RankedText(ranks=r, sigma=sigma)
        wide.append(r)
        wide_sa.append(si.build_sa_dc3(t).sa)
        wide_sigma.append(sigma)
    out["wide_ranks"], out["wide_offs"] = pack(wide, np.int64)
    out["wide_sa"], _ = pack(wide_sa, np.int32)
    out["wide_sigma"] = np.asarray(wide_sigma, np.int64)

    # --- sparse table: values, queries, answers (rmq.py:30-58) --------------
    qr = random.Random(8)
    sv, sq_i, sq_j, sq_ans, sq_vo, sq_qo = [], [], [], [], [0], [0]
    for case in range(60):
        n = qr.randrange(1, 300) if case < 50 else qr.randrange(1000, 20000)
        lo, hi = (-5, 6) if case % 3 == 0 else (0, 40)
        vals = [qr.randrange(lo, hi) for _ in range(n)]
        st = rmq.SparseTable(vals)
        qs = [(qr.randrange(n), qr.randrange(n)) for _ in range(400)]
        sv.append(vals)
        sq_i += [a for a, _ in qs]
        sq_j += [b for _, b in qs]
        sq_ans += [st.query(a, b) for a, b in qs]
        sq_vo.append(sq_vo[-1] + n)
        sq_qo.append(sq_qo[-1] + len(qs))
    out["rmq_values"] = np.concatenate([np.asarray(v, np.int64) for v in sv])
    out["rmq_voffs"] = np.asarray(sq_vo, np.int64)
    out["rmq_qi"] = np.asarray(sq_i, np.int64)
    out["rmq_qj"] = np.asarray(sq_j, np.int64)
    out["rmq_ans"] = np.asarray(sq_ans, np.int64)
    out["rmq_qoffs"] = np.asarray(sq_qo, np.int64)

    # --- lcp_query (overlap.py:58-69) ---------------------------------------
    lr = random.Random(9)
    lq_text, lq_i, lq_j, lq_ans, lq_qo = [], [], [], [], [0]
    for _ in range(30):
        s = random_dna(lr, lr.randrange(1, 1500))
        eng = LcpQueryEngine.build(encode(DnaSequence("t", s)))
        qs = [(lr.randrange(len(s)), lr.randrange(len(s))) for _ in range(200)]
        lq_text.append(encode(DnaSequence("t", s)).ranks)
        lq_i += [a for a, _ in qs]
        lq_j += [b for _, b in qs]
        lq_ans += [lcp_query(eng, a, b) for a, b in qs]
        lq_qo.append(lq_qo[-1] + len(qs))
    out["lcpq_ranks"], out["lcpq_offs"] = pack(lq_text, np.uint8)
    out["lcpq_qi"] = np.asarray(lq_i, np.int64)
    out["lcpq_qj"] = np.asarray(lq_j, np.int64)
    out["lcpq_ans"] = np.asarray(lq_ans, np.int64)
    out["lcpq_qoffs"] = np.asarray(lq_qo, np.int64)

    # --- longest_overlap (overlap.py:110-152) -------------------------------
    orr = random.Random(10)
    pairs = [("ATTGCTAC", "GCTA"), ("AAAA", "TTTT"), ("", "GCTA"), ("ATTGCTAC", ""),
             ("A", "A"), ("AAAA", "AAAA"), ("ACGT" * 30, "CGTA" * 30)]
    for _ in range(240):
        a = random_dna(orr, orr.randrange(0, 300))
        b = random_dna(orr, orr.randrange(0, 300))
        if orr.random() < 0.3:
            blk = random_dna(orr, orr.randrange(1, 60))
            a = a[: len(a) // 2] + blk + a[len(a) // 2:]
            b = b[: len(b) // 3] + blk + b[len(b) // 3:]
        pairs.append((a, b))
    res = []
    for a, b in pairs:
        r = longest_overlap(DnaSequence("a", a), DnaSequence("b", b))
        res.append((r.length, r.pos_a, r.pos_b))
    ov_a, ov_ao = pack([np.frombuffer(a.encode(), np.uint8) for a, _ in pairs], np.uint8)
    ov_b, ov_bo = pack([np.frombuffer(b.encode(), np.uint8) for _, b in pairs], np.uint8)
    out["ov_a"], out["ov_aoffs"], out["ov_b"], out["ov_boffs"] = ov_a, ov_ao, ov_b, ov_bo
    out["ov_ans"] = np.asarray(res, np.int64)

    # --- C1: two 100 kbp random sequences (BASELINE.json configs[0]) --------
    a = gen_random(100_000, 1)
    b = gen_random(100_000, 2)
    r = longest_overlap(a, b)
    out["c1_ans"] = np.asarray([r.length, r.pos_a, r.pos_b], np.int64)
    gen = saix.GeneralizedText.build(a, b).to_ranked_text()
    ix = si.build_sa_dc3(gen)
    c1_lcp = si.build_lcp(gen, ix).lcp
    out["c1_sa_sha256"] = np.frombuffer(sha(ix.sa).encode(), np.uint8)
    out["c1_lcp_sha256"] = np.frombuffer(sha(c1_lcp).encode(), np.uint8)
    out["c1_seq_sha256"] = np.frombuffer(
        hashlib.sha256((a.residues + "|" + b.residues).encode()).hexdigest().encode(), np.uint8)

    np.savez_compressed(OUT, **out)
    print("wrote", OUT, os.path.getsize(OUT), "bytes")


if __name__ == "__main__":
    main()
