"""Pin the C oracle (oracle/) to the reference before trusting it.

Every vector in tests/golden/reference_vectors.npz was produced by running
the reference saix package itself (tests/golden/make_golden.py); the known
answers below are the reference tests' own fixtures
(test_suffix_index.py:11-40,133-134,154-169,203-214; test_rmq.py:20-57;
test_overlap.py:22-26,68-97).
"""

import hashlib
import random

import numpy as np
import pytest

import oracle
from conftest import cases

FIX = "ATTGCTAC"
LUT = {"A": 1, "C": 2, "G": 3, "T": 4}


def ranks(s):
    return np.array([LUT[c] for c in s], np.int64)


def naive_sa(r):
    r = list(r)
    return sorted(range(len(r)), key=lambda i: r[i:])


def naive_lcp(r, sa):
    out = [0] * len(sa)
    for k in range(1, len(sa)):
        a, b, h = sa[k - 1], sa[k], 0
        while a + h < len(r) and b + h < len(r) and r[a + h] == r[b + h]:
            h += 1
        out[k] = h
    return out


def lcs_dp(a, b):
    best, pa, pb = 0, 0, 0
    prev = [0] * (len(b) + 1)
    for i in range(1, len(a) + 1):
        cur = [0] * (len(b) + 1)
        for j in range(1, len(b) + 1):
            if a[i - 1] == b[j - 1]:
                cur[j] = prev[j - 1] + 1
                L = cur[j]
                if L > best or (L == best and (i - L, j - L) < (pa, pb)):
                    best, pa, pb = L, i - L, j - L
        prev = cur
    return (best, pa, pb) if best else (0, 0, 0)


class TestKnownAnswers:
    def test_fixture_sa_rank_lcp(self):
        sa, rank = oracle.dc3(ranks(FIX), 4)
        assert sa.tolist() == [6, 0, 7, 4, 3, 5, 2, 1]
        assert (rank + 1).tolist() == [2, 8, 7, 5, 4, 6, 1, 3]
        assert oracle.lcp(ranks(FIX), sa, rank).tolist() == [0, 1, 0, 1, 0, 0, 1, 1]

    def test_fixture_probe(self):
        p = oracle.dc3_probe(ranks(FIX), 4)
        sr = {int(q): int(p["sample_rank"][q]) for q in (1, 2, 4, 5, 7)}
        assert sr == {1: 5, 2: 4, 4: 2, 5: 3, 7: 1}
        assert p["mod1"].tolist() == [1, 4, 7] and p["mod2"].tolist() == [2, 5]
        assert p["sorted_nonsamples"].tolist() == [6, 0, 3]

    def test_degenerate(self):
        assert oracle.dc3(ranks("AAAA"), 4)[0].tolist() == [3, 2, 1, 0]
        sa, rk = oracle.dc3(ranks("AAAA"), 4)
        assert oracle.lcp(ranks("AAAA"), sa, rk).tolist() == [0, 1, 2, 3]
        assert oracle.dc3(ranks("A"), 4)[0].tolist() == [0]
        assert oracle.dc3(ranks(""), 4)[0].tolist() == []
        p = oracle.dc3_probe(ranks("A"), 4)
        assert int(p["sample_rank"][1]) == 1 and p["sorted_samples"].tolist() == []

    def test_rmq_fixtures(self):
        row = [0, 1, 0, 1, 0, 0, 1, 1]
        t = oracle.sparse_build(row)
        assert oracle.sparse_query(row, t, [1, 4, 7], [7, 6, 1]).tolist() == [2, 4, 2]
        tie = [2, 1, 1, 1, 2]
        assert oracle.sparse_query(tie, oracle.sparse_build(tie), [0, 2], [4, 4]).tolist() == [1, 2]
        with pytest.raises(IndexError):
            oracle.sparse_query(row, t, [0], [8])

    def test_overlap_fixtures(self):
        assert oracle.longest_overlap("ATTGCTAC", "GCTA") == (4, 3, 0)
        assert oracle.longest_overlap("AAAA", "TTTT") == (0, 0, 0)
        assert oracle.longest_overlap("", "GCTA") == (0, 0, 0)

    def test_lcp_query_fixture(self):
        r = ranks(FIX)
        sa, rk = oracle.dc3(r, 4)
        lcp = oracle.lcp(r, sa, rk)
        assert oracle.lcp_query(r, sa, rk, lcp, [6, 3], [0, 3]).tolist() == [1, 5]


class TestGoldenVectors:
    def test_dc3_lcp_and_probes(self, golden):
        g = golden
        for c, r in cases(g, "dna_ranks", "dna_offs"):
            r = r.astype(np.int64)
            sl = slice(g["dna_offs"][c], g["dna_offs"][c + 1])
            sa, rank = oracle.dc3(r, 4)
            assert np.array_equal(sa, g["dna_sa"][sl]), c
            assert np.array_equal(rank, g["dna_rank"][sl]), c
            assert np.array_equal(oracle.lcp(r, sa, rank), g["dna_lcp"][sl]), c
            p = oracle.dc3_probe(r, 4)
            for key in ("triple_text", "sample_rank", "sorted_samples", "sorted_nonsamples"):
                offs = g[f"dna_{key}_offs" if key != "triple_text" else "dna_triple_offs"]
                want = g[f"dna_{key}"][offs[c]:offs[c + 1]]
                assert np.array_equal(p[key], want), (c, key)
            assert p["depth"] == int(g["dna_depth"][c]), c

    def test_wide_alphabet(self, golden):
        g = golden
        for c, r in cases(g, "wide_ranks", "wide_offs"):
            sl = slice(g["wide_offs"][c], g["wide_offs"][c + 1])
            assert np.array_equal(oracle.dc3(r, int(g["wide_sigma"][c]))[0], g["wide_sa"][sl])

    def test_sparse_table(self, golden):
        g = golden
        vo, qo = g["rmq_voffs"], g["rmq_qoffs"]
        for c in range(len(vo) - 1):
            v = g["rmq_values"][vo[c]:vo[c + 1]]
            qi, qj = g["rmq_qi"][qo[c]:qo[c + 1]], g["rmq_qj"][qo[c]:qo[c + 1]]
            want = g["rmq_ans"][qo[c]:qo[c + 1]]
            assert np.array_equal(oracle.sparse_query(v, oracle.sparse_build(v), qi, qj), want)
            assert np.array_equal(oracle.argmin_blocked(v, qi, qj), want)

    def test_lcp_query(self, golden):
        g = golden
        qo = g["lcpq_qoffs"]
        for c, r in cases(g, "lcpq_ranks", "lcpq_offs"):
            r = r.astype(np.int64)
            sa, rk = oracle.dc3(r, 4)
            lcp = oracle.lcp(r, sa, rk)
            got = oracle.lcp_query(r, sa, rk, lcp, g["lcpq_qi"][qo[c]:qo[c + 1]],
                                   g["lcpq_qj"][qo[c]:qo[c + 1]])
            assert np.array_equal(got, g["lcpq_ans"][qo[c]:qo[c + 1]]), c

    def test_longest_overlap(self, golden):
        g = golden
        ao, bo = g["ov_aoffs"], g["ov_boffs"]
        for c in range(len(ao) - 1):
            a = g["ov_a"][ao[c]:ao[c + 1]].tobytes()
            b = g["ov_b"][bo[c]:bo[c + 1]].tobytes()
            assert oracle.longest_overlap(a, b) == tuple(int(x) for x in g["ov_ans"][c]), c

    def test_c1_config(self, golden):
        """BASELINE configs[0]: 2 x 100 kbp, answer and SA/LCP hashes."""
        from paper_1404_3448_b200.sequence import gen_random
        a, b = gen_random(100_000, 1), gen_random(100_000, 2)
        seq_hash = hashlib.sha256((a.residues + "|" + b.residues).encode()).hexdigest()
        assert seq_hash == golden["c1_seq_sha256"].tobytes().decode()
        assert oracle.longest_overlap(a.residues, b.residues) == tuple(int(x) for x in golden["c1_ans"])
        lut = np.zeros(256, np.int64)
        for k, ch in enumerate("ACGT", 2):
            lut[ord(ch)] = k
        gsa = np.concatenate([lut[np.frombuffer(a.residues.encode(), np.uint8)], [1],
                              lut[np.frombuffer(b.residues.encode(), np.uint8)]])
        sa, rank = oracle.dc3(gsa, 5)
        lcp = oracle.lcp(gsa, sa, rank)
        assert hashlib.sha256(sa.tobytes()).hexdigest() == golden["c1_sa_sha256"].tobytes().decode()
        assert hashlib.sha256(lcp.tobytes()).hexdigest() == golden["c1_lcp_sha256"].tobytes().decode()


class TestAgainstBruteForce:
    def test_exhaustive_short_texts(self):
        for k in range(1, 7):
            for code in range(4 ** k):
                r = [(code // 4 ** p) % 4 + 1 for p in range(k)]
                sa, rank = oracle.dc3(r, 4)
                want = naive_sa(r)
                assert sa.tolist() == want, r
                assert oracle.lcp(r, sa, rank).tolist() == naive_lcp(r, want), r

    def test_random_overlap_vs_dp(self):
        rng = random.Random(10)
        for _ in range(150):
            a = "".join(rng.choice("ACGT") for _ in range(rng.randrange(0, 80)))
            b = "".join(rng.choice("ACGT") for _ in range(rng.randrange(0, 80)))
            assert oracle.longest_overlap(a, b) == lcs_dp(a, b), (a, b)

    def test_batch_threads_equal_serial(self):
        rng = random.Random(3)
        seqs, offs = [], [0]
        pairs = []
        for _ in range(40):
            a = "".join(rng.choice("ACGT") for _ in range(rng.randrange(1, 200)))
            b = "".join(rng.choice("ACGT") for _ in range(rng.randrange(1, 200)))
            pairs.append((a, b))
            for s in (a, b):
                seqs.append(s)
                offs.append(offs[-1] + len(s))
        buf = np.frombuffer("".join(seqs).encode(), np.uint8)
        got = oracle.overlap_batch(buf, offs, threads=4)
        assert [tuple(x) for x in got.tolist()] == [oracle.longest_overlap(a, b) for a, b in pairs]
