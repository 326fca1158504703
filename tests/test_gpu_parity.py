"""Parity of the CUDA path (through the C ABI) against the reference's golden
vectors and the pinned C oracle.  Bit-exact: every array and answer is
integer/index data, so equality is the only tolerance."""

import hashlib
import random

import numpy as np
import pytest

import oracle
import paper_1404_3448_b200 as sx
from conftest import cases
from paper_1404_3448_b200.sequence import DnaSequence, RankedText, encode, gen_random

pytestmark = pytest.mark.gpu

FIX = "ATTGCTAC"
FIX_SA = [6, 0, 7, 4, 3, 5, 2, 1]


def text_of(s):
    return encode(DnaSequence("t", s))


def rdna(rng, n):
    return "".join(rng.choice("ACGT") for _ in range(n))


# ------------------------------------------------------------------ DC3

class TestDc3:
    def test_fixture(self):
        sa = sx.build_sa_dc3(text_of(FIX))
        assert sa.sa.tolist() == FIX_SA
        assert (sa.rank + 1).tolist() == [2, 8, 7, 5, 4, 6, 1, 3]
        assert sa.sa.dtype == np.int64 and not sa.sa.flags.writeable

    def test_degenerate(self):
        assert sx.build_sa_dc3(text_of("")).sa.tolist() == []
        assert sx.build_sa_dc3(text_of("A")).sa.tolist() == [0]
        assert sx.build_sa_dc3(text_of("AAAA")).sa.tolist() == [3, 2, 1, 0]
        assert sx.build_sa_dc3(text_of("AC")).sa.tolist() == [0, 1]

    def test_golden_vectors(self, golden):
        g = golden
        for c, r in cases(g, "dna_ranks", "dna_offs"):
            sl = slice(g["dna_offs"][c], g["dna_offs"][c + 1])
            t = RankedText(r.astype(np.int64), 4)
            ix = sx.build_sa_dc3(t)
            assert np.array_equal(ix.sa, g["dna_sa"][sl]), c
            assert np.array_equal(ix.rank, g["dna_rank"][sl]), c
            assert np.array_equal(sx.build_lcp(t, ix).lcp, g["dna_lcp"][sl]), c

    def test_golden_probes(self, golden):
        """Level-0 introspection (prepare_dc3_workspace, suffix_index.py:
        425-449) on every golden text."""
        g = golden
        for c, r in cases(g, "dna_ranks", "dna_offs"):
            t = RankedText(r.astype(np.int64), 4)
            ws = sx.prepare_dc3_workspace(t)
            for key, offk in (("triple_text", "dna_triple_offs"),
                              ("sample_rank", "dna_sample_rank_offs"),
                              ("sorted_samples", "dna_sorted_samples_offs"),
                              ("sorted_nonsamples", "dna_sorted_nonsamples_offs")):
                o = g[offk]
                assert np.array_equal(getattr(ws, key), g[f"dna_{key}"][o[c]:o[c + 1]]), (c, key)
            assert ws.depth == int(g["dna_depth"][c]), c
            assert sx.merge_sample_nonsample(ws, t).sa.tolist() == \
                g["dna_sa"][g["dna_offs"][c]:g["dna_offs"][c + 1]].tolist()

    def test_wide_alphabet(self, golden):
        g = golden
        for c, r in cases(g, "wide_ranks", "wide_offs"):
            sl = slice(g["wide_offs"][c], g["wide_offs"][c + 1])
            t = RankedText(r, int(g["wide_sigma"][c]))
            assert np.array_equal(sx.build_sa_dc3(t).sa, g["wide_sa"][sl]), c

    def test_sample_ranks_fixtures(self):
        assert sx.sample_ranks(text_of(FIX)) == {1: 5, 2: 4, 4: 2, 5: 3, 7: 1}
        assert sx.sample_ranks(text_of("A")) == {1: 1}
        got = sx.sample_ranks(text_of("AAAA"))
        assert got[1] > got[2] > got[4]

    def test_workspace_fixture(self):
        ws = sx.prepare_dc3_workspace(text_of(FIX))
        assert ws.mod1.tolist() == [1, 4, 7] and ws.mod2.tolist() == [2, 5]
        assert ws.nonsample.tolist() == [0, 3, 6]
        assert ws.sorted_nonsamples.tolist() == [6, 0, 3]
        assert sx.merge_sample_nonsample(ws, text_of(FIX)).sa.tolist() == FIX_SA
        one = sx.prepare_dc3_workspace(text_of("A"))
        assert one.sorted_samples.tolist() == []
        assert sx.merge_sample_nonsample(one, text_of("A")).sa.tolist() == [0]

    def test_exhaustive_short(self):
        for k in range(1, 7):
            for code in range(4 ** k):
                r = np.array([(code // 4 ** p) % 4 + 1 for p in range(k)], np.int64)
                got = sx.build_sa_dc3(RankedText(r, 4))
                want_sa, _ = oracle.dc3(r, 4)
                assert np.array_equal(got.sa, want_sa), r

    def test_random_corpus_vs_oracle(self):
        rng = random.Random(20240601)
        for _ in range(120):
            n = rng.randrange(1, 10_001)
            t = encode(gen_random(n, rng.randrange(1 << 62)))
            ix = sx.build_sa_dc3(t)
            sa, rank = oracle.dc3(t.ranks, 4)
            assert np.array_equal(ix.sa, sa) and np.array_equal(ix.rank, rank), n
            assert np.array_equal(sx.build_lcp(t, ix).lcp, oracle.lcp(t.ranks, sa, rank)), n

    @pytest.mark.parametrize("s", ["A" * 5000, "AC" * 3000, "ACGT" * 2000, "AAAAT" * 1500,
                                   "A" * 3000 + "C" + "A" * 3000])
    def test_repetitive(self, s):
        t = text_of(s)
        ix = sx.build_sa_dc3(t)
        sa, rank = oracle.dc3(t.ranks, 4)
        assert np.array_equal(ix.sa, sa)
        assert np.array_equal(sx.build_lcp(t, ix).lcp, oracle.lcp(t.ranks, sa, rank))

    def test_recursion_depth_bounded(self):
        import math
        for s in ["A" * 200, "ACGT" * 64, rdna(random.Random(3), 3000)]:
            ws = sx.prepare_dc3_workspace(text_of(s))
            assert ws.depth <= math.ceil(math.log(max(len(s), 2), 1.5)) + 1
            assert ws.depth == oracle.dc3_probe(text_of(s).ranks, 4)["depth"]

    def test_lcp_from_uploaded_suffix_array(self):
        t = text_of(rdna(random.Random(4), 1500))
        sa, rank = oracle.dc3(t.ranks, 4)
        host_sa = sx.SuffixArray.from_order(sa)     # no device copy attached
        assert np.array_equal(sx.build_lcp(t, host_sa).lcp, oracle.lcp(t.ranks, sa, rank))


# ------------------------------------------------------------------ RMQ

class TestSparseTable:
    ROW = [0, 1, 0, 1, 0, 0, 1, 1]

    def test_fixtures(self):
        st = sx.SparseTable(self.ROW)
        assert st.query(1, 7) == 2 and st.query(4, 6) == 4 and st.query(7, 1) == 2
        assert sx.SparseTable([5]).query(0, 0) == 0
        tie = sx.SparseTable([2, 1, 1, 1, 2])
        assert tie.query(0, 4) == 1 and tie.query(2, 4) == 2
        with pytest.raises(IndexError):
            st.query(0, 8)
        with pytest.raises(IndexError):
            st.query(-1, 3)
        with pytest.raises(ValueError):
            sx.SparseTable([])

    def test_golden(self, golden):
        g = golden
        vo, qo = g["rmq_voffs"], g["rmq_qoffs"]
        for c in range(len(vo) - 1):
            v = g["rmq_values"][vo[c]:vo[c + 1]]
            st = sx.SparseTable(v)
            got = st.query_batch(g["rmq_qi"][qo[c]:qo[c + 1]], g["rmq_qj"][qo[c]:qo[c + 1]])
            assert np.array_equal(got, g["rmq_ans"][qo[c]:qo[c + 1]]), c
            if c < 20:
                flat = np.concatenate(st.table)
                assert np.array_equal(flat, oracle.sparse_build(v)), c

    def test_exhaustive_small(self):
        rng = random.Random(8)
        for _ in range(60):
            n = rng.randrange(1, 65)
            vals = [rng.randrange(0, 10) for _ in range(n)]
            st = sx.SparseTable(vals)
            ii, jj = np.meshgrid(np.arange(n), np.arange(n), indexing="ij")
            got = st.query_batch(ii.ravel(), jj.ravel())
            assert np.array_equal(got, oracle.argmin_blocked(vals, ii.ravel(), jj.ravel()))

    @pytest.mark.parametrize("lo,hi", [(0, 40), (-(1 << 40), 1 << 40), (-(1 << 62), 1 << 62)])
    def test_all_layouts(self, lo, hi):
        rng = np.random.default_rng(5)
        v = rng.integers(lo, hi, size=20_000)
        qi, qj = rng.integers(0, v.shape[0], size=(2, 20_000))
        assert np.array_equal(sx.SparseTable(v).query_batch(qi, qj), oracle.argmin_blocked(v, qi, qj))

    def test_batch_bounds(self):
        st = sx.SparseTable(self.ROW)
        with pytest.raises(IndexError):
            st.query_batch([0, 1], [3, 99])


class TestLcpQuery:
    def test_fixtures(self):
        eng = sx.LcpQueryEngine.build(text_of(FIX))
        assert sx.lcp_query(eng, 6, 0) == 1 and sx.lcp_query(eng, 3, 3) == 5
        with pytest.raises(IndexError):
            sx.lcp_query(sx.LcpQueryEngine.build(text_of("ACGT")), 0, 4)
        with pytest.raises(ValueError):
            sx.LcpQueryEngine.build(text_of("ACGT"), rmq_kind="nope")

    def test_golden(self, golden):
        g = golden
        qo = g["lcpq_qoffs"]
        for c, r in cases(g, "lcpq_ranks", "lcpq_offs"):
            eng = sx.LcpQueryEngine.build(RankedText(r.astype(np.int64), 4))
            got = sx.lcp_query_batch(eng, g["lcpq_qi"][qo[c]:qo[c + 1]], g["lcpq_qj"][qo[c]:qo[c + 1]])
            assert np.array_equal(got, g["lcpq_ans"][qo[c]:qo[c + 1]]), c

    def test_exhaustive_small(self):
        rng = random.Random(9)
        for _ in range(20):
            s = rdna(rng, rng.randrange(1, 60))
            t = text_of(s)
            eng = sx.LcpQueryEngine.build(t, rmq_kind="cartesian")
            ii, jj = np.meshgrid(np.arange(len(s)), np.arange(len(s)), indexing="ij")
            sa, rank = oracle.dc3(t.ranks, 4)
            want = oracle.lcp_query(t.ranks, sa, rank, oracle.lcp(t.ranks, sa, rank), ii.ravel(), jj.ravel())
            assert np.array_equal(sx.lcp_query_batch(eng, ii.ravel(), jj.ravel()), want)


# ------------------------------------------------------------------ overlap

class TestLongestOverlap:
    def test_fixtures(self):
        A, B = DnaSequence("A", FIX), DnaSequence("B", "GCTA")
        assert sx.longest_overlap(A, B) == sx.OverlapResult(4, 3, 0)
        assert sx.longest_overlap(DnaSequence("a", "AAAA"), DnaSequence("b", "TTTT")) == \
            sx.OverlapResult(0, 0, 0)
        assert sx.longest_overlap(DnaSequence("a", ""), B) == sx.OverlapResult(0, 0, 0)
        assert sx.longest_overlap(A, DnaSequence("b", "")) == sx.OverlapResult(0, 0, 0)

    def test_golden(self, golden):
        g = golden
        ao, bo = g["ov_aoffs"], g["ov_boffs"]
        for c in range(len(ao) - 1):
            a = DnaSequence("a", g["ov_a"][ao[c]:ao[c + 1]].tobytes().decode())
            b = DnaSequence("b", g["ov_b"][bo[c]:bo[c + 1]].tobytes().decode())
            r = sx.longest_overlap(a, b)
            assert (r.length, r.pos_a, r.pos_b) == tuple(int(x) for x in g["ov_ans"][c]), c

    def test_residue_errors_match_reference(self):
        with pytest.raises(sx.SequenceError, match="'X' at position 2"):
            sx.longest_overlap(DnaSequence("a", "ACXT"), DnaSequence("b", "ACGT"))
        with pytest.raises(sx.SequenceError, match="record 'b'.*'N' at position 1"):
            sx.longest_overlap(DnaSequence("a", "ACGT"), DnaSequence("b", "ANGT"))
        r = sx.longest_overlap(DnaSequence("a", "ACNNT"), DnaSequence("b", "GNNTA"), sx.NPolicy.KEEP)
        assert r == sx.OverlapResult(3, 2, 1)

    def test_c1_config(self, golden):
        a, b = gen_random(100_000, 1), gen_random(100_000, 2)
        r = sx.longest_overlap(a, b)
        assert (r.length, r.pos_a, r.pos_b) == tuple(int(x) for x in golden["c1_ans"])
        gen = sx.GeneralizedText.build(a, b).to_ranked_text()
        ix = sx.build_sa_dc3(gen)
        lcp = sx.build_lcp(gen, ix).lcp
        assert hashlib.sha256(ix.sa.tobytes()).hexdigest() == golden["c1_sa_sha256"].tobytes().decode()
        assert hashlib.sha256(lcp.tobytes()).hexdigest() == golden["c1_lcp_sha256"].tobytes().decode()

    def test_planted_blocks_vs_oracle(self):
        rng = np.random.default_rng(77)
        for p in range(20):
            a = gen_random(10_000, 2 * p + 100, (0.3, 0.2, 0.2, 0.3)).residues
            b = list(gen_random(10_000, 2 * p + 101, (0.3, 0.2, 0.2, 0.3)).residues)
            L = int(rng.integers(32, 257))
            x, y = rng.integers(0, 10_000 - L, size=2)
            b[y:y + L] = a[x:x + L]
            b = "".join(b)
            r = sx.longest_overlap(DnaSequence("a", a), DnaSequence("b", b))
            assert (r.length, r.pos_a, r.pos_b) == oracle.longest_overlap(a, b)


class TestLargeAlphabets:
    """Bucket-sort naming / mod-0 split (bsort.cuh): small buckets, medium
    (CTA-sorted) buckets and the oversize-bucket fallback."""

    @pytest.mark.parametrize("n,sigma,hot", [(60_000, 5000, 0.0), (60_000, 5000, 0.05),
                                             (60_000, 5000, 0.5), (30_000, 70_000, 0.02)])
    def test_skewed_wide_text_vs_oracle(self, n, sigma, hot):
        rng = np.random.default_rng(n + sigma)
        r = rng.integers(1, sigma + 1, size=n)
        r[rng.random(n) < hot] = 1                      # one hot symbol -> one big bucket
        t = RankedText(r, sigma)
        ix = sx.build_sa_dc3(t)
        sa, rank = oracle.dc3(r, sigma)
        assert np.array_equal(ix.sa, sa) and np.array_equal(ix.rank, rank)
        assert np.array_equal(sx.build_lcp(t, ix).lcp, oracle.lcp(r, sa, rank))


class TestDirectLcp:
    """Word-compare LCP (lcp.cu k_lcp_direct): 2-bit packed and byte texts,
    the capped-entry extension, the separator clamp and the Kasai fallback."""

    @pytest.mark.parametrize("n", [2, 3, 31, 32, 33, 63, 64, 65, 95, 96, 97, 1000, 4097])
    def test_pack_tails(self, n):
        t = encode(gen_random(n, 900 + n))
        ix = sx.build_sa_dc3(t)
        sa, rank = oracle.dc3(t.ranks, 4)
        assert np.array_equal(sx.build_lcp(t, ix).lcp, oracle.lcp(t.ranks, sa, rank))

    @pytest.mark.parametrize("rep", [257, 400, 1500])
    def test_long_repeat_extension(self, rep):
        s = list(gen_random(100_000, 5).residues)
        s[60_000:60_000 + rep] = s[10_000:10_000 + rep]       # capped entries, < n/64 of them
        t = text_of("".join(s))
        ix = sx.build_sa_dc3(t)
        sa, rank = oracle.dc3(t.ranks, 4)
        assert np.array_equal(sx.build_lcp(t, ix).lcp, oracle.lcp(t.ranks, sa, rank))

    @pytest.mark.parametrize("sigma", [5, 20, 255])
    def test_byte_text(self, sigma):
        rng = np.random.default_rng(sigma)
        r = rng.integers(1, sigma + 1, size=50_000)
        r[30_000:30_700] = r[1_000:1_700]
        t = RankedText(r, sigma)
        ix = sx.build_sa_dc3(t)
        sa, rank = oracle.dc3(r, sigma)
        assert np.array_equal(sx.build_lcp(t, ix).lcp, oracle.lcp(r, sa, rank))

    @pytest.mark.parametrize("L", [300, 2000])
    def test_overlap_long_block(self, L):
        a = gen_random(100_000, 11).residues
        b = list(gen_random(100_000, 12).residues)
        b[50_000:50_000 + L] = a[7_000:7_000 + L]
        b = "".join(b)
        r = sx.longest_overlap(DnaSequence("a", a), DnaSequence("b", b))
        assert (r.length, r.pos_a, r.pos_b) == oracle.longest_overlap(a, b)
        assert r.length >= L

    def test_overlap_block_at_separator(self):
        # A ends and B starts with the same block: matches run up to the separator
        blk = gen_random(700, 3).residues
        a = gen_random(5_000, 1).residues + blk
        b = blk + gen_random(5_000, 2).residues
        r = sx.longest_overlap(DnaSequence("a", a), DnaSequence("b", b))
        assert (r.length, r.pos_a, r.pos_b) == oracle.longest_overlap(a, b)

    def test_overlap_keep_n_byte_path(self):
        rng = random.Random(9)
        a = "".join(rng.choice("ACGTN") for _ in range(20_000))
        b = list("".join(rng.choice("ACGTN") for _ in range(20_000)))
        b[9_000:9_500] = a[100:600]
        b = "".join(b)
        r = sx.longest_overlap(DnaSequence("a", a), DnaSequence("b", b), sx.NPolicy.KEEP)
        assert (r.length, r.pos_a, r.pos_b) == oracle.longest_overlap(a, b, keep_n=True)
        assert r.length >= 500


class TestDeepLevels:
    """Recursing u32 levels (wide-level finish from the child's order), wide
    naming by (c0, c1) bucket sort with in-run c2 fix-up, and its fallback."""

    def test_repeated_blocks_deep_recursion(self):
        rng = np.random.default_rng(11)
        blocks = [rng.integers(1, 5, size=int(rng.integers(50, 400))) for _ in range(40)]
        parts = [blocks[int(rng.integers(0, 40))] for _ in range(3000)]
        r = np.concatenate(parts)[: 1 << 20]
        t = RankedText(r, 4)
        ws = sx.prepare_dc3_workspace(t)
        assert ws.depth >= 4
        ix = sx.build_sa_dc3(t)
        sa, rank = oracle.dc3(r, 4)
        assert np.array_equal(ix.sa, sa) and np.array_equal(ix.rank, rank)
        assert np.array_equal(sx.build_lcp(t, ix).lcp, oracle.lcp(r, sa, rank))

    @pytest.mark.parametrize("hot", [0, 40, 200])
    def test_wide_alphabet_repeats(self, hot):
        rng = np.random.default_rng(12 + hot)
        sigma = 1 << 22
        r = rng.integers(1, sigma + 1, size=120_000)
        r[50_000:52_000] = r[10_000:12_000]                  # equal (c0, c1, c2) runs
        for k in range(hot):                                  # one (c0, c1) pair `hot` times
            r[70_000 + 3 * k: 70_000 + 3 * k + 2] = (7, 9)
        t = RankedText(r, sigma)
        ix = sx.build_sa_dc3(t)
        sa, rank = oracle.dc3(r, sigma)
        assert np.array_equal(ix.sa, sa) and np.array_equal(ix.rank, rank)


class TestTieResolution:
    """Levels whose names are almost all distinct resolve the few tied samples
    by prefix doubling on the recursion string instead of recursing."""

    @pytest.mark.parametrize("reps", [(300,), (257, 1200, 40), (2000, 2000)])
    def test_sparse_repeats(self, reps):
        rng = np.random.default_rng(sum(reps))
        r = rng.integers(1, 5, size=1 << 20)
        for k, L in enumerate(reps):                     # copies of earlier stretches
            src, dst = 1000 + 7919 * k, 600_000 + 50_000 * k
            r[dst:dst + L] = r[src:src + L]
        t = RankedText(r, 4)
        ix = sx.build_sa_dc3(t)
        from paper_1404_3448_b200 import _lib
        trace = _lib.dc3_trace()
        assert trace[-1][3] < trace[-1][2], trace      # deepest level had ties: resolved, not recursed
        sa, rank = oracle.dc3(r, 4)
        assert np.array_equal(ix.sa, sa) and np.array_equal(ix.rank, rank)
        assert np.array_equal(sx.build_lcp(t, ix).lcp, oracle.lcp(r, sa, rank))

    def test_many_copies_of_one_block(self):
        """One block repeated 40 times: long tied groups (the doubling still
        converges; > 4096 copies would fall back to recursion)."""
        rng = np.random.default_rng(3)
        r = rng.integers(1, 5, size=1 << 19)
        blk = r[:500].copy()
        for k in range(40):
            r[100_000 + 9000 * k: 100_000 + 9000 * k + 500] = blk
        t = RankedText(r, 4)
        ix = sx.build_sa_dc3(t)
        sa, rank = oracle.dc3(r, 4)
        assert np.array_equal(ix.sa, sa) and np.array_equal(ix.rank, rank)

    def test_overlap_pairs_with_ties(self):
        seqs, offs = c4_pairs_local(200, 4000)
        want = oracle.overlap_batch(seqs, offs, threads=4)
        ob = sx.OverlapBatch(seqs, offs)
        ob.run_device()
        assert np.array_equal(ob.results(), want)


def c4_pairs_local(n, length):
    from paper_1404_3448_b200.workloads import c4_pairs
    return c4_pairs(0, n, length=length)
