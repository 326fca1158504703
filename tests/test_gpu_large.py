"""Full-size parity at BASELINE.json's configurations.

C2 (10 Mbp pair) is compared array-for-array with the C oracle; larger
inputs use size-independent properties: the suffix array is a permutation,
adjacent suffixes are strictly increasing (Burkhardt-Kaerkkaeinen checker
via ISA), and LCP equals the oracle's Kasai on the GPU's own SA."""

import numpy as np
import pytest

import oracle
import paper_1404_3448_b200 as sx
from paper_1404_3448_b200.sequence import encode, gen_random

pytestmark = pytest.mark.gpu


def sa_is_correct(t: np.ndarray, sa: np.ndarray, rank: np.ndarray) -> bool:
    """O(n) suffix-array checker: permutation + adjacent order via ISA."""
    n = t.shape[0]
    if not np.array_equal(np.sort(sa), np.arange(n)):
        return False
    if not np.array_equal(rank[sa], np.arange(n)):
        return False
    a, b = sa[:-1], sa[1:]
    ca, cb = t[a], t[b]
    # rank of the suffix one position later; suffix n (empty) ranks lowest (-1)
    ra = np.where(a + 1 < n, rank[np.minimum(a + 1, n - 1)], -1)
    rb = np.where(b + 1 < n, rank[np.minimum(b + 1, n - 1)], -1)
    return bool(np.all((ca < cb) | ((ca == cb) & (ra < rb))))


def test_c2_pair_full_pipeline_vs_oracle():
    """BASELINE configs[1]: 2 x 10 Mbp, SA/LCP/answer against the C oracle."""
    a, b = gen_random(10_000_000, 11), gen_random(10_000_000, 12)
    gen = sx.GeneralizedText.build(a, b).to_ranked_text()
    ix = sx.build_sa_dc3(gen)
    sa, rank = oracle.dc3(gen.ranks, gen.sigma)
    assert np.array_equal(ix.sa, sa)
    assert np.array_equal(ix.rank, rank)
    lcp = sx.build_lcp(gen, ix).lcp
    assert np.array_equal(lcp, oracle.lcp(gen.ranks, sa, rank))
    r = sx.longest_overlap(a, b)
    assert (r.length, r.pos_a, r.pos_b) == oracle.longest_overlap(a.residues, b.residues)


@pytest.mark.parametrize("n", [1 << 24, 1 << 26])
def test_large_random_sa_properties(n):
    """2^24: the byte levels gather their records (text + ranks <= 128 MB);
    2^26: both byte levels take the bucketed-scatter path (k_srec_emit ->
    refine -> window) and the top level is too large for direct scatters."""
    t = encode(gen_random(n, 1))
    ix = sx.build_sa_dc3(t)
    assert sa_is_correct(t.ranks, ix.sa, ix.rank)
    lcp = sx.build_lcp(t, ix).lcp
    assert np.array_equal(lcp, oracle.lcp(t.ranks, ix.sa, ix.rank))


def test_rmq_sweep_prefix():
    """C5 shape at reduced n: batched query_sparse and lcp_query vs oracle."""
    t = encode(gen_random(1 << 22, 1))
    eng = sx.LcpQueryEngine.build(t)
    rng = np.random.default_rng(2026)
    q = rng.integers(0, t.n, size=(1_000_000, 2))
    got = sx.query_sparse_batch(eng.rmq, q[:, 0], q[:, 1])
    want = oracle.argmin_blocked(eng.lcp.lcp, q[:, 0], q[:, 1])
    assert np.array_equal(got, want)
    lq = sx.lcp_query_batch(eng, q[:200_000, 0], q[:200_000, 1])
    assert np.array_equal(lq, oracle.lcp_query(t.ranks, eng.sa.sa, eng.sa.rank, eng.lcp.lcp,
                                               q[:200_000, 0], q[:200_000, 1]))


def test_long_repeat_text():
    """Repetitive input: long LCPs exercise the chunk-seeded Kasai."""
    s = "ACGTTGCA" * 25_000 + "A" * 100_000
    t = encode(sx.DnaSequence("r", s))
    ix = sx.build_sa_dc3(t)
    sa, rank = oracle.dc3(t.ranks, 4)
    assert np.array_equal(ix.sa, sa)
    assert np.array_equal(sx.build_lcp(t, ix).lcp, oracle.lcp(t.ranks, sa, rank))


@pytest.mark.parametrize("n,copies,seglen", [(300_000, 1500, 40), (120_000, 300, 25), (60_000, 40, 80)])
def test_window_naming_with_planted_repeats(n, copies, seglen):
    """Level-0 window naming with a few percent of tied 21-character windows:
    the ties go through prefix doubling (resolve_ties), the result must equal
    the oracle's DC3 exactly."""
    rng = np.random.default_rng(n + copies)
    t = rng.integers(1, 5, n)
    seg = rng.integers(1, 5, seglen)
    for p in rng.integers(0, n - seglen, copies):
        t[p:p + seglen] = seg
    text = sx.RankedText(ranks=t, sigma=4)
    got = sx.build_sa_dc3(text)
    sa, rank = oracle.dc3(t, 4)
    assert np.array_equal(got.sa, sa)
    assert np.array_equal(got.rank, rank)
    assert np.array_equal(sx.build_lcp(text, got).lcp, oracle.lcp(t, sa, rank))


@pytest.mark.parametrize("sigma", [5, 6, 7])
def test_window_naming_wider_alphabets(sigma):
    rng = np.random.default_rng(sigma)
    t = rng.integers(1, sigma + 1, 200_000)
    t[rng.integers(0, len(t), 50)] = 1  # a rare low character (separator-like)
    text = sx.RankedText(ranks=t, sigma=sigma)
    sa, rank = oracle.dc3(t, sigma)
    assert np.array_equal(sx.build_sa_dc3(text).sa, sa)
