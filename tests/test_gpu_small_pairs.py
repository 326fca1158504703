"""Scalar longest_overlap (overlap.py:110-152) on pairs small enough for the
on-chip pair kernel (SmallPairPipeline): equal to the C oracle and to the
multi-pass DC3 pipeline on the same pair, over every length split, planted
overlaps, keep-N, repeats, the size boundary and residue errors."""

import numpy as np
import pytest

import oracle
import paper_1404_3448_b200 as sx
from paper_1404_3448_b200.overlap import ONCHIP_RESIDUES, OverlapPipeline, _ascii
from paper_1404_3448_b200.sequence import DnaSequence, NPolicy, SequenceError

pytestmark = pytest.mark.gpu


def _rand(rng, n, alpha="ACGT"):
    return "".join(rng.choice(list(alpha), size=n))


def _check(a: str, b: str, keep=False):
    pol = NPolicy.KEEP if keep else NPolicy.REJECT
    r = sx.longest_overlap(DnaSequence("a", a), DnaSequence("b", b), pol)
    want = oracle.longest_overlap(a, b, keep_n=keep)
    assert (r.length, r.pos_a, r.pos_b) == want, (len(a), len(b))
    return r


def test_random_splits_vs_oracle():
    rng = np.random.default_rng(7)
    for _ in range(60):
        tot = int(rng.integers(2, ONCHIP_RESIDUES))
        la = int(rng.integers(1, tot))
        lb = tot - la
        a, b = _rand(rng, la), _rand(rng, lb)
        if rng.random() < 0.5 and min(la, lb) > 40:   # planted shared block
            k = int(rng.integers(8, min(la, lb) // 2))
            s = int(rng.integers(0, la - k))
            t = int(rng.integers(0, lb - k))
            b = b[:t] + a[s:s + k] + b[t + k:]
        _check(a, b)


def _pipeline_run(a: str, b: str, onchip: bool, keep=False):
    """saix_longest_overlap through the C ABI (OverlapPipeline); onchip=False
    forces the multi-pass DC3 pipeline for pairs the pair kernel would take."""
    from paper_1404_3448_b200 import _lib
    L = _lib.load()
    prev = L.saix_overlap_batch_set_onchip(int(onchip))
    try:
        pol = NPolicy.KEEP if keep else NPolicy.REJECT
        return OverlapPipeline(len(a), len(b)).run(np.frombuffer(a.encode(), np.uint8),
                                                   np.frombuffer(b.encode(), np.uint8), pol)
    finally:
        L.saix_overlap_batch_set_onchip(prev)


def test_size_boundary_both_paths_agree():
    rng = np.random.default_rng(11)
    for tot in (ONCHIP_RESIDUES - 2, ONCHIP_RESIDUES - 1, ONCHIP_RESIDUES, ONCHIP_RESIDUES + 1):
        la = tot // 2
        a, b = _rand(rng, la), _rand(rng, tot - 1 - la)   # |A| + 1 + |B| = tot
        r = _check(a, b)
        for onchip in (True, False):
            got = _pipeline_run(a, b, onchip)
            assert (r.length, r.pos_a, r.pos_b) == tuple(int(v) for v in got[:3]), (tot, onchip)


def test_c_abi_routes_small_pairs_with_the_pipeline_conventions():
    """saix_longest_overlap on a small pair (on-chip route) returns what the
    multi-pass pipeline returns: the answer and the first illegal residue as a
    generalized-text position (B's residue k at |A| + 1 + k)."""
    rng = np.random.default_rng(9)
    for la, lb in ((1, 1), (3000, 5000), (10000, 10000), (17, 20000)):
        a, b = _rand(rng, la), _rand(rng, lb)
        on, off = _pipeline_run(a, b, True), _pipeline_run(a, b, False)
        assert np.array_equal(on, off)
        assert tuple(int(v) for v in on[:3]) == oracle.longest_overlap(a, b)
    a, b = _rand(rng, 900, "ACGTN"), _rand(rng, 700, "ACGTN")
    assert np.array_equal(_pipeline_run(a, b, True, keep=True), _pipeline_run(a, b, False, keep=True))
    for a, b in (("ACGXT", "ACGT"), ("ACGT", "ACGTTGX"), ("ACNGT", "AC")):
        on, off = _pipeline_run(a, b, True), _pipeline_run(a, b, False)
        assert int(on[3]) == int(off[3]) != np.iinfo(np.int64).max, (a, b, on, off)


def test_repeats_and_tiny():
    _check("A", "A")
    _check("A", "C")
    _check("ACGT" * 2000, "ACGT" * 1500)           # long periodic: ties broken by position
    _check("A" * 9000, "A" * 9000)                 # one-letter run (work-bound fallback if any)
    _check("AC" * 5000, "CA" * 5000)


def test_keep_n_and_errors():
    rng = np.random.default_rng(3)
    a = _rand(rng, 3000, "ACGTN")
    b = _rand(rng, 2500, "ACGTN")
    _check(a, b, keep=True)
    with pytest.raises(SequenceError) as ea:
        sx.longest_overlap(DnaSequence("ra", "ACGTNAC"), DnaSequence("rb", "ACGX"))
    assert str(ea.value) == ("record 'ra': residue 'N' at position 4 not allowed "
                             "under policy=reject")
    with pytest.raises(SequenceError) as eb:
        sx.longest_overlap(DnaSequence("ra", "ACGTAC"), DnaSequence("rb", "ACGXT"))
    assert str(eb.value) == ("record 'rb': residue 'X' at position 3 not allowed "
                             "under policy=reject")
    with pytest.raises(SequenceError) as ek:
        sx.longest_overlap(DnaSequence("ra", "ACGTNAC"), DnaSequence("rb", "AC-G"), NPolicy.KEEP)
    assert "residue '-' at position 2" in str(ek.value)


def test_many_calls_reuse_one_pipeline():
    from paper_1404_3448_b200 import overlap as ov
    rng = np.random.default_rng(5)
    for _ in range(20):
        _check(_rand(rng, int(rng.integers(1, 500))), _rand(rng, int(rng.integers(1, 500))))
    assert len(ov._SMALL) == 1
