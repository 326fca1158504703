"""Level-0 window naming of DNA texts by the MSD record sort (csrc/wsort.cuh).

The path runs for byte texts with ranks 1..4 (sigma <= 4), N < 2^29 and
>= 2^20 samples; it must give exactly the reference's SA / rank
(suffix_index.py:395-399) on every text, including the ones that stress its
own conventions: windows reaching past the end (0-filled digits + a flag;
texts ending in long A runs), every N mod 3 (padding sample), tied windows
(prefix-doubling rounds), skewed prefix buckets (variable P3 capacity) and
texts that leave the path (16-bit bin overflow -> generic window sort;
too many ties -> triple naming + recursion)."""

import numpy as np
import pytest

import oracle
import paper_1404_3448_b200 as sx
from paper_1404_3448_b200 import _lib
from paper_1404_3448_b200.sequence import RankedText

pytestmark = pytest.mark.gpu

N0 = (1 << 21) + 12345  # >= 2^20 samples


def _random(n, seed, alphabet=(1, 2, 3, 4)):
    rng = np.random.default_rng(seed)
    return np.asarray(alphabet, np.uint8)[rng.integers(0, len(alphabet), n)]


def _check(ranks, sigma=4, naming=2):
    t = RankedText(ranks=ranks.astype(np.int64), sigma=sigma)
    ix = sx.build_sa_dc3(t)
    got_naming = _lib.dc3_naming()
    sa, rank = oracle.dc3(ranks, sigma)
    assert np.array_equal(ix.sa, sa)
    assert np.array_equal(ix.rank, rank)
    if naming is not None:
        assert got_naming == naming, got_naming


@pytest.mark.parametrize("extra", [0, 1, 2])
def test_random_every_n_mod_3(extra):
    _check(_random(N0 + extra, 5 + extra))


@pytest.mark.parametrize("tail", [1, 2, 7, 20, 21, 22, 40])
def test_end_windows_after_a_run(tail):
    """0-filled end windows equal to full windows of A's: the flag and the
    reversed position order them as suffixes (shorter first)."""
    t = _random(N0, 11)
    t[-tail:] = 1
    _check(t)


def test_end_windows_repeat_the_tail():
    """The last 20 characters also occur earlier followed by A's."""
    t = _random(N0, 12)
    t[1000:1020] = t[-20:]
    t[1020:1060] = 1
    t[-41:-21] = t[-20:]
    _check(t)


@pytest.mark.parametrize("sigma", [2, 3])
def test_small_alphabets(sigma):
    """sigma 3 stays on the path; binary text has ~m/2 tied windows (2^21
    windows for 1.4M samples) and takes the recursion."""
    _check(_random(N0, 20 + sigma, tuple(range(1, sigma + 1))), sigma=sigma, naming=2 if sigma == 3 else None)


def test_skewed_text_larger_buckets():
    """Weights (0.5, 0.2, 0.2, 0.1): the AAAAAAAA bucket holds ~5.5k records
    (P3 capacity above its 4096 minimum, one CTA per SM) and its sub-buckets
    reach past 32 records (the CTA bitonic)."""
    rng = np.random.default_rng(31)
    t = (rng.choice(4, size=N0, p=[0.5, 0.2, 0.2, 0.1]) + 1).astype(np.uint8)
    _check(t)


def test_two_letter_text_leaves_the_path():
    """A/T only: 2^21 windows for 1.4M samples, mostly tied -> recursion."""
    _check(_random(N0, 31, (1, 4)), naming=None)


def test_planted_repeats_tie_rounds():
    """Some hundred planted copies: tied 21-character windows resolved by the
    prefix-doubling rounds (fewer than m/32 ties)."""
    t = _random(N0, 41)
    rng = np.random.default_rng(42)
    for _ in range(300):
        L = int(rng.integers(40, 400))
        s, d = (int(x) for x in rng.integers(0, N0 - L, 2))
        t[d:d + L] = t[s:s + L]
    _check(t)


def test_periodic_text_leaves_the_path():
    """A period-7 text: almost every window is tied -> recursion."""
    base = np.array([1, 2, 3, 4, 4, 2, 1], np.uint8)
    t = np.tile(base, N0 // 7 + 1)[:N0].copy()
    t[N0 // 2] = 3
    _check(t, naming=None)


def test_homopolymer_leaves_the_path():
    """One fine bin takes every sample (16-bit bin overflow)."""
    t = np.ones(N0, np.uint8)
    t[::4099] = 2
    _check(t, naming=None)


def test_matches_lcp_and_overlap_pipeline():
    """The SA feeds Kasai exactly like the other paths."""
    t = _random(N0, 51)
    rt = RankedText(ranks=t.astype(np.int64), sigma=4)
    ix = sx.build_sa_dc3(rt)
    assert _lib.dc3_naming() == 2
    lcp = sx.build_lcp(rt, ix).lcp
    assert np.array_equal(lcp, oracle.lcp(t, ix.sa, ix.rank))


def test_homopolymer_run_in_random_text():
    """A 4000-base A run: its windows fill one fine bucket (within P3's
    capacity) and one sub-bucket far past WS_BIG_SUB -> the pass is
    discarded (the generic window sort or the recursion take over), and the
    answer stays exact."""
    t = _random(N0, 61)
    t[N0 // 3:N0 // 3 + 4000] = 1
    _check(t, naming=None)


def _gsa(a, b):
    """GeneralizedText ranks (overlap.py:83-95): A+1, separator 1, B+1."""
    return np.concatenate([a + 1, [1], b + 1]).astype(np.uint8)


@pytest.mark.parametrize("la", [1 << 20, 7, 40])
def test_generalized_text_separator(la):
    """sigma 5 with one separator (the C2 text): windows reaching the
    separator stop there like end windows; A of 7 / 40 residues puts the
    separator among the first windows."""
    a = _random(la, 71)
    b = _random(N0 - la, 72)
    _check(_gsa(a, b), sigma=5)


def test_generalized_text_stop_order():
    """An end window and a separator window with equal 0-filled keys: the
    nearer stop orders first (A ends ...CGT|, B ends ...CGTAAAAAAA)."""
    a = _random(1 << 20, 81)
    b = _random(N0 - (1 << 20), 82)
    a[-3:] = [2, 3, 4]
    b[-10:-7] = [2, 3, 4]
    b[-7:] = 1
    _check(_gsa(a, b), sigma=5)


def test_sigma5_with_two_separators_leaves_the_path():
    """Two rank-1 characters: not a single separator -> generic window sort."""
    a = _random(N0, 91) + 1
    a[[100, 200]] = 1
    _check(a.astype(np.uint8), sigma=5, naming=None)
