"""SuffixIndexer (the C3 throughput path: pinned upload, DC3 + LCP, SA download
overlapped with the LCP kernel, LCP download) against the C oracle's DC3 and
Kasai (suffix_index.py:395-399, 479-506), over repeated steps that reuse the
buffers."""

import numpy as np
import pytest

import oracle
from paper_1404_3448_b200.suffix_index import SuffixIndexer

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n,sigma,seed", [(1, 4, 0), (1000, 4, 1), (300_001, 4, 2), (200_000, 20, 3)])
def test_indexer_staged_matches_oracle(n, sigma, seed):
    ix = SuffixIndexer(n, sigma)
    for step in range(2):
        t = np.random.default_rng(seed * 10 + step).integers(1, sigma + 1, n)
        ix.stage(t)
        ix.run_staged()
        sa, rank = oracle.dc3(t.astype(np.int64), sigma)
        assert np.array_equal(ix.hsa.numpy()[:n].astype(np.int64), sa)
        assert np.array_equal(ix.hlcp.numpy()[:n].astype(np.int64), oracle.lcp(t.astype(np.int64), sa, rank))
