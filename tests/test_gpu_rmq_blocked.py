"""The L2-resident blocked RMQ layout (csrc/rmq.cu, SAIX_SPARSE_BLOCKED) at
its seams: 32-value blocks, 1024-value superblocks, value spans at the
254 limit (255 keeps the full table), ties across every part of a query
(left scan, next block's suffix entry, superblock table, previous block's
prefix entry, right scan), and the per-level reference table built on
demand.  Answers are the reference's leftmost argmin (rmq.py:48-58)."""

import ctypes

import numpy as np
import pytest

import oracle
import paper_1404_3448_b200 as sx
from paper_1404_3448_b200 import _lib

pytestmark = pytest.mark.gpu


def _edge_queries(n, rng, extra=4000):
    """Queries whose ends sit on and around every block / superblock seam,
    plus random ones."""
    marks = sorted({x for b in range(0, n + 1024, 32) for x in (b - 1, b, b + 1) if 0 <= x < n})
    marks = np.array(marks[:600], dtype=np.int64)
    qi = np.concatenate([np.repeat(marks, 3), rng.integers(0, n, extra)])
    qj = np.concatenate([np.tile(marks[::-1][:len(marks)], 3)[:3 * len(marks)], rng.integers(0, n, extra)])
    return qi, qj


@pytest.mark.parametrize("n", [1, 2, 31, 32, 33, 1023, 1024, 1025, 4097, 70_001, (1 << 20) + 7])
def test_blocked_sizes(n):
    rng = np.random.default_rng(n)
    vals = rng.integers(0, 30, n)
    st = sx.SparseTable(vals)
    assert st.plan.mode == _lib.SPARSE_BLOCKED
    qi, qj = _edge_queries(n, rng)
    assert np.array_equal(st.query_batch(qi, qj), oracle.argmin_blocked(vals, qi, qj))


@pytest.mark.parametrize("span,mode", [(254, "blocked"), (255, "full")])
def test_value_span_limit(span, mode):
    rng = np.random.default_rng(span)
    n = 50_000
    vals = rng.integers(0, span + 1, n) - 7
    vals[[3, 4000]] = [-7, span - 7]  # both extremes present
    st = sx.SparseTable(vals)
    assert (st.plan.mode == _lib.SPARSE_BLOCKED) == (mode == "blocked")
    qi, qj = _edge_queries(n, rng)
    assert np.array_equal(st.query_batch(qi, qj), oracle.argmin_blocked(vals, qi, qj))


def test_ties_everywhere_leftmost():
    """Few distinct values: the minimum occurs in several parts of most
    queries; the leftmost position must win."""
    rng = np.random.default_rng(9)
    n = 300_000
    vals = rng.integers(0, 3, n)
    st = sx.SparseTable(vals)
    qi, qj = _edge_queries(n, rng, extra=20_000)
    assert np.array_equal(st.query_batch(qi, qj), oracle.argmin_blocked(vals, qi, qj))


def test_reference_table_on_demand():
    """SparseTable.table (the reference's per-level argmin layout) from a
    blocked table equals the oracle's level build."""
    vals = np.random.default_rng(4).integers(0, 9, 3000)
    st = sx.SparseTable(vals)
    assert st.plan.mode == _lib.SPARSE_BLOCKED
    assert np.array_equal(np.concatenate(st.table), oracle.sparse_build(vals))


def test_lcp_query_through_blocked_table():
    """lcp_query over an engine whose RMQ is the blocked layout."""
    from paper_1404_3448_b200.sequence import encode, gen_random
    t = encode(gen_random(200_000, 3))
    eng = sx.LcpQueryEngine.build(t)
    assert eng.rmq.plan.mode == _lib.SPARSE_BLOCKED
    rng = np.random.default_rng(5)
    qi, qj = rng.integers(0, t.n, 20_000), rng.integers(0, t.n, 20_000)
    want = oracle.lcp_query(t.ranks, eng.sa.sa, eng.sa.rank, eng.lcp.lcp, qi, qj)
    assert np.array_equal(sx.lcp_query_batch(eng, qi, qj), want)


def test_plan_blocked_abi():
    L = _lib.load()
    p = _lib.SparsePlan()
    assert L.saix_sparse_plan_blocked(1 << 26, 0, 24, ctypes.byref(p)) == 0
    assert p.mode == _lib.SPARSE_BLOCKED and p.levels == 27
    assert L.saix_sparse_plan_blocked(1 << 26, 0, 300, ctypes.byref(p)) == 0
    assert p.mode == _lib.SPARSE_PACK32 or p.mode == _lib.SPARSE_PACK64
