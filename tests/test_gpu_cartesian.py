"""GPU parity of the Cartesian-tree RMQ engine (rmq.py:61-251): tree, tour
and ±1 structure equal the reference's (tests/golden/cartesian_cases.npz),
the reference's own test expectations (tests/test_rmq.py of the reference)
hold, and large inputs equal the C oracle / the sparse table."""

import os
import random

import numpy as np
import pytest

import oracle
from conftest import ROOT
from paper_1404_3448_b200 import rmq

pytestmark = pytest.mark.gpu

GOLD = os.path.join(ROOT, "tests", "golden", "cartesian_cases.npz")
LCP_ROW = [0, 1, 0, 2, 1, 3, 0, 1]


@pytest.fixture(scope="module")
def gold():
    return dict(np.load(GOLD))


def random_pm1(rng, m):
    arr = [rng.randrange(-3, 4)]
    for _ in range(m - 1):
        arr.append(arr[-1] + rng.choice((-1, 1)))
    return arr


def test_golden_tree_tour_pm1_and_answers(gold):
    for k in range(int(gold["count"])):
        v = gold[f"v{k}"]
        ct = rmq.CartesianRmq(v)
        assert np.array_equal(ct.tree.parent, gold[f"parent{k}"]), k
        assert np.array_equal(ct.tree.left, gold[f"left{k}"])
        assert np.array_equal(ct.tree.right, gold[f"right{k}"])
        assert ct.tree.root == int(gold[f"root{k}"])
        assert np.array_equal(ct.tour.tour_nodes, gold[f"nodes{k}"])
        assert np.array_equal(ct.tour.tour_depths, gold[f"depths{k}"])
        assert np.array_equal(ct.tour.first_visit, gold[f"first{k}"])
        assert ct.pm1.block == int(gold[f"block{k}"])
        assert np.array_equal(ct.pm1.block_argmin, gold[f"bargmin{k}"])
        assert np.array_equal(ct.pm1.block_min, gold[f"bmin{k}"])
        assert np.array_equal(ct.pm1.types, gold[f"types{k}"])
        assert np.array_equal(ct.query_batch(gold[f"qi{k}"], gold[f"qj{k}"]), gold[f"ans{k}"])


class TestCartesianTree:
    def test_middle_minimum(self):
        tree = rmq.build_cartesian([2, 1, 3])
        assert tree.root == 1
        assert tree.left[1] == 0 and tree.right[1] == 2

    def test_tie_breaks_left(self):
        assert rmq.build_cartesian([1, 1]).root == 0

    def test_empty_rejected(self):
        with pytest.raises(ValueError):
            rmq.build_cartesian([])

    def test_inorder_is_identity_and_heap_property(self):
        rng = random.Random(1)
        for _ in range(40):
            n = rng.randrange(1, 60)
            vals = [rng.randrange(0, 8) for _ in range(n)]
            tree = rmq.build_cartesian(vals)
            order = []

            def walk(x):
                if x < 0:
                    return
                walk(int(tree.left[x]))
                order.append(x)
                walk(int(tree.right[x]))
            walk(tree.root)
            assert order == list(range(n))
            for x in range(n):
                p = int(tree.parent[x])
                if p >= 0:
                    assert vals[p] <= vals[x]


class TestEulerTour:
    def test_single_node(self):
        tour = rmq.euler_tour(rmq.build_cartesian([5]))
        assert tour.tour_nodes.tolist() == [0]
        assert tour.tour_depths.tolist() == [0]
        assert tour.first_visit.tolist() == [0]

    def test_invariants_random(self):
        rng = random.Random(2)
        for _ in range(30):
            n = rng.randrange(1, 200)
            vals = [rng.randrange(0, 10) for _ in range(n)]
            tour = rmq.euler_tour(rmq.build_cartesian(vals))
            assert len(tour.tour_nodes) == 2 * n - 1
            if n > 1:
                assert set(np.abs(np.diff(tour.tour_depths)).tolist()) == {1}
            assert tour.tour_depths[0] == 0
            for v in range(n):
                f = int(tour.first_visit[v])
                assert tour.tour_nodes[f] == v and v not in tour.tour_nodes[:f].tolist()


class TestPlusMinusOne:
    def test_identity(self):
        arr = random_pm1(random.Random(2), 50)
        pm = rmq.build_pm1(arr)
        for i in range(len(arr)):
            assert rmq.query_pm1(pm, i, i) == i

    def test_rejects_non_unit_steps(self):
        with pytest.raises(ValueError):
            rmq.build_pm1([0, 2, 1])
        with pytest.raises(ValueError):
            rmq.build_pm1([])

    def test_path_shaped_tree_full_range(self):
        tour = rmq.euler_tour(rmq.build_cartesian(list(range(30))))
        pm = rmq.build_pm1(tour.tour_depths)
        full = rmq.query_pm1(pm, 0, len(tour.tour_depths) - 1)
        assert full == oracle.scan_argmin(tour.tour_depths, 0, len(tour.tour_depths) - 1)
        assert full == int(tour.first_visit[0])

    def test_many_random_queries_match_scan(self):
        rng = random.Random(3)
        for _ in range(20):
            m = rng.randrange(1, 700)
            arr = random_pm1(rng, m)
            pm = rmq.build_pm1(arr)
            qi = np.array([rng.randrange(m) for _ in range(200)])
            qj = np.array([rng.randrange(m) for _ in range(200)])
            want = [oracle.scan_argmin(arr, int(a), int(b)) for a, b in zip(qi, qj)]
            assert pm.query_batch(qi, qj).tolist() == want

    def test_block_types_sound(self):
        rng = random.Random(4)
        for _ in range(20):
            arr = random_pm1(rng, rng.randrange(20, 400))
            pm = rmq.build_pm1(arr)
            b = pm.block
            assert b == max(1, (len(arr).bit_length() - 1) // 2)
            assert len(pm.inblock) <= 2 ** max(b - 1, 0)
            for code, table in pm.inblock.items():
                # the step pattern's walk (bit k set: step k goes down), then
                # every in-block range's leftmost argmin by the scan oracle
                walk = np.cumsum([0] + [-1 if (code >> k) & 1 else 1 for k in range(b - 1)])
                for i in range(b):
                    for j in range(i, b):
                        assert int(table[i, j]) == oracle.scan_argmin(walk, i, j), (code, i, j)
            for blk in range(len(pm.types)):
                lo = blk * b
                hi = min(len(arr), lo + b)
                for i in range(lo, hi):
                    for j in range(i, hi):
                        assert pm._inblock_query(blk, i - lo, j - lo) == oracle.scan_argmin(arr, i, j)


class TestLcaPipeline:
    def test_lcp_row_query(self):
        assert rmq.rmq_via_lca(LCP_ROW, 1, 7) == 2

    def test_identity(self):
        assert rmq.rmq_via_lca([3, 1, 2], 2, 2) == 2

    def test_agrees_with_sparse_exhaustive(self):
        rng = random.Random(5)
        for _ in range(30):
            n = rng.randrange(1, 65)
            vals = [rng.randrange(0, 6) for _ in range(n)]
            st = rmq.SparseTable(vals)
            ct = rmq.CartesianRmq(vals)
            qi = np.array([i for i in range(n) for j in range(i, n)])
            qj = np.array([j for i in range(n) for j in range(i, n)])
            want = [oracle.scan_argmin(vals, int(a), int(b)) for a, b in zip(qi, qj)]
            assert st.query_batch(qi, qj).tolist() == want
            assert ct.query_batch(qi, qj).tolist() == want

    def test_bounds_checked(self):
        ct = rmq.CartesianRmq([1, 2, 3])
        with pytest.raises(IndexError):
            ct.query(0, 3)


@pytest.mark.parametrize("n,hi", [(100_000, 60), (1 << 20, 5), (3_000_001, 1 << 40)])
def test_large_matches_oracle_and_sparse(n, hi):
    rng = np.random.default_rng(n)
    vals = rng.integers(0, hi, n)
    ct = rmq.CartesianRmq(vals)
    parent, left, right, root, nodes, depths, first = oracle.cartesian(vals)
    assert np.array_equal(ct.tree.parent, parent)
    assert np.array_equal(ct.tree.left, left) and np.array_equal(ct.tree.right, right)
    assert ct.tree.root == root
    assert np.array_equal(ct.tour.tour_nodes, nodes)
    assert np.array_equal(ct.tour.tour_depths, depths)
    assert np.array_equal(ct.tour.first_visit, first)
    qi, qj = rng.integers(0, n, 20000), rng.integers(0, n, 20000)
    assert np.array_equal(ct.query_batch(qi, qj), rmq.SparseTable(vals).query_batch(qi, qj))


def test_monotone_and_constant_arrays():
    for vals in (np.arange(5000), np.arange(5000)[::-1].copy(), np.zeros(5000, np.int64)):
        ct = rmq.CartesianRmq(vals)
        parent, left, right, root, nodes, depths, first = oracle.cartesian(vals)
        assert np.array_equal(ct.tree.parent, parent) and ct.tree.root == root
        assert np.array_equal(ct.tour.tour_nodes, nodes)


def test_lcp_engine_cartesian_kind_matches_sparse():
    from paper_1404_3448_b200 import LcpQueryEngine, encode, lcp_query, lcp_query_batch
    from paper_1404_3448_b200.sequence import gen_random
    t = encode(gen_random(50_000, 3))
    es = LcpQueryEngine.build(t)
    ec = LcpQueryEngine.build(t, rmq_kind="cartesian")
    assert isinstance(ec.rmq, rmq.CartesianRmq)
    rng = np.random.default_rng(1)
    qi, qj = rng.integers(0, t.n, 5000), rng.integers(0, t.n, 5000)
    qj[:50] = qi[:50]
    assert np.array_equal(lcp_query_batch(ec, qi, qj), lcp_query_batch(es, qi, qj))
    assert lcp_query(ec, 7, 7) == t.n - 7
    with pytest.raises(IndexError):
        lcp_query(ec, 0, t.n)
