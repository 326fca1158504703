"""Cartesian-tree / Euler-tour oracle (oracle_cartesian, a C restatement of
rmq.py:91-152) pinned against the reference's own outputs
(tests/golden/cartesian_cases.npz, made by make_cartesian_golden.py)."""

import os

import numpy as np
import pytest

import oracle
from conftest import ROOT

GOLD = os.path.join(ROOT, "tests", "golden", "cartesian_cases.npz")


@pytest.fixture(scope="module")
def gold():
    return dict(np.load(GOLD))


def test_oracle_tree_and_tour_match_reference(gold):
    for k in range(int(gold["count"])):
        parent, left, right, root, nodes, depths, first = oracle.cartesian(gold[f"v{k}"])
        assert np.array_equal(parent, gold[f"parent{k}"]), k
        assert np.array_equal(left, gold[f"left{k}"])
        assert np.array_equal(right, gold[f"right{k}"])
        assert root == int(gold[f"root{k}"])
        assert np.array_equal(nodes, gold[f"nodes{k}"])
        assert np.array_equal(depths, gold[f"depths{k}"])
        assert np.array_equal(first, gold[f"first{k}"])


def test_reference_answers_are_leftmost_argmins(gold):
    for k in range(int(gold["count"])):
        v = gold[f"v{k}"]
        for a, b, ans in zip(gold[f"qi{k}"], gold[f"qj{k}"], gold[f"ans{k}"]):
            assert oracle.scan_argmin(v, int(a), int(b)) == int(ans)
