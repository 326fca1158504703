"""The large-sweep RMQ checker (oracle.argmin_sparse_blocked, used for the
full 10^8-query C5 parity) agrees with the plain leftmost-argmin scan
(oracle.argmin_blocked) and with the reference's own RMQ fixtures
(test_rmq.py:20-23, 54-57)."""

import numpy as np
import pytest

import oracle


def test_reference_fixtures():
    row = [0, 3, 1, 4, 0, 2, 1, 0]
    assert oracle.argmin_sparse_blocked([2, 1, 1, 1, 2], [0, 2], [4, 4]).tolist() == [1, 2]
    assert oracle.argmin_sparse_blocked(row, [0], [0]).tolist() == [0]


@pytest.mark.parametrize("n", [1, 2, 63, 64, 65, 127, 128, 129, 1000, 70_000])
def test_matches_scan(n):
    rng = np.random.default_rng(n)
    for hi in (3, 40):
        v = rng.integers(0, hi, n)
        q = rng.integers(0, n, (5000, 2))
        want = oracle.argmin_blocked(v, q[:, 0], q[:, 1])
        for threads in (1, 3):
            assert np.array_equal(oracle.argmin_sparse_blocked(v, q[:, 0], q[:, 1], threads=threads), want)


def test_out_of_range():
    with pytest.raises(IndexError):
        oracle.argmin_sparse_blocked([1, 2, 3], [0], [3])
