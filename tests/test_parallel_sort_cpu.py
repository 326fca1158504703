"""Host-side parts of the parallel-sort mirror (parallel_sort.py:38-91):
config validation and chunk planning, exactly as the reference tests them
(test_parallel_sort.py:128-159)."""

import pytest

from paper_1404_3448_b200 import parallel_sort as ps


def test_config_validation():
    with pytest.raises(ValueError):
        ps.SortConfig(digit_bits=0)
    with pytest.raises(ValueError):
        ps.SortConfig(digit_bits=3, total_bits=32)
    with pytest.raises(ValueError):
        ps.SortConfig(chunk_size=0)
    with pytest.raises(ValueError):
        ps.SortConfig(workers=0)
    with pytest.raises(ValueError):
        ps.SortConfig(total_bits=64)


def test_plan_covers_input():
    plan = ps.plan_chunks(10, ps.SortConfig(chunk_size=3))
    assert plan.boundaries == ((0, 3), (3, 6), (6, 9), (9, 10))
    assert plan.chunk_size == 3
    assert ps.plan_chunks(0, ps.SortConfig()).boundaries == ()


def test_chunk32_flag():
    assert ps.SortConfig(chunk_size=32).chunk_is_multiple_of_32
    assert ps.SortConfig(chunk_size=4096).chunk_is_multiple_of_32
    assert not ps.SortConfig(chunk_size=31).chunk_is_multiple_of_32
