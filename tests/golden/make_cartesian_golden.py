"""Generate Cartesian-tree / Euler-tour / ±1-RMQ golden cases by running the
REFERENCE saix.rmq.

Run in the dev container (the reference exists only there):

    cd /tmp && PYTHONDONTWRITEBYTECODE=1 NUMBA_CACHE_DIR=/tmp/numba_cache \
        python /root/repo/tests/golden/make_cartesian_golden.py

Writes tests/golden/cartesian_cases.npz: for each value array its tree
(parent, left, right, root), tour (nodes, depths, first_visit), the ±1
structure of the tour depths (block, block_argmin, block_min, types) and
CartesianRmq answers to seeded queries.
"""

from __future__ import annotations

import os
import random
import sys

import numpy as np

REF = "/root/reference/pkg/src"
OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "cartesian_cases.npz")

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
sys.dont_write_bytecode = True
sys.path.insert(0, REF)

from saix import rmq  # noqa: E402


def main():
    rng = random.Random(61251)
    arrays = [[5], [2, 1, 3], [1, 1], [3, 1, 2], list(range(30)), list(range(30, 0, -1)), [0] * 40,
              [0, 2, 1, 3, 0, 2], [7, 7, 3, 3, 9, 1, 1, 8]]
    for _ in range(40):
        n = rng.randrange(1, 3000)
        hi = rng.choice([2, 5, 60, 10 ** 6])
        arrays.append([rng.randrange(0, hi) for _ in range(n)])
    for _ in range(5):  # negative values
        arrays.append([rng.randrange(-50, 50) for _ in range(rng.randrange(1, 500))])
    out = {"count": np.array(len(arrays))}
    for k, vals in enumerate(arrays):
        tree = rmq.build_cartesian(vals)
        tour = rmq.euler_tour(tree)
        pm = rmq.PlusMinusOneRmq(tour.tour_depths)
        ct = rmq.CartesianRmq(vals)
        n = len(vals)
        qi = np.array([rng.randrange(n) for _ in range(100)], np.int64)
        qj = np.array([rng.randrange(n) for _ in range(100)], np.int64)
        ans = np.array([ct.query(int(a), int(b)) for a, b in zip(qi, qj)], np.int64)
        out.update({f"v{k}": np.array(vals, np.int64), f"parent{k}": tree.parent, f"left{k}": tree.left,
                    f"right{k}": tree.right, f"root{k}": np.array(tree.root), f"nodes{k}": tour.tour_nodes,
                    f"depths{k}": tour.tour_depths, f"first{k}": tour.first_visit, f"block{k}": np.array(pm.block),
                    f"bargmin{k}": pm.block_argmin, f"bmin{k}": pm.block_min, f"types{k}": pm.types,
                    f"qi{k}": qi, f"qj{k}": qj, f"ans{k}": ans})
    np.savez_compressed(OUT, **out)
    print("wrote", OUT, len(arrays), "cases")


if __name__ == "__main__":
    main()
