"""Synthetic inputs of BASELINE.json's configurations (host-side generators).

C4 ("batch of 100k synthetic 10 kbp noncoding-like pairs") has no generator
in the reference; SURVEY.md section 8(d) fixes a builder-chosen definition,
implemented here: pair p is A_p = gen_random(10_000, 2p+100, W),
B_p = gen_random(10_000, 2p+101, W) with W = (0.3, 0.2, 0.2, 0.3) (AT-rich,
40% GC), plus one planted shared block: with default_rng(10**7 + p),
L ~ U{32..256}, x, y ~ U{0..10^4-L}, B_p[y:y+L] = A_p[x:x+L].
"""

from __future__ import annotations

import numpy as np

from .sequence import gen_random

C4_WEIGHTS = (0.3, 0.2, 0.2, 0.3)
C4_LEN = 10_000


def c4_pair(p: int, length: int = C4_LEN) -> tuple[bytes, bytes]:
    a = gen_random(length, 2 * p + 100, C4_WEIGHTS).residues.encode()
    b = bytearray(gen_random(length, 2 * p + 101, C4_WEIGHTS).residues.encode())
    rng = np.random.default_rng(10 ** 7 + p)
    L = int(rng.integers(32, 257))
    x, y = (int(v) for v in rng.integers(0, length - L + 1, size=2))
    b[y:y + L] = a[x:x + L]
    return a, bytes(b)


def c4_pairs(p0: int, p1: int, length: int = C4_LEN) -> tuple[np.ndarray, np.ndarray]:
    """Pairs [p0, p1) packed as (ASCII bytes, int64[2P+1] offsets)."""
    n = p1 - p0
    seqs = np.empty(2 * n * length, dtype=np.uint8)
    for k, p in enumerate(range(p0, p1)):
        a, b = c4_pair(p, length)
        seqs[2 * k * length:(2 * k + 1) * length] = np.frombuffer(a, np.uint8)
        seqs[(2 * k + 1) * length:(2 * k + 2) * length] = np.frombuffer(b, np.uint8)
    offs = np.arange(2 * n + 1, dtype=np.int64) * length
    return seqs, offs

def _chunk(args):
    return c4_pairs(*args)


def c4_generate(lo: int, hi: int, length: int = C4_LEN, workers: int | None = None):
    """Pairs [lo, hi) packed like c4_pairs, generated in 1000-pair chunks on
    the host's cores (process pool)."""
    import concurrent.futures as cf
    import os
    chunks = [(a, min(a + 1000, hi), length) for a in range(lo, hi, 1000)]
    if not chunks:
        return np.zeros(0, np.uint8), np.zeros(1, np.int64)
    if len(chunks) == 1:
        return c4_pairs(*chunks[0])
    with cf.ProcessPoolExecutor(max_workers=workers or min(32, os.cpu_count() or 4)) as ex:
        parts = list(ex.map(_chunk, chunks))
    seqs = np.concatenate([p[0] for p in parts])
    offs, base = [np.zeros(1, np.int64)], 0
    for _s, o in parts:
        offs.append(o[1:] + base)
        base += int(o[-1])
    return seqs, np.concatenate(offs)


from .distributed import shard  # noqa: E402,F401  (re-exported for bench.py)
