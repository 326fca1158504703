"""Per-call latency of the scalar reference entry point longest_overlap
(overlap.py:110-152) on C4-shaped pairs (2 x 10 kbp): the on-chip single-pair
path (SmallPairPipeline) vs the multi-pass DC3 pipeline (OverlapPipeline) on
the same pairs, host ASCII in / answer out, answers compared.
usage: python tools/scalar_probe.py [calls]"""

import json
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_1404_3448_b200 as sx  # noqa: E402
from paper_1404_3448_b200.overlap import OverlapPipeline, _ascii  # noqa: E402
from paper_1404_3448_b200.sequence import DnaSequence  # noqa: E402
from paper_1404_3448_b200.workloads import c4_pairs  # noqa: E402

calls = int(sys.argv[1]) if len(sys.argv) > 1 else 200
seqs, offs = c4_pairs(0, calls)
pairs = []
for p in range(calls):
    a = seqs[offs[2 * p]:offs[2 * p + 1]].tobytes().decode()
    b = seqs[offs[2 * p + 1]:offs[2 * p + 2]].tobytes().decode()
    pairs.append((DnaSequence("a", a), DnaSequence("b", b)))

for a, b in pairs[:5]:
    sx.longest_overlap(a, b)          # warm-up (allocations, first launch)
t0 = time.perf_counter()
small = [sx.longest_overlap(a, b) for a, b in pairs]
t_small = (time.perf_counter() - t0) / calls

# the multi-pass DC3 pipeline (saix_longest_overlap with the on-chip route off)
from paper_1404_3448_b200 import _lib  # noqa: E402
L = _lib.load()
prev = L.saix_overlap_batch_set_onchip(0)
pipe = OverlapPipeline(len(pairs[0][0]), len(pairs[0][1]))
for a, b in pairs[:5]:
    pipe.run(_ascii(a), _ascii(b))
t0 = time.perf_counter()
big = [pipe.run(_ascii(a), _ascii(b)) for a, b in pairs]
t_big = (time.perf_counter() - t0) / calls
L.saix_overlap_batch_set_onchip(prev)

same = all((r.length, r.pos_a, r.pos_b) == tuple(int(v) for v in g[:3]) for r, g in zip(small, big))
print(json.dumps({"calls": calls, "pair_residues": int(offs[2] - offs[0]),
                  "onchip_us_per_call": round(t_small * 1e6, 1), "dc3_pipeline_us_per_call": round(t_big * 1e6, 1),
                  "speedup": round(t_big / t_small, 2), "answers_equal": same}))
