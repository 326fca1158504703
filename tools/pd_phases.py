"""Phase breakdown of the on-chip pair kernel (SAIX_PD_CLOCKS=1): SM cycles
per phase summed over CTAs, as a share of the total."""
import ctypes
import os
import sys

os.environ["SAIX_PD_CLOCKS"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1404_3448_b200 as sx  # noqa: E402
from paper_1404_3448_b200 import _lib  # noqa: E402
from paper_1404_3448_b200.workloads import c4_generate  # noqa: E402

k = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
seqs, offs = c4_generate(0, k)
ob = sx.OverlapBatch(seqs, offs)
ob.run_device()
torch.cuda.synchronize()
c = np.zeros(17, np.int64)
_lib.load().saix_overlap_batch_phase_clocks(c.ctypes.data_as(ctypes.c_void_p), 17)
extra, c = c[12:], c[:12]
names = ["load", "bucket counts", "scan", "scatter", "in-bucket sort", "big buckets", "ranks",
         "non-samples", "merge", "lcp pass 1", "runs pass 2", "pair fetch"]
tot = c.sum()
print(f"{k} pairs; cycles per pair per CTA: {tot / k:.0f}")
for nm, v in sorted(zip(names, c), key=lambda x: -x[1]):
    print(f"  {nm:16s} {100 * v / tot:5.1f}%  {v / k:9.0f} cycles/pair")
print(f"in-bucket: slowest thread {extra[0] / k:.0f} cycles/pair, mean thread {extra[1] / k:.0f}")
print(f"in-bucket: lane steps {extra[2] / k:.0f} per pair, warp steps {extra[3] / k:.0f} per pair "
      f"({extra[3] / k / 16:.1f} per warp), queue build {extra[4] / k:.0f} cycles/pair (thread 0)")
