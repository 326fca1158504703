"""One saix_overlap_batch call over the first K C4 pairs under
cudaProfilerStart/Stop (for ncu --profile-from-start off)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1404_3448_b200 as sx  # noqa: E402
from paper_1404_3448_b200.workloads import c4_generate  # noqa: E402

k = int(sys.argv[1]) if len(sys.argv) > 1 else 4000
seqs, offs = c4_generate(0, k)
ob = sx.OverlapBatch(seqs, offs)
ob.run_device()
ob.run_device()
torch.cuda.synchronize()
torch.cuda.profiler.start()
ob.run_device()
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print(ob.results()[:3])
