"""Run one workload step under cudaProfilerStart/Stop (for ncu --profile-from-start off)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1404_3448_b200 as sx
from paper_1404_3448_b200.sequence import gen_random, RankedText
from paper_1404_3448_b200.suffix_index import DeviceText, dc3_device, lcp_device

what = sys.argv[1] if len(sys.argv) > 1 else "c2"
if what == "c5":
    import bench
    wl = bench.C5(0)
    wl.step_device(); wl.step_device()
    torch.cuda.synchronize()
    torch.cuda.profiler.start(); wl.step_device(); torch.cuda.synchronize(); torch.cuda.profiler.stop()
elif what == "c4":
    from paper_1404_3448_b200.workloads import c4_generate
    seqs, offs = c4_generate(0, 100_000)  # the whole C4 batch (on-chip pair DC3: one launch)
    ob = sx.OverlapBatch(seqs, offs)
    ob.run_device(); ob.run_device()
    torch.cuda.synchronize()
    torch.cuda.profiler.start(); ob.run_device(); torch.cuda.synchronize(); torch.cuda.profiler.stop()
elif what == "c2":
    a, b = gen_random(10_000_000, 11), gen_random(10_000_000, 12)
    ha = np.frombuffer(a.residues.encode(), np.uint8); hb = np.frombuffer(b.residues.encode(), np.uint8)
    p = sx.OverlapPipeline(len(ha), len(hb))
    p.run(ha, hb); p.run(ha, hb)
    torch.cuda.synchronize()
    torch.cuda.profiler.start(); p.run_device(); torch.cuda.synchronize(); torch.cuda.profiler.stop()
    print(p.res.cpu())
else:
    # the C3 bench path: SuffixIndexer (SA + LCP, no ISA)
    from paper_1404_3448_b200.suffix_index import SuffixIndexer
    n = int(what)
    ix = SuffixIndexer(n, 4)
    ix.stage(np.random.default_rng(1).integers(1, 5, size=n).astype(np.uint8))
    ix.run_staged(); ix.run_device(); torch.cuda.synchronize()
    torch.cuda.profiler.start(); ix.run_device(); torch.cuda.synchronize(); torch.cuda.profiler.stop()
