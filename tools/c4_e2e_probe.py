"""C4 end-to-end breakdown: the 2 GB pinned H2D alone, the device-resident
step, and run_from_host at several chunk counts (CUDA events, after warm-up)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1404_3448_b200 as sx  # noqa: E402
from paper_1404_3448_b200.workloads import c4_generate  # noqa: E402

seqs, offs = c4_generate(0, 100_000)
ob = sx.OverlapBatch(seqs, offs)
h = torch.from_numpy(seqs).pin_memory()
hout = torch.empty(3 * 100_000, dtype=torch.int64, pin_memory=True)


def ev():
    e = torch.cuda.Event(enable_timing=True)
    e.record()
    return e


def timed(fn, reps=4):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        e0 = ev()
        fn()
        e1 = ev()
        torch.cuda.synchronize()
        ts.append((e0.elapsed_time(e1), (time.perf_counter() - t0) * 1e3))
    return min(t[0] for t in ts), min(t[1] for t in ts)


print("H2D 2 GB         events %.2f ms wall %.2f ms" % timed(lambda: ob.seqs_dev[: h.numel()].copy_(h, non_blocking=True)))
print("device step      events %.2f ms wall %.2f ms" % timed(ob.run_device))
for ch in (8, 16, 32, 64):
    def step(ch=ch):
        ob.run_from_host(h, stream_chunks=ch)
        hout.copy_(ob.out[: 3 * 100_000], non_blocking=True)
    print(f"e2e chunks={ch:3d}   events %.2f ms wall %.2f ms" % timed(step))
