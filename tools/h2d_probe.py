"""Pinned host -> device copy rate for the C4 input size (2 GB), the e2e
ceiling of the batched-pairs step: CUDA events around one copy, then the
same bytes split over 2 / 4 concurrent streams (several copy engines)."""
import torch

n = 2_000_000_000
h = torch.empty(n, dtype=torch.uint8).pin_memory()
d = torch.empty(n, dtype=torch.uint8, device="cuda")
for _ in range(2):
    d.copy_(h, non_blocking=True)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(3):
    d.copy_(h, non_blocking=True)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 3
print(f"H2D 2 GB: {ms:.2f} ms  {n / ms / 1e6:.1f} GB/s")
for k in (2, 4):
    ss = [torch.cuda.Stream() for _ in range(k)]
    part = n // k
    cur = torch.cuda.current_stream()
    torch.cuda.synchronize()
    e0.record()
    for _ in range(3):
        for i, s in enumerate(ss):
            s.wait_stream(cur)
            with torch.cuda.stream(s):
                d[i * part:(i + 1) * part].copy_(h[i * part:(i + 1) * part], non_blocking=True)
        for s in ss:
            cur.wait_stream(s)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 3
    print(f"H2D 2 GB over {k} streams: {ms:.2f} ms  {n / ms / 1e6:.1f} GB/s")
# D2H for the C3 e2e leg
e0.record()
for _ in range(3):
    h.copy_(d, non_blocking=True)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 3
print(f"D2H 2 GB: {ms:.2f} ms  {n / ms / 1e6:.1f} GB/s")
