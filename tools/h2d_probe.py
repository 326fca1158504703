"""Pinned host -> device copy rate for the C4 input size (2 GB), the e2e
ceiling of the batched-pairs step: CUDA events around one copy."""
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
