"""Ad-hoc stage timing (development aid, not the bench contract)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1404_3448_b200 as sx
from paper_1404_3448_b200 import _lib
from paper_1404_3448_b200.suffix_index import DeviceText, dc3_device, lcp_device
from paper_1404_3448_b200.sequence import encode, gen_random, RankedText

def ev():
    e = torch.cuda.Event(enable_timing=True); e.record(); return e

def time_text(r, sigma, reps=3):
    t = RankedText(r, sigma) if not isinstance(r, RankedText) else r
    dt = DeviceText(t)
    for _ in range(reps):
        torch.cuda.synchronize()
        e0 = ev(); ix = dc3_device(dt); e1 = ev(); lcp = lcp_device(ix); e2 = ev()
        torch.cuda.synchronize()
        print(f"  n={t.n:>11} dc3 {e0.elapsed_time(e1):8.2f} ms ({t.n/e0.elapsed_time(e1)/1e3:8.1f} Mb/s)  lcp {e1.elapsed_time(e2):7.2f} ms", flush=True)

for n in [int(x) for x in sys.argv[1:]] or [1 << 20, 10**7]:
    g = np.random.default_rng(1).integers(1, 5, size=n)
    print("random", n); time_text(g, 4)
a, b = gen_random(10_000_000, 11), gen_random(10_000_000, 12)
ha = np.frombuffer(a.residues.encode(), np.uint8); hb = np.frombuffer(b.residues.encode(), np.uint8)
p = sx.OverlapPipeline(len(ha), len(hb))
for i in range(4):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    res = p.run(ha, hb); t1 = time.perf_counter()
    print("C2 pipeline e2e", res, f"{(t1-t0)*1e3:.2f} ms", flush=True)
p.a[:len(ha)].copy_(torch.from_numpy(ha)); p.b[:len(hb)].copy_(torch.from_numpy(hb))
for i in range(3):
    torch.cuda.synchronize(); e0 = ev(); p.run_device(); e1 = ev(); torch.cuda.synchronize()
    print(f"C2 device {e0.elapsed_time(e1):.2f} ms", flush=True)
