"""Phase timing of save_index / load_index at n = 2^26 (host path breakdown)."""
import io, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1404_3448_b200 import _lib, index_store as ist
from paper_1404_3448_b200.overlap import LcpQueryEngine
from paper_1404_3448_b200.sequence import encode, gen_random

n = 1 << 26
eng = LcpQueryEngine.build(encode(gen_random(n, 21)))
def tm(label, fn):
    torch.cuda.synchronize(); t0 = time.perf_counter(); r = fn(); torch.cuda.synchronize()
    print(f"{label:28s} {1e3*(time.perf_counter()-t0):9.1f} ms", flush=True); return r
for rep in range(3):
    sink = io.BytesIO()
    tm("save_index BytesIO", lambda: ist.save_index(eng, sink))
    sink.seek(0)
    tm("load_index BytesIO", lambda: ist.load_index(sink))
    tm("save_index file", lambda: ist.save_index(eng, "/tmp/x.saix"))
    tm("load_index file", lambda: ist.load_index("/tmp/x.saix"))
    sink.seek(0)
    img = tm("_read_image", lambda: ist._read_image(sink))
    tm("unpack_index", lambda: ist.unpack_index(img))
os.remove("/tmp/x.saix")
