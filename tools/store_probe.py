"""Time the device .saix kernels (pack, CRC-32, unpack) at n = 2^k."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1404_3448_b200 import _lib, index_store
from paper_1404_3448_b200.overlap import LcpQueryEngine
from paper_1404_3448_b200.sequence import encode, gen_random

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 27
eng = LcpQueryEngine.build(encode(gen_random(n, 5)))
L = _lib.load()
t = torch
blob = index_store.pack_index(eng)
payload = 40 + 17 * n
ws = _lib.workspace(max(L.saix_crc32_workspace_bytes(payload), L.saix_index_unpack_workspace_bytes(n)))
from paper_1404_3448_b200.suffix_index import _device_index_of
ix = _device_index_of(eng.text, eng.sa)
lcp = eng.lcp._dev[1]
text_d = _lib.empty(n, t.uint8)
sa_d, lcp_d, isa_d = (_lib.empty(n, t.int32) for _ in range(3))
crc = _lib.empty(1, t.int32)
s = _lib.stream_ptr()

def pack():
    _lib.check(L.saix_index_pack(_lib.ptr(ix.text.t), _lib.ptr(ix.sa), _lib.ptr(lcp), n, 4, 0, _lib.ptr(blob),
                                 _lib.ptr(ws), ws.numel(), s))
def crc32():
    _lib.check(L.saix_crc32(_lib.ptr(blob), payload, _lib.ptr(crc), _lib.ptr(ws), ws.numel(), s))
def unpack():
    _lib.check(L.saix_index_unpack(_lib.ptr(blob), n, _lib.ptr(text_d), _lib.ptr(sa_d), _lib.ptr(lcp_d),
                                   _lib.ptr(isa_d), _lib.ptr(ws), ws.numel(), s))

out = {"n": n}
for name, fn, algo in (("crc32", crc32, 17.0 * n), ("pack", pack, 9.0 * n + 17 * n + 17 * n),
                       ("unpack", unpack, 17.0 * n + 17 * n + 13 * n)):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); reps = 10
    for _ in range(reps):
        fn()
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    out[name] = {"ms": round(ms, 3), "GBps_algo": round(algo / ms / 1e6, 1)}
assert np.array_equal(_lib.u32_to_i64_host(sa_d, n), eng.sa.sa)
assert np.array_equal(_lib.u32_to_i64_host(isa_d, n), eng.sa.rank)
print(json.dumps(out))
