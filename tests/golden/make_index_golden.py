"""Generate .saix golden files by running the REFERENCE saix.index_store.

Run in the dev container (the reference exists only there):

    cd /tmp && PYTHONDONTWRITEBYTECODE=1 NUMBA_CACHE_DIR=/tmp/numba_cache \
        python /root/repo/tests/golden/make_index_golden.py

Imports the reference from /root/reference/pkg/src (read-only) and writes
tests/golden/index_files.npz: for each case the exact bytes the reference's
save_index writes (blob_<k>) plus the source string and N policy.
"""

from __future__ import annotations

import io
import os
import random
import sys

import numpy as np

REF = "/root/reference/pkg/src"
OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "index_files.npz")

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
sys.dont_write_bytecode = True
sys.path.insert(0, REF)

from saix import index_store  # noqa: E402
from saix.overlap import LcpQueryEngine  # noqa: E402
from saix.sequence import DnaSequence, NPolicy, encode, gen_random  # noqa: E402


def main():
    rng = random.Random(1404)
    cases = [("", "reject"), ("A", "reject"), ("ATTGCTAC", "reject"), ("GATTACA", "reject"),
             ("ACGTN", "keep"), ("NNNNACGTNNAC" * 5, "keep"), (gen_random(300, 5).residues, "reject"),
             ("A" * 500, "reject")]
    for _ in range(6):
        cases.append(("".join(rng.choice("ACGT") for _ in range(rng.randrange(1, 3000))), "reject"))
    cases.append(("".join(rng.choice("ACGTN") for _ in range(2000)), "keep"))
    out = {}
    for k, (s, pol) in enumerate(cases):
        policy = NPolicy.KEEP if pol == "keep" else NPolicy.REJECT
        engine = LcpQueryEngine.build(encode(DnaSequence("t", s), policy))
        sink = io.BytesIO()
        index_store.save_index(engine, sink)
        out[f"blob_{k}"] = np.frombuffer(sink.getvalue(), np.uint8)
        out[f"text_{k}"] = np.frombuffer(s.encode(), np.uint8)
        out[f"keep_{k}"] = np.array(pol == "keep")
    out["count"] = np.array(len(cases))
    np.savez_compressed(OUT, **out)
    print("wrote", OUT, len(cases), "cases")


if __name__ == "__main__":
    main()
