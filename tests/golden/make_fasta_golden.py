"""Generate FASTA golden cases by running the REFERENCE saix.sequence.

Run in the dev container (the reference exists only there):

    cd /tmp && PYTHONDONTWRITEBYTECODE=1 NUMBA_CACHE_DIR=/tmp/numba_cache \
        python /root/repo/tests/golden/make_fasta_golden.py

Imports the reference from /root/reference/pkg/src (read-only) and writes
tests/golden/fasta_cases.json: for each (input text, policy) the records
parse_fasta returns (id, residues, description) and the ranks encode gives
for each record, or the SequenceError message it raises.
"""

from __future__ import annotations

import json
import os
import random
import sys

REF = "/root/reference/pkg/src"
OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "fasta_cases.json")

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
sys.dont_write_bytecode = True
sys.path.insert(0, REF)

from saix.sequence import NPolicy, SequenceError, encode, parse_fasta, write_fasta, DnaSequence  # noqa: E402


def random_fasta(rng: random.Random, keep: bool) -> str:
    alpha = "ACGTN" if keep else "ACGT"
    lines = []
    for r in range(rng.randrange(1, 6)):
        desc = rng.choice(["", " some description", "\tx", "  two  spaces "])
        lines.append(f">{rng.choice([' ', ''])}rec{r}{desc}{rng.choice(['', ' ', '\\r'])}")
        seq = "".join(rng.choice(alpha + alpha.lower()) for _ in range(rng.randrange(0, 400)))
        w = rng.randrange(1, 90)
        for i in range(0, len(seq), w):
            pre = rng.choice(["", "", " ", "\t"])
            post = rng.choice(["", "", " ", "\r", "\x0b", "\x1c"])
            lines.append(pre + seq[i:i + w] + post)
            if rng.random() < 0.1:
                lines.append(rng.choice(["", "   ", "\r", "\t\t"]))
    text = "\n".join(lines)
    return text + rng.choice(["", "\n", "\n\n", "\r\n"])


def main():
    fixed = [
        "", "\n", "   \n\n", ">a\nACGT\n", ">a\nACGT", ">a desc\nacgt\nAC\n>b\n>c x y\nGG\n",
        ">a\r\nAC\r\nGT\r\n", ">\nACGT\n", ">   \nAC\n", "ACGT\n>a\nAC\n", "\n\nAC\n", ">a\nACGX\n",
        ">a\nAC GT\n", ">a\nACN\n", ">a\nAC\n>b\nTTnT\n", ">a\n\tACGT  \n", ">id\tdesc\nA\n",
        ">a\nAC\rGT\n", ">a b  c\nA\n", ">a\n>b\n", ">x\nA\x0cC\n", ">x\n\x1cAC\x1f\n", ">x\n-\n",
        ">x\nAC\n\n\n   \n>y\nGT\n", "  >x\nAC\n", ">x\nAC\n>\n", ">a\nacgtn\nACGTN\n",
    ]
    rng = random.Random(14043448)
    cases = []
    for text in fixed:
        for pol in ("reject", "keep"):
            cases.append((text, pol))
    for _ in range(60):
        keep = rng.random() < 0.5
        cases.append((random_fasta(rng, keep), "keep" if keep else "reject"))
    # round trips of write_fasta output
    for _ in range(5):
        recs = [DnaSequence(f"s{k}", "".join(rng.choice("ACGT") for _ in range(rng.randrange(0, 300))),
                            rng.choice(["", "d e s c"])) for k in range(rng.randrange(1, 5))]
        cases.append((write_fasta(recs, width=rng.randrange(1, 80)), "reject"))
    out = []
    for text, pol in cases:
        policy = NPolicy.KEEP if pol == "keep" else NPolicy.REJECT
        entry = {"input": text, "policy": pol}
        try:
            recs = parse_fasta(text, policy)
            entry["records"] = [[r.id, r.residues, r.description] for r in recs]
            entry["ranks"] = [encode(r, policy).ranks.tolist() for r in recs]
            entry["error"] = None
        except SequenceError as e:
            entry["records"] = None
            entry["error"] = str(e)
        out.append(entry)
    with open(OUT, "w") as f:
        json.dump(out, f)
    print("wrote", OUT, len(out), "cases;", sum(e["error"] is not None for e in out), "errors")


if __name__ == "__main__":
    main()
