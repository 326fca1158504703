"""FASTA ingest oracle (oracle_fasta, a C restatement of parse_fasta +
encode, sequence.py:77-157) pinned against the reference's own outputs
(tests/golden/fasta_cases.json, made by tests/golden/make_fasta_golden.py)."""

import json
import os

import pytest

import oracle
from conftest import ROOT

CASES = os.path.join(ROOT, "tests", "golden", "fasta_cases.json")


@pytest.fixture(scope="module")
def cases():
    with open(CASES) as f:
        return json.load(f)


def test_oracle_matches_reference_records_and_errors(cases):
    for c in cases:
        keep = c["policy"] == "keep"
        recs, err = oracle.fasta(c["input"].encode("ascii"), keep)
        assert err == c["error"], (c["input"][:80], err, c["error"])
        if err is None:
            assert [[r, s.decode(), d] for r, s, d in recs] == c["records"]


def test_oracle_ranks_match_reference_encode(cases):
    for c in cases:
        if c["error"] is not None:
            continue
        recs, _ = oracle.fasta(c["input"].encode("ascii"), c["policy"] == "keep", as_ranks=True)
        assert [list(s) for _, s, _ in recs] == c["ranks"]


def test_golden_covers_error_kinds(cases):
    errs = [c["error"] for c in cases if c["error"]]
    assert any("empty FASTA header" in e for e in errs)
    assert any("before any '>' header" in e for e in errs)
    assert any("illegal residue" in e for e in errs)
