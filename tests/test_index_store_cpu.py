""".saix files on the CPU side: the oracle's file image against the
reference's own save_index output (tests/golden/index_files.npz, made by
tests/golden/make_index_golden.py), and load_index's header checks, which
run on the host before anything touches the device (index_store.py:99-116;
mirrors the reference's tests/test_index_store.py::TestCorruption)."""

import io
import os
import struct
import zlib

import numpy as np
import pytest

import oracle
from conftest import ROOT
from paper_1404_3448_b200 import index_store

INDEX_GOLDEN = os.path.join(ROOT, "tests", "golden", "index_files.npz")


@pytest.fixture(scope="module")
def blobs():
    g = np.load(INDEX_GOLDEN)
    out = []
    for k in range(int(g["count"])):
        out.append((g[f"text_{k}"].tobytes().decode(), bool(g[f"keep_{k}"]), g[f"blob_{k}"].tobytes()))
    return out


def test_golden_files_are_well_formed(blobs):
    for s, keep, blob in blobs:
        n = len(s)
        assert blob[:8] == b"SAIX1\x00\x00\x00"
        version, flags, nn, sigma = struct.unpack_from("<4Q", blob, 8)
        assert (version, nn) == (1, n)
        assert sigma == (5 if keep else 4)
        assert flags == (1 if keep else 0)
        assert len(blob) == 40 + 17 * n + 8
        assert struct.unpack_from("<Q", blob, len(blob) - 8)[0] == zlib.crc32(blob[:-8])


def test_oracle_file_image_matches_reference(blobs):
    for s, keep, blob in blobs:
        ranks = oracle.dna_ranks(s, keep)
        sigma = 5 if keep else 4
        if len(s):
            sa, rank = oracle.dc3(ranks, sigma)
            lcp = oracle.lcp(ranks, sa, rank)
        else:
            sa = lcp = np.zeros(0, np.int64)
        assert oracle.index_file(ranks, sigma, sa, lcp) == blob


def test_fixture_sections(blobs):
    s, _, blob = blobs[2]
    assert s == "ATTGCTAC"
    assert list(blob[40:48]) == [1, 4, 4, 3, 2, 4, 1, 2]
    assert np.frombuffer(blob, dtype="<u8", count=8, offset=48).tolist() == [6, 0, 7, 4, 3, 5, 2, 1]


def test_bad_magic(blobs):
    blob = bytearray(blobs[2][2])
    blob[0] ^= 0xFF
    with pytest.raises(index_store.BadMagicError):
        index_store.load_index(io.BytesIO(bytes(blob)))


def test_unsupported_version(blobs):
    blob = bytearray(blobs[2][2])
    blob[8] = 9
    with pytest.raises(index_store.UnsupportedVersionError):
        index_store.load_index(io.BytesIO(bytes(blob)))


def test_truncation(blobs):
    blob = blobs[2][2]
    for cut in (0, 5, 20, 47, len(blob) - 1):
        with pytest.raises(index_store.TruncatedFileError):
            index_store.load_index(io.BytesIO(blob[:cut]))


def test_truncation_with_inflated_n(blobs):
    blob = bytearray(blobs[2][2])
    blob[24:32] = struct.pack("<Q", 1 << 40)
    with pytest.raises(index_store.TruncatedFileError):
        index_store.load_index(io.BytesIO(bytes(blob)))


def test_errors_are_distinct_types():
    kinds = {index_store.BadMagicError, index_store.UnsupportedVersionError,
             index_store.ChecksumError, index_store.TruncatedFileError}
    assert len(kinds) == 4
    for kind in kinds:
        assert issubclass(kind, index_store.IndexFileError)


def test_path_errors(tmp_path, blobs):
    p = tmp_path / "bad.saix"
    p.write_bytes(b"SAIX0" + bytes(50))
    with pytest.raises(index_store.BadMagicError):
        index_store.load_index(p)


def test_oracle_index_load_roundtrip(blobs):
    for s, keep, blob in blobs:
        ranks, sigma, sa, rank, lcp = oracle.index_load(blob)
        assert ranks.tolist() == oracle.dna_ranks(s, keep).tolist()
        assert oracle.index_file(ranks, sigma, sa, lcp) == blob
        if len(s):
            assert rank[sa].tolist() == list(range(len(s)))
    bad = bytearray(blobs[3][2])
    bad[45] ^= 4
    with pytest.raises(ValueError):
        oracle.index_load(bytes(bad))
