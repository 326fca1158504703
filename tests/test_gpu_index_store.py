"""GPU parity of .saix persistence (index_store.py:65-134): the device-packed
file equals the reference's save_index bytes (tests/golden/index_files.npz),
device load returns the reference's arrays, and the reference's own test
expectations (tests/test_index_store.py of the reference) hold; at large n the
device CRC is checked against zlib.crc32 of the same bytes."""

import io
import os
import random
import zlib

import numpy as np
import pytest

import oracle
from conftest import ROOT
from paper_1404_3448_b200 import _lib, index_store
from paper_1404_3448_b200.overlap import LcpQueryEngine, lcp_query, lcp_query_batch
from paper_1404_3448_b200.sequence import DnaSequence, NPolicy, encode, gen_random

pytestmark = pytest.mark.gpu

INDEX_GOLDEN = os.path.join(ROOT, "tests", "golden", "index_files.npz")


def engine_for(s, policy=NPolicy.REJECT):
    return LcpQueryEngine.build(encode(DnaSequence("t", s), policy))


def saved_bytes(engine):
    sink = io.BytesIO()
    count = index_store.save_index(engine, sink)
    blob = sink.getvalue()
    assert count == len(blob)
    return blob


@pytest.fixture(scope="module")
def blobs():
    g = np.load(INDEX_GOLDEN)
    return [(g[f"text_{k}"].tobytes().decode(), bool(g[f"keep_{k}"]), g[f"blob_{k}"].tobytes())
            for k in range(int(g["count"]))]


class TestGoldenFiles:
    def test_save_matches_reference_bytes(self, blobs):
        for s, keep, blob in blobs:
            eng = engine_for(s, NPolicy.KEEP if keep else NPolicy.REJECT)
            assert saved_bytes(eng) == blob, s[:40]

    def test_load_matches_reference_arrays(self, blobs):
        for s, keep, blob in blobs:
            n = len(s)
            eng = index_store.load_index(io.BytesIO(blob))
            want_sa = np.frombuffer(blob, "<u8", n, 40 + n).astype(np.int64)
            want_lcp = np.frombuffer(blob, "<u8", n, 40 + 9 * n).astype(np.int64)
            assert eng.text.ranks.tolist() == oracle.dna_ranks(s, keep).tolist()
            assert eng.sa.sa.tolist() == want_sa.tolist()
            rank = np.empty(n, np.int64)
            rank[want_sa] = np.arange(n)
            assert eng.sa.rank.tolist() == rank.tolist()
            assert eng.lcp.lcp.tolist() == want_lcp.tolist()

    def test_loaded_engine_answers_queries(self, blobs):
        rng = np.random.default_rng(3)
        for s, keep, blob in blobs:
            n = len(s)
            if n == 0:
                continue
            eng = index_store.load_index(io.BytesIO(blob))
            qi, qj = rng.integers(0, n, 200), rng.integers(0, n, 200)
            sa = eng.sa.sa
            want = oracle.lcp_query(oracle.dna_ranks(s, keep), sa, eng.sa.rank, eng.lcp.lcp, qi, qj)
            assert lcp_query_batch(eng, qi, qj).tolist() == want.tolist()


class TestSaveLoad:
    def test_fixture_sections(self):
        blob = saved_bytes(engine_for("ATTGCTAC"))
        assert blob[:8] == b"SAIX1\x00\x00\x00"
        assert (int.from_bytes(blob[24:32], "little"), int.from_bytes(blob[32:40], "little")) == (8, 4)
        assert list(blob[40:48]) == [1, 4, 4, 3, 2, 4, 1, 2]
        assert np.frombuffer(blob, dtype="<u8", count=8, offset=48).tolist() == [6, 0, 7, 4, 3, 5, 2, 1]

    def test_roundtrip_preserves_queries(self):
        engine = index_store.load_index(io.BytesIO(saved_bytes(engine_for("ATTGCTAC"))))
        assert lcp_query(engine, 6, 0) == 1
        assert lcp_query(engine, 3, 3) == 5

    def test_empty_text(self):
        engine = index_store.load_index(io.BytesIO(saved_bytes(engine_for(""))))
        assert engine.text.n == 0
        assert engine.sa.sa.tolist() == []
        assert engine.rmq is None

    def test_save_is_deterministic(self):
        assert saved_bytes(engine_for("ACGTACGT")) == saved_bytes(engine_for("ACGTACGT"))

    def test_path_based_io(self, tmp_path):
        path = tmp_path / "x.saix"
        engine = engine_for("GATTACA")
        written = index_store.save_index(engine, path)
        assert path.stat().st_size == written
        assert index_store.load_index(path).text == engine.text

    def test_n_flag_set_for_wide_alphabet(self):
        plain = saved_bytes(engine_for("ACGT"))
        wide = saved_bytes(engine_for("ACGTN", NPolicy.KEEP))
        assert int.from_bytes(plain[16:24], "little") == 0
        assert int.from_bytes(wide[16:24], "little") == 1

    def test_random_roundtrips_exact(self):
        rng = random.Random(0)
        for _ in range(30):
            engine = LcpQueryEngine.build(encode(gen_random(rng.randrange(0, 400), rng.randrange(10**6))))
            loaded = index_store.load_index(io.BytesIO(saved_bytes(engine)))
            assert loaded.text == engine.text
            assert loaded.sa.sa.tolist() == engine.sa.sa.tolist()
            assert loaded.sa.rank.tolist() == engine.sa.rank.tolist()
            assert loaded.lcp.lcp.tolist() == engine.lcp.lcp.tolist()

    def test_cartesian_kind_and_bad_kind(self):
        blob = saved_bytes(engine_for("ATTGCTAC"))
        assert lcp_query(index_store.load_index(io.BytesIO(blob), "cartesian"), 3, 3) == 5
        with pytest.raises(ValueError):
            index_store.load_index(io.BytesIO(blob), "bogus")

    def test_host_only_engine_is_saved_identically(self):
        eng = engine_for("GATTACAGATTACA")
        host = LcpQueryEngine.from_parts(eng.text, type(eng.sa)(n=eng.sa.n, sa=eng.sa.sa, rank=eng.sa.rank),
                                         type(eng.lcp)(eng.lcp.lcp))
        assert saved_bytes(host) == saved_bytes(eng)

    def test_sigma_over_255_rejected(self):
        from paper_1404_3448_b200.sequence import RankedText
        t = RankedText(ranks=np.array([1, 300, 2], np.int64), sigma=300)
        eng = LcpQueryEngine.build(t)
        with pytest.raises(ValueError):
            index_store.save_index(eng, io.BytesIO())


class TestCorruption:
    def test_single_byte_payload_corruption_detected(self):
        blob = bytearray(saved_bytes(engine_for("ATTGCTACGGA")))
        rng = random.Random(1)
        for _ in range(50):
            pos = rng.randrange(40, len(blob) - 8)
            flipped = blob.copy()
            flipped[pos] ^= 1 + rng.randrange(255)
            with pytest.raises(index_store.ChecksumError):
                index_store.load_index(io.BytesIO(bytes(flipped)))

    def test_crc_field_corruption_detected(self):
        blob = bytearray(saved_bytes(engine_for("ACGTTGCA")))
        blob[-3] ^= 1  # high (always-zero) half of the stored u64
        with pytest.raises(index_store.ChecksumError):
            index_store.load_index(io.BytesIO(bytes(blob)))

    def test_trailing_bytes_ignored(self):
        blob = saved_bytes(engine_for("ACGTTGCA"))
        eng = index_store.load_index(io.BytesIO(blob + b"junk"))
        assert eng.sa.sa.tolist() == engine_for("ACGTTGCA").sa.sa.tolist()


def test_oracle_values_survive_roundtrip():
    rng = random.Random(2)
    for _ in range(10):
        s = "".join(rng.choice("ACGT") for _ in range(rng.randrange(1, 200)))
        loaded = index_store.load_index(io.BytesIO(saved_bytes(engine_for(s))))
        ranks = oracle.dna_ranks(s)
        sa, rank = oracle.dc3(ranks, 4)
        assert loaded.sa.sa.tolist() == sa.tolist()
        qi = np.array([rng.randrange(len(s)) for _ in range(20)])
        qj = np.array([rng.randrange(len(s)) for _ in range(20)])
        want = oracle.lcp_query(ranks, sa, rank, oracle.lcp(ranks, sa, rank), qi, qj)
        assert lcp_query_batch(loaded, qi, qj).tolist() == want.tolist()


class TestDeviceCrc:
    @pytest.mark.parametrize("nbytes", [0, 1, 15, 255, 256, 257, 4095, 65535, 65536, 65537,
                                        3 * 65536 + 5, 1 << 20, 10_000_019])
    def test_crc_matches_zlib(self, nbytes):
        t = _lib.torch()
        rng = np.random.default_rng(nbytes)
        host = rng.integers(0, 256, nbytes + 16, dtype=np.uint8)
        dev = _lib.to_device(host)
        L = _lib.load()
        for off in (0, 1, 7):
            if off and nbytes > (1 << 20):
                continue
            out = _lib.empty(1, t.int32)
            ws = _lib.workspace(L.saix_crc32_workspace_bytes(nbytes))
            _lib.check(L.saix_crc32(_lib.ptr(dev) + off, nbytes, _lib.ptr(out), _lib.ptr(ws), ws.numel(),
                                    _lib.stream_ptr()), "saix_crc32")
            got = int(out.cpu().numpy().view(np.uint32)[0])
            assert got == zlib.crc32(host[off:off + nbytes].tobytes()), (nbytes, off)


@pytest.mark.parametrize("n", [1 << 20, (1 << 24) + 3])
def test_large_roundtrip(n):
    seq = gen_random(n, 11)
    eng = LcpQueryEngine.build(encode(seq))
    blob = saved_bytes(eng)
    assert len(blob) == 40 + 17 * n + 8
    assert int.from_bytes(blob[-8:], "little") == zlib.crc32(blob[:-8])
    assert np.frombuffer(blob, "<u8", n, 40 + n).astype(np.int64).tolist()[:1000] == eng.sa.sa[:1000].tolist()
    loaded = index_store.load_index(io.BytesIO(blob))
    assert np.array_equal(loaded.sa.sa, eng.sa.sa)
    assert np.array_equal(loaded.sa.rank, eng.sa.rank)
    assert np.array_equal(loaded.lcp.lcp, eng.lcp.lcp)
    assert np.array_equal(np.frombuffer(blob, "<u8", n, 40 + 9 * n).astype(np.int64), eng.lcp.lcp)


def _recrc(blob: bytearray) -> bytes:
    blob[-8:] = zlib.crc32(bytes(blob[:-8])).to_bytes(8, "little")
    return bytes(blob)


def test_crafted_bad_rank_rejected():
    blob = bytearray(saved_bytes(engine_for("ACGTACGT")))
    blob[41] = 0  # rank 0 with a valid checksum
    with pytest.raises(ValueError):
        index_store.load_index(io.BytesIO(_recrc(blob)))


def test_crafted_sa_out_of_range_rejected():
    blob = bytearray(saved_bytes(engine_for("ACGTACGT")))
    blob[48:56] = (99).to_bytes(8, "little")  # sa[0] = 99 >= n
    with pytest.raises(IndexError):
        index_store.load_index(io.BytesIO(_recrc(blob)))


def test_crafted_large_lcp_loads_like_reference():
    # the reference loads any lcp value (index_store.py:128-131); so do we
    blob = bytearray(saved_bytes(engine_for("ACGTACGT")))
    n = 8
    blob[40 + 9 * n + 8: 40 + 9 * n + 16] = (1000).to_bytes(8, "little")  # lcp[1] = 1000 > n
    loaded = index_store.load_index(io.BytesIO(_recrc(blob)))
    assert int(loaded.lcp.lcp[1]) == 1000


def sx_build_lcp(eng):
    from paper_1404_3448_b200.suffix_index import build_lcp
    return build_lcp(eng.text, eng.sa).lcp


def test_sigma_above_255_header_loads_like_reference():
    # one byte per rank in the file whatever sigma says; the reference keeps
    # the header's sigma (index_store.py:126) and so does the device text
    blob = bytearray(saved_bytes(engine_for("ATTGCTAC")))
    blob[32:40] = (300).to_bytes(8, "little")
    loaded = index_store.load_index(io.BytesIO(_recrc(blob)))
    assert loaded.text.sigma == 300
    ref = engine_for("ATTGCTAC")
    assert loaded.sa.sa.tolist() == ref.sa.sa.tolist()
    # test_overlap.py:22-26 answers on ATTGCTAC
    assert lcp_query(loaded, 3, 3) == 5 and lcp_query(loaded, 6, 0) == 1
    assert sx_build_lcp(loaded).tolist() == ref.lcp.lcp.tolist()


def test_widen_matches_host():
    t = _lib.torch()
    rng = np.random.default_rng(5)
    for n in (1, 3, 4, 5, 1000, 1 << 20):
        a = rng.integers(0, 1 << 32, n, dtype=np.uint64).astype(np.uint32)
        assert np.array_equal(_lib.widen_i64_host(_lib.to_device(a.view(np.int32)), n), a.astype(np.int64))
        b = rng.integers(0, 256, n, dtype=np.uint8)
        assert np.array_equal(_lib.widen_i64_host(_lib.to_device(b), n), b.astype(np.int64))
