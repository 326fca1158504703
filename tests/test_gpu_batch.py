"""Batched longest_overlap (C4 path): equals the scalar reference answer for
every pair, across waves, ragged / empty pairs and residue errors."""

import numpy as np
import pytest

import oracle
import paper_1404_3448_b200 as sx
from paper_1404_3448_b200.sequence import DnaSequence
from paper_1404_3448_b200.workloads import c4_pairs

pytestmark = pytest.mark.gpu


def golden_pairs(g):
    ao, bo = g["ov_aoffs"], g["ov_boffs"]
    out = []
    for c in range(len(ao) - 1):
        a = g["ov_a"][ao[c]:ao[c + 1]].tobytes().decode()
        b = g["ov_b"][bo[c]:bo[c + 1]].tobytes().decode()
        out.append((DnaSequence("a", a), DnaSequence("b", b)))
    return out


def test_golden_pairs_as_one_batch(golden):
    pairs = golden_pairs(golden)
    got = sx.longest_overlap_batch(pairs)
    want = [tuple(int(x) for x in r) for r in golden["ov_ans"]]
    assert [(r.length, r.pos_a, r.pos_b) for r in got] == want


def test_c4_pairs_vs_oracle_and_waves():
    seqs, offs = c4_pairs(0, 64, length=3000)
    want = oracle.overlap_batch(seqs, offs, threads=4)
    ob = sx.OverlapBatch(seqs, offs)
    ob.run_device()
    assert np.array_equal(ob.results(), want)
    small = sx.OverlapBatch(seqs, offs, wave_residues=20_000)   # many waves
    assert len(small.waves) > 4
    small.run_device()
    assert np.array_equal(small.results(), want)


def test_ragged_and_empty_pairs():
    rng = np.random.default_rng(4)
    pairs = []
    for _ in range(50):
        la, lb = (int(v) for v in rng.integers(0, 400, size=2))
        if rng.random() < 0.1:
            la = 0
        a = "".join(rng.choice(list("ACGT"), size=la))
        b = "".join(rng.choice(list("ACGT"), size=lb))
        pairs.append((DnaSequence("a", a), DnaSequence("b", b)))
    got = sx.longest_overlap_batch(pairs)
    for (a, b), r in zip(pairs, got):
        assert (r.length, r.pos_a, r.pos_b) == oracle.longest_overlap(a.residues, b.residues)


def test_first_bad_pair_raises_like_reference():
    pairs = [(DnaSequence("a0", "ACGT"), DnaSequence("b0", "GT")),
             (DnaSequence("a1", "ACGT"), DnaSequence("b1", "GXT")),
             (DnaSequence("a2", "NNN"), DnaSequence("b2", "AC"))]
    with pytest.raises(sx.SequenceError, match="record 'b1'.*'X' at position 1"):
        sx.longest_overlap_batch(pairs)
    ok = sx.longest_overlap_batch([(DnaSequence("a", ""), DnaSequence("b", "XYZ"))])
    assert ok == [sx.OverlapResult(0, 0, 0)]


def test_many_short_pairs_two_partition_passes():
    """> 256 pairs per wave: the pair-id partition takes two LSD passes."""
    seqs, offs = c4_pairs(0, 1500, length=300)
    want = oracle.overlap_batch(seqs, offs, threads=4)
    ob = sx.OverlapBatch(seqs, offs)
    ob.run_device()
    assert np.array_equal(ob.results(), want)


def test_keep_n_pairs_byte_compare():
    rng = np.random.default_rng(5)
    pairs = []
    for _ in range(40):
        a = "".join(rng.choice(list("ACGTN"), size=1500))
        b = list("".join(rng.choice(list("ACGTN"), size=1500)))
        b[300:700] = a[900:1300]
        pairs.append((DnaSequence("a", a), DnaSequence("b", "".join(b))))
    got = sx.longest_overlap_batch(pairs, sx.NPolicy.KEEP)
    for (a, b), r in zip(pairs, got):
        assert (r.length, r.pos_a, r.pos_b) == oracle.longest_overlap(a.residues, b.residues, keep_n=True)
        assert r.length >= 400


def test_repetitive_pairs_kasai_fallback():
    """Most adjacent LCPs exceed the direct-compare cap: the Phi/PLCP path."""
    pairs = [(DnaSequence("a", "A" * 3000), DnaSequence("b", "A" * 2000 + "C")),
             (DnaSequence("a", "ACG" * 900), DnaSequence("b", "CGA" * 700)),
             (DnaSequence("a", "AC" * 10), DnaSequence("b", "GT" * 10))]
    got = sx.longest_overlap_batch(pairs)
    for (a, b), r in zip(pairs, got):
        assert (r.length, r.pos_a, r.pos_b) == oracle.longest_overlap(a.residues, b.residues)


def test_full_wave_c4_scale():
    """One full 2^27-residue wave of C4 pairs (byte levels on the bucketed
    scatter, planted repeats -> tie resolution at the wide level); a spread
    subset of pairs against the oracle."""
    seqs, offs = c4_pairs(0, 6700)
    ob = sx.OverlapBatch(seqs, offs)
    assert len(ob.waves) == 1
    ob.run_device()
    got = ob.results()
    idx = list(range(0, 6700, 23))
    for p in idx:
        a = seqs[offs[2 * p]:offs[2 * p + 1]].tobytes()
        b = seqs[offs[2 * p + 1]:offs[2 * p + 2]].tobytes()
        assert tuple(int(x) for x in got[p]) == oracle.longest_overlap(a, b), p


# ---------------------------------------------------------------- on-chip path
# saix_overlap_batch runs every pair of <= 20,480 GSA residues in one CTA
# (csrc/pairdc3.cu) and sends longer / over-budget pairs to the wave-global
# DC3; both must give the reference's answer (overlap.py:110-152).

def _rnd(rng, k, alpha=b"ACGT"):
    return np.frombuffer(alpha, np.uint8)[rng.integers(0, len(alpha), k)].tobytes()


def _batch(pairs_bytes, keep=False):
    seqs = np.frombuffer(b"".join(a + b for a, b in pairs_bytes), np.uint8)
    offs = [0]
    for a, b in pairs_bytes:
        offs += [offs[-1] + len(a), offs[-1] + len(a) + len(b)]
    return seqs, np.asarray(offs, np.int64)


def _run(seqs, offs, keep=False, onchip=True):
    from paper_1404_3448_b200 import _lib
    L = _lib.load()
    prev = L.saix_overlap_batch_set_onchip(int(onchip))
    try:
        ob = sx.OverlapBatch(seqs, offs, sx.NPolicy.KEEP if keep else sx.NPolicy.REJECT)
        ob.run_device()
        return ob.results()
    finally:
        L.saix_overlap_batch_set_onchip(prev)


def test_onchip_equals_wave_global_and_oracle():
    seqs, offs = c4_pairs(0, 3000)
    want = oracle.overlap_batch(seqs, offs, threads=8)
    assert np.array_equal(_run(seqs, offs, onchip=True), want)
    from paper_1404_3448_b200 import _lib
    assert _lib.load().saix_overlap_batch_last_fallbacks() == 0   # all C4 pairs stayed on chip
    assert np.array_equal(_run(seqs[: offs[600]], offs[:601], onchip=False), want[:300])
    assert _lib.load().saix_overlap_batch_last_fallbacks() == 300


def test_onchip_small_pairs_every_length_mod3():
    rng = np.random.default_rng(11)
    pairs = []
    for la in range(1, 25):
        for lb in range(1, 25):
            a = _rnd(rng, la)
            b = _rnd(rng, lb, b"AC")
            pairs.append((a, b))
    seqs, offs = _batch(pairs)
    want = oracle.overlap_batch(seqs, offs, threads=8)
    assert np.array_equal(_run(seqs, offs), want)


def test_onchip_mixed_with_fallback_pairs():
    """Poly-A and tandem-repeat pairs (buckets / comparisons over the on-chip
    bounds), pairs longer than 20,480 residues, pairs right at the limit,
    empty sides and ordinary pairs in one call."""
    rng = np.random.default_rng(12)

    def rnd(k, alpha=b"ACGT"):
        return _rnd(rng, k, alpha)

    pairs = [
        (b"A" * 9000, b"A" * 8000 + b"C"),                      # one huge bucket
        (b"ACGT" * 2500, b"TACG" * 2400),                       # long periodic repeats
        (rnd(15000), rnd(12000)),                                # longer than the on-chip limit
        (rnd(10239), rnd(10240)),                                # n = 20480 exactly
        (rnd(10240), rnd(10240)),                                # n = 20481
        (b"", rnd(50)), (rnd(50), b""),
        (rnd(5000), rnd(5000)),
        (b"AT" * 300 + rnd(3000), rnd(2000) + b"AT" * 280),       # bucket of ~200 samples
        (rnd(10000, b"AT"), rnd(10000, b"AT")),                   # two-letter text: big buckets, long LCPs
    ]
    a, b = rnd(10000), bytearray(rnd(10000))
    b[4000:4256] = a[1234:1490]                                   # planted block of 256
    pairs.append((a, bytes(b)))
    seqs, offs = _batch(pairs)
    want = oracle.overlap_batch(seqs, offs, threads=8)
    got = _run(seqs, offs)
    assert np.array_equal(got, want), np.flatnonzero(np.any(got != want, axis=1))
    assert tuple(got[-1]) >= (256,)


def test_onchip_keep_n_and_reject():
    rng = np.random.default_rng(13)
    pairs = []
    for _ in range(30):
        a = _rnd(rng, 4000, b"ACGTN")
        b = bytearray(_rnd(rng, 3000, b"ACGTN"))
        b[100:400] = a[2000:2300]
        pairs.append((a, bytes(b)))
    seqs, offs = _batch(pairs)
    want = oracle.overlap_batch(seqs, offs, keep_n=True, threads=8)
    assert np.array_equal(_run(seqs, offs, keep=True), want)
    ob = sx.OverlapBatch(seqs, offs)                             # REJECT: the first N in the batch
    ob.run_device()
    first = int(np.flatnonzero(seqs == ord("N"))[0])
    assert ob.first_bad() == first


@pytest.mark.parametrize("stream_chunks", [0, 1, 7, 32, 700])
def test_run_from_host_chunks_match_device_run(stream_chunks):
    """H2D overlapped with the pairs (run_from_host): one launch gated on the
    copy engine's per-chunk counts (saix_overlap_batch_stream, 1..700
    chunks), or one launch per chunk (0) -- the device-resident answers, and
    an illegal residue in a later chunk reported at its absolute offset."""
    import torch
    seqs, offs = c4_pairs(0, 700)
    want = oracle.overlap_batch(seqs, offs, threads=8)
    ob = sx.OverlapBatch(seqs, offs, chunks=5)
    assert len(ob.chunks) == 5
    host = torch.from_numpy(seqs.copy()).pin_memory()
    ob.seqs_dev.zero_()
    ob.run_from_host(host, stream_chunks=stream_chunks)
    assert np.array_equal(ob.results(), want)
    bad_at = int(offs[2 * 650 + 1]) + 17
    host[bad_at] = ord("Q")
    ob.run_from_host(host, stream_chunks=stream_chunks)
    assert ob.first_bad() == bad_at


def test_stream_entry_rejects_blocking_copy_stream():
    """saix_overlap_batch_stream refuses a copy stream the legacy default
    stream could serialise behind the gated kernel (a deadlock otherwise):
    no stream, the launch stream itself, or a blocking stream (the
    per-thread default stream, handle 2)."""
    import torch
    from paper_1404_3448_b200 import _lib
    seqs, offs = c4_pairs(0, 3)
    ob = sx.OverlapBatch(seqs, offs)
    host = torch.from_numpy(seqs.copy()).pin_memory()
    a, b, o, od = ob._calls["waves"][0]
    L = _lib.load()
    cur = torch.cuda.current_stream().cuda_stream
    for cs in (None, cur, 2):
        rc = L.saix_overlap_batch_stream(_lib.ptr(ob.seqs_dev), host.data_ptr(), o.ctypes.data, _lib.ptr(od), b - a,
                                         2, 0, _lib.ptr(ob.out), _lib.ptr(ob.bad), _lib.ptr(ob.ws), ob.ws.numel(),
                                         cur, cs)
        assert rc == _lib.SAIX_EINVAL, cs
    assert b"NonBlocking" in L.saix_last_error()
    ob.run_from_host(host)  # the default path still works afterwards
    assert np.array_equal(ob.results(), oracle.overlap_batch(seqs, offs))


@pytest.mark.parametrize("stream_chunks", [4, 64])
def test_run_from_host_ramped_chunk_plan(stream_chunks):
    """A batch big enough for the streamed chunk plan's ramps (chunks of 296,
    592, 1184 pairs at both ends around the uniform ones, pd::stream_plan):
    answers equal the oracle, and an illegal residue inside the last, smallest
    chunk is reported at its absolute offset."""
    import torch
    seqs, offs = c4_pairs(0, 5000)
    want = oracle.overlap_batch(seqs, offs, threads=16)
    ob = sx.OverlapBatch(seqs, offs)
    host = torch.from_numpy(seqs.copy()).pin_memory()
    ob.seqs_dev.zero_()
    ob.run_from_host(host, stream_chunks=stream_chunks)
    assert np.array_equal(ob.results(), want)
    bad_at = int(offs[2 * 4990]) + 5
    host[bad_at] = ord("Z")
    ob.run_from_host(host, stream_chunks=stream_chunks)
    assert ob.first_bad() == bad_at
