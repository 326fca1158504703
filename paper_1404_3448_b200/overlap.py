"""LCP queries and longest-overlap search on the B200 -- drop-in for
``saix.overlap`` (overlap.py:28-180).

``longest_overlap`` runs end to end on the device: ASCII A and B are copied
once, encoded into the generalized text on the GPU, and DC3, Kasai LCP and
the two-pass overlap scan run back to back on one stream; only the three
result integers (plus the residue-check word) come back.
"""

from __future__ import annotations

import ctypes
import json
from dataclasses import dataclass, field
from typing import Any, Literal

import numpy as np

from . import _lib
from .rmq import CartesianRmq, SparseTable
from .sequence import (DnaSequence, NPolicy, RankedText, SequenceError, alphabet, encode,
                       residue_error)
from .suffix_index import (LcpArray, SuffixArray, _device_index_of, build_lcp, build_sa_dc3)

RmqKind = Literal["sparse", "cartesian"]

SEPARATOR_RANK = 1  # between the padding sentinel 0 and every residue rank
INT64_MAX = np.iinfo(np.int64).max


@dataclass(frozen=True, eq=False)
class LcpQueryEngine:
    """Text + suffix array + LCP array + RMQ over the LCP (overlap.py:28-55)."""

    text: RankedText
    sa: SuffixArray
    lcp: LcpArray
    rmq: SparseTable | CartesianRmq | None
    _isa_dev: Any = field(default=None, repr=False, compare=False)

    @classmethod
    def build(cls, text: RankedText, rmq_kind: RmqKind = "sparse",
              sa: SuffixArray | None = None) -> "LcpQueryEngine":
        sa = sa or build_sa_dc3(text)
        lcp = build_lcp(text, sa)
        return cls.from_parts(text, sa, lcp, rmq_kind)

    @classmethod
    def from_parts(cls, text: RankedText, sa: SuffixArray, lcp: LcpArray,
                   rmq_kind: RmqKind = "sparse") -> "LcpQueryEngine":
        if rmq_kind not in ("sparse", "cartesian"):
            raise ValueError(f"unknown rmq kind {rmq_kind!r}")
        if text.n == 0:
            return cls(text=text, sa=sa, lcp=lcp, rmq=None)
        if rmq_kind == "cartesian":  # the reference's parity engine (rmq.py:239-251), on the device
            return cls(text=text, sa=sa, lcp=lcp, rmq=CartesianRmq(lcp.lcp))
        dev_vals = (lcp._dev[1], 4) if lcp._dev is not None else None
        rmq = SparseTable(lcp.lcp, _device_values=dev_vals)
        isa = _device_index_of(text, sa).isa
        return cls(text=text, sa=sa, lcp=lcp, rmq=rmq, _isa_dev=isa)


def lcp_query_batch(engine: LcpQueryEngine, i, j) -> np.ndarray:
    """Vectorised ``lcp_query`` (overlap.py:58-69): one device kernel."""
    n = engine.text.n
    qi = np.ascontiguousarray(i, dtype=np.int64)
    qj = np.ascontiguousarray(j, dtype=np.int64)
    if qi.shape != qj.shape:
        raise ValueError("i and j must have the same shape")
    if qi.size == 0:
        return np.zeros(qi.shape, np.int64)
    if n == 0:
        raise IndexError(f"positions ({int(qi.ravel()[0])}, {int(qj.ravel()[0])}) "
                         f"out of bounds for length 0")
    st = engine.rmq
    if isinstance(st, CartesianRmq):  # overlap.py:58-69 through the Cartesian engine
        fi, fj = qi.ravel(), qj.ravel()
        bad = np.flatnonzero((fi < 0) | (fi >= n) | (fj < 0) | (fj >= n))
        if bad.size:
            raise IndexError(f"positions ({int(fi[bad[0]])}, {int(fj[bad[0]])}) out of bounds for length {n}")
        ri, rj = engine.sa.rank[fi], engine.sa.rank[fj]
        lo, hi = np.minimum(ri, rj), np.maximum(ri, rj)
        same = fi == fj
        k = st.query_batch(np.where(same, 0, lo + 1), np.where(same, 0, hi))
        return np.where(same, n - fi, engine.lcp.lcp[k]).reshape(qi.shape)
    t = _lib.torch()
    L = _lib.load()
    di, dj = _lib.to_device(qi.ravel()), _lib.to_device(qj.ravel())
    out = t.empty(qi.size, dtype=t.int64, device=di.device)
    st._err.zero_()
    rc = L.saix_lcp_query(ctypes.byref(st.plan), _lib.ptr(st._table), _lib.ptr(st._vals), st._vbytes,
                          _lib.ptr(engine._isa_dev), _lib.ptr(di), _lib.ptr(dj), qi.size, _lib.ptr(out),
                          _lib.ptr(st._err), _lib.stream_ptr())
    _lib.check(rc, "saix_lcp_query")
    res = out.cpu().numpy()
    if int(st._err.item()):
        f = qi.ravel(), qj.ravel()
        bad = np.flatnonzero((f[0] < 0) | (f[0] >= n) | (f[1] < 0) | (f[1] >= n))[0]
        raise IndexError(f"positions ({int(f[0][bad])}, {int(f[1][bad])}) out of bounds for length {n}")
    return res.reshape(qi.shape)


def lcp_query(engine: LcpQueryEngine, i: int, j: int) -> int:
    """Longest common prefix of suffix(i) and suffix(j) (overlap.py:58-69)."""
    n = engine.text.n
    if not (0 <= i < n) or not (0 <= j < n):
        raise IndexError(f"positions ({i}, {j}) out of bounds for length {n}")
    return int(lcp_query_batch(engine, np.array([i]), np.array([j]))[0])


@dataclass(frozen=True, eq=False)
class GeneralizedText:
    """encode(A)+1 ++ [separator 1] ++ encode(B)+1 (overlap.py:72-98)."""

    ranks: np.ndarray
    boundary: int
    len_a: int
    len_b: int
    sigma: int

    @classmethod
    def build(cls, a: DnaSequence, b: DnaSequence,
              policy: NPolicy = NPolicy.REJECT) -> "GeneralizedText":
        ra, rb = encode(a, policy), encode(b, policy)
        ranks = np.concatenate([ra.ranks + 1, np.array([SEPARATOR_RANK], np.int64), rb.ranks + 1])
        return cls(ranks=ranks, boundary=ra.n, len_a=ra.n, len_b=rb.n,
                   sigma=max(ra.sigma, rb.sigma) + 1)

    def to_ranked_text(self) -> RankedText:
        return RankedText(ranks=self.ranks, sigma=self.sigma)


@dataclass(frozen=True)
class OverlapResult:
    """Longest common substring of A and B; zero length pins positions to 0."""

    length: int
    pos_a: int
    pos_b: int


def _ascii(seq: DnaSequence) -> np.ndarray:
    return np.frombuffer(seq.residues.encode("ascii"), dtype=np.uint8)


class OverlapPipeline:
    """Reusable device buffers for the end-to-end pair pipeline
    (saix_longest_overlap): ASCII in, (length, pos_a, pos_b) out."""

    def __init__(self, na: int, nb: int):
        t = _lib.torch()
        L = _lib.load()
        dev = _lib.device()
        self.na, self.nb = na, nb
        self.a = t.empty(max(na, 1), dtype=t.uint8, device=dev)
        self.b = t.empty(max(nb, 1), dtype=t.uint8, device=dev)
        self.res = t.zeros(4, dtype=t.int64, device=dev)  # out3 + bad_pos
        self.ws = _lib.workspace(L.saix_longest_overlap_workspace_bytes(na, nb))
        # pinned host staging: the e2e path copies host ASCII in and 32 B out
        self.ha = t.empty(max(na, 1), dtype=t.uint8, pin_memory=True)
        self.hb = t.empty(max(nb, 1), dtype=t.uint8, pin_memory=True)
        self.hres = t.empty(4, dtype=t.int64, pin_memory=True)

    def run_device(self, policy: NPolicy = NPolicy.REJECT) -> None:
        """Run on the already-resident self.a / self.b (no host traffic)."""
        L = _lib.load()
        rc = L.saix_longest_overlap(_lib.ptr(self.a), self.na, _lib.ptr(self.b), self.nb,
                                    int(policy is NPolicy.KEEP), _lib.ptr(self.res),
                                    _lib.ptr(self.res) + 24, _lib.ptr(self.ws), self.ws.numel(),
                                    _lib.stream_ptr())
        _lib.check(rc, "saix_longest_overlap")

    def stage(self, a_host: np.ndarray, b_host: np.ndarray) -> None:
        """Copy host ASCII into the pinned staging buffers (outside timing)."""
        self.ha.numpy()[: self.na] = a_host
        self.hb.numpy()[: self.nb] = b_host

    def run_staged(self, policy: NPolicy = NPolicy.REJECT) -> np.ndarray:
        """Pinned host -> device, pipeline, result -> pinned host (e2e step)."""
        self.a[: self.na].copy_(self.ha[: self.na], non_blocking=True)
        self.b[: self.nb].copy_(self.hb[: self.nb], non_blocking=True)
        self.run_device(policy)
        self.hres.copy_(self.res, non_blocking=True)
        _lib.torch().cuda.current_stream().synchronize()
        return self.hres.numpy().copy()

    def run(self, a_host, b_host, policy: NPolicy = NPolicy.REJECT) -> np.ndarray:
        """Host ASCII in, host int64[4] (length, pos_a, pos_b, bad_pos) out."""
        self.stage(a_host, b_host)
        return self.run_staged(policy)


_PIPES: "OrderedDict[tuple, OverlapPipeline]" = None  # type: ignore[assignment]
_PIPES_LOCK = None
_PIPES_MAX = 4


def _pipeline(na: int, nb: int) -> "OverlapPipeline":
    """A reusable OverlapPipeline for this (|A|, |B|, device, thread): repeated
    calls reuse its workspace and pinned staging buffers instead of
    allocating them per call (small LRU)."""
    global _PIPES, _PIPES_LOCK
    import threading
    from collections import OrderedDict
    if _PIPES_LOCK is None:
        _PIPES, _PIPES_LOCK = OrderedDict(), threading.Lock()
    key = (na, nb, _lib.torch().cuda.current_device(), threading.get_ident())
    with _PIPES_LOCK:
        p = _PIPES.pop(key, None)
        if p is None:
            p = OverlapPipeline(na, nb)
        _PIPES[key] = p
        while len(_PIPES) > _PIPES_MAX:
            _PIPES.popitem(last=False)
    return p


# Largest pair (|A| + 1 + |B| generalized-text residues) the on-chip pair
# kernel solves in one CTA (pd::NMAX, csrc/pairdc3.cu)
ONCHIP_RESIDUES = 20480


class SmallPairPipeline:
    """``longest_overlap`` of one pair of up to ONCHIP_RESIDUES residues
    through the on-chip pair kernel (saix_overlap_batch, one pair): a single
    launch instead of the multi-pass DC3 pipeline.  One instance serves every
    pair shape: buffers are sized for the largest pair, A and B are copied
    back to back into one pinned staging buffer and moved with one H2D copy."""

    def __init__(self):
        t = _lib.torch()
        L = _lib.load()
        dev = _lib.device()
        cap = ONCHIP_RESIDUES
        self.seqs = t.empty(cap, dtype=t.uint8, device=dev)
        self.res = t.zeros(4, dtype=t.int64, device=dev)     # out3 + bad offset
        self.hseqs = t.empty(cap, dtype=t.uint8, pin_memory=True)
        self.hres = t.empty(4, dtype=t.int64, pin_memory=True)
        # workspace for the largest pair, whatever its A/B split
        need = max(L.saix_overlap_batch_workspace_bytes(
            np.array([0, na, cap - 1], dtype=np.int64).ctypes.data, 1) for na in (1, cap // 2, cap - 2))
        self.ws = _lib.workspace(need)

    def run(self, a_host: np.ndarray, b_host: np.ndarray, policy: NPolicy = NPolicy.REJECT) -> np.ndarray:
        """Host ASCII in, host int64[4] (length, pos_a, pos_b, bad) out, bad in
        saix_longest_overlap's convention (generalized-text position: B's
        residue k at |A| + 1 + k; INT64_MAX when every residue is legal)."""
        na, nb = len(a_host), len(b_host)
        h = self.hseqs.numpy()
        h[:na] = a_host
        h[na: na + nb] = b_host
        self.seqs[: na + nb].copy_(self.hseqs[: na + nb], non_blocking=True)
        offs = np.array([0, na, na + nb], dtype=np.int64)
        r = self.res
        rc = _lib.load().saix_overlap_batch(_lib.ptr(self.seqs), offs.ctypes.data, 1, int(policy is NPolicy.KEEP),
                                            _lib.ptr(r), _lib.ptr(r) + 24, _lib.ptr(self.ws), self.ws.numel(),
                                            _lib.stream_ptr())
        _lib.check(rc, "saix_overlap_batch")
        self.hres.copy_(r, non_blocking=True)
        _lib.torch().cuda.current_stream().synchronize()
        out = self.hres.numpy().copy()
        if out[3] != INT64_MAX and out[3] >= na:   # batch offsets put B right after A
            out[3] += 1
        return out


_SMALL: dict = {}


def _small_pipeline() -> SmallPairPipeline:
    import threading
    key = (_lib.torch().cuda.current_device(), threading.get_ident())
    p = _SMALL.get(key)
    if p is None:
        p = _SMALL[key] = SmallPairPipeline()
    return p


def longest_overlap(a: DnaSequence, b: DnaSequence,
                    policy: NPolicy = NPolicy.REJECT) -> OverlapResult:
    """Longest common substring of A and B via the generalized suffix array
    (overlap.py:110-152), ties to the smallest A position then B position.
    Pairs of up to ONCHIP_RESIDUES residues run in one CTA's shared memory
    (SmallPairPipeline), longer ones through the device DC3 pipeline."""
    if len(a) == 0 or len(b) == 0:
        return OverlapResult(0, 0, 0)
    ha, hb = _ascii(a), _ascii(b)
    if len(ha) + len(hb) + 1 <= ONCHIP_RESIDUES:
        res = _small_pipeline().run(ha, hb, policy)
    else:
        res = _pipeline(len(ha), len(hb)).run(ha, hb, policy)
    bad = int(res[3])
    if bad != INT64_MAX:
        if bad < len(ha):
            raise residue_error(a, bad, policy)
        raise residue_error(b, bad - len(ha) - 1, policy)
    return OverlapResult(int(res[0]), int(res[1]), int(res[2]))


class OverlapBatch:
    """Batched ``longest_overlap`` over many independent pairs on the device
    (saix_overlap_batch).  Pairs are packed as ASCII into ``seqs`` with
    ``offs`` (int64[2P+1]: pair p is A = seqs[offs[2p]:offs[2p+1]], B =
    seqs[offs[2p+1]:offs[2p+2]]).  Every pair of up to 20,480 GSA residues
    runs its whole pipeline in one CTA's shared memory; one call covers all
    pairs unless ``wave_residues`` (or SAIX_WAVE_RESIDUES) splits the batch
    into calls of at most that many residues.

    ``run_device`` works on the device-resident copy of ``seqs``;
    ``run_from_host`` streams pinned host ASCII in chunks on a copy stream,
    each chunk's pairs starting as soon as its bytes have landed (the H2D of
    chunk k+1 overlaps the pairs of chunk k)."""

    def __init__(self, seqs: np.ndarray, offs: np.ndarray, policy: NPolicy = NPolicy.REJECT,
                 wave_residues: int | None = None, chunks: int = 8):
        if wave_residues is None:
            import os
            wave_residues = int(os.environ.get("SAIX_WAVE_RESIDUES", 1 << 62))
        t = _lib.torch()
        L = _lib.load()
        dev = _lib.device()
        self.offs = np.ascontiguousarray(offs, dtype=np.int64)
        self.P = (len(self.offs) - 1) // 2
        self.keep_n = int(policy is NPolicy.KEEP)
        self.policy = policy
        self.waves = self._split(lambda p, q: self.offs[2 * (q + 1)] - self.offs[2 * p] <= wave_residues)
        per = max(1, -(-self.P // max(1, chunks)))
        self.chunks = [(p, min(p + per, self.P)) for p in range(0, self.P, per)]
        self.seqs_dev = _lib.to_device(np.ascontiguousarray(seqs, dtype=np.uint8))
        self.out = t.zeros(max(3 * self.P, 3), dtype=t.int64, device=dev)
        self.bad = t.zeros(max(len(self.waves), len(self.chunks), 1), dtype=t.int64, device=dev)
        self._calls = {}
        for kind, spans in (("waves", self.waves), ("chunks", self.chunks)):
            calls = []
            for a, b in spans:
                o = np.ascontiguousarray(self.offs[2 * a: 2 * b + 1] - self.offs[2 * a])
                calls.append((a, b, o, _lib.to_device(o)))   # host copy + resident device copy
            self._calls[kind] = calls
        ws = max((L.saix_overlap_batch_workspace_bytes(o.ctypes.data, b - a)
                  for calls in self._calls.values() for a, b, o, _d in calls), default=256)
        self.ws = _lib.workspace(ws)
        self.h2d_bytes = int(self.offs[-1])
        self._last = "waves"
        self._copy_stream = None

    def _split(self, fits):
        spans, p = [], 0
        while p < self.P:
            q = p + 1
            while q < self.P and fits(p, q):
                q += 1
            spans.append((p, q))
            p = q
        return spans

    def _call(self, k: int, a: int, b: int, o: np.ndarray, od, L, s) -> None:
        rc = L.saix_overlap_batch_dev(_lib.ptr(self.seqs_dev) + int(self.offs[2 * a]), o.ctypes.data,
                                      _lib.ptr(od), b - a, self.keep_n, _lib.ptr(self.out) + 24 * a,
                                      _lib.ptr(self.bad) + 8 * k, _lib.ptr(self.ws), self.ws.numel(), s)
        _lib.check(rc, "saix_overlap_batch")

    def run_device(self) -> None:
        """All waves on the device-resident ASCII (no host traffic)."""
        L = _lib.load()
        s = _lib.stream_ptr()
        self._last = "waves"
        for k, (a, b, o, od) in enumerate(self._calls["waves"]):
            self._call(k, a, b, o, od, L, s)

    def run_from_host(self, host_seqs, stream_chunks: int = 32) -> None:
        """Copy pinned host ASCII (a uint8 torch tensor laid out like
        ``seqs``) to the device and run the pairs as their bytes land: one
        kernel launch per wave whose CTAs wait on the copy engine's per-chunk
        counts (saix_overlap_batch_stream); ``stream_chunks=0`` uses one
        launch per chunk instead."""
        t = _lib.torch()
        L = _lib.load()
        cur = t.cuda.current_stream()
        if self._copy_stream is None:
            self._copy_stream = t.cuda.Stream()   # a pool stream: cudaStreamNonBlocking
        cs = self._copy_stream
        if stream_chunks:
            self._last = "waves"
            base = host_seqs.data_ptr()
            for k, (a, b, o, od) in enumerate(self._calls["waves"]):
                lo = int(self.offs[2 * a])
                rc = L.saix_overlap_batch_stream(_lib.ptr(self.seqs_dev) + lo, base + lo, o.ctypes.data,
                                                 _lib.ptr(od), b - a, int(stream_chunks), self.keep_n,
                                                 _lib.ptr(self.out) + 24 * a, _lib.ptr(self.bad) + 8 * k,
                                                 _lib.ptr(self.ws), self.ws.numel(), cur.cuda_stream,
                                                 cs.cuda_stream)
                _lib.check(rc, "saix_overlap_batch_stream")
            return
        cs.wait_stream(cur)  # the previous step's kernels are done with seqs_dev
        events = []
        with t.cuda.stream(cs):
            for a, b, _o, _d in self._calls["chunks"]:
                lo, hi = int(self.offs[2 * a]), int(self.offs[2 * b])
                self.seqs_dev[lo:hi].copy_(host_seqs[lo:hi], non_blocking=True)
                ev = t.cuda.Event()
                ev.record(cs)
                events.append(ev)
        s = cur.cuda_stream
        self._last = "chunks"
        for k, ((a, b, o, od), ev) in enumerate(zip(self._calls["chunks"], events)):
            cur.wait_event(ev)
            self._call(k, a, b, o, od, L, s)

    def first_bad(self) -> int | None:
        """Smallest seqs offset of an illegal residue in the last run, or None."""
        calls = self._calls[self._last]
        bad = self.bad[: len(calls)].cpu().numpy()
        hit = [int(v) + int(self.offs[2 * a]) for v, (a, _b, _o, _d) in zip(bad, calls) if v != INT64_MAX]
        return min(hit) if hit else None

    def results(self) -> np.ndarray:
        """(P, 3) int64 host array; raises SequenceError like the reference."""
        pos = self.first_bad()
        if pos is not None:
            raise SequenceError(f"illegal residue at packed offset {pos} "
                                f"(policy={self.policy.value})")
        return self.out[: 3 * self.P].cpu().numpy().reshape(self.P, 3)


def pack_pairs(pairs) -> tuple[np.ndarray, np.ndarray]:
    """[(A, B), ...] DnaSequences -> (ASCII bytes, int64[2P+1] offsets)."""
    chunks, offs = [], [0]
    for a, b in pairs:
        for s in (a, b):
            raw = np.frombuffer(s.residues.encode("ascii"), dtype=np.uint8)
            chunks.append(raw)
            offs.append(offs[-1] + raw.shape[0])
    seqs = np.concatenate(chunks) if chunks else np.zeros(0, np.uint8)
    return seqs, np.asarray(offs, dtype=np.int64)


def longest_overlap_batch(pairs, policy: NPolicy = NPolicy.REJECT) -> list[OverlapResult]:
    """Equals ``[longest_overlap(a, b, policy) for a, b in pairs]`` (including
    the SequenceError of the first offending pair), computed as batched waves."""
    pairs = list(pairs)
    if not pairs:
        return []
    seqs, offs = pack_pairs(pairs)
    ob = OverlapBatch(seqs, offs, policy)
    ob.run_device()
    pos = ob.first_bad()
    if pos is not None:
        pi = int(np.searchsorted(offs, pos, side="right") - 1)  # sequence index 2p or 2p+1
        seq = pairs[pi // 2][pi % 2]
        raise residue_error(seq, pos - int(offs[pi]), policy)
    res = ob.out[: 3 * len(pairs)].cpu().numpy().reshape(len(pairs), 3)
    return [OverlapResult(int(x), int(y), int(z)) for x, y, z in res]


def overlap_report(result: OverlapResult, a: DnaSequence, b: DnaSequence) -> tuple[str, str]:
    """Human summary + one-object JSON record (overlap.py:155-173)."""
    sub = a.residues[result.pos_a:result.pos_a + result.length]
    if sub != b.residues[result.pos_b:result.pos_b + result.length]:
        raise ValueError("overlap result does not match the given sequences")
    record = {"length": result.length, "posA": result.pos_a, "posB": result.pos_b,
              "substring": sub}
    if result.length:
        human = (f"overlap of {result.length} residues: {a.id}[{result.pos_a}] "
                 f"= {b.id}[{result.pos_b}] = {sub!r}")
    else:
        human = f"no overlap between {a.id} and {b.id}"
    return human, json.dumps(record)


def parse_overlap_record(payload: str) -> OverlapResult:
    """Inverse of the JSON half of overlap_report (overlap.py:176-180)."""
    rec = json.loads(payload)
    return OverlapResult(length=rec["length"], pos_a=rec["posA"], pos_b=rec["posB"])


__all__ = ["GeneralizedText", "LcpQueryEngine", "OverlapBatch", "OverlapPipeline", "OverlapResult",
           "longest_overlap_batch", "pack_pairs",
           "SequenceError", "alphabet", "lcp_query", "lcp_query_batch", "longest_overlap",
           "overlap_report", "parse_overlap_record"]
