"""FASTA ingest on the device: the reference's
``parse_fasta`` + ``encode`` (sequence.py:77-157) over raw FASTA bytes in
HBM, so a file goes host -> device once at 1 byte per base and comes out as
device-resident residues (upper-cased ASCII) or ranks (A1 C2 G3 T4, N5)
ready for the suffix-array path.

``parse_fasta(str)`` runs through here and returns the reference's records
and SequenceError messages exactly; ``ingest_fasta`` is the throughput entry
(bytes, a path, or a device uint8 tensor) that keeps the residues on the
device.  Semantics are the reference's for a ``str`` source (lines end at
'\\n'; a file is read in binary, so a lone '\\r' is not a line break).
"""

from __future__ import annotations

import os
from dataclasses import dataclass, field
from pathlib import Path
from typing import Any

import numpy as np

from . import _lib
from .sequence import DnaSequence, NPolicy, RankedText, SequenceError, alphabet


@dataclass(eq=False)
class FastaIngest:
    """Records of one FASTA input with their residues resident on the device.

    ``residues``: device uint8 tensor, ranks when ``as_ranks`` else upper-cased
    ASCII, records concatenated; record r is ``residues[offsets[r]:offsets[r+1]]``.
    """

    residues: Any
    offsets: np.ndarray
    ids: list[str]
    descriptions: list[str]
    policy: NPolicy
    as_ranks: bool
    _host: Any = field(default=None, repr=False)

    def __len__(self) -> int:
        return len(self.ids)

    @property
    def total_residues(self) -> int:
        return int(self.offsets[-1]) if len(self.offsets) else 0

    def _host_bytes(self) -> np.ndarray:
        if self._host is None:
            n = self.total_residues
            self._host = self.residues[:n].cpu().numpy() if n else np.zeros(0, np.uint8)
        return self._host

    def records(self) -> list[DnaSequence]:
        """The reference's parse_fasta result (one D2H of all residues)."""
        h = self._host_bytes()
        if self.as_ranks:
            h = np.frombuffer(b"?ACGTN", np.uint8)[h]
        o = self.offsets
        return [DnaSequence(self.ids[r], h[o[r]:o[r + 1]].tobytes().decode("ascii"), self.descriptions[r])
                for r in range(len(self.ids))]

    def ranked(self, r: int) -> RankedText:
        """encode(record r) as a RankedText whose device copy is already
        resident (build_sa_dc3 / LcpQueryEngine.build reuse it)."""
        from .suffix_index import DeviceText
        if not self.as_ranks:
            raise ValueError("ingest_fasta(..., as_ranks=True) keeps ranks on the device")
        a, b = int(self.offsets[r]), int(self.offsets[r + 1])
        dev = self.residues[a:b] if b > a else self.residues[:0]
        ranks = _lib.widen_i64_host(dev, b - a) if b > a else np.zeros(0, np.int64)
        text = RankedText._checked(ranks, len(alphabet(self.policy)))
        object.__setattr__(text, "_dev", DeviceText.resident(text, dev))
        return text


def _as_device_bytes(data):
    """(device uint8 tensor, host uint8 view or None) for bytes-like input, an
    ASCII str of FASTA text, a pathlib.Path (read in binary straight into the
    pinned staging buffer), or a CUDA uint8 tensor."""
    t = _lib.torch()
    if isinstance(data, t.Tensor):
        if data.dtype != t.uint8 or not data.is_cuda:
            raise TypeError("device FASTA input must be a CUDA uint8 tensor")
        return data.contiguous(), None
    if isinstance(data, Path):
        with open(data, "rb") as fh:
            size = os.fstat(fh.fileno()).st_size
            buf = _lib.staging(max(size, 1))
            view = memoryview(buf.numpy())[:size]
            got = 0
            while got < size:
                k = fh.readinto(view[got:])
                if not k:
                    break
                got += k
        host = np.frombuffer(view[:got], np.uint8)
    else:
        if isinstance(data, str):
            data = data.encode("ascii")
        host = np.frombuffer(data, np.uint8)
    return _lib.to_device(host), host


def _error(info, host, dev, ids) -> SequenceError:
    pos, line, kind, start, nh = (int(x) for x in info)
    if kind == 1:
        return SequenceError(f"line {line + 1}: empty FASTA header")
    if nh == 0:
        return SequenceError(f"line {line + 1}: sequence data before any '>' header")
    byte = int(host[pos]) if host is not None else int(dev[pos].item())
    ch = chr(byte).upper()
    return SequenceError(f"record {ids[nh - 1]!r}, line {line + 1}: illegal residue {ch!r} at column {pos - start + 1}")


def ingest_fasta(data, policy: NPolicy = NPolicy.REJECT, as_ranks: bool = True) -> FastaIngest:
    """Parse + validate (+ encode) FASTA on the device.  ``data``: bytes, an
    ASCII str of FASTA text, a ``pathlib.Path``, or a CUDA uint8 tensor.  Raises the
    reference's SequenceError (same message) for the first malformed line."""
    _lib.device()
    t = _lib.torch()
    L = _lib.load()
    dev, host = _as_device_bytes(data)
    B = int(dev.numel()) if host is None else int(host.shape[0])
    st = _lib.stream_ptr()
    lines = np.zeros(1, np.int64)
    ws0 = _lib.workspace(((B + 16383) // 16384 + 8) * 4 + 1024)
    _lib.check(L.saix_fasta_lines(_lib.ptr(dev), B, lines.ctypes.data, _lib.ptr(ws0), ws0.numel(), st),
               "saix_fasta_lines")
    nl = int(lines[0])
    ws = _lib.workspace(L.saix_fasta_workspace_bytes(B, nl))
    counts = np.zeros(4, np.int64)
    _lib.check(L.saix_fasta_scan(_lib.ptr(dev), B, nl, counts.ctypes.data, _lib.ptr(ws), ws.numel(), st),
               "saix_fasta_scan")
    nres, nrec, nhdr = (int(x) for x in counts[:3])
    res = _lib.empty(nres, t.uint8)
    rec = _lib.empty(nrec + 1, t.int32)
    hdr = _lib.empty(nhdr, t.uint8)
    hoff = _lib.empty(nrec + 1, t.int32)
    info = np.zeros(5, np.int64)
    _lib.check(L.saix_fasta_emit(_lib.ptr(dev), B, nl, int(policy is NPolicy.KEEP), int(as_ranks), _lib.ptr(res),
                                 _lib.ptr(rec), _lib.ptr(hdr), _lib.ptr(hoff), info.ctypes.data, _lib.ptr(ws),
                                 ws.numel(), st), "saix_fasta_emit")
    offsets = _lib.widen_i64_host(rec, nrec + 1)
    hb = hdr[:nhdr].cpu().numpy().tobytes() if nhdr else b""
    ho = _lib.widen_i64_host(hoff, nrec + 1)
    ids, descs = [], []
    for r in range(nrec):
        rid, _, desc = hb[ho[r]:ho[r + 1]].decode("utf-8", "surrogateescape").partition(" ")
        ids.append(rid)
        descs.append(desc.strip())
    if info[0] >= 0:
        raise _error(info, host, dev, ids)
    return FastaIngest(residues=res, offsets=offsets, ids=ids, descriptions=descs, policy=policy,
                       as_ranks=as_ranks)
