"""``.saix`` index files (the reference's ``saix.index_store``,
index_store.py:1-134) written from and read into device buffers.

Same layout, names, return values and exceptions as the reference:

    magic "SAIX1\\0\\0\\0" | u64 version=1 | u64 flags (bit 0: alphabet has N)
    | u64 n | u64 sigma | text (n rank bytes) | sa (n x u64) | lcp (n x u64)
    | u64 zlib.crc32 of everything above

``save_index`` packs the file image on the device from the engine's resident
text / SA / LCP (u32 -> little-endian u64) and computes its CRC-32 there
(``saix_index_pack``); the host only writes the bytes out.  ``load_index``
checks the header on the host (magic, version, length: the reference's order
of checks, index_store.py:108-121), uploads the image once, and verifies the
CRC, narrows SA / LCP and rebuilds the inverse suffix array on the device
(``saix_index_unpack``); the engine it returns keeps those device buffers, so
the RMQ build and every query after the load start on the device.
"""

from __future__ import annotations

import struct
from pathlib import Path
from typing import BinaryIO

import numpy as np

from . import _lib
from .overlap import LcpQueryEngine, RmqKind
from .sequence import RankedText
from .suffix_index import DeviceIndex, DeviceText, LcpArray, SuffixArray, _device_index_of

MAGIC = b"SAIX1\x00\x00\x00"
VERSION = 1
FLAG_N_ALPHABET = 1 << 0

_U64 = struct.Struct("<Q")
_HEADER = len(MAGIC) + 4 * _U64.size


class IndexFileError(Exception):
    """Base class for unreadable index files (index_store.py:40-41)."""


class BadMagicError(IndexFileError):
    pass


class UnsupportedVersionError(IndexFileError):
    pass


class ChecksumError(IndexFileError):
    pass


class TruncatedFileError(IndexFileError):
    pass


def _open_sink(destination):
    if isinstance(destination, (str, Path)):
        return open(destination, "wb"), True
    return destination, False


def _ws(nbytes: int):
    return _lib.workspace(int(nbytes))


def _device_lcp(engine: LcpQueryEngine, n: int):
    lcp = engine.lcp
    if lcp._dev is not None:
        return lcp._dev[1]
    return _lib.to_device(np.asarray(lcp.lcp).astype(np.uint32).view(np.int32))


def pack_index(engine: LcpQueryEngine):
    """The file image of ``engine`` as a device uint8 tensor (CRC included)."""
    text = engine.text
    if text.sigma > 255:
        raise ValueError("index format stores one rank per byte; sigma must be <= 255")
    n = text.n
    if len(engine.lcp) != n or engine.sa.n != n:
        raise ValueError("engine parts do not match the text length")
    flags = FLAG_N_ALPHABET if text.sigma >= 5 else 0
    _lib.device()
    L = _lib.load()
    ix = _device_index_of(text, engine.sa)
    lcp = _device_lcp(engine, n)
    total = int(L.saix_index_bytes(n))
    out = _lib.empty(total, _lib.torch().uint8)
    ws = _ws(L.saix_crc32_workspace_bytes(total))
    _lib.check(L.saix_index_pack(_lib.ptr(ix.text.t), _lib.ptr(ix.sa), _lib.ptr(lcp), n, int(text.sigma), flags,
                                 _lib.ptr(out), _lib.ptr(ws), ws.numel(), _lib.stream_ptr()), "saix_index_pack")
    return out[:total]


def save_index(engine: LcpQueryEngine, destination: str | Path | BinaryIO) -> int:
    """Write an engine's text, suffix array, and lcp array; returns bytes
    written (index_store.py:65-88)."""
    image_d = pack_index(engine)
    total = int(image_d.shape[0])
    host = _lib.staging(total)
    host[:total].copy_(image_d)
    sink, owned = _open_sink(destination)
    try:
        sink.write(memoryview(host.numpy())[:total])
    finally:
        if owned:
            sink.close()
    return total


def _check_prefix(head) -> int:
    """index_store.py:99-112: the reference's checks on the first 48 bytes
    (length, magic, version), in its order; returns n."""
    if len(head) < _HEADER + _U64.size:
        raise TruncatedFileError(f"file is {len(head)} bytes; shorter than any valid index")
    if bytes(head[:len(MAGIC)]) != MAGIC:
        raise BadMagicError(f"bad magic {bytes(head[:len(MAGIC)])!r}")
    version, _flags, n, _sigma = (_U64.unpack_from(head, len(MAGIC) + k * _U64.size)[0] for k in range(4))
    if version != VERSION:
        raise UnsupportedVersionError(f"unsupported version {version}")
    return int(n)


def _check_header(blob) -> int:
    """index_store.py:99-116: prefix checks, then the length n implies."""
    n = _check_prefix(blob)
    expected = _HEADER + n + 2 * 8 * n + _U64.size
    if len(blob) < expected:
        raise TruncatedFileError(f"file is {len(blob)} bytes; need {expected} for n={n}")
    return n


def _read_image(fh):
    """The file image from a binary stream -- read straight into the pinned
    staging buffer when the stream supports readinto (else fh.read()), with
    the reference's checks on what was read.  Returns a bytes-like image of
    exactly the checked length."""
    seekable = hasattr(fh, "readinto") and hasattr(fh, "seekable") and fh.seekable()
    if not seekable:
        blob = fh.read()
        n = _check_header(blob)
        return memoryview(blob)[:_HEADER + 17 * n + _U64.size]
    head = fh.read(_HEADER + _U64.size)
    n = _check_prefix(head)
    total = _HEADER + 17 * n + _U64.size
    here = fh.tell()
    size = fh.seek(0, 2) - here + len(head)
    fh.seek(here)
    if size < total:  # checked before any buffer is sized from the header's n
        fh.read()
        raise TruncatedFileError(f"file is {size} bytes; need {total} for n={n}")
    buf = _lib.staging(total)
    view = memoryview(buf.numpy())[:total]
    view[:len(head)] = head
    got = len(head)
    while got < total:
        k = fh.readinto(view[got:])
        if not k:
            break
        got += k
    if got < total:
        raise TruncatedFileError(f"file is {got} bytes; need {total} for n={n}")
    fh.read()  # the reference consumes the whole stream; trailing bytes are ignored
    return view


def unpack_index(blob, rmq_kind: RmqKind = "sparse") -> LcpQueryEngine:
    """An engine from a file image (bytes-like) whose parts stay on the device."""
    n = _check_header(blob)
    sigma = _U64.unpack_from(blob, len(MAGIC) + 3 * _U64.size)[0]
    _lib.device()
    t = _lib.torch()
    L = _lib.load()
    payload = _HEADER + 17 * n
    dev_blob = _lib.to_device(np.frombuffer(blob, dtype=np.uint8, count=payload + _U64.size))
    text_d = _lib.empty(n, t.uint8)
    sa_d, lcp_d, isa_d = (_lib.empty(n, t.int32) for _ in range(3))
    ws = _ws(L.saix_index_unpack_workspace_bytes(n))
    rc = L.saix_index_unpack(_lib.ptr(dev_blob), n, _lib.ptr(text_d), _lib.ptr(sa_d), _lib.ptr(lcp_d),
                             _lib.ptr(isa_d), _lib.ptr(ws), ws.numel(), _lib.stream_ptr())
    if rc != 0:
        msg = L.saix_last_error().decode()
        if "checksum" in msg:
            raise ChecksumError("checksum mismatch; file is corrupt")
        if "out of range" in msg:
            raise IndexError(f"index entries out of range for n={n}")
        _lib.check(rc, "saix_index_unpack")
    if n:
        # RankedText's 1..sigma check (sequence.py:55-62), on the device
        mm = t.empty(2, dtype=t.int64, device=text_d.device)
        _lib.check(L.saix_minmax(_lib.ptr(text_d), 1, n, _lib.ptr(mm), _lib.stream_ptr()), "saix_minmax")
        lo, hi = (int(x) for x in mm.cpu().tolist())
        if lo < 1 or hi > sigma:
            raise ValueError("ranks must lie in 1..sigma")
    text = RankedText._checked(_lib.widen_i64_host(text_d, n), int(sigma))
    # the file stores one byte per rank whatever the header's sigma (the
    # reference loads sigma > 255 files too); device texts with sigma > 255
    # are u32, so widen on the device
    dt = DeviceText.resident(text, text_d if int(sigma) <= 255 else text_d.to(t.int32))
    object.__setattr__(text, "_dev", dt)
    ix = DeviceIndex(dt, sa_d, isa_d)
    sa = _lib.widen_i64_host(sa_d, n)
    rank = _lib.widen_i64_host(isa_d, n) if n else sa.copy()
    sa_struct = SuffixArray(n=n, sa=sa, rank=rank, _dev=ix)
    lcp = LcpArray(_lib.widen_i64_host(lcp_d, n), _dev=(ix, lcp_d))
    return LcpQueryEngine.from_parts(text, sa_struct, lcp, rmq_kind)


def load_index(source: str | Path | BinaryIO, rmq_kind: RmqKind = "sparse") -> LcpQueryEngine:
    """Read an index file back into an engine, rebuilding the RMQ structure
    (index_store.py:91-134)."""
    if isinstance(source, (str, Path)):
        with open(source, "rb") as fh:
            image = _read_image(fh)
    else:
        image = _read_image(source)
    return unpack_index(image, rmq_kind)
