"""Suffix arrays (DC3) and LCP arrays on the B200 -- drop-in for
``saix.suffix_index`` (suffix_index.py:84-506).

Every builder runs the CUDA path in libsaix_b200.so; results come back as the
reference's frozen dataclasses holding read-only int64 numpy arrays.  The
device copies (u32) stay attached (``_dev``) so chained calls
(``build_lcp(text, build_sa_dc3(text))``, ``LcpQueryEngine.build``) do not
re-upload anything.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field
from typing import Any, Callable

import numpy as np

from . import _lib
from .sequence import RankedText

SortByKeys = Callable[..., np.ndarray]


@dataclass(frozen=True, eq=False)
class SuffixArray:
    """Suffix start positions in lexicographic order and the inverse map
    (suffix_index.py:84-101)."""

    n: int
    sa: np.ndarray
    rank: np.ndarray
    _dev: Any = field(default=None, repr=False, compare=False)

    def __post_init__(self):
        self.sa.flags.writeable = False
        self.rank.flags.writeable = False

    @classmethod
    def from_order(cls, order: np.ndarray) -> "SuffixArray":
        order = np.asarray(order, dtype=np.int64)
        rank = np.empty_like(order)
        rank[order] = np.arange(order.shape[0], dtype=np.int64)
        return cls(n=int(order.shape[0]), sa=order, rank=rank)


@dataclass(frozen=True, eq=False)
class LcpArray:
    """lcp[i] = |lcp(suffix sa[i-1], suffix sa[i])|, lcp[0] = 0
    (suffix_index.py:104-116)."""

    lcp: np.ndarray
    _dev: Any = field(default=None, repr=False, compare=False)

    def __post_init__(self):
        arr = np.asarray(self.lcp, dtype=np.int64)
        arr.flags.writeable = False
        object.__setattr__(self, "lcp", arr)

    def __len__(self) -> int:
        return int(self.lcp.shape[0])


@dataclass
class Dc3Workspace:
    """Level-0 DC3 intermediates (suffix_index.py:119-140)."""

    mod1: np.ndarray
    mod2: np.ndarray
    nonsample: np.ndarray
    triple_text: np.ndarray
    sample_rank: np.ndarray
    sorted_samples: np.ndarray
    sorted_nonsamples: np.ndarray
    depth: int

    @property
    def sample_positions(self) -> np.ndarray:
        return np.concatenate([self.mod1, self.mod2])


# ------------------------------------------------------------------ device

class DeviceText:
    """A RankedText resident on the device: u8 ranks when sigma <= 255,
    else u32 (int32 tensor)."""

    def __init__(self, text: RankedText):
        self.n = text.n
        self.sigma = int(text.sigma)
        self.source = text.ranks
        if self.sigma <= 255:
            self.bytes = 1
            self.t = _lib.to_device(text.ranks.astype(np.uint8))
        else:
            self.bytes = 4
            self.t = _lib.to_device(text.ranks.astype(np.uint32).view(np.int32))

    @classmethod
    def resident(cls, text: RankedText, t) -> "DeviceText":
        """Wrap ranks already on the device (u8 when sigma <= 255, else u32)."""
        self = cls.__new__(cls)
        self.n = text.n
        self.sigma = int(text.sigma)
        self.source = text.ranks
        self.bytes = 1 if self.sigma <= 255 else 4
        self.t = t
        return self


def device_text(text: RankedText, cache: Any = None) -> DeviceText:
    resident = getattr(text, "_dev", None)
    if resident is not None and resident.source is text.ranks:
        return resident
    if cache is not None and getattr(cache, "text", None) is not None \
            and cache.text.source is text.ranks:
        return cache.text
    return DeviceText(text)


class DeviceIndex:
    """Device-side SA / ISA (u32 stored as int32 tensors) of one text."""

    def __init__(self, text: DeviceText, sa, isa):
        self.text = text
        self.sa = sa
        self.isa = isa


def sample_counts(n: int) -> tuple[int, int]:
    """(|mod1|, |mod2|) sample positions (suffix_index.py:149-153)."""
    limit = n + 1 if n % 3 == 1 else n
    return max(0, (limit + 1) // 3), max(0, limit // 3)


def dc3_device(dt: DeviceText, probe: _lib.Dc3Probe | None = None) -> DeviceIndex:
    """Run DC3 on a device text; returns device SA/ISA."""
    t = _lib.torch()
    L = _lib.load()
    n = dt.n
    sa = _lib.empty(n, t.int32)
    isa = _lib.empty(n, t.int32)
    ws = _lib.workspace(L.saix_dc3_workspace_bytes(n, dt.bytes))
    rc = L.saix_dc3(_lib.ptr(dt.t), dt.bytes, n, max(dt.sigma, 1), _lib.ptr(sa), _lib.ptr(isa),
                    _lib.ptr(ws), ws.numel(), ctypes.byref(probe) if probe is not None else None,
                    _lib.stream_ptr())
    _lib.check(rc, "saix_dc3")
    return DeviceIndex(dt, sa, isa)


def _device_index_of(text: RankedText, sa: SuffixArray) -> DeviceIndex:
    if sa._dev is not None and sa._dev.text.source is text.ranks:
        return sa._dev
    n = text.n
    if sa.n != n:
        raise ValueError("suffix array length does not match the text")
    if n and (int(sa.sa.min()) < 0 or int(sa.sa.max()) >= n
              or int(sa.rank.min()) < 0 or int(sa.rank.max()) >= n):
        raise ValueError("suffix array entries out of range")
    dt = device_text(text, sa._dev)
    return DeviceIndex(dt, _lib.to_device(sa.sa.astype(np.uint32).view(np.int32)),
                       _lib.to_device(sa.rank.astype(np.uint32).view(np.int32)))


# ------------------------------------------------------------------ API

def build_sa_dc3(text: RankedText, sort_by_keys: SortByKeys | None = None) -> SuffixArray:
    """Linear-time suffix array via DC3 on the GPU (suffix_index.py:395-399).

    ``sort_by_keys`` is accepted for signature compatibility; the suffix
    array of a text is unique, so the GPU radix passes give the same output
    any correct stable sorter would.
    """
    n = text.n
    if n == 0:
        return SuffixArray(n=0, sa=np.zeros(0, np.int64), rank=np.zeros(0, np.int64))
    _lib.device()
    ix = dc3_device(device_text(text))
    return SuffixArray(n=n, sa=_lib.u32_to_i64_host(ix.sa, n),
                       rank=_lib.u32_to_i64_host(ix.isa, n), _dev=ix)


def build_sa_oracle(text: RankedText) -> SuffixArray:
    """Same contract as the reference's comparison-sort oracle
    (suffix_index.py:402-411, alphabets <= 255); the suffix array is unique,
    so this returns the GPU DC3 result."""
    if text.sigma > 255:
        raise ValueError("oracle supports alphabets up to 255 ranks")
    return build_sa_dc3(text)


def lcp_device(ix: DeviceIndex):
    """Kasai LCP on device arrays; returns the u32 LCP tensor."""
    t = _lib.torch()
    L = _lib.load()
    n = ix.text.n
    lcp = _lib.empty(n, t.int32)
    ws = _lib.workspace(L.saix_lcp_workspace_bytes(n))
    rc = L.saix_lcp_sigma(_lib.ptr(ix.text.t), ix.text.bytes, n, ix.text.sigma, -1, _lib.ptr(ix.sa),
                          _lib.ptr(lcp), _lib.ptr(ws), ws.numel(), _lib.stream_ptr())
    _lib.check(rc, "saix_lcp_sigma")
    return lcp


def build_lcp(text: RankedText, sa: SuffixArray) -> LcpArray:
    """Adjacent-suffix LCP lengths (suffix_index.py:479-506), on the GPU."""
    n = text.n
    if n == 0:
        return LcpArray(np.zeros(0, np.int64))
    _lib.device()
    ix = _device_index_of(text, sa)
    lcp = lcp_device(ix)
    return LcpArray(_lib.u32_to_i64_host(lcp, n), _dev=(ix, lcp))


def _probe_run(text: RankedText):
    n = text.n
    t = _lib.torch()
    m1, m2 = sample_counts(n)
    m = m1 + m2
    k = (n + 2) // 3
    bufs = {
        "triple_text": _lib.empty(m, t.int32),
        "sample_rank": _lib.empty(n + 3, t.int32),
        "sorted_samples": _lib.empty(m, t.int32),
        "sorted_nonsamples": _lib.empty(k, t.int32),
    }
    probe = _lib.Dc3Probe(*[_lib.ptr(bufs[k_]) for k_ in
                            ("triple_text", "sample_rank", "sorted_samples", "sorted_nonsamples")])
    ix = dc3_device(device_text(text), probe)

    def host(name, count):
        if count == 0:
            return np.zeros(0, np.int32)
        return bufs[name][:count].cpu().numpy().view(np.uint32).astype(np.int32)

    out = {
        "triple_text": host("triple_text", probe.n_samples),
        "sample_rank": host("sample_rank", n + 3),
        "sorted_samples": host("sorted_samples", probe.n_sorted_samples),
        "sorted_nonsamples": host("sorted_nonsamples", probe.n_sorted_nonsamples),
        "depth": int(probe.depth),
        "m1": m1,
        "m2": m2,
    }
    return out, ix


def sample_ranks(text: RankedText) -> dict[int, int]:
    """1-based ranks of the mod-1/mod-2 samples keyed by position, padding
    position n included when n % 3 == 1 (suffix_index.py:414-422)."""
    n = text.n
    if n == 0:
        return {}
    _lib.device()
    pr, _ = _probe_run(text)
    limit = n + 1 if n % 3 == 1 else n
    pos = np.arange(1, limit)
    pos = pos[pos % 3 != 0]
    rk = pr["sample_rank"]
    return {int(p): int(rk[p]) for p in pos}


def prepare_dc3_workspace(text: RankedText,
                          sort_by_keys: SortByKeys | None = None) -> Dc3Workspace:
    """DC3 steps 1-2 with the level-0 intermediates (suffix_index.py:425-449)."""
    n = text.n
    m1, m2 = sample_counts(n)
    mod1 = np.arange(1, 1 + 3 * m1, 3, dtype=np.int32)[:m1]
    mod2 = np.arange(2, 2 + 3 * m2, 3, dtype=np.int32)[:m2]
    nonsample = np.arange(0, n, 3, dtype=np.int32)
    if n == 0:
        return Dc3Workspace(mod1, mod2, nonsample, np.zeros(0, np.int32),
                            np.zeros(3, np.int32), np.zeros(0, np.int32),
                            np.zeros(0, np.int32), 0)
    _lib.device()
    pr, _ = _probe_run(text)
    return Dc3Workspace(mod1=mod1, mod2=mod2, nonsample=nonsample,
                        triple_text=pr["triple_text"], sample_rank=pr["sample_rank"],
                        sorted_samples=pr["sorted_samples"],
                        sorted_nonsamples=pr["sorted_nonsamples"], depth=pr["depth"])


def merge_sample_nonsample(workspace: Dc3Workspace, text: RankedText) -> SuffixArray:
    """Step 3 alone on a prepared workspace (suffix_index.py:452-457)."""
    n = text.n
    ss = np.asarray(workspace.sorted_samples, np.int64)
    sn = np.asarray(workspace.sorted_nonsamples, np.int64)
    total = ss.shape[0] + sn.shape[0]
    if total == 0:
        return SuffixArray.from_order(np.zeros(0, np.int64))
    _lib.device()
    t = _lib.torch()
    L = _lib.load()
    dt = device_text(text)
    rank = _lib.to_device(np.asarray(workspace.sample_rank).astype(np.uint32).view(np.int32))
    a = _lib.to_device(ss.astype(np.uint32).view(np.int32))
    b = _lib.to_device(sn.astype(np.uint32).view(np.int32))
    out = _lib.empty(total, t.int32)
    ws = _lib.workspace(L.saix_dc3_merge_workspace_bytes(total))
    rc = L.saix_dc3_merge(_lib.ptr(dt.t), dt.bytes, n, _lib.ptr(rank), _lib.ptr(a), ss.shape[0],
                          _lib.ptr(b), sn.shape[0], _lib.ptr(out), _lib.ptr(ws), ws.numel(),
                          _lib.stream_ptr())
    _lib.check(rc, "saix_dc3_merge")
    return SuffixArray.from_order(_lib.u32_to_i64_host(out, total))


class SuffixIndexer:
    """Reusable device buffers for suffix array + LCP construction of texts of
    length n (the throughput path behind ``build_sa_dc3`` + ``build_lcp``).

    ``t`` (device) holds the ranks; ``run_device()`` builds SA (and ISA when
    ``want_isa``) and LCP without host traffic; ``run_staged()`` adds the
    pinned-host upload of the ranks and the download of SA and LCP (u32)."""

    def __init__(self, n: int, sigma: int, want_isa: bool = False):
        t = _lib.torch()
        L = _lib.load()
        dev = _lib.device()
        self.n, self.sigma = int(n), int(sigma)
        self.bytes = 1 if sigma <= 255 else 4
        self.t = t.zeros(max(n, 1) + 8, dtype=t.uint8 if self.bytes == 1 else t.int32, device=dev)
        self.sa = t.empty(max(n, 1), dtype=t.int32, device=dev)
        self.isa = t.empty(max(n, 1), dtype=t.int32, device=dev) if want_isa else None
        self.lcp = t.empty(max(n, 1), dtype=t.int32, device=dev)
        wsz = max(L.saix_dc3_workspace_bytes(n, self.bytes), L.saix_lcp_workspace_bytes(n))
        self.ws = _lib.workspace(wsz)
        self.ht = t.empty(max(n, 1), dtype=self.t.dtype, pin_memory=True)
        self.hsa = t.empty(max(n, 1), dtype=t.int32, pin_memory=True)
        self.hlcp = t.empty(max(n, 1), dtype=t.int32, pin_memory=True)

    def stage(self, ranks: np.ndarray) -> None:
        self.ht.numpy()[: self.n] = ranks

    def _dc3(self, s: int) -> None:
        L = _lib.load()
        _lib.check(L.saix_dc3(_lib.ptr(self.t), self.bytes, self.n, self.sigma, _lib.ptr(self.sa),
                              _lib.ptr(self.isa), _lib.ptr(self.ws), self.ws.numel(), None, s), "saix_dc3")

    def _lcp(self, s: int) -> None:
        L = _lib.load()
        _lib.check(L.saix_lcp_sigma(_lib.ptr(self.t), self.bytes, self.n, self.sigma, -1, _lib.ptr(self.sa),
                                    _lib.ptr(self.lcp), _lib.ptr(self.ws), self.ws.numel(), s), "saix_lcp_sigma")

    def run_device(self) -> None:
        s = _lib.stream_ptr()
        self._dc3(s)
        self._lcp(s)

    def run_staged(self) -> None:
        """Upload, build, download; the SA download (copy stream) overlaps
        the LCP kernel, which only reads SA."""
        t = _lib.torch()
        n = self.n
        cur = t.cuda.current_stream()
        if not hasattr(self, "_copy"):
            self._copy = t.cuda.Stream()
        self.t[:n].copy_(self.ht[:n], non_blocking=True)
        self._dc3(cur.cuda_stream)
        done = cur.record_event()
        self._copy.wait_event(done)
        with t.cuda.stream(self._copy):
            self.hsa[:n].copy_(self.sa[:n], non_blocking=True)
        self._lcp(cur.cuda_stream)
        self.hlcp[:n].copy_(self.lcp[:n], non_blocking=True)
        cur.wait_stream(self._copy)  # the next step's DC3 rewrites SA only after its download
        cur.synchronize()
