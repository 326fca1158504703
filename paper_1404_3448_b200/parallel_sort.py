"""The reference's split-kernel sort engine (``saix.parallel_sort``,
parallel_sort.py:1-293) on the B200: same names, signatures, config
validation, return types and errors; the compute runs on the device.

* ``exclusive_scan``  -> ``saix_exclusive_scan_i64`` (device block scan)
* ``split_by_bit``    -> ``saix_split_by_bit`` (device scan + stable scatter);
  the returned ``SplitState`` holds the same per-lane arrays
* ``radix_sort`` / ``chunked_sort`` -> ``saix_radix_sort_i64`` (onesweep LSD
  radix, 8-bit digits): a stable ascending sort of the keys alone is unique,
  so digit width, chunk size and worker count cannot change the result
  (the reference states the same invariance, parallel_sort.py:11-18)
* ``parallel_build_sa`` -> the device DC3 (``build_sa_dc3``): "DC3 with all
  sorting passes on the chunked engine; equals the serial build"
  (parallel_sort.py:288-293), including the engine's 63-bit packed-key limit.

Host work is limited to argument validation (the reference's ValueErrors).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib
from .sequence import RankedText
from .suffix_index import SuffixArray, build_sa_dc3

MAX_KEY_BITS = 63  # keys are held in signed 64-bit lanes (parallel_sort.py:33)


@dataclass(frozen=True)
class SortConfig:
    """Engine knobs: digit width, key width, chunking, and worker count
    (parallel_sort.py:38-62; same validation)."""

    digit_bits: int = 1
    total_bits: int = 32
    chunk_size: int = 4096
    workers: int = 1

    def __post_init__(self):
        if self.digit_bits < 1:
            raise ValueError("digit_bits must be >= 1")
        if self.total_bits < 1 or self.total_bits > MAX_KEY_BITS:
            raise ValueError(f"total_bits must be in 1..{MAX_KEY_BITS}")
        if self.total_bits % self.digit_bits:
            raise ValueError("total_bits must be a multiple of digit_bits")
        if self.chunk_size < 1:
            raise ValueError("chunk_size must be >= 1")
        if self.workers < 1:
            raise ValueError("workers must be >= 1")

    @property
    def chunk_is_multiple_of_32(self) -> bool:
        return self.chunk_size % 32 == 0


@dataclass(frozen=True)
class SplitState:
    """Per-lane state of one split pass (parallel_sort.py:65-78)."""

    bits: np.ndarray
    zero_flags: np.ndarray
    scanned: np.ndarray
    zero_total: int
    dest: np.ndarray


@dataclass(frozen=True)
class ChunkPlan:
    """Contiguous, disjoint chunk boundaries covering the input exactly."""

    boundaries: tuple[tuple[int, int], ...]
    chunk_size: int
    workers: int


def plan_chunks(n: int, config: SortConfig) -> ChunkPlan:
    """parallel_sort.py:88-91."""
    cs = config.chunk_size
    bounds = tuple((s, min(s + cs, n)) for s in range(0, n, cs))
    return ChunkPlan(boundaries=bounds, chunk_size=cs, workers=config.workers)


def _as_keys(values) -> np.ndarray:
    return np.ascontiguousarray(values, dtype=np.int64)


def _ws(n: int):
    return _lib.workspace(_lib.load().saix_psort_workspace_bytes(max(int(n), 1)))


def _check_width_device(keys_dev, n: int, total_bits: int) -> None:
    """_check_width (parallel_sort.py:98-106) with the min / max reduced on
    the device."""
    if n == 0:
        return
    t = _lib.torch()
    mm = t.empty(2, dtype=t.int64, device=keys_dev.device)
    _lib.check(_lib.load().saix_minmax(_lib.ptr(keys_dev), 8, n, _lib.ptr(mm), _lib.stream_ptr()), "saix_minmax")
    lo, hi = (int(x) for x in mm.cpu().tolist())
    if lo < 0:
        raise ValueError("keys must be nonnegative")
    if hi >> total_bits:
        raise ValueError(f"key {hi} exceeds the configured width of {total_bits} bits")


def exclusive_scan(values) -> np.ndarray:
    """Prefix sums with out[0] = 0 (parallel_sort.py:110-131), on the device."""
    vals = _as_keys(values)
    n = len(vals)
    if n == 0:
        return vals.copy()
    _lib.device()
    src = _lib.to_device(vals)
    out = _lib.empty(n, _lib.torch().int64)
    ws = _ws(n)
    _lib.check(_lib.load().saix_exclusive_scan_i64(_lib.ptr(src), n, _lib.ptr(out), _lib.ptr(ws), ws.numel(),
                                                   _lib.stream_ptr()), "saix_exclusive_scan_i64")
    return out[:n].cpu().numpy()


def split_by_bit(keys, bit: int) -> tuple[np.ndarray, SplitState]:
    """Stable partition by one bit: zero-bit keys first, order preserved
    (parallel_sort.py:150-163)."""
    keys = _as_keys(keys)
    n = len(keys)
    if n == 0:
        e = np.zeros(0, np.int64)
        return keys.copy(), SplitState(bits=e, zero_flags=e.copy(), scanned=e.copy(), zero_total=0, dest=e.copy())
    _lib.device()
    t = _lib.torch()
    src = _lib.to_device(keys)
    out, bits, zf, sc, dest = (_lib.empty(n, t.int64) for _ in range(5))
    zt = _lib.empty(1, t.int64)
    ws = _ws(n)
    _lib.check(_lib.load().saix_split_by_bit(_lib.ptr(src), n, int(bit), _lib.ptr(out), _lib.ptr(bits), _lib.ptr(zf),
                                             _lib.ptr(sc), _lib.ptr(dest), _lib.ptr(zt), _lib.ptr(ws), ws.numel(),
                                             _lib.stream_ptr()), "saix_split_by_bit")
    host = lambda a: a[:n].cpu().numpy()  # noqa: E731
    return host(out), SplitState(bits=host(bits), zero_flags=host(zf), scanned=host(sc),
                                 zero_total=int(zt[0].item()), dest=host(dest))


def _device_sort(keys: np.ndarray, total_bits: int) -> np.ndarray:
    n = len(keys)
    _lib.device()
    src = _lib.to_device(keys)
    _check_width_device(src, n, total_bits)
    out = _lib.empty(n, _lib.torch().int64)
    ws = _ws(n)
    _lib.check(_lib.load().saix_radix_sort_i64(_lib.ptr(src), n, int(total_bits), _lib.ptr(out), _lib.ptr(ws),
                                               ws.numel(), _lib.stream_ptr()), "saix_radix_sort_i64")
    return out[:n].cpu().numpy()


def radix_sort(keys, config: SortConfig | None = None) -> np.ndarray:
    """Ascending stable sort of nonnegative integer keys (parallel_sort.py:195-203)."""
    config = config or SortConfig()
    keys = _as_keys(keys)
    if len(keys) == 0:
        return keys.copy()
    return _device_sort(keys, config.total_bits)


def chunked_sort(keys, config: SortConfig | None = None) -> np.ndarray:
    """Output equals radix_sort for every configuration (parallel_sort.py:215-254)."""
    config = config or SortConfig()
    keys = _as_keys(keys)
    if len(keys) == 0:
        return keys.copy()
    return _device_sort(keys, config.total_bits)


def _engine_key_check(text: RankedText, config: SortConfig, sa: SuffixArray | None = None) -> None:
    """The engine's packed-key limit (parallel_sort.py:270-279): each sorting
    pass packs (key, lane index) and sizes the key by the pass's actual
    maximum; a pass whose key bits + index bits, rounded up to the digit
    width, exceeds 63 raises.  Level 0 uses the text's actual maxima (triple
    keys t[1:], non-sample characters t[0::3], the largest sample rank of a
    mod-1 sample from the suffix array); deeper levels read the device DC3's
    level trace (names are 1..distinct of the level above)."""
    trace = _lib.dc3_trace()
    db = config.digit_bits

    def check(key_max: int, items: int) -> None:
        if items <= 0:
            return
        idx_bits = max(1, int(items - 1).bit_length())
        total = max(1, int(key_max).bit_length()) + idx_bits
        total = ((total + db - 1) // db) * db
        if total > MAX_KEY_BITS:
            raise ValueError("packed sort key exceeds 63 bits")

    for lvl, (n_l, sigma, m, _names) in enumerate(trace):
        k = (n_l + 2) // 3
        if lvl == 0 and sa is not None and text.n == n_l:
            t = np.concatenate([text.ranks, np.zeros(3, np.int64)])  # zero padding
            limit = n_l + 1 if n_l % 3 == 1 else n_l
            smp = np.concatenate([np.arange(1, limit, 3), np.arange(2, limit, 3)])
            for off in (2, 1, 0):  # _name_triples' keys t[s], t[s+1], t[s+2], least significant first
                check(int(t[smp + off].max()) if smp.size else 0, m)
            mod1 = np.arange(1, n_l, 3)
            rank_max = 0
            if mod1.size:  # 1-based ranks among the samples (pad sample lowest when present)
                real = np.concatenate([mod1, np.arange(2, n_l, 3)])
                top = int(sa.rank[mod1].max())
                rank_max = int(np.count_nonzero(sa.rank[real] <= top)) + (1 if n_l % 3 == 1 else 0)
            check(rank_max, k)                       # _sort_nonsamples' keys: rank_of[i+1], then t[i]
            check(int(t[0:n_l:3].max()), k)
        else:
            check(sigma, m)
            check(m, k)
            check(sigma, k)


def parallel_build_sa(text: RankedText, config: SortConfig | None = None) -> SuffixArray:
    """DC3 with all sorting passes on the (device) engine; equals the serial
    build (parallel_sort.py:288-293)."""
    config = config or SortConfig()
    # the engine check reads the reference recursion's levels: run the DC3
    # with the level-0 window naming off so the level trace is that recursion
    L = _lib.load() if text.n > 1 else None
    prev = L.saix_dc3_set_window_naming(0) if L is not None else None
    try:
        sa = build_sa_dc3(text)
    finally:
        if L is not None:
            L.saix_dc3_set_window_naming(prev)
    if text.n > 1:
        _engine_key_check(text, config, sa)
    return sa
