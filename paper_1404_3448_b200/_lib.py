"""ctypes binding of libsaix_b200.so (include/saix_b200.h) + device plumbing.

PyTorch is used only for device memory, streams and host<->device copies.
There is no CPU fallback: every compute call needs the CUDA library and a
visible GPU and raises RuntimeError otherwise.
"""

from __future__ import annotations

import ctypes
import os
import warnings

import numpy as np

from . import _build

_c = ctypes
_vp = _c.c_void_p
_i64 = _c.c_int64
_int = _c.c_int

SAIX_OK = 0
SAIX_EINVAL = -22
SAIX_ERANGE = -34
SAIX_ENOSPC = -28
SAIX_ECUDA = -100
SAIX_ESEQ = -101
SAIX_ENCCL = -102

SPARSE_PACK32, SPARSE_PACK64, SPARSE_INDEX, SPARSE_BLOCKED = 0, 1, 2, 3


class Dc3Probe(_c.Structure):
    _fields_ = [
        ("triple_text", _vp),
        ("sample_rank", _vp),
        ("sorted_samples", _vp),
        ("sorted_nonsamples", _vp),
        ("n_samples", _i64),
        ("n_sorted_samples", _i64),
        ("n_sorted_nonsamples", _i64),
        ("depth", _c.c_int32),
        ("reserved", _c.c_int32),
    ]


class ProfEntry(_c.Structure):
    _fields_ = [("name", _c.c_char * 64), ("launches", _i64), ("total_ms", _c.c_double),
                ("bytes", _c.c_double)]


class SparsePlan(_c.Structure):
    _fields_ = [
        ("n", _i64),
        ("value_bias", _i64),
        ("table_bytes", _i64),
        ("levels", _c.c_int32),
        ("mode", _c.c_int32),
        ("index_bits", _c.c_int32),
        ("value_bits", _c.c_int32),
    ]


# name -> (restype, argtypes); mirrors include/saix_b200.h exactly
SIGNATURES = {
    "saix_last_error": (_c.c_char_p, []),
    "saix_abi_version": (_int, []),
    "saix_prof_enable": (None, [_int]),
    "saix_prof_collect": (_int, [_c.POINTER(ProfEntry), _int]),
    "saix_encode_gsa": (_int, [_vp, _i64, _vp, _i64, _int, _vp, _vp, _vp]),
    "saix_encode": (_int, [_vp, _i64, _int, _vp, _vp, _vp]),
    "saix_dc3_workspace_bytes": (_c.c_size_t, [_i64, _int]),
    "saix_dc3": (_int, [_vp, _int, _i64, _i64, _vp, _vp, _vp, _c.c_size_t,
                        _c.POINTER(Dc3Probe), _vp]),
    "saix_dc3_merge_workspace_bytes": (_c.c_size_t, [_i64]),
    "saix_dc3_merge": (_int, [_vp, _int, _i64, _vp, _vp, _i64, _vp, _i64, _vp, _vp, _c.c_size_t, _vp]),
    "saix_lcp_workspace_bytes": (_c.c_size_t, [_i64]),
    "saix_lcp": (_int, [_vp, _int, _i64, _vp, _vp, _vp, _vp, _c.c_size_t, _vp]),
    "saix_lcp_sigma": (_int, [_vp, _int, _i64, _i64, _i64, _vp, _vp, _vp, _c.c_size_t, _vp]),
    "saix_dc3_trace": (_int, [_vp, _int]),
    "saix_dc3_naming": (_int, []),
    "saix_psort_workspace_bytes": (_c.c_size_t, [_i64]),
    "saix_exclusive_scan_i64": (_int, [_vp, _i64, _vp, _vp, _c.c_size_t, _vp]),
    "saix_split_by_bit": (_int, [_vp, _i64, _int, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _c.c_size_t, _vp]),
    "saix_radix_sort_i64": (_int, [_vp, _i64, _int, _vp, _vp, _c.c_size_t, _vp]),
    "saix_minmax": (_int, [_vp, _int, _i64, _vp, _vp]),
    "saix_widen_i64": (_int, [_vp, _int, _i64, _vp, _vp]),
    "saix_cartesian_workspace_bytes": (_c.c_size_t, [_i64]),
    "saix_cartesian_build": (_int, [_vp, _int, _i64, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _c.c_size_t, _vp]),
    "saix_pm1_build": (_int, [_vp, _i64, _int, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "saix_pm1_query_begin": (_int, [_int, _vp, _vp, _vp, _vp, _vp, _i64, _vp, _vp, _vp, _vp]),
    "saix_pm1_query_end": (_int, [_vp, _int, _vp, _vp, _vp, _vp, _i64, _vp, _vp]),
    "saix_fasta_lines": (_int, [_vp, _i64, _vp, _vp, _c.c_size_t, _vp]),
    "saix_fasta_workspace_bytes": (_c.c_size_t, [_i64, _i64]),
    "saix_fasta_scan": (_int, [_vp, _i64, _i64, _vp, _vp, _c.c_size_t, _vp]),
    "saix_fasta_emit": (_int, [_vp, _i64, _i64, _int, _int, _vp, _vp, _vp, _vp, _vp, _vp, _c.c_size_t, _vp]),
    "saix_dc3_set_window_naming": (_int, [_int]),
    "saix_crc32_workspace_bytes": (_c.c_size_t, [_i64]),
    "saix_crc32": (_int, [_vp, _i64, _vp, _vp, _c.c_size_t, _vp]),
    "saix_index_bytes": (_i64, [_i64]),
    "saix_index_pack": (_int, [_vp, _vp, _vp, _i64, _i64, _i64, _vp, _vp, _c.c_size_t, _vp]),
    "saix_index_unpack_workspace_bytes": (_c.c_size_t, [_i64]),
    "saix_index_unpack": (_int, [_vp, _i64, _vp, _vp, _vp, _vp, _vp, _c.c_size_t, _vp]),
    "saix_sparse_plan_make": (_int, [_i64, _i64, _i64, _c.POINTER(SparsePlan)]),
    "saix_comm_unique_id": (_int, [_vp]),
    "saix_comm_init": (_int, [_c.POINTER(_vp), _int, _vp, _int, _int]),
    "saix_comm_destroy": (_int, [_vp]),
    "saix_comm_allgather_i64": (_int, [_vp, _vp, _i64, _vp, _vp]),
    "saix_comm_allreduce_min_i64": (_int, [_vp, _vp, _vp, _i64, _vp]),
    "saix_sparse_plan_blocked": (_int, [_i64, _i64, _i64, _c.POINTER(SparsePlan)]),
    "saix_sparse_build": (_int, [_c.POINTER(SparsePlan), _vp, _int, _vp, _vp]),
    "saix_sparse_query": (_int, [_c.POINTER(SparsePlan), _vp, _vp, _int, _vp, _vp, _i64,
                                 _vp, _vp, _vp, _vp]),
    "saix_lcp_query": (_int, [_c.POINTER(SparsePlan), _vp, _vp, _int, _vp, _vp, _vp, _i64,
                              _vp, _vp, _vp]),
    "saix_overlap_workspace_bytes": (_c.c_size_t, [_i64]),
    "saix_overlap_scan": (_int, [_vp, _vp, _i64, _i64, _vp, _vp, _c.c_size_t, _vp]),
    "saix_longest_overlap_workspace_bytes": (_c.c_size_t, [_i64, _i64]),
    "saix_longest_overlap": (_int, [_vp, _i64, _vp, _i64, _int, _vp, _vp, _vp, _c.c_size_t, _vp]),
    "saix_overlap_batch_workspace_bytes": (_c.c_size_t, [_vp, _i64]),
    "saix_overlap_batch": (_int, [_vp, _vp, _i64, _int, _vp, _vp, _vp, _c.c_size_t, _vp]),
    "saix_overlap_batch_dev": (_int, [_vp, _vp, _vp, _i64, _int, _vp, _vp, _vp, _c.c_size_t, _vp]),
    "saix_overlap_batch_stream": (_int, [_vp, _vp, _vp, _vp, _i64, _int, _int, _vp, _vp, _vp, _c.c_size_t, _vp,
                                         _vp]),
    "saix_overlap_batch_set_onchip": (_int, [_int]),
    "saix_overlap_batch_last_fallbacks": (_i64, []),
    "saix_overlap_batch_phase_clocks": (_int, [_vp, _int]),
}

_lib = None


def lib_path() -> str:
    return _build.LIB


def load(build_if_missing: bool = True):
    """Load libsaix_b200.so (building it in-tree when nvcc is available)."""
    global _lib
    if _lib is not None:
        return _lib
    path = _build.LIB
    if not os.path.exists(path) and build_if_missing and os.path.exists(_build.NVCC):
        _build.build()
    if not os.path.exists(path):
        raise RuntimeError(
            f"libsaix_b200.so not found at {path}; build it with "
            "`python -c 'import __graft_entry__; __graft_entry__.build()'` "
            "(there is no CPU fallback)")
    L = _c.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    _lib = L
    return L


def check(rc: int, what: str = "") -> None:
    if rc == SAIX_OK:
        return
    msg = load().saix_last_error().decode(errors="replace")
    if rc == SAIX_ERANGE:
        raise IndexError(msg or what)
    if rc == SAIX_EINVAL:
        raise ValueError(msg or what)
    raise RuntimeError(f"{what}: saix error {rc}: {msg}")


# ------------------------------------------------------------------ torch

_torch = None


def torch():
    global _torch
    if _torch is None:
        import torch as t
        _torch = t
    return _torch


def device():
    t = torch()
    if not t.cuda.is_available():
        raise RuntimeError("paper_1404_3448_b200 needs a CUDA device (B200); "
                           "there is no CPU fallback")
    load()
    return t.device("cuda", t.cuda.current_device())


def stream_ptr() -> int:
    return torch().cuda.current_stream().cuda_stream


def ptr(t) -> int | None:
    return None if t is None else t.data_ptr()


def empty(n: int, dtype, dev=None):
    t = torch()
    return t.empty(max(int(n), 1), dtype=dtype, device=dev or device())


def workspace(nbytes: int):
    return empty(nbytes, torch().uint8)


def to_device(arr: np.ndarray, dev=None):
    """Host numpy -> device tensor (pinned staging for large arrays)."""
    t = torch()
    arr = np.ascontiguousarray(arr)
    if not arr.flags.writeable:   # read-only host data (e.g. file bytes): only ever copied from
        with warnings.catch_warnings():
            warnings.simplefilter("ignore", UserWarning)
            h = t.from_numpy(arr)
    else:
        h = t.from_numpy(arr)
    if h.numel() == 0:
        return t.empty(1, dtype=h.dtype, device=dev or device())
    return h.to(dev or device(), non_blocking=False)


def to_host(t_dev, n: int | None = None, dtype=np.int64) -> np.ndarray:
    """Device tensor -> host numpy (widened to `dtype`)."""
    if n is not None:
        t_dev = t_dev[:n]
    a = t_dev.cpu().numpy()
    if n == 0:
        a = a[:0]
    return a.astype(dtype, copy=False) if a.dtype != dtype else a


def widen_i64_host(t_dev, n: int) -> np.ndarray:
    """u8 / u32 device array (uint8 / int32 tensor) -> host int64, widened on
    the device (saix_widen_i64) so the download is the only host work."""
    if n == 0:
        return np.zeros(0, np.int64)
    t = torch()
    src_bytes = 1 if t_dev.dtype == t.uint8 else 4
    out = t.empty(n, dtype=t.int64, device=t_dev.device)
    check(load().saix_widen_i64(ptr(t_dev), src_bytes, n, ptr(out), stream_ptr()), "saix_widen_i64")
    host = t.empty(n, dtype=t.int64, pin_memory=True)   # torch caches pinned blocks across calls
    host.copy_(out)
    return host.numpy()


_staging = {}


def staging(nbytes: int):
    """A reusable pinned host uint8 buffer of at least nbytes (grown in powers
    of two): file images pass through it at full PCIe / C2C speed instead of
    page-faulting into fresh pageable memory."""
    t = torch()
    buf = _staging.get("b")
    if buf is None or buf.numel() < nbytes:
        size = 1 << max(20, (int(nbytes) - 1).bit_length())
        _staging.pop("b", None)
        buf = t.empty(size, dtype=t.uint8, pin_memory=True)
        _staging["b"] = buf
    return buf


def u32_to_i64_host(t_dev, n: int) -> np.ndarray:
    """u32 device array (stored in an int32 tensor) -> host int64."""
    return widen_i64_host(t_dev, n)


def prof_enable(on: bool = True) -> None:
    load().saix_prof_enable(int(on))


def prof_collect() -> list[dict]:
    """Per-kernel CUDA-event totals since prof_enable (synchronizes)."""
    L = load()
    buf = (ProfEntry * 256)()
    n = L.saix_prof_collect(buf, 256)
    return [{"name": buf[i].name.decode(), "launches": int(buf[i].launches),
             "ms": float(buf[i].total_ms), "bytes": float(buf[i].bytes)} for i in range(min(n, 256))]


def dc3_naming() -> int:
    """Level-0 naming path of the last DC3 level 0 on this thread (0 triples,
    1 generic window sort, 2 DNA window sort)."""
    return int(load().saix_dc3_naming())


def dc3_trace() -> list[tuple[int, int, int, int]]:
    """(N, sigma, m, distinct names) per level of the last DC3 on this thread."""
    import numpy as np
    out = np.zeros(4 * 64, np.int64)
    k = load().saix_dc3_trace(out.ctypes.data, 64)
    return [tuple(int(x) for x in out[4 * i: 4 * i + 4]) for i in range(min(k, 64))]
