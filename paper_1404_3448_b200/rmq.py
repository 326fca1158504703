"""Sparse-table range-minimum queries on the B200 -- drop-in for the
``SparseTable`` half of ``saix.rmq`` (rmq.py:24-58, 254-259).

The table lives on the device as packed (value, index) entries (u32 when
value range + index bits fit 32, else u64).  ``query`` keeps
the reference's scalar signature (inclusive range, swapped if i > j, leftmost
argmin, IndexError out of range); ``query_batch`` / ``query_sparse_batch`` are
the throughput path: one kernel over arrays of queries.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib


def _check_range(n: int, i: int, j: int) -> tuple[int, int]:
    if not (0 <= i < n) or not (0 <= j < n):
        raise IndexError(f"query ({i}, {j}) out of bounds for length {n}")
    return (i, j) if i <= j else (j, i)


class SparseTable:
    """Indices of window minima for every power-of-two window width."""

    def __init__(self, values, _device_values=None):
        values = np.asarray(values, dtype=np.int64)
        if values.shape[0] == 0:
            raise ValueError("cannot build a sparse table over an empty array")
        self.values = values
        n = int(values.shape[0])
        L = _lib.load()
        if _device_values is not None:          # plan from a device min / max, no host pass
            t = _lib.torch()
            mm = t.empty(2, dtype=t.int64, device=_device_values[0].device)
            _lib.check(L.saix_minmax(_lib.ptr(_device_values[0]), _device_values[1], n, _lib.ptr(mm),
                                     _lib.stream_ptr()), "saix_minmax")
            vmin, vmax = (int(x) for x in mm.cpu().tolist())
        else:
            vmin, vmax = int(values.min()), int(values.max())
        plan = _lib.SparsePlan()
        _lib.check(L.saix_sparse_plan_make(n, vmin, vmax, ctypes.byref(plan)), "saix_sparse_plan_make")
        self.plan = plan
        _lib.device()
        t = _lib.torch()
        if _device_values is not None:          # (tensor, value_bytes) already on device
            self._vals, self._vbytes = _device_values
        else:
            self._vals, self._vbytes = _lib.to_device(values), 8
        self._table = _lib.workspace(plan.table_bytes)
        rc = L.saix_sparse_build(ctypes.byref(plan), _lib.ptr(self._vals), self._vbytes,
                                 _lib.ptr(self._table), _lib.stream_ptr())
        _lib.check(rc, "saix_sparse_build")
        self._err = t.zeros(1, dtype=t.int32, device=self._table.device)
        self._table_host = None

    @property
    def n(self) -> int:
        return int(self.plan.n)

    @property
    def table(self) -> list[np.ndarray]:
        """The reference layout: per level, int64 argmin indices."""
        if self._table_host is None:
            raw = self._table.cpu().numpy()
            n, ib = self.n, self.plan.index_bits
            mode = self.plan.mode
            dt = np.uint64 if mode == _lib.SPARSE_PACK64 else np.uint32
            flat = raw[: self.plan.table_bytes].view(dt)
            levels, off = [], 0
            for k in range(self.plan.levels):
                ln = n - (1 << k) + 1
                e = flat[off: off + ln].astype(np.uint64)
                idx = e if mode == _lib.SPARSE_INDEX else e & np.uint64((1 << ib) - 1)
                levels.append(idx.astype(np.int64))
                off += ln
            self._table_host = levels
        return self._table_host

    def query_device(self, qi, qj, want_values: bool = False):
        """Batched query on device int64 tensors; returns device tensors."""
        t = _lib.torch()
        L = _lib.load()
        q = int(qi.numel())
        out = t.empty(max(q, 1), dtype=t.int64, device=self._table.device)
        outv = t.empty(max(q, 1), dtype=t.int64, device=self._table.device) if want_values else None
        self._err.zero_()
        rc = L.saix_sparse_query(ctypes.byref(self.plan), _lib.ptr(self._table), _lib.ptr(self._vals),
                                 self._vbytes, _lib.ptr(qi), _lib.ptr(qj), q, _lib.ptr(out),
                                 _lib.ptr(outv), _lib.ptr(self._err), _lib.stream_ptr())
        _lib.check(rc, "saix_sparse_query")
        return out[:q], (outv[:q] if outv is not None else None)

    def query_batch(self, i, j) -> np.ndarray:
        """Vectorised ``query`` over equal-length integer arrays."""
        qi = np.ascontiguousarray(i, dtype=np.int64)
        qj = np.ascontiguousarray(j, dtype=np.int64)
        if qi.shape != qj.shape:
            raise ValueError("i and j must have the same shape")
        if qi.size == 0:
            return np.zeros(qi.shape, np.int64)
        out, _ = self.query_device(_lib.to_device(qi.ravel()), _lib.to_device(qj.ravel()))
        res = out.cpu().numpy()
        if int(self._err.item()):
            bad = np.flatnonzero((qi.ravel() < 0) | (qi.ravel() >= self.n)
                                 | (qj.ravel() < 0) | (qj.ravel() >= self.n))[0]
            raise IndexError(f"query ({int(qi.ravel()[bad])}, {int(qj.ravel()[bad])}) "
                             f"out of bounds for length {self.n}")
        return res.reshape(qi.shape)

    def query(self, i: int, j: int) -> int:
        i, j = _check_range(self.n, int(i), int(j))
        return int(self.query_batch(np.array([i]), np.array([j]))[0])


class DeviceSparseTable(SparseTable):
    """SparseTable over a device-resident array (u32 or int64), e.g. the LCP
    array the GPU just built: planned from a device min/max, never copied to
    the host.  ``values`` (host) is materialised lazily for API parity."""

    def __init__(self, values_dev, value_bytes: int, n: int):  # noqa: D401 - no super().__init__
        t = _lib.torch()
        L = _lib.load()
        if n <= 0:
            raise ValueError("cannot build a sparse table over an empty array")
        mm = t.empty(2, dtype=t.int64, device=values_dev.device)
        _lib.check(L.saix_minmax(_lib.ptr(values_dev), value_bytes, n, _lib.ptr(mm), _lib.stream_ptr()),
                   "saix_minmax")
        vmin, vmax = (int(x) for x in mm.tolist())
        plan = _lib.SparsePlan()
        _lib.check(L.saix_sparse_plan_make(n, vmin, vmax, ctypes.byref(plan)), "saix_sparse_plan_make")
        self.plan = plan
        self._vals, self._vbytes = values_dev, value_bytes
        self._table = _lib.workspace(plan.table_bytes)
        self._err = t.zeros(1, dtype=t.int32, device=values_dev.device)
        self._table_host = None
        self._values_host = None
        self.rebuild()

    def rebuild(self) -> None:
        """Re-run the table build kernels (the values are unchanged)."""
        L = _lib.load()
        _lib.check(L.saix_sparse_build(ctypes.byref(self.plan), _lib.ptr(self._vals), self._vbytes,
                                       _lib.ptr(self._table), _lib.stream_ptr()), "saix_sparse_build")

    @property
    def values(self) -> np.ndarray:
        if self._values_host is None:
            a = self._vals[: self.n].cpu().numpy()
            self._values_host = (a.view(np.uint32) if self._vbytes == 4 else a).astype(np.int64)
        return self._values_host


def build_sparse(values) -> SparseTable:
    return SparseTable(values)


def query_sparse(st: SparseTable, i: int, j: int) -> int:
    return st.query(i, j)


def query_sparse_batch(st: SparseTable, i, j) -> np.ndarray:
    """Equals ``[query_sparse(st, a, b) for a, b in zip(i, j)]``."""
    return st.query_batch(i, j)
