"""Range-minimum queries on the B200 -- drop-in for ``saix.rmq``: the
``SparseTable`` engine (rmq.py:24-58, 254-259) and the Cartesian-tree /
Euler-tour / ±1 engine (rmq.py:61-251, end of this file).

The table lives on the device as packed (value, index) entries (u32 when
value range + index bits fit 32, else u64).  ``query`` keeps
the reference's scalar signature (inclusive range, swapped if i > j, leftmost
argmin, IndexError out of range); ``query_batch`` / ``query_sparse_batch`` are
the throughput path: one kernel over arrays of queries.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field
from typing import Any

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
        _lib.check(L.saix_sparse_plan_blocked(n, vmin, vmax, ctypes.byref(plan)), "saix_sparse_plan_blocked")
        self.plan = plan
        self._vrange = (vmin, vmax)
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

    def _full_table(self):
        """(plan, device table) in the per-level layout; a blocked query table
        (SAIX_SPARSE_BLOCKED) gets a full one built on demand."""
        if self.plan.mode != _lib.SPARSE_BLOCKED:
            return self.plan, self._table
        L = _lib.load()
        plan = _lib.SparsePlan()
        _lib.check(L.saix_sparse_plan_make(self.n, self._vrange[0], self._vrange[1], ctypes.byref(plan)),
                   "saix_sparse_plan_make")
        tab = _lib.workspace(plan.table_bytes)
        _lib.check(L.saix_sparse_build(ctypes.byref(plan), _lib.ptr(self._vals), self._vbytes, _lib.ptr(tab),
                                       _lib.stream_ptr()), "saix_sparse_build")
        return plan, tab

    @property
    def table(self) -> list[np.ndarray]:
        """The reference layout: per level, int64 argmin indices."""
        if self._table_host is None:
            plan, tab = self._full_table()
            raw = tab.cpu().numpy()
            n, ib = self.n, plan.index_bits
            mode = plan.mode
            dt = np.uint64 if mode == _lib.SPARSE_PACK64 else np.uint32
            flat = raw[: plan.table_bytes].view(dt)
            levels, off = [], 0
            for k in range(plan.levels):
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
        _lib.check(L.saix_sparse_plan_blocked(n, vmin, vmax, ctypes.byref(plan)), "saix_sparse_plan_blocked")
        self.plan = plan
        self._vrange = (vmin, vmax)
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


# ------------------------------------------------------- Cartesian pipeline
# The reference's second RMQ engine (rmq.py:61-251): Cartesian tree -> Euler
# tour -> ±1 RMQ, built on the device (csrc/cartesian.cu); same classes,
# fields, values and query answers.


@dataclass
class CartesianTree:
    """Min-heap binary tree whose in-order traversal is 0..n-1; ties break so
    the leftmost minimum becomes the ancestor (rmq.py:61-72)."""

    values: np.ndarray
    parent: np.ndarray
    left: np.ndarray
    right: np.ndarray
    root: int
    _tour: Any = field(default=None, repr=False, compare=False)


@dataclass
class EulerTour:
    """Depth-first tour (node on entry and after each child; rmq.py:75-88)."""

    tour_nodes: np.ndarray
    tour_depths: np.ndarray
    first_visit: np.ndarray
    _dev: Any = field(default=None, repr=False, compare=False)  # (nodes, depths, first) int32 tensors


def _cartesian_device(values: np.ndarray):
    t = _lib.torch()
    L = _lib.load()
    n = int(values.shape[0])
    _lib.device()
    vals = _lib.to_device(values)
    parent, left, right, first = (_lib.empty(n, t.int32) for _ in range(4))
    nodes, depths = (_lib.empty(2 * n - 1, t.int32) for _ in range(2))
    root = np.zeros(1, np.int64)
    ws = _lib.workspace(L.saix_cartesian_workspace_bytes(n))
    _lib.check(L.saix_cartesian_build(_lib.ptr(vals), 8, n, _lib.ptr(parent), _lib.ptr(left), _lib.ptr(right),
                                      _lib.ptr(nodes), _lib.ptr(depths), _lib.ptr(first), root.ctypes.data,
                                      _lib.ptr(ws), ws.numel(), _lib.stream_ptr()), "saix_cartesian_build")
    i32 = lambda x, k: x[:k].cpu().numpy().astype(np.int64)  # noqa: E731  (signed: -1 = none)
    tour = EulerTour(tour_nodes=i32(nodes, 2 * n - 1), tour_depths=i32(depths, 2 * n - 1),
                     first_visit=i32(first, n), _dev=(nodes, depths, first))
    tree = CartesianTree(values=values, parent=i32(parent, n), left=i32(left, n), right=i32(right, n),
                         root=int(root[0]), _tour=tour)
    return tree


def build_cartesian(values) -> CartesianTree:
    """Cartesian tree of ``values`` (rmq.py:91-117) on the device."""
    values = np.asarray(values, dtype=np.int64)
    if len(values) == 0:
        raise ValueError("cannot build a Cartesian tree over an empty array")
    return _cartesian_device(values)


def euler_tour(tree: CartesianTree) -> EulerTour:
    """Euler tour of a Cartesian tree (rmq.py:120-152); the device builds it
    with the tree, from the same nearest-value links."""
    if tree._tour is None:
        tree._tour = _cartesian_device(np.asarray(tree.values, dtype=np.int64))._tour
    return tree._tour


class PlusMinusOneRmq:
    """O(1) RMQ over an array whose adjacent entries differ by exactly 1
    (rmq.py:155-236): blocks of b = max(1, floor(log2 m / 2)), per-block
    leftmost argmin / min / step-pattern type, one in-block table per present
    type, a sparse table over block minima -- all built on the device."""

    def __init__(self, depths, _device_depths=None):
        depths = np.asarray(depths, dtype=np.int64)
        m = len(depths)
        if m == 0:
            raise ValueError("cannot build over an empty array")
        t = _lib.torch()
        L = _lib.load()
        _lib.device()
        self.depths = depths
        self.block = b = max(1, (m.bit_length() - 1) // 2)
        if b > 16:
            raise ValueError("array too large for the ±1 engine")
        nblocks = (m + b - 1) // b
        d0 = int(depths[0])
        if _device_depths is not None and d0 == 0:
            dd = _device_depths
        else:  # argmin is shift-invariant: store depths - depths[0] (|.| < m) as int32
            dd = _lib.to_device((depths - d0).astype(np.int32))
        self._d = dd
        bargmin, bmin, types = (_lib.empty(nblocks, t.int32) for _ in range(3))
        ncodes = 1 << (b - 1)
        present = _lib.empty(((ncodes + 3) & ~3) + 4, t.uint8)
        tab = _lib.empty(ncodes * b * b, t.uint8)
        bad = np.zeros(1, np.int32)
        _lib.check(L.saix_pm1_build(_lib.ptr(dd), m, b, _lib.ptr(bargmin), _lib.ptr(bmin), _lib.ptr(types),
                                    _lib.ptr(present), _lib.ptr(tab), bad.ctypes.data, _lib.stream_ptr()),
                   "saix_pm1_build")
        if bad[0]:
            raise ValueError("adjacent entries must differ by exactly 1")
        self._bargmin, self._types, self._tab = bargmin, types, tab
        self.block_argmin = bargmin[:nblocks].cpu().numpy().astype(np.int64)
        self.block_min = bmin[:nblocks].cpu().numpy().astype(np.int64) + d0
        self.block_sparse = SparseTable(self.block_min)
        self.types = types[:nblocks].cpu().numpy().astype(np.int64)
        flags = present[:ncodes].cpu().numpy()
        tabs = tab[:ncodes * b * b].cpu().numpy().reshape(ncodes, b, b)
        self.inblock: dict[int, np.ndarray] = {int(c): tabs[c].astype(np.int64) for c in np.flatnonzero(flags)}

    def _inblock_query(self, blk: int, lo: int, hi: int) -> int:
        return blk * self.block + int(self.inblock[int(self.types[blk])][lo, hi])

    def _query_device(self, qi, qj, first=None, nodes=None) -> np.ndarray:
        t = _lib.torch()
        L = _lib.load()
        q = int(qi.shape[0])
        di, dj = _lib.to_device(qi), _lib.to_device(qj)
        lo, hi = _lib.empty(q, t.int64), _lib.empty(q, t.int64)
        cand = _lib.empty(3 * q, t.int32)
        st = _lib.stream_ptr()
        _lib.check(L.saix_pm1_query_begin(self.block, _lib.ptr(self._types), _lib.ptr(self._tab),
                                          _lib.ptr(first) if first is not None else None, _lib.ptr(di),
                                          _lib.ptr(dj), q, _lib.ptr(lo), _lib.ptr(hi), _lib.ptr(cand), st),
                   "saix_pm1_query_begin")
        mid, _ = self.block_sparse.query_device(lo[:q], hi[:q])
        out = _lib.empty(q, t.int64)
        _lib.check(L.saix_pm1_query_end(_lib.ptr(self._d), self.block, _lib.ptr(self._bargmin), _lib.ptr(mid),
                                        _lib.ptr(cand), _lib.ptr(nodes) if nodes is not None else None, q,
                                        _lib.ptr(out), st), "saix_pm1_query_end")
        return out[:q].cpu().numpy()

    def query_batch(self, i, j) -> np.ndarray:
        qi = np.ascontiguousarray(i, dtype=np.int64).ravel()
        qj = np.ascontiguousarray(j, dtype=np.int64).ravel()
        m = len(self.depths)
        if qi.size and (qi.min() < 0 or qi.max() >= m or qj.min() < 0 or qj.max() >= m):
            bad = np.flatnonzero((qi < 0) | (qi >= m) | (qj < 0) | (qj >= m))[0]
            raise IndexError(f"query ({int(qi[bad])}, {int(qj[bad])}) out of bounds for length {m}")
        if qi.size == 0:
            return np.zeros(0, np.int64)
        return self._query_device(qi, qj)

    def query(self, i: int, j: int) -> int:
        i, j = _check_range(len(self.depths), int(i), int(j))
        return int(self.query_batch(np.array([i]), np.array([j]))[0])


class CartesianRmq:
    """Range minima answered as LCAs: tree + tour + ±1 RMQ, built once on the
    device (rmq.py:239-251)."""

    def __init__(self, values):
        self.values = np.asarray(values, dtype=np.int64)
        self.tree = build_cartesian(self.values)
        self.tour = euler_tour(self.tree)
        self.pm1 = PlusMinusOneRmq(self.tour.tour_depths, _device_depths=self.tour._dev[1])

    def query_batch(self, i, j) -> np.ndarray:
        qi = np.ascontiguousarray(i, dtype=np.int64).ravel()
        qj = np.ascontiguousarray(j, dtype=np.int64).ravel()
        n = len(self.values)
        if qi.size and (qi.min() < 0 or qi.max() >= n or qj.min() < 0 or qj.max() >= n):
            bad = np.flatnonzero((qi < 0) | (qi >= n) | (qj < 0) | (qj >= n))[0]
            raise IndexError(f"query ({int(qi[bad])}, {int(qj[bad])}) out of bounds for length {n}")
        if qi.size == 0:
            return np.zeros(0, np.int64)
        nodes, _, first = self.tour._dev
        return self.pm1._query_device(qi, qj, first=first, nodes=nodes)

    def query(self, i: int, j: int) -> int:
        i, j = _check_range(len(self.values), int(i), int(j))
        return int(self.query_batch(np.array([i]), np.array([j]))[0])


def build_pm1(depths) -> PlusMinusOneRmq:
    return PlusMinusOneRmq(depths)


def query_pm1(structure: PlusMinusOneRmq, i: int, j: int) -> int:
    return structure.query(i, j)


def rmq_via_lca(values, i: int, j: int) -> int:
    """One-shot build-and-query through the Cartesian pipeline (rmq.py:266-268)."""
    return CartesianRmq(values).query(i, j)
