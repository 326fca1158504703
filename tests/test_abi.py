"""CPU checks of the C-ABI boundary: the library loads, exports exactly what
include/saix_b200.h declares, and its host-only planning entry points behave.
No compute calls (there is no GPU here)."""

import ctypes
import os
import re
import subprocess

import pytest

from paper_1404_3448_b200 import _build, _lib

HEADER = os.path.join(os.path.dirname(_build.PKG), "include", "saix_b200.h")


def declared():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"SAIX_API\s+[\w\s\*]*?\b(saix_\w+)\s*\(", src)))


def test_header_declares_entry_points():
    names = declared()
    assert "saix_dc3" in names and "saix_lcp" in names and "saix_longest_overlap" in names
    assert len(names) >= 17


def test_library_exports_every_declared_symbol():
    _lib.load()
    out = subprocess.run(["nm", "-D", "--defined-only", _build.LIB], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r"\bT (saix_\w+)", out))
    assert set(declared()) <= exported
    # and nothing undeclared leaks out of the C ABI
    assert exported <= set(declared())


def test_bindings_cover_header():
    assert set(_lib.SIGNATURES) == set(declared())


def test_sm100a_code_object():
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _build.LIB],
                         capture_output=True, text=True, check=True).stdout
    assert "sm_100a" in out


def test_version_and_error_string():
    L = _lib.load()
    assert L.saix_abi_version() == 1
    assert isinstance(L.saix_last_error(), bytes)


def test_sparse_plan_layouts():
    L = _lib.load()
    p = _lib.SparsePlan()
    # LCP-like values at 2^26 pack into 32 bits (5 value bits + 26 index bits)
    assert L.saix_sparse_plan_make(1 << 26, 0, 24, ctypes.byref(p)) == 0
    assert p.mode == _lib.SPARSE_PACK32 and p.levels == 27 and p.index_bits == 26
    lens = sum((1 << 26) - (1 << k) + 1 for k in range(27))
    assert p.table_bytes == 4 * lens
    assert L.saix_sparse_plan_make(1000, -5, 1 << 40, ctypes.byref(p)) == 0
    assert p.mode == _lib.SPARSE_PACK64 and p.levels == 10
    assert L.saix_sparse_plan_make(1000, -(1 << 62), 1 << 62, ctypes.byref(p)) == 0
    assert p.mode == _lib.SPARSE_INDEX
    assert L.saix_sparse_plan_make(0, 0, 0, ctypes.byref(p)) == _lib.SAIX_EINVAL
    assert b"empty" in L.saix_last_error()


@pytest.mark.parametrize("n", [0, 1, 2, 8, 1000, 20_000_001, 1 << 28])
def test_workspace_planners_monotone(n):
    L = _lib.load()
    a = L.saix_dc3_workspace_bytes(n, 1)
    b = L.saix_dc3_workspace_bytes(n + 1000, 1)
    assert 0 < a <= b
    # worst-case recursion: persistent per-level arrays (tt, SAc, ISAc, child SA)
    # ~ 12 * sum(N_l) = 36 n, plus the largest level's temps (records and bucketed-scatter staging)
    assert a < 96 * max(n, 1) + (1 << 24)
    assert L.saix_lcp_workspace_bytes(n) > 0
    assert L.saix_overlap_workspace_bytes(n) > 0
    assert L.saix_longest_overlap_workspace_bytes(n // 2, n - n // 2) >= a


def test_invalid_arguments_rejected_without_gpu():
    L = _lib.load()
    assert L.saix_dc3(None, 3, 10, 4, None, None, None, 0, None, None) == _lib.SAIX_EINVAL
    assert L.saix_lcp(None, 1, -1, None, None, None, None, 0, None) == _lib.SAIX_EINVAL


def test_product_never_imports_oracle():
    pkg = _build.PKG
    for root, _, files in os.walk(pkg):
        for f in files:
            if f.endswith(".py"):
                src = open(os.path.join(root, f)).read()
                assert "import oracle" not in src and "from oracle" not in src, f
