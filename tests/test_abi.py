"""CPU-side checks of the C-ABI library: it builds, loads, exports every
symbol include/mm.h declares, and rejects bad arguments before touching the
GPU (no compute call is made here)."""
from __future__ import annotations

import ctypes
import os
import re
import subprocess

import pytest

import paper_1506_04383_b200 as mm
from paper_1506_04383_b200 import _build, mulment

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    _build.build()
    return mm.load()


def header_symbols():
    src = open(os.path.join(ROOT, "include", "mm.h")).read()
    return sorted(set(re.findall(r"^MM_API [^(]*?\b(mm_[a-z_0-9]+)\(", src, flags=re.M)))


def test_header_declares_the_four_entry_points():
    syms = header_symbols()
    for s in ["mm_build_hierarchy", "mm_sweep", "mm_layout", "mm_energy"]:
        assert s in syms


def test_library_exports_every_declared_symbol(lib):
    out = subprocess.check_output(["nm", "-D", "--defined-only", mm.LIB_PATH]).decode()
    exported = set(re.findall(r" T (mm_[a-z_0-9]+)", out))
    missing = [s for s in header_symbols() if s not in exported]
    assert not missing, missing
    assert sorted(header_symbols()) == sorted(mulment.EXPORTS)


def test_library_is_sm100a_only(lib):
    out = subprocess.check_output(["/usr/local/cuda/bin/cuobjdump", "--list-elf", mm.LIB_PATH]).decode()
    assert "sm_100a" in out
    for other in ["sm_90", "sm_80", "sm_103"]:
        assert other not in out


def test_status_strings_and_version(lib):
    assert mm.mulment.status_name(0) == "MM_OK"
    assert mm.mulment.status_name(-3) == "MM_ERR_NONFINITE"
    assert lib.mm_version().decode().startswith("mm_b200")


def test_argument_errors_before_any_launch(lib):
    n0 = lib.mm_launch_count()
    # NULL S
    rc = lib.mm_sweep(None, 2, 0.1, 0.0, None, None, None, None, None, 0, None)
    assert rc == mulment.MM_ERR_INVALID_ARGUMENT
    assert b"S is NULL" in lib.mm_last_error()
    # bad dim / negative q with a syntactically valid S (fake device pointers, never dereferenced)
    s = mulment.mm_sset(4, 6, 0x1000, 0x2000, 0x3000, 0x4000)
    rc = lib.mm_sweep(ctypes.byref(s), 4, 0.1, 0.0, None, 0x5000, 0x6000, None, None, 0, None)
    assert rc == mulment.MM_ERR_UNSUPPORTED
    rc = lib.mm_sweep(ctypes.byref(s), 2, 0.1, -1.0, None, 0x5000, 0x6000, None, None, 0, None)
    assert rc == mulment.MM_ERR_UNSUPPORTED
    # aliasing x_out == x_in
    rc = lib.mm_sweep(ctypes.byref(s), 2, 0.1, 0.0, None, 0x5000, 0x5000, None, None, 0, None)
    assert rc == mulment.MM_ERR_INVALID_ARGUMENT and b"alias" in lib.mm_last_error()
    # misaligned float4 coordinates for dim 3
    rc = lib.mm_sweep(ctypes.byref(s), 3, 0.1, 0.0, None, 0x5008, 0x6000, None, None, 0, None)
    assert rc == mulment.MM_ERR_INVALID_ARGUMENT and b"aligned" in lib.mm_last_error()
    # energy needs a host output
    rc = lib.mm_energy(ctypes.byref(s), 2, 0.1, 0.0, 0x5000, None, None)
    assert rc == mulment.MM_ERR_INVALID_ARGUMENT
    # layout: h = 0 needs x_init; negative sweeps rejected
    sw = (ctypes.c_int32 * 1)(5)
    rep = mulment.mm_layout_report()
    rc = lib.mm_layout(None, ctypes.byref(s), 2, 0.1, 0.0, 0, sw, 1, 1, 1000, None, 0x6000, ctypes.byref(rep), None)
    assert rc == mulment.MM_ERR_INVALID_ARGUMENT
    swn = (ctypes.c_int32 * 1)(-1)
    rc = lib.mm_layout(None, ctypes.byref(s), 2, 0.1, 0.0, 0, swn, 1, 1, 1000, 0x5000, 0x6000, None, None)
    assert rc == mulment.MM_ERR_INVALID_ARGUMENT
    # hierarchy: bad dim, bad graph
    g = mulment.mm_graph(4, 6, 0x1000, 0x2000, None)
    h = ctypes.c_void_p()
    assert lib.mm_build_hierarchy(ctypes.byref(g), None, 5, 1, 10, 8, 8, ctypes.byref(h), None) == \
        mulment.MM_ERR_UNSUPPORTED
    assert lib.mm_build_hierarchy(None, None, 2, 1, 10, 8, 8, ctypes.byref(h), None) == \
        mulment.MM_ERR_INVALID_ARGUMENT
    # mm_sweeps: NULL S, bad K, aliasing
    rc = lib.mm_sweeps(None, 2, 0.1, 0.0, None, 0x5000, 0x6000, 3, None, None)
    assert rc == mulment.MM_ERR_INVALID_ARGUMENT
    rc = lib.mm_sweeps(ctypes.byref(s), 2, 0.1, 0.0, None, 0x5000, 0x6000, -1, None, None)
    assert rc == mulment.MM_ERR_INVALID_ARGUMENT
    rc = lib.mm_sweeps(ctypes.byref(s), 2, 0.1, 0.0, None, 0x5000, 0x5000, 3, None, None)
    assert rc == mulment.MM_ERR_INVALID_ARGUMENT and b"alias" in lib.mm_last_error()
    # mm_prolong: bad dim, negative size, NULL parent, aliasing, misaligned float4
    assert lib.mm_prolong(8, 4, 0x1000, 0x5000, None, 1, 0, 0x6000, None) == mulment.MM_ERR_UNSUPPORTED
    assert lib.mm_prolong(-1, 2, 0x1000, 0x5000, None, 1, 0, 0x6000, None) == mulment.MM_ERR_INVALID_ARGUMENT
    assert lib.mm_prolong(8, 2, None, 0x5000, None, 1, 0, 0x6000, None) == mulment.MM_ERR_INVALID_ARGUMENT
    assert lib.mm_prolong(8, 2, 0x1000, 0x5000, None, 1, 0, 0x5000, None) == mulment.MM_ERR_INVALID_ARGUMENT
    assert lib.mm_prolong(8, 3, 0x1000, 0x5008, None, 1, 0, 0x6000, None) == mulment.MM_ERR_INVALID_ARGUMENT
    assert lib.mm_prolong(0, 2, None, None, None, 1, 0, None, None) == mulment.MM_OK  # empty: nothing to do
    # mm_sweep: a caller workspace that is not 256-B aligned
    rc = lib.mm_sweep(ctypes.byref(s), 2, 0.1, 0.0, None, 0x5000, 0x6000, None, 0x7010, 1 << 40, None)
    assert rc == mulment.MM_ERR_INVALID_ARGUMENT and b"256-B" in lib.mm_last_error()
    assert lib.mm_launch_count() == n0  # nothing was launched


def test_workspace_query(lib):
    b = ctypes.c_size_t()
    assert lib.mm_sweep_workspace(65536, 2, None, ctypes.byref(b)) == 0 and b.value > 65536 * 8
    ap = mulment.mm_approx(1000, 0x1000, 0x2000)
    b2 = ctypes.c_size_t()
    assert lib.mm_sweep_workspace(65536, 3, ctypes.byref(ap), ctypes.byref(b2)) == 0 and b2.value > 0
    assert lib.mm_sweep_workspace(0, 2, None, ctypes.byref(b)) == mulment.MM_ERR_INVALID_ARGUMENT


def test_product_path_has_no_oracle_or_fallback():
    """The CUDA package never imports oracle/ and has no CPU code path."""
    pkg = os.path.join(ROOT, "paper_1506_04383_b200")
    for f in os.listdir(pkg):
        if f.endswith(".py"):
            src = open(os.path.join(pkg, f)).read()
            assert "import oracle" not in src and "from oracle" not in src, f
    for f in os.listdir(os.path.join(pkg, "csrc")):
        if f.endswith((".cu", ".cuh")):
            src = open(os.path.join(pkg, "csrc", f)).read()
            assert "mm_oracle.h" not in src and "or_sweep" not in src, f
