"""The C-ABI library loads without a GPU and exports every symbol the header
declares; the product package never touches the oracle."""

import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "tilemesh_b200.h")


def declared():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|int64_t|const char \*)\s*(tm_\w+)\s*\(", src, re.M)))


def test_library_exports_header_symbols():
    from paper_1604_03570_b200 import _native

    L = _native.load()
    names = declared()
    assert len(names) >= 14
    for n in names:
        assert hasattr(L, n), n
    assert set(names) == set(_native.EXPORTS)
    out = subprocess.run(["nm", "-D", "--defined-only", _native.LIB_PATH], capture_output=True, text=True).stdout
    for n in names:
        assert re.search(rf"\bT {n}$", out, re.M), n
    assert L.tm_abi_version() == _native.ABI_VERSION


def test_library_is_sm100a():
    from paper_1604_03570_b200 import _native

    out = subprocess.run(["cuobjdump", "--list-elf", _native.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["cuobjdump", "-sass", _native.LIB_PATH], capture_output=True, text=True).stdout
    assert "UTMALDG" in sass  # TMA plane staging in the sweep kernels


def test_invalid_arguments_are_rejected_on_host():
    from paper_1604_03570_b200 import _native

    L = _native.load()
    h = ctypes.c_void_p()
    assert L.tm_copy_plan_create(None, -1, 1, ctypes.byref(h)) == _native.TM_ERR_INVALID
    assert b"bad arguments" in L.tm_last_error()
    with pytest.raises(ValueError):
        _native.check(L.tm_sweep_plan_create(None, -3, ctypes.byref(h)), "tm_sweep_plan_create")


def test_product_package_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_1604_03570_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                text = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"^\s*(from|import)\s+oracle\b", text, re.M), f
                assert "liboracle" not in text, f
