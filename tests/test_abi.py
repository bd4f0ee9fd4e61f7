"""The C-ABI library loads and exports every symbol include/omp_b200.h declares (no GPU needed)."""

import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "omp_b200.h")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:ompStatus_t|int64_t|int|float|const char\s*\*)\s*(\w+)\s*\(", text, flags=re.M)))


@pytest.fixture(scope="module")
def lib():
    from paper_2407_06434_b200 import build, _lib
    build.build()
    return _lib.load()


def test_header_declares_the_boundary():
    fns = declared_functions()
    for name in ("ompCreate", "ompBatch", "ompBatchHost", "ompDensify", "ompDestroy", "ompGetErrorString",
                 "ompGetErrorDetail", "omp_batch", "ompCorrelate", "ompGetGram", "ompGetFactor"):
        assert name in fns


def test_library_exports_every_declared_symbol(lib):
    from paper_2407_06434_b200 import _lib
    fns = declared_functions()
    assert set(fns) == set(_lib.SIGNATURES), "binding signatures out of sync with the header"
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (\w+)$", out, flags=re.M))
    missing = [f for f in fns if f not in exported]
    assert not missing, missing
    for f in fns:
        getattr(lib, f)


def test_error_strings_and_sm100a_code(lib):
    for s in range(7):
        assert lib.ompGetErrorString(s).startswith(b"OMP_")
    from paper_2407_06434_b200 import _lib
    sass = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in sass


def test_invalid_arguments_fail_before_any_launch(lib):
    import ctypes
    h = ctypes.c_void_p()
    assert lib.ompCreate(None, 0, None, 1, 1, 1, 0, None) == 1
    assert lib.ompCreate(ctypes.byref(h), 0, None, 4, 4, 4, 0, None) == 1
    assert lib.ompCreate(ctypes.byref(h), 0, ctypes.c_void_p(16), 4, 4, 2, 0, None) == 1  # lda < M
    assert lib.ompBatch(None, None, 1, 1, 1, 0.0, None, 1, None, 1, None, None, None, None) == 1
    assert lib.ompDestroy(None) == 1
