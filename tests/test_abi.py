"""The C-ABI library loads on CPU and exports every symbol include/modmcache.h declares."""
import ctypes
import re
import subprocess
from pathlib import Path

import pytest

from paper_2503_11972_b200 import _native, build

ROOT = Path(__file__).resolve().parents[1]


def declared_functions():
    text = (ROOT / "include" / "modmcache.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(mc_[a-z0-9_]+)\s*\(", text)))


@pytest.fixture(scope="module")
def lib():
    build.build()
    return _native.load()


def test_header_declares_expected_api():
    fns = declared_functions()
    assert set(fns) == set(_native.EXPORTED), fns


def test_library_exports_every_declared_symbol(lib):
    for name in declared_functions():
        assert hasattr(lib, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", str(_native.LIB_PATH)], capture_output=True, text=True)
    exported = set(re.findall(r" T (mc_\w+)", out.stdout))
    assert set(declared_functions()) <= exported


def test_version_and_error_string_without_gpu(lib):
    assert b"sm_100a" in lib.mc_version()
    h = ctypes.c_void_p()
    rc = lib.mc_create(ctypes.byref(h), 0, 8, 0)  # capacity 0 is rejected before any CUDA call
    assert rc == -1
    assert b"capacity" in lib.mc_last_error()


def test_library_is_sm100a_only():
    out = subprocess.run(["cuobjdump", "--list-elf", str(_native.LIB_PATH)], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    arches = set(re.findall(r"sm_(\d+a?)", out.stdout))
    assert arches == {"100a"}, arches
