"""The C-ABI library builds for sm_100a, loads without a GPU, and exports
every function include/raspvisor_b200.h declares."""

import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "raspvisor_b200.h")


def _declared():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:[\w\s\*]+?)\b(rasp_\w+)\s*\(", text, re.M)))


@pytest.fixture(scope="module")
def lib_path():
    from paper_2604_12902_b200 import build
    return build.build()


def test_header_declares_the_boundary():
    names = _declared()
    for want in ("rasp_run", "rasp_workspace_bytes", "rasp_histogram", "rasp_validate",
                 "rasp_error_string", "rasp_last_cuda_error", "rasp_abi_version"):
        assert want in names


def test_library_exports_every_declared_symbol(lib_path):
    lib = ctypes.CDLL(lib_path)
    for name in _declared():
        assert hasattr(lib, name), name
    from paper_2604_12902_b200 import _native
    assert set(_native.EXPORTS) == set(_declared())


def test_abi_version_and_error_strings(lib_path):
    from paper_2604_12902_b200 import _native
    lib = _native.load()
    assert lib.rasp_abi_version() == _native.ABI_VERSION
    assert lib.rasp_error_string(-2).decode().startswith("batch or geometry")
    # parameter validation happens before any CUDA call
    p = _native.RaspParams(0, 8, 1, 1)
    b = _native.RaspBatch()
    rc = lib.rasp_run(ctypes.byref(p), ctypes.byref(b), ctypes.byref(b), 1, 1, 0, None, 0, None)
    assert rc == -1


def test_sass_is_sm100a(lib_path):
    """The shipped kernels are sm_100a SASS (not PTX JIT, not another arch)."""
    out = subprocess.run(["cuobjdump", "--list-elf", lib_path], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout
