"""The checked build (kernel bounds and lane-ownership checks compiled in,
-DRASP_CHECKED=1) over every kernel family -- the substitute for
compute-sanitizer, which is closed on this project's GPU pool.  See
tests/check_workload.py for what each kind launches; every run is also
checked against the CPU oracle."""

import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KINDS = ("mx", "big", "refill", "big64", "hbm", "enum", "aux")


@pytest.fixture(scope="module")
def checked_lib():
    from paper_2604_12902_b200 import build
    return build.build(checked=True)


def test_checked_library_reports_itself(checked_lib):
    import ctypes
    lib = ctypes.CDLL(checked_lib)
    lib.rasp_error_string.restype = ctypes.c_char_p
    assert lib.rasp_checked_build() == 1
    from paper_2604_12902_b200 import _native
    assert _native.load().rasp_checked_build() == 0   # the product library carries no checks
    assert lib.rasp_error_string(-7).decode().startswith("kernel bounds")


@pytest.mark.gpu
@pytest.mark.parametrize("kind", KINDS)
def test_kernels_pass_the_checks(checked_lib, kind):
    env = dict(os.environ, RASP_LIBRARY=checked_lib)
    out = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "check_workload.py"), kind],
                         capture_output=True, text=True, timeout=900, cwd=ROOT, env=env)
    log = out.stdout + out.stderr
    assert out.returncode == 0, log[-4000:]
    assert f"check workload {kind}: ok (checked build: 1)" in log, log[-4000:]
