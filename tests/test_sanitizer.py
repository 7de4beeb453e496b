"""compute-sanitizer over every kernel family of the engine.

memcheck (out-of-bounds / misaligned device accesses), racecheck (shared-
memory hazards between threads: the tiles are shared by a warp's lanes, the
stmatrix/ldmatrix row moves cross lanes) and synccheck (barrier, warp-sync
and vote usage) on small batches of each kind -- see tests/sanitize_workload.py,
which also checks the results against the oracle.  The reference needs no
such check (disjoint stripes, hypervisor.py:1-9); these kernels share tiles,
use atomics and a last-block epoch planner, so they get the tool."""

import os
import shutil
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SAN = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"

CASES = [(tool, kind) for tool, kinds in (
    ("memcheck", ("mx", "big", "big64", "hbm", "enum", "aux")),
    ("racecheck", ("mx", "big", "enum", "aux")),
    ("synccheck", ("mx", "big", "enum")),
) for kind in kinds]


@pytest.mark.parametrize("tool,kind", CASES, ids=[f"{t}-{k}" for t, k in CASES])
def test_sanitizer_clean(tool, kind):
    if not os.path.exists(SAN):
        pytest.fail("compute-sanitizer not found")
    cmd = [SAN, "--tool", tool, "--error-exitcode", "86", "--print-limit", "20",
           sys.executable, os.path.join(ROOT, "tests", "sanitize_workload.py"), kind]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=1200, cwd=ROOT)
    log = out.stdout + out.stderr
    assert out.returncode == 0, log[-4000:]
    assert f"sanitize workload {kind}: ok" in log, log[-4000:]
    assert "ERROR SUMMARY: 0 errors" in log, log[-4000:]
    if tool == "racecheck":
        assert "RACECHECK SUMMARY: 0 hazards" in log or "0 hazards" in log, log[-4000:]
