"""Build the in-tree CUDA engine library for sm_100a.

    python -m paper_2604_12902_b200.build [--force] [-v]

Produces paper_2604_12902_b200/_lib/libraspvisor_b200.so (git-ignored; it
travels to the GPU box with the repo snapshot).
"""

from __future__ import annotations

import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")
OUT = os.path.join(PKG, "_lib", "libraspvisor_b200.so")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-shared", "-Xcompiler", "-fPIC",
    "--expt-relaxed-constexpr",
]


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


# the checked build: kernel bounds/ownership checks compiled in (tests only)
OUT_CHECKED = os.path.join(PKG, "_lib", "libraspvisor_b200_checked.so")


def _stale(out: str = OUT) -> bool:
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    deps = sources() + glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.h")) + \
        glob.glob(os.path.join(INCLUDE, "*.h"))
    return any(os.path.getmtime(f) > t for f in deps)


def build(force: bool = False, verbose: bool = False, checked: bool = False) -> str:
    """Compile every csrc/*.cu to an object in parallel (the kernel
    instantiations are split by HBM word type), then link the shared library.
    checked=True builds the variant with the kernel checks (-DRASP_CHECKED=1)."""
    out = OUT_CHECKED if checked else OUT
    if not force and not _stale(out):
        return out
    os.makedirs(os.path.dirname(out), exist_ok=True)
    nvcc = os.environ.get("NVCC", "nvcc")
    obj_dir = os.path.join(os.path.dirname(out), "obj_checked" if checked else "obj")
    os.makedirs(obj_dir, exist_ok=True)
    compile_flags = [f for f in NVCC_FLAGS if f != "-shared"] + (["-DRASP_CHECKED=1"] if checked else [])
    jobs = []
    for src in sources():
        obj = os.path.join(obj_dir, os.path.basename(src)[:-3] + ".o")
        cmd = [nvcc, *compile_flags, f"-I{INCLUDE}", "-c", "-o", obj, src]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
            print(" ".join(cmd), file=sys.stderr)
        jobs.append((subprocess.Popen(cmd), obj, cmd))
    objs = []
    for proc, obj, cmd in jobs:
        if proc.wait() != 0:
            raise subprocess.CalledProcessError(proc.returncode, cmd)
        objs.append(obj)
    link = [nvcc, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o", out + ".tmp", *objs, "-ldl"]
    subprocess.run(link, check=True)
    os.replace(out + ".tmp", out)
    return out


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, checked="--checked" in sys.argv))
