"""Synthetic c0 batches for the throughput configs (host side).

Generator G (frozen): every machine's program fills all of
memory (2m = n); even cells hold opcodes uniform in {1..7}, odd cells hold
operands uniform in [0, n) with BNZ operands rounded down to even; the input
tape holds ell uniform w-bit words; i = a = u0 = y = 0.  This is the c0 shape
of raspvisor/machine.py:289-309 (init_config) with a random program.

The draw order below is part of the definition: the same seed gives the same
batch on every host, so CPU and GPU consume identical c0 arrays.
"""

from __future__ import annotations

import numpy as np

from .machine import MachineParams, natural_dtype


def synthetic_c0(d: int, params: MachineParams, seed: int = 0, dtype=None) -> dict:
    """Generator G.  Returns SoA arrays iw, ac [d]; M [d,n]; u [d,ell+1];
    y [d,s+1] in `dtype` (default: the natural width of params.w)."""
    w, n, ell, s = params.w, params.n, params.ell, params.s
    dt = np.dtype(dtype) if dtype is not None else natural_dtype(w)
    rng = np.random.default_rng(seed)
    half = n // 2
    ops = rng.integers(1, 8, (d, half), dtype=np.uint64)
    opr = rng.integers(0, n, (d, half), dtype=np.uint64)
    opr = np.where(ops == 5, opr & ~np.uint64(1), opr)
    M = np.zeros((d, n), dt)
    M[:, 0:2 * half:2] = ops
    M[:, 1:2 * half:2] = opr
    mask = (1 << w) - 1
    M &= dt.type(mask)   # a no-op unless w is too small to hold n or 7
    u = np.zeros((d, ell + 1), dt)
    u[:, 1:] = rng.integers(0, mask, (d, ell), dtype=np.uint64, endpoint=True)
    return {
        "iw": np.zeros(d, dt),
        "ac": np.zeros(d, dt),
        "M": M,
        "u": u,
        "y": np.zeros((d, s + 1), dt),
    }
