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


def random_configs(count: int, params: MachineParams, rng: np.random.Generator, dtype=None) -> dict:
    """Well-formed mid-run configurations (not c0): arbitrary i, a, cursors and
    tapes, opcode cells biased into [0, 9) -- the distribution of the
    reference's differential corpus (selftest.py:32-95), drawn as SoA arrays.
    Used to exercise every step case at scale."""
    w, n, ell, s = params.w, params.n, params.ell, params.s
    top = (1 << w) - 1
    dt = np.dtype(dtype) if dtype is not None else natural_dtype(w)

    def words(shape):
        return rng.integers(0, top, shape, dtype=np.uint64, endpoint=True)

    M = words((count, n))
    half = (n + 1) // 2
    ops = rng.integers(0, 9, (count, half), dtype=np.uint64) % np.uint64(top + 1 if w < 64 else 1 << 63)
    keep = rng.random((count, half)) < 0.8
    M[:, 0::2] = np.where(keep, ops, M[:, 0::2])
    u = np.concatenate([rng.integers(0, ell + 1, (count, 1), dtype=np.uint64), words((count, ell))], 1)
    y = np.concatenate([rng.integers(0, s + 1, (count, 1), dtype=np.uint64), words((count, s))], 1)
    near = rng.integers(0, 2 * n, count, dtype=np.uint64) & np.uint64(top)
    i = np.where(rng.random(count) < 0.7, near, words(count))
    small = rng.integers(0, min(top + 1, 10), count, dtype=np.uint64)
    a = np.where(rng.random(count) < 0.5, small, words(count))
    return {"iw": i.astype(dt), "ac": a.astype(dt), "M": M.astype(dt), "u": u.astype(dt),
            "y": y.astype(dt)}
