"""Drop-in replacement for the reference's numba kernel.

The reference's batch operator ``raspvisor.hypervisor.run_batch``
(hypervisor.py:265-323) packs configurations into uint64 SoA arrays and calls
``_worker(iw, ac, M, u, y, status, steps, tau_h, g, W, q, rounds, tau_max,
wmask, n, ell, s)`` once per worker stripe (hypervisor.py:305-314, kernel
hypervisor.py:128-164).  ``worker`` below has exactly that signature and runs
the whole batch through the C ABI (``rasp_run``, include/raspvisor_b200.h) on
the GPU, writing the results back into the caller's arrays in place, as the
numba kernel does.  ``install(hypervisor_module)`` swaps it in, so the
reference's own ``run_batch`` -- argument checks, packing, histogram, SlotView
-- runs unchanged on top of the B200 engine:

    from raspvisor import hypervisor
    from paper_2604_12902_b200 import dropin
    dropin.install(hypervisor)
    res = hypervisor.run_batch(configs, params, hypervisor.BatchConfig(tau_max=1024, workers=1))

The engine runs a batch in one call, so it must receive all of it: one worker
(``workers=1``), or stripe 0 of W when the other stripes are empty.
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _native
from .errors import NativeError

_FIELDS = ("iw", "ac", "M", "u", "y", "status", "steps", "tau_h")


def worker(iw, ac, M, u, y, status, steps, tau_h, g, W, q, rounds, tau_max, wmask, n, ell, s):
    """hypervisor.py:128-164 on the GPU: same arrays (uint64 words, int8
    status, int64 steps/tau_h), same in-place result.  `rounds` is implied by
    tau_max (the reference derives it as ceil(tau_max / q), hv:297)."""
    d = int(iw.shape[0])
    if int(W) != 1 or int(g) != 0:
        if d <= int(g):
            return   # an empty stripe
        raise NativeError("the B200 engine runs the whole batch in one call: use workers=1")
    if d == 0:
        return
    lib = _native.load()
    w = int(wmask).bit_length()
    p = _native.RaspParams(w, int(n), int(ell), int(s))
    dev = torch.device("cuda", torch.cuda.current_device())
    host = dict(iw=iw, ac=ac, M=M, u=u, y=y, status=status, steps=steps, tau_h=tau_h)
    t = {k: torch.from_numpy(np.ascontiguousarray(a)).to(dev) for k, a in host.items()}
    b = _native.RaspBatch(*(t[k].data_ptr() for k in _FIELDS), d, 8, 0)
    need = lib.rasp_workspace_bytes(ctypes.byref(p), d)
    ws = torch.empty(max(int(need), 256), dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)
    with torch.cuda.device(dev):
        rc = lib.rasp_run(ctypes.byref(p), ctypes.byref(b), ctypes.byref(b), int(tau_max), max(int(q), 1), 0,
                          ws.data_ptr(), ws.numel(), stream.cuda_stream)
    _native.check(rc, "rasp_run")
    for k, a in host.items():   # results land in the caller's arrays, as with the numba kernel
        a[...] = t[k].cpu().numpy().reshape(a.shape)


def install(hypervisor_module) -> None:
    """Route ``hypervisor_module.run_batch``'s kernel calls to ``worker``."""
    hypervisor_module._worker = worker
