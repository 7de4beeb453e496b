"""Busy-beaver style search over a batch of programs.

The reference's `raspvisor bb-search` (cli.py:184-234) runs chunks of sampled
programs with zero inputs through run_batch and keeps a min-heap of
(tau_h, -sample_index, source) for the K longest halting runs (cli.py:218-226),
reported by sorted(best, reverse=True).  Here the run and the selection both
stay on the device: rasp_run, then rasp_topk (radix select over tau_h), so
only K (index, tau_h) pairs and two counters come back per chunk.  Program
sampling and pretty-printing (lang.py, lowering.py, sampler.py) are outside the
hot path: callers pass program words.
"""

from __future__ import annotations

import heapq
from dataclasses import dataclass

import numpy as np
import torch

from .engine import DeviceBatch
from .hypervisor import get_engine
from .machine import MachineParams


@dataclass
class SearchReport:
    sampled: int
    halted: int
    best: list            # [(tau_h, sample_index)], longest first, ties to the lower index


def top_halting(batch: DeviceBatch, k: int, tau_max: int, stream=None) -> list:
    """[(tau_h, index)] of the k longest halting runs in a finished batch."""
    eng = get_engine(batch.params, batch.iw.device)
    idx, tau = eng.topk(batch, k, tau_max, stream)
    pairs = torch.stack([tau, idx], 1).cpu().numpy()
    return [(int(t), int(i)) for t, i in pairs if i >= 0]


def bb_search(programs, params: MachineParams, tau_max: int, top: int = 3, chunk: int = 1 << 20,
              epoch: int = 64, device=None) -> SearchReport:
    """Run programs[i] (rows of program words, inputs all zero) to halt or
    tau_max in device chunks; keep the `top` longest halting runs over all
    chunks with the reference's ordering (tau_h desc, sample index asc)."""
    progs = programs if torch.is_tensor(programs) else torch.from_numpy(np.ascontiguousarray(programs))
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    eng = get_engine(params, dev)
    d = int(progs.shape[0])
    best: list = []   # min-heap of (tau_h, -index), as cli.py:195
    halted = 0
    empty_inputs = torch.empty((0, 0), dtype=progs.dtype, device=dev)
    for lo in range(0, d, chunk):
        hi = min(d, lo + chunk)
        pdev = progs[lo:hi].to(dev, non_blocking=True)
        b = DeviceBatch.empty(hi - lo, params, dev, word_bytes=pdev.element_size(), fresh=True)
        eng.init_c0(pdev, empty_inputs, b)
        eng.run(b, tau_max, epoch, fresh=True)
        halted += int((b.status == 1).sum().item())
        for tau_h, j in top_halting(b, top, tau_max):
            item = (tau_h, -(lo + j))
            if len(best) < top:
                heapq.heappush(best, item)
            elif item > best[0]:
                heapq.heapreplace(best, item)
    ranked = sorted(best, reverse=True)
    return SearchReport(sampled=d, halted=halted, best=[(t, -ni) for t, ni in ranked])
