"""Refill kernel against the epochs on a workload/budget grid (analysis only):
    python scripts/refill_policy.py
Times one out-of-place fresh run (CUDA events, best of 3 after a warm-up) of
bench.make_c0's batches at several budgets with $RASP_REFILL=1 (the refill
kernel takes the whole budget) and =0 (epochs, the config's first epoch)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2604_12902_b200.engine import DeviceBatch  # noqa: E402
from paper_2604_12902_b200.hypervisor import get_engine  # noqa: E402
from paper_2604_12902_b200.machine import MachineParams  # noqa: E402


def timed(eng, src, dst, tau, epoch):
    best = 1e9
    for _ in range(4):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        eng.run(src, tau, epoch, out=dst, fresh=True)
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b))
    return best


dev = torch.device("cuda:0")
CFGS = os.environ.get("CFGS", "c5 paper").split()
TAUS = [int(t) for t in os.environ.get("TAUS", "256 512 1024 2048").split()]
MINS = os.environ.get("MINS", "12").split()
for cfg in CFGS:
    taus = TAUS
    d, w, n, ell, s, _, _ = bench.CONFIGS[cfg][:7]
    p = MachineParams(w=w, n=n, ell=ell, s=s)
    c0 = bench.make_c0(cfg, d, p, 0)
    eng = get_engine(p, dev)
    src = DeviceBatch.from_arrays(c0, p, dev)
    dst = DeviceBatch.empty(d, p, dev, fresh=False)
    for tau in taus:
        os.environ["RASP_REFILL"] = "0"
        ep = timed(eng, src, dst, tau, bench.DEFAULT_EPOCH[cfg])
        os.environ["RASP_REFILL"] = "1"
        rf = []
        for m in MINS:
            os.environ["RASP_REFILL_MIN"] = m
            rf.append(f"min {m}: {timed(eng, src, dst, tau, tau):.3f}")
        print(f"{cfg} tau {tau}: epochs {ep:.3f} ms; refill " + ", ".join(rf), flush=True)
