"""Time the reference's own numba kernel (raspvisor.hypervisor._worker) against
the C port (oracle/rasp_oracle.c) on identical c0 arrays, and check they agree.

Build-container only (needs /root/reference):
    NUMBA_CACHE_DIR=/tmp/numba_cache python oracle/compare_reference.py
Numbers are recorded in DESIGN.md §6 to show the CPU baseline is not a strawman.
"""
import os
import sys
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, "/root/reference/pkg/src")
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

from raspvisor import hypervisor as H  # noqa: E402

from oracle import oracle  # noqa: E402
from paper_2604_12902_b200.machine import MachineParams  # noqa: E402
from paper_2604_12902_b200.workload import synthetic_c0  # noqa: E402


def ref_worker(c0, p, tau, W, q=64):
    """hv:295-314 dispatch of the reference kernel on pre-packed arrays."""
    d = c0["iw"].shape[0]
    a = {k: np.ascontiguousarray(v.astype(np.uint64)) for k, v in c0.items()}
    status = np.zeros(d, np.int8)
    steps = np.zeros(d, np.int64)
    tau_h = np.full(d, -1, np.int64)
    rounds = (tau + q - 1) // q
    args = (np.uint64(p.mask), np.uint64(p.n), np.uint64(p.ell), np.uint64(p.s))
    H._warm_kernel()
    t0 = time.perf_counter()
    if W == 1:
        H._worker(a["iw"], a["ac"], a["M"], a["u"], a["y"], status, steps, tau_h, 0, 1, q, rounds, tau, *args)
    else:
        with ThreadPoolExecutor(W) as ex:
            fs = [ex.submit(H._worker, a["iw"], a["ac"], a["M"], a["u"], a["y"], status, steps, tau_h,
                            g, W, q, rounds, tau, *args) for g in range(W)]
            for f in fs:
                f.result()
    dt = time.perf_counter() - t0
    a.update(status=status, steps=steps, tau_h=tau_h)
    return a, dt


def main():
    cores = len(os.sched_getaffinity(0))
    for name, (d, w, n, ell, s, tau) in {"c2": (1 << 16, 16, 64, 8, 8, 1024),
                                         "c5": (1 << 14, 32, 256, 32, 32, 1024)}.items():
        p = MachineParams(w=w, n=n, ell=ell, s=s, mu=1)
        c0 = synthetic_c0(d, p, seed=0)
        for W in (1, cores):
            ref, tr = min((ref_worker(c0, p, tau, W) for _ in range(3)), key=lambda x: x[1])
            best = 1e9
            for _ in range(3):
                t0 = time.perf_counter()
                port = oracle.worker_arrays(c0, w, n, ell, s, tau, epoch=64, workers=W)
                best = min(best, time.perf_counter() - t0)
            for k in ("iw", "ac", "M", "u", "y", "status", "steps", "tau_h"):
                assert np.array_equal(ref[k], port[k]), (name, W, k)
            st = int(ref["steps"].sum())
            print(f"{name} d={d} W={W}: reference numba {st / tr:.3e} steps/s, "
                  f"C port {st / best:.3e} steps/s (port/ref {tr / best:.2f}x), identical results")


if __name__ == "__main__":
    main()
