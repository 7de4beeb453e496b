"""Randomised geometries: every tile kind, word width, power-of-two or not,
in place or out of place, fresh or mid-run, against the CPU oracle."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _case(seed):
    rng = np.random.default_rng(seed)
    w = int(rng.choice([2, 3, 5, 8, 12, 16, 20, 24, 31, 32, 40, 64]))
    n = int(rng.choice([2, 3, 7, 16, 30, 64, 100, 128, 250, 256, 300, 511, 1024]))
    ell = int(rng.integers(1, min(40, (1 << min(w, 20)) - 1) + 1))
    s = int(rng.integers(1, min(40, (1 << min(w, 20)) - 1) + 1))
    d = int(rng.integers(1, 1500))
    tau = int(rng.choice([0, 1, 5, 64, 300, 2000]))
    epoch = int(rng.choice([1, 3, 16, 64, 500]))
    return w, n, ell, s, d, tau, epoch, bool(rng.integers(0, 2)), bool(rng.integers(0, 2))


@pytest.mark.parametrize("seed", range(120))
def test_random_geometry(seed):
    import torch

    from oracle import oracle
    from paper_2604_12902_b200.engine import DeviceBatch
    from paper_2604_12902_b200.hypervisor import get_engine
    from paper_2604_12902_b200.machine import MachineParams
    from paper_2604_12902_b200.workload import random_configs
    w, n, ell, s, d, tau, epoch, inplace, midrun = _case(seed)
    p = MachineParams(w=w, n=n, ell=ell, s=s)
    rng = np.random.default_rng(1000 + seed)
    c0 = random_configs(d, p, rng, dtype=np.uint64)
    k = max(1, d // 4)                      # some machines loop forever
    if n >= 4:
        c0["M"][:k, :4] = np.array([1, 1, 5, 0], np.uint64) & np.uint64((1 << w) - 1)
        c0["iw"][:k] = 0
    want = {f: np.ascontiguousarray(c0[f].astype(np.uint64)) for f in ("iw", "ac", "M", "u", "y")}
    steps0 = rng.integers(0, 2 * tau + 2, d).astype(np.int64) if midrun else np.zeros(d, np.int64)
    status0 = (rng.random(d) < 0.1).astype(np.int8) if midrun else np.zeros(d, np.int8)
    want.update(status=status0.copy(), steps=steps0.copy(), tau_h=np.full(d, -1, np.int64))
    oracle.oracle_run(want["iw"], want["ac"], want["M"], want["u"], want["y"], want["status"],
                      want["steps"], want["tau_h"], w, n, ell, s, tau)
    dev = torch.device("cuda:0")
    eng = get_engine(p, dev)
    arrays = dict(c0, status=status0, steps=steps0, tau_h=np.full(d, -1, np.int64))
    src = DeviceBatch.from_arrays(arrays, p, dev)
    if inplace:
        eng.run(src, tau, epoch, fresh=not midrun)
        got = src.to_numpy()
    else:
        dst = DeviceBatch.empty(d, p, dev, fresh=False)
        eng.run(src, tau, epoch, out=dst, fresh=not midrun)
        got = dst.to_numpy()
        chk = src.to_numpy()   # the input is untouched
        for f in ("iw", "ac", "M", "u", "y"):
            assert np.array_equal(chk[f].astype(np.uint64), c0[f].astype(np.uint64)), f
    for f in ("iw", "ac", "M", "u", "y", "status", "steps", "tau_h"):
        g = got[f].astype(np.uint64) if f in ("iw", "ac", "M", "u", "y") else got[f]
        np.testing.assert_array_equal(g, want[f], err_msg=f"case {_case(seed)} field {f}")
