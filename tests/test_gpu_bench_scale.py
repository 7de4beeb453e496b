"""Parity at bench scale for the big-machine (u32/u64 cell) paths.

The bench rows C5, paper and paper6 run machines whose state is too large for
the small shared-memory tiles (w > 16, ~1 KB of memory each): they run on the
epoch kernel's one-warp BIG tiles (u32/u64 cells, output tape written straight
to HBM), where each warp claims many tiles per epoch (the tile-claim loop, the
next-tile L2 prefetch, PRI stores across tiles).  These tests build bench.py's exact inputs
(bench.make_c0), run them the way bench.py does (out-of-place, fresh, on the
bench's first-epoch setting) and compare with the CPU oracle
(oracle/rasp_oracle.c, pinned to the reference by tests/test_oracle_golden.py):

* C5 in full: 2^20 machines, w32 n256 l32 s32, cap 1024 -- every field;
* paper: a seeded 2^16 sample of its 2^20 machines (tau 10^4);
* paper6: a seeded 4096 sample of its 2^20 machines (tau 10^6);
* mid-run configurations (arbitrary i, a, cursors, tapes, statuses, step
  counts) at w64, w32 and w24 with d far above the resident lanes, so every
  warp takes many tiles (per-lane budgets, untouched machines);
* the reference's uint64 layout for a C5 sample (cells of 8 bytes).

Reference contract: hypervisor.py:265-323 (run_batch) / :128-164 (_worker);
tests/test_hypervisor.py:27-43 is the reference's own batch-vs-scalar check.
"""

import os

import numpy as np
import pytest

from golden_io import FIELDS, RESULTS

pytestmark = pytest.mark.gpu

CORES = len(os.sched_getaffinity(0))


@pytest.fixture(scope="module")
def env():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device")
    import bench
    from paper_2604_12902_b200.machine import MachineParams
    return torch, bench, MachineParams


def _run_like_bench(torch, p, c0, tau, epoch):
    """bench.py's step: out-of-place fresh run of a resident batch."""
    from paper_2604_12902_b200.engine import DeviceBatch
    from paper_2604_12902_b200.hypervisor import get_engine
    dev = torch.device("cuda:0")
    eng = get_engine(p, dev)
    src = DeviceBatch.from_arrays(c0, p, dev)
    dst = DeviceBatch.empty(src.d, p, dev, fresh=False)
    fused = torch.empty(102, dtype=torch.int64, device=dev)
    eng.run(src, tau, epoch, out=dst, fresh=True, hist=fused)
    hist = eng.histogram(dst).cpu().numpy()
    np.testing.assert_array_equal(fused.cpu().numpy(), hist)   # counted in the run == re-read
    out = dst.to_numpy()
    return out, hist


def _check(got, want, idx=None, tag=""):
    for k in RESULTS:
        g = got[k] if idx is None else got[k][idx]
        if k in FIELDS:
            g = g.astype(np.uint64)
        np.testing.assert_array_equal(g, want[k], err_msg=f"{tag} field {k}")


def _resident_lane_bound(p, word_bytes):
    """Upper bound on lanes resident at once: a machine's M and tape rows
    must fit in shared memory (<= 228 KB per SM, 148 SMs)."""
    per = (p.n + p.ell + 1) * word_bytes
    return 148 * (228 * 1024 // per + 1)


def test_c5_full_batch(env):
    torch, bench, MP = env
    from oracle import oracle
    d, w, n, ell, s, tau, _ = bench.CONFIGS["c5"]
    p = MP(w=w, n=n, ell=ell, s=s, mu=1)
    c0 = bench.make_c0("c5", d, p, seed=0)
    assert d > 8 * _resident_lane_bound(p, 4)   # every lane runs many machines
    got, hist = _run_like_bench(torch, p, c0, tau, bench.DEFAULT_EPOCH["c5"])
    want = oracle.worker_arrays(c0, w, n, ell, s, tau, workers=CORES)
    _check(got, want, tag="c5")
    st, th = want["status"], want["tau_h"]
    ref_hist = [int(((st == 1) & (th == k)).sum()) for k in range(100)] + \
        [int(((st == 1) & (th >= 100)).sum()), int((st == 2).sum())]
    assert list(hist) == ref_hist


@pytest.mark.parametrize("cfg,sample", [("paper", 1 << 16), ("paper6", 4096)])
def test_paper_rows_sample(env, cfg, sample):
    torch, bench, MP = env
    from oracle import oracle
    d, w, n, ell, s, tau, _ = bench.CONFIGS[cfg]
    p = MP(w=w, n=n, ell=ell, s=s, mu=1)
    c0 = bench.make_c0(cfg, d, p, seed=0)
    got, _ = _run_like_bench(torch, p, c0, tau, bench.DEFAULT_EPOCH[cfg])
    idx = np.sort(np.random.default_rng(11).choice(d, sample, replace=False))
    want = oracle.worker_arrays({k: c0[k][idx] for k in FIELDS}, w, n, ell, s, tau, workers=CORES)
    _check(got, want, idx, tag=cfg)
    # whole-batch invariants (hv:153-164)
    st, steps, th = got["status"], got["steps"], got["tau_h"]
    assert set(np.unique(st)) <= {1, 2}
    assert (th[st == 1] == steps[st == 1]).all() and (steps[st == 2] == tau).all()


@pytest.mark.parametrize("shape", [(64, 128, 8, 8), (32, 256, 32, 32), (32, 250, 10, 2), (24, 200, 6, 5)])
def test_midrun_many_machines_per_lane(env, shape):
    """Mid-run inputs (random i, a, cursors, tapes; statuses 0/1/2 and prior
    step counts) in place and out of place, several budgets."""
    torch, bench, MP = env
    from oracle import oracle
    from paper_2604_12902_b200 import hypervisor as H
    from paper_2604_12902_b200.workload import random_configs
    w, n, ell, s = shape
    p = MP(w=w, n=n, ell=ell, s=s, mu=1)
    d = 1 << 18
    assert d > 4 * _resident_lane_bound(p, p.dtype.itemsize)
    rng = np.random.default_rng(w + n)
    c0 = random_configs(d, p, rng)
    status = rng.choice(np.array([0, 0, 0, 0, 1, 2], np.int8), d)
    steps = rng.integers(0, 300, d).astype(np.int64)
    tau_h = np.where(status == 1, steps, -1).astype(np.int64)
    for tau in (0, 7, 300):
        want = {k: c0[k].astype(np.uint64) for k in FIELDS}
        want.update(status=status.copy(), steps=steps.copy(), tau_h=tau_h.copy())
        oracle.oracle_run(want["iw"], want["ac"], want["M"], want["u"], want["y"], want["status"],
                          want["steps"], want["tau_h"], w, n, ell, s, tau, 64, CORES)
        arrays = dict(c0, status=status, steps=steps, tau_h=tau_h)
        res = H.run_arrays(arrays, p, H.BatchConfig(tau_max=tau, epoch=16, memory_budget_words=1 << 40))
        _check({k: getattr(res.slots, k) for k in RESULTS}, want, tag=f"{shape} tau={tau} in-place")
        # out of place through the engine (input untouched, every field written)
        from paper_2604_12902_b200.engine import DeviceBatch
        from paper_2604_12902_b200.hypervisor import get_engine
        dev = torch.device("cuda:0")
        src = DeviceBatch.from_arrays(arrays, p, dev)
        dst = DeviceBatch.empty(d, p, dev, fresh=False)
        get_engine(p, dev).run(src, tau, 16, out=dst)
        _check(dst.to_numpy(), want, tag=f"{shape} tau={tau} out-of-place")
        np.testing.assert_array_equal(src.M.cpu().numpy(), c0["M"])


def test_fresh_many_machines_w64(env):
    torch, bench, MP = env
    from oracle import oracle
    from paper_2604_12902_b200.workload import synthetic_c0
    p = MP(w=64, n=128, ell=8, s=8, mu=1)
    d = 1 << 17
    c0 = synthetic_c0(d, p, seed=5)
    got, hist = _run_like_bench(torch, p, c0, 1024, 64)
    want = oracle.worker_arrays(c0, p.w, p.n, p.ell, p.s, 1024, workers=CORES)
    _check(got, want, tag="w64 fresh")


def test_uint64_layout_c5_sample(env):
    """The reference's own uint64 arrays at the C5 geometry (8-byte cells)."""
    torch, bench, MP = env
    from oracle import oracle
    from paper_2604_12902_b200 import hypervisor as H
    p = MP(w=32, n=256, ell=32, s=32, mu=1)
    c0 = {k: v.astype(np.uint64) for k, v in bench.make_c0("c5", 1 << 15, p, seed=3).items()}
    res = H.run_arrays(c0, p, H.BatchConfig(tau_max=1024, epoch=64, memory_budget_words=1 << 40))
    assert res.slots.M.dtype == np.uint64
    want = oracle.worker_arrays(c0, p.w, p.n, p.ell, p.s, 1024, workers=CORES)
    _check({k: getattr(res.slots, k) for k in RESULTS}, want, tag="u64 layout")


@pytest.mark.parametrize("family", ["bb", "paper", "paper100"])
def test_device_packer_matches_reference_c0(env, family):
    """rasp_init_c0 against the c0 the reference's init_config built
    (m:289-309) from the same program and input words (tests/golden/packer.npz)."""
    torch, bench, MP = env
    from golden_io import GOLDEN
    from paper_2604_12902_b200.engine import DeviceBatch
    from paper_2604_12902_b200.hypervisor import get_engine
    z = np.load(os.path.join(GOLDEN, "packer.npz"))
    p = MP(w=32, n=250, ell=10, s=2, mu=10)
    prog = z[f"{family}_prog"].astype(np.uint32)
    inp = z[f"{family}_inp"].astype(np.uint32)
    dev = torch.device("cuda:0")
    out = DeviceBatch.empty(prog.shape[0], p, dev, fresh=False)
    get_engine(p, dev).init_c0(torch.from_numpy(prog).to(dev), torch.from_numpy(inp).to(dev), out)
    got = out.to_numpy()
    for k in FIELDS:
        np.testing.assert_array_equal(got[k].astype(np.uint64), z[f"{family}_c0_{k}"], err_msg=f"{family} {k}")
    assert not got["status"].any() and not got["steps"].any() and (got["tau_h"] == -1).all()
