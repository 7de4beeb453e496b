"""The per-lane refill kernel for big machines (rasp_kernels.cuh, refill_kernel).

Fresh runs of big-tile machines (u32/u64 cells, tile > 16 KB) whose budget is
a multiple of the unrolled block run in one launch in which every lane takes
a new machine as soon as its own stops.  Each case here forces
that path ($RASP_REFILL=1, read per run), checks it launched exactly one
kernel, and compares every field and the fused histogram with the CPU oracle
(oracle/rasp_oracle.c, pinned to the reference) and with the epoch path
($RASP_REFILL=0) on the same input.  Geometries cover power-of-two and
residue-carrying n, u32 and u64 cells, HBM words narrower/wider than the
cells (the synchronous row loads with conversion), tapes longer than 32
cells (the two-pass row load), batches smaller than a warp and far larger
than the resident lanes, in place and out of place, and refill thresholds
from 1 to 32.  Reference contract: hypervisor.py:128-164 (_worker).
"""

import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

FIELDS = ("iw", "ac", "M", "u", "y")
RESULTS = FIELDS + ("status", "steps", "tau_h")

# w, n, ell, s, d, tau, word dtype, in place, refill_min
CASES = [
    (32, 256, 32, 32, 20000, 1024, np.uint32, False, None),   # C5 shape, many machines per lane
    (32, 256, 32, 32, 7, 64, np.uint32, True, None),          # fewer machines than lanes
    (32, 250, 16, 16, 6000, 512, np.uint32, False, None),     # n not a power of two (carried residues)
    (24, 300, 40, 20, 3000, 320, np.uint32, True, None),      # ell > 32: two-pass row load
    (48, 128, 8, 8, 4000, 256, np.uint64, False, None),       # u64 cells
    (64, 96, 12, 12, 3000, 160, np.uint64, True, None),       # u64, full width, n not a power of two
    (32, 256, 32, 32, 5000, 1024, np.uint64, False, None),    # HBM words wider than the cells
    (20, 512, 8, 8, 3000, 2048, np.uint32, False, 1),         # refill at every free lane
    (32, 256, 32, 32, 5000, 512, np.uint32, True, 32),        # refill only when the warp is empty
    (31, 1024, 4, 4, 2000, 16, np.uint32, False, None),       # one block of steps
]


def _inputs(case, seed):
    from paper_2604_12902_b200.machine import MachineParams
    from paper_2604_12902_b200.workload import random_configs
    w, n, ell, s, d = case[:5]
    p = MachineParams(w=w, n=n, ell=ell, s=s)
    rng = np.random.default_rng(seed)
    c0 = random_configs(d, p, rng, dtype=np.uint64)
    k = max(1, d // 5)                      # some machines loop until the budget
    c0["M"][:k, :4] = np.array([1, 1, 5, 0], np.uint64) & np.uint64((1 << w) - 1)
    c0["iw"][:k] = 0
    perm = rng.permutation(d)
    for f in FIELDS:
        c0[f] = np.ascontiguousarray(c0[f][perm])
    return p, c0


def _oracle(c0, p, tau):
    from oracle import oracle
    d = c0["iw"].shape[0]
    want = {f: np.ascontiguousarray(c0[f].astype(np.uint64)) for f in FIELDS}
    want.update(status=np.zeros(d, np.int8), steps=np.zeros(d, np.int64), tau_h=np.full(d, -1, np.int64))
    oracle.oracle_run(want["iw"], want["ac"], want["M"], want["u"], want["y"], want["status"],
                      want["steps"], want["tau_h"], p.w, p.n, p.ell, p.s, tau)
    return want


def _run(torch, p, c0, tau, word, inplace, refill, rmin=None, epoch=None):
    from paper_2604_12902_b200 import _native
    from paper_2604_12902_b200.engine import DeviceBatch
    from paper_2604_12902_b200.hypervisor import get_engine
    dev = torch.device("cuda:0")
    d = c0["iw"].shape[0]
    arrays = {f: c0[f].astype(word) for f in FIELDS}
    arrays.update(status=np.zeros(d, np.int8), steps=np.zeros(d, np.int64), tau_h=np.full(d, -1, np.int64))
    eng = get_engine(p, dev)
    wb = np.dtype(word).itemsize
    src = DeviceBatch.from_arrays(arrays, p, dev, word_bytes=wb)
    dst = src if inplace else DeviceBatch.empty(d, p, dev, word_bytes=wb, fresh=False)
    hist = torch.empty(102, dtype=torch.int64, device=dev)
    old = {k: os.environ.get(k) for k in ("RASP_REFILL", "RASP_REFILL_MIN")}
    os.environ["RASP_REFILL"] = "1" if refill else "0"
    if rmin is not None:
        os.environ["RASP_REFILL_MIN"] = str(rmin)
    try:
        eng.warm(wb, True)
        torch.cuda.synchronize()
        n0 = _native.load().rasp_launch_count()
        eng.run(src, tau, epoch or max(tau, 1), out=None if inplace else dst, fresh=True, hist=hist)
        torch.cuda.synchronize()
        launches = _native.load().rasp_launch_count() - n0
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    return dst.to_numpy(), hist.cpu().numpy(), launches


def _hist_of(want):
    h = np.zeros(102, np.int64)
    for st, th in zip(want["status"], want["tau_h"]):
        if st == 1:
            h[min(int(th), 100)] += 1
        elif st == 2:
            h[101] += 1
    return h


@pytest.fixture(scope="module")
def torch_mod():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device")
    return torch


@pytest.mark.parametrize("case", CASES, ids=lambda c: f"w{c[0]}n{c[1]}l{c[2]}d{c[4]}t{c[5]}{np.dtype(c[6]).name}"
                         f"{'ip' if c[7] else 'oop'}r{c[8]}")
def test_refill_matches_oracle_and_epochs(torch_mod, case):
    torch = torch_mod
    w, n, ell, s, d, tau, word, inplace, rmin = case
    p, c0 = _inputs(case, seed=w * 1000 + n)
    want = _oracle(c0, p, tau)
    got, hist, launches = _run(torch, p, c0, tau, word, inplace, True, rmin)
    # out of place: two tape copies and the one refill launch; in place: one launch
    assert launches == (1 if inplace else 3), launches
    for f in RESULTS:
        g = got[f].astype(np.uint64) if f in FIELDS else got[f]
        np.testing.assert_array_equal(g, want[f], err_msg=f"{case} field {f}")
    np.testing.assert_array_equal(hist, _hist_of(want))
    epo, hist_e, launches_e = _run(torch, p, c0, tau, word, inplace, False, epoch=16)
    assert launches_e > launches or tau <= 16
    for f in RESULTS:
        np.testing.assert_array_equal(epo[f], got[f], err_msg=f"{case} field {f} (epoch path)")
    np.testing.assert_array_equal(hist_e, hist)


# w, n, ell, s, d, tau, first epoch, word dtype, in place
SURVIVOR_CASES = [
    (32, 256, 32, 32, 20000, 1000, 48, np.uint32, False),    # budget not a multiple of the block
    (32, 250, 40, 16, 8000, 3000, 320, np.uint32, True),     # carried residues, two-pass loads
    (64, 128, 8, 8, 4000, 700, 100, np.uint64, False),       # u64 cells; K0 = 112
]


@pytest.mark.parametrize("case", SURVIVOR_CASES, ids=lambda c: f"w{c[0]}n{c[1]}t{c[5]}k{c[6]}")
def test_refill_first_epoch_with_survivors(torch_mod, case):
    """$RASP_REFILL=1: the refill kernel runs the first epoch (K0 = the first-epoch
    length rounded up to the block) and appends the machines still running
    to the survivor list; the epoch kernel runs the rest of the budget."""
    torch = torch_mod
    w, n, ell, s, d, tau, epoch, word, inplace = case
    p, c0 = _inputs((w, n, ell, s, d), seed=n + tau)
    want = _oracle(c0, p, tau)
    got, hist, launches = _run(torch, p, c0, tau, word, inplace, True, epoch=epoch)
    assert launches > (1 if inplace else 3), launches   # survivors continued on later epochs
    for f in RESULTS:
        g = got[f].astype(np.uint64) if f in FIELDS else got[f]
        np.testing.assert_array_equal(g, want[f], err_msg=f"{case} field {f}")
    np.testing.assert_array_equal(hist, _hist_of(want))


def test_refill_not_used_where_it_loses(torch_mod):
    """Auto mode runs the refill kernel only when it takes the whole budget in
    one launch (tau a multiple of the block, at most 2048) on 16-byte aligned
    machine rows; longer budgets keep the epochs (the paper row: 2.21 ms on
    epochs, 2.60+ refilled), and so do misaligned rows (n = 250 words)."""
    torch = torch_mod
    case = (32, 256, 32, 32, 3000, 4096, np.uint32, True, None)
    p, c0 = _inputs(case, seed=7)
    old = os.environ.pop("RASP_REFILL", None)
    try:
        from paper_2604_12902_b200 import _native
        from paper_2604_12902_b200.engine import DeviceBatch
        from paper_2604_12902_b200.hypervisor import get_engine
        dev = torch.device("cuda:0")
        eng = get_engine(p, dev)
        eng.warm(4, True)
        for tau, refilled in ((4096, False), (1024, True), (1000, False)):
            arrays = {f: c0[f].astype(np.uint32) for f in FIELDS}
            arrays.update(status=np.zeros(3000, np.int8), steps=np.zeros(3000, np.int64),
                          tau_h=np.full(3000, -1, np.int64))
            src = DeviceBatch.from_arrays(arrays, p, dev, word_bytes=4)
            torch.cuda.synchronize()
            n0 = _native.load().rasp_launch_count()
            eng.run(src, tau, 16, fresh=True)
            torch.cuda.synchronize()
            assert (_native.load().rasp_launch_count() - n0 == 1) == refilled, tau
        # misaligned rows (n * 4 bytes not a multiple of 16): epochs at any budget
        p2, c2 = _inputs((32, 250, 16, 16, 3000), seed=9)
        eng2 = get_engine(p2, dev)
        eng2.warm(4, True)
        arrays = {f: c2[f].astype(np.uint32) for f in FIELDS}
        src = DeviceBatch.from_arrays(arrays, p2, dev, word_bytes=4)
        torch.cuda.synchronize()
        n0 = _native.load().rasp_launch_count()
        eng2.run(src, 1024, 16, fresh=True)
        torch.cuda.synchronize()
        assert _native.load().rasp_launch_count() - n0 > 1
    finally:
        if old is not None:
            os.environ["RASP_REFILL"] = old
