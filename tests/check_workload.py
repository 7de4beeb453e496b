"""Small workloads for the checked build of the engine (tests/test_checked_build.py).

    RASP_LIBRARY=paper_2604_12902_b200/_lib/libraspvisor_b200_checked.so \
        python tests/check_workload.py <kind>

compute-sanitizer is closed on the GPU pool this project runs on (runs under
it left GPUs needing a reset), so its checks are compiled into the kernels
instead (-DRASP_CHECKED=1, csrc/rasp_kernels.cuh): every shared access within
the block's dynamic window, every cell access of a step within the lane's own
column (the ownership rule that makes the tiles race-free), every machine
index and compaction slot within the batch.  Each kind launches one family of
the engine's kernels and checks the results against the CPU oracle, so a run
that passes the checks but is wrong also fails.
Kinds:
  mx      u16 cells, lane-column tiles moved with stmatrix/ldmatrix (C2 shape),
          out of place (tile-wise u/y copies) and in place
  big     u32 cells, one-warp BIG tiles with PRI straight to HBM (C5 shape),
          several tiles per warp (the claim loop and the next-tile prefetch)
  refill  the per-lane refill kernel for fresh big machines (C5 shape; n not a
          power of two with a tape longer than 32 cells)
  big64   u64 cells (w = 64) BIG tiles, mid-run inputs (per-lane budgets)
  hbm     tiles in HBM (n too large for shared memory)
  enum    the exhaustive-enumeration kernel (config 4 domain, a few programs)
  aux     histogram, top-k (radix select), init_c0 packer, generator, validate,
          pack/unpack
"""

from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

FIELDS = ("iw", "ac", "M", "u", "y")
RESULTS = FIELDS + ("status", "steps", "tau_h")


def _check(got, want, tag):
    for k in RESULTS:
        g = np.asarray(got[k])
        if k in FIELDS:
            g = g.astype(np.uint64)
        if not np.array_equal(g, want[k]):
            raise SystemExit(f"{tag}: field {k} differs from the oracle")


def run_batch_kind(w, n, ell, s, d, tau, epoch, midrun=False, seed=0):
    import torch

    from oracle import oracle
    from paper_2604_12902_b200.engine import DeviceBatch
    from paper_2604_12902_b200.hypervisor import BatchConfig, get_engine, run_arrays
    from paper_2604_12902_b200.machine import MachineParams
    from paper_2604_12902_b200.workload import random_configs, synthetic_c0
    p = MachineParams(w=w, n=n, ell=ell, s=s, mu=1)
    rng = np.random.default_rng(seed)
    c0 = random_configs(d, p, rng) if midrun else synthetic_c0(d, p, seed=seed)
    arrays = dict(c0)
    want = {k: c0[k].astype(np.uint64) for k in FIELDS}
    if midrun:
        st = rng.choice(np.array([0, 0, 0, 1, 2], np.int8), d)
        sp = rng.integers(0, 2 * tau + 1, d).astype(np.int64)
        th = np.where(st == 1, sp, -1).astype(np.int64)
        arrays.update(status=st, steps=sp, tau_h=th)
        want.update(status=st.copy(), steps=sp.copy(), tau_h=th.copy())
    else:
        want.update(status=np.zeros(d, np.int8), steps=np.zeros(d, np.int64), tau_h=np.full(d, -1, np.int64))
    oracle.oracle_run(want["iw"], want["ac"], want["M"], want["u"], want["y"], want["status"], want["steps"],
                      want["tau_h"], w, n, ell, s, tau, 64, 1)
    # in place, through the public host surface
    res = run_arrays(arrays, p, BatchConfig(tau_max=tau, epoch=epoch, memory_budget_words=1 << 40))
    _check({k: getattr(res.slots, k) for k in RESULTS}, want, f"w{w} n{n} in-place")
    # out of place through the engine (the first epoch copies tapes tile by tile)
    dev = torch.device("cuda:0")
    src = DeviceBatch.from_arrays(arrays, p, dev)
    dst = DeviceBatch.empty(d, p, dev, fresh=False)
    get_engine(p, dev).run(src, tau, epoch, out=dst, fresh=not midrun)
    _check(dst.to_numpy(), want, f"w{w} n{n} out-of-place")


def run_enum():
    import torch

    from oracle import oracle
    from paper_2604_12902_b200.enumeration import C4, enumerate_device
    cnt = 64
    rec = torch.empty(cnt, dtype=torch.uint64, device="cuda:0")
    st = torch.zeros(1, dtype=torch.uint64, device="cuda:0")
    enumerate_device(C4, 1000, cnt, rec, st)
    want, steps = oracle.enumerate_records(C4.m, C4.opcode_bits, C4.operand_bits, C4.w, C4.n, C4.tau_max, 1000, cnt)
    if not np.array_equal(rec.cpu().numpy(), want) or int(st.cpu().numpy()[0]) != steps:
        raise SystemExit("enum: records differ from the oracle")


def run_aux():
    import torch

    from paper_2604_12902_b200.engine import DeviceBatch
    from paper_2604_12902_b200.hypervisor import get_engine
    from paper_2604_12902_b200.machine import MachineParams, init_batch
    from paper_2604_12902_b200.sharding import histogram_np
    dev = torch.device("cuda:0")
    p = MachineParams(w=16, n=64, ell=8, s=8, mu=1)
    eng = get_engine(p, dev)
    b = eng.generate(DeviceBatch.empty(3000, p, dev, fresh=False), seed=3)
    eng.run(b, 300, 16, fresh=True)
    h = eng.histogram(b).cpu().numpy()
    st, th = b.status.cpu().numpy(), b.tau_h.cpu().numpy()
    if not np.array_equal(h, histogram_np(st, th)):
        raise SystemExit("aux: histogram differs")
    idx, tau = eng.topk(b, 10, 300)
    order = sorted(((int(th[j]), -j) for j in range(len(st)) if st[j] == 1), reverse=True)[:10]
    if [int(v) for v in tau.cpu().numpy()] != [t for t, _ in order]:
        raise SystemExit("aux: top-k differs")
    if eng.validate(b).any():
        raise SystemExit("aux: validate flagged a valid batch")
    rng = np.random.default_rng(4)
    progs = rng.integers(0, 1 << 16, (500, 30), dtype=np.uint64).astype(np.uint16)
    xs = rng.integers(0, 1 << 16, (500, 4), dtype=np.uint64).astype(np.uint16)
    out = DeviceBatch.empty(500, p, dev, fresh=False)
    eng.init_c0(torch.from_numpy(progs).to(dev), torch.from_numpy(xs).to(dev), out)
    want = init_batch(progs, xs, p)
    got = out.to_numpy()
    for k in FIELDS:
        if not np.array_equal(got[k], want[k]):
            raise SystemExit(f"aux: init_c0 field {k} differs")
    wide = DeviceBatch.empty(500, p, dev, word_bytes=8, fresh=False)
    eng.convert(out, wide)
    back = DeviceBatch.empty(500, p, dev, fresh=False)
    eng.convert(wide, back)
    for k in FIELDS:
        if not torch.equal(getattr(back, k), getattr(out, k)):
            raise SystemExit(f"aux: pack/unpack round trip differs in {k}")


def main(kind):
    import torch
    torch.cuda.set_device(0)
    if kind == "mx":
        run_batch_kind(16, 64, 8, 8, 512, 200, 16)
    elif kind == "big":
        os.environ["RASP_REFILL"] = "0"                     # the epoch kernel's big tiles
        run_batch_kind(32, 256, 32, 32, 1 << 16, 48, 24)   # > 2 tiles per resident warp (888)
    elif kind == "refill":
        os.environ["RASP_REFILL"] = "1"                     # the per-lane refill kernel
        run_batch_kind(32, 256, 32, 32, 1 << 16, 256, 256)  # whole budget, ~70 machines per resident warp
        run_batch_kind(32, 256, 32, 32, 20000, 256, 24)     # first epoch of 32, survivors on epochs
        run_batch_kind(32, 250, 40, 16, 20000, 320, 16)     # carried residues, two-pass row loads
    elif kind == "big64":
        run_batch_kind(64, 128, 8, 8, 256, 60, 8, midrun=True)
    elif kind == "hbm":
        run_batch_kind(32, 4000, 4, 2, 64, 40, 8, midrun=True)
    elif kind == "enum":
        run_enum()
    elif kind == "aux":
        run_aux()
    else:
        raise SystemExit(f"unknown kind {kind}")
    torch.cuda.synchronize()
    from paper_2604_12902_b200 import _native
    print(f"check workload {kind}: ok (checked build: {_native.load().rasp_checked_build()})")


if __name__ == "__main__":
    main(sys.argv[1])
