"""C3-scale parity (SURVEY §8c plan, §8e): 2^24 machines of the C2 shape.

* Partition invariance: the whole batch run at once and the same machines run
  as G = 2, 4, 8 contiguous shards (shard_bounds) give byte-identical results
  (the 1/2/4/8-GPU requirement, checked on one device shard by shard).
* A seeded 2^20-machine sample of the batch equals the CPU oracle.
"""

import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

D = 1 << 24
TAU = 1024


@pytest.fixture(scope="module")
def c3():
    import torch

    from paper_2604_12902_b200.engine import DeviceBatch
    from paper_2604_12902_b200.hypervisor import get_engine
    from paper_2604_12902_b200.machine import MachineParams
    p = MachineParams(w=16, n=64, ell=8, s=8)
    dev = torch.device("cuda:0")
    eng = get_engine(p, dev)
    c0 = eng.generate(DeviceBatch.empty(D, p, dev), seed=0)
    whole = DeviceBatch.empty(D, p, dev)
    eng.run(c0, TAU, 64, out=whole, fresh=True)
    torch.cuda.synchronize()
    return p, dev, eng, c0, whole


@pytest.mark.parametrize("world", [2, 4, 8])
def test_partition_invariance(c3, world):
    import torch

    from paper_2604_12902_b200.engine import DeviceBatch
    from paper_2604_12902_b200.sharding import shard_bounds
    p, dev, eng, c0, whole = c3
    for rank in range(world):
        lo, hi = shard_bounds(D, world, rank)
        shard = eng.generate(DeviceBatch.empty(hi - lo, p, dev), seed=0, first_machine=lo)
        for k in ("iw", "ac", "M", "u", "y"):
            assert torch.equal(getattr(shard, k), getattr(c0, k)[lo:hi]), (world, rank, k)
        eng.run(shard, TAU, 64, fresh=True)
        for k in ("iw", "ac", "M", "u", "y", "status", "steps", "tau_h"):
            assert torch.equal(getattr(shard, k), getattr(whole, k)[lo:hi]), (world, rank, k)
        del shard


def test_sample_matches_oracle(c3):
    import torch

    from oracle.oracle import oracle_run
    p, dev, eng, c0, whole = c3
    rng = np.random.default_rng(20)
    idx = np.sort(rng.choice(D, 1 << 20, replace=False))
    it = torch.from_numpy(idx).to(dev)
    a = {k: getattr(c0, k).index_select(0, it).cpu().numpy().astype(np.uint64)
         for k in ("iw", "ac", "M", "u", "y")}
    d = idx.size
    st, sp, th = np.zeros(d, np.int8), np.zeros(d, np.int64), np.full(d, -1, np.int64)
    oracle_run(a["iw"], a["ac"], a["M"], a["u"], a["y"], st, sp, th, p.w, p.n, p.ell, p.s, TAU,
               workers=os.cpu_count() or 1)
    got = {k: getattr(whole, k).index_select(0, it).cpu().numpy() for k in
           ("iw", "ac", "M", "u", "y", "status", "steps", "tau_h")}
    for k in ("iw", "ac", "M", "u", "y"):
        np.testing.assert_array_equal(got[k].astype(np.uint64), a[k], err_msg=k)
    np.testing.assert_array_equal(got["status"], st)
    np.testing.assert_array_equal(got["steps"], sp)
    np.testing.assert_array_equal(got["tau_h"], th)


def test_histogram_and_topk_at_scale(c3):
    """Device histogram and top-K over the 16M results equal numpy's."""
    from paper_2604_12902_b200.search import top_halting
    from paper_2604_12902_b200.sharding import histogram_np
    p, dev, eng, c0, whole = c3
    status = whole.status.cpu().numpy()
    tau_h = whole.tau_h.cpu().numpy()
    np.testing.assert_array_equal(eng.histogram(whole).cpu().numpy(), histogram_np(status, tau_h))
    hal = np.nonzero(status == 1)[0]
    order = np.lexsort((hal, -tau_h[hal]))[:100]
    assert top_halting(whole, 100, TAU) == [(int(tau_h[hal[o]]), int(hal[o])) for o in order]
