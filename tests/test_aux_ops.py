"""Auxiliary boundary ops: rasp_topk (bb-search's top-K, cli.py:195-230),
rasp_pack/rasp_unpack (uint64 <-> natural width, hv:280-284) and the NCCL
shard collectives through NativeComm."""

import heapq

import numpy as np
import pytest

from golden_io import load_family


def heap_topk(status, tau_h, k, first_index=0):
    """The reference's selection, literally: a min-heap of (tau_h, -index)
    fed in index order (cli.py:218-226), reported sorted(reverse=True)."""
    best = []
    for pos in range(len(status)):
        if status[pos] == 1:
            item = (int(tau_h[pos]), -(first_index + pos))
            if len(best) < k:
                heapq.heappush(best, item)
            elif item > best[0]:
                heapq.heapreplace(best, item)
    return [(t, -ni) for t, ni in sorted(best, reverse=True)]


def numpy_topk(status, tau_h, k):
    """Same selection by a stable sort (tau_h desc, index asc)."""
    idx = np.nonzero(status == 1)[0]
    order = np.lexsort((idx, -tau_h[idx]))[:k]
    return [(int(tau_h[idx[o]]), int(idx[o])) for o in order]


@pytest.mark.parametrize("seed", range(5))
def test_numpy_topk_matches_heap(seed):
    rng = np.random.default_rng(seed)
    d = 3000
    status = rng.integers(0, 3, d).astype(np.int8)
    tau_h = np.where(status == 1, rng.integers(0, 50, d), -1)
    for k in (1, 3, 17, 2000, 5000):
        assert numpy_topk(status, tau_h, k) == heap_topk(status, tau_h, k)


# ------------------------------------------------------------------------- GPU
def _batch_of(status, tau_h):
    import torch

    from paper_2604_12902_b200.engine import DeviceBatch
    from paper_2604_12902_b200.machine import MachineParams
    p = MachineParams(w=16, n=4, ell=1, s=1)
    b = DeviceBatch.empty(len(status), p, "cuda:0")
    b.status.copy_(torch.from_numpy(np.ascontiguousarray(status)))
    b.tau_h.copy_(torch.from_numpy(np.ascontiguousarray(tau_h.astype(np.int64))))
    return b


@pytest.mark.gpu
@pytest.mark.parametrize("case", ["random", "ties", "few", "none", "all_tied", "deep", "one"])
def test_topk_matches_heap(case):
    from paper_2604_12902_b200.search import top_halting
    rng = np.random.default_rng(len(case) * 7919 + ord(case[0]))
    d, tau_max = 200_000, 1024
    status = rng.integers(0, 3, d).astype(np.int8)
    tau_h = rng.integers(0, tau_max + 1, d)
    if case == "ties":
        tau_h = rng.integers(0, 4, d)
    elif case == "few":
        status[:] = 2
        status[rng.choice(d, 5, replace=False)] = 1
    elif case == "none":
        status[:] = 2
    elif case == "all_tied":
        status[:] = 1
        tau_h[:] = 7
    elif case == "deep":
        tau_max = 10 ** 6
        tau_h = rng.integers(0, tau_max + 1, d)
        tau_h[rng.choice(d, 50, replace=False)] = tau_max
    elif case == "one":
        d = 1
        status, tau_h = np.array([1], np.int8), np.array([0])
    tau_h = np.where(status == 1, tau_h, -1)
    b = _batch_of(status, tau_h)
    for k in (1, 3, 10, 100, 2048):
        assert top_halting(b, k, tau_max) == heap_topk(status, tau_h, k), (case, k)


@pytest.mark.gpu
def test_topk_large_batch():
    from paper_2604_12902_b200.search import top_halting
    rng = np.random.default_rng(7)
    d = 1 << 24
    status = (rng.random(d) < 0.8).astype(np.int8)
    status[status == 0] = 2
    tau_h = np.where(status == 1, rng.geometric(0.02, d), -1)
    tau_h = np.minimum(tau_h, 100_000)
    b = _batch_of(status, tau_h)
    assert top_halting(b, 64, 100_000) == numpy_topk(status, tau_h, 64)


@pytest.mark.gpu
def test_topk_errors():
    import torch

    from paper_2604_12902_b200.errors import NativeError
    from paper_2604_12902_b200.hypervisor import get_engine
    b = _batch_of(np.ones(4, np.int8), np.arange(4))
    eng = get_engine(b.params, torch.device("cuda:0"))
    with pytest.raises(NativeError):
        eng.topk(b, 4097, 10)
    idx, tau = eng.topk(b, 0, 10)
    assert idx.numel() == 0 and tau.numel() == 0


@pytest.mark.gpu
def test_bb_search_on_golden_programs():
    """The BB fixtures (t/test_lowering.py:179-187: tau_h 1727, 1409, 1387)
    mixed into random short programs: bb_search's ranking equals the
    reference's heap over the oracle's results, and the fixtures top it."""
    from oracle.oracle import oracle_run
    from paper_2604_12902_b200.machine import MachineParams
    from paper_2604_12902_b200.search import bb_search
    (g,) = load_family("bb")
    p = MachineParams(w=g.w, n=g.n, ell=g.ell, s=g.s)
    rng = np.random.default_rng(3)
    rand = np.zeros((3000, p.n), np.uint64)
    rand[:, 0:40:2] = rng.integers(0, 8, (3000, 20))
    rand[:, 1:40:2] = rng.integers(0, 40, (3000, 20))
    progs = np.concatenate([rand[:1000], g.c0["M"], rand[1000:]])
    tau_max = 10 ** 5
    rep = bb_search(progs.astype(np.uint32), p, tau_max=tau_max, top=5, chunk=1024)
    d = progs.shape[0]
    c0 = dict(iw=np.zeros(d, np.uint64), ac=np.zeros(d, np.uint64), M=progs.copy(),
              u=np.zeros((d, p.ell + 1), np.uint64), y=np.zeros((d, p.s + 1), np.uint64),
              status=np.zeros(d, np.int8), steps=np.zeros(d, np.int64), tau_h=np.full(d, -1, np.int64))
    oracle_run(c0["iw"], c0["ac"], c0["M"], c0["u"], c0["y"], c0["status"], c0["steps"], c0["tau_h"],
               p.w, p.n, p.ell, p.s, tau_max, workers=8)
    assert rep.sampled == d
    assert rep.halted == int((c0["status"] == 1).sum())
    assert rep.best == heap_topk(c0["status"], c0["tau_h"], 5)
    assert rep.best[:3] == [(1727, 1000), (1409, 1001), (1387, 1002)]


@pytest.mark.gpu
@pytest.mark.parametrize("w,wb", [(8, 1), (16, 2), (32, 4), (12, 2), (64, 8)])
def test_pack_unpack_roundtrip_and_run(w, wb):
    """uint64 (reference layout) -> natural width -> run -> back to uint64
    equals running on the uint64 arrays directly."""
    import torch

    from paper_2604_12902_b200.engine import DeviceBatch
    from paper_2604_12902_b200.hypervisor import get_engine
    from paper_2604_12902_b200.machine import MachineParams
    from paper_2604_12902_b200.workload import random_configs
    p = MachineParams(w=w, n=24, ell=5, s=4)
    arr = random_configs(5000, p, np.random.default_rng(w), dtype=np.uint64)
    dev = torch.device("cuda:0")
    eng = get_engine(p, dev)
    wide = DeviceBatch.from_arrays(arr, p, dev, word_bytes=8)
    nat = DeviceBatch.empty(wide.d, p, dev, word_bytes=wb)
    eng.convert(wide, nat)
    back = DeviceBatch.empty(wide.d, p, dev, word_bytes=8)
    eng.convert(nat, back)
    for k in ("iw", "ac", "M", "u", "y", "status", "steps", "tau_h"):
        assert torch.equal(getattr(back, k), getattr(wide, k)), k
    eng.run(wide, 300, 8)
    eng.run(nat, 300, 8)
    eng.convert(nat, back)
    for k in ("iw", "ac", "M", "u", "y", "status", "steps", "tau_h"):
        assert torch.equal(getattr(back, k), getattr(wide, k)), k


@pytest.mark.gpu
def test_pack_rejects_narrow_destination():
    import torch

    from paper_2604_12902_b200.engine import DeviceBatch
    from paper_2604_12902_b200.errors import NativeError
    from paper_2604_12902_b200.hypervisor import get_engine
    from paper_2604_12902_b200.machine import MachineParams
    p = MachineParams(w=16, n=8, ell=2, s=2)
    dev = torch.device("cuda:0")
    a = DeviceBatch.empty(10, p, dev, word_bytes=8)
    b = DeviceBatch.empty(10, p, dev, word_bytes=1)
    with pytest.raises(NativeError):
        get_engine(p, dev).convert(a, b)


@pytest.mark.gpu
def test_native_comm_single_rank():
    """rasp_nccl_* / rasp_shard_* on a one-rank communicator: the all-reduce
    is the identity and the gather places the shard into the full batch."""
    import torch

    from paper_2604_12902_b200._native import RASP_GATHER_CONFIG, RASP_GATHER_OUTPUT, RASP_GATHER_RESULTS
    from paper_2604_12902_b200.engine import DeviceBatch
    from paper_2604_12902_b200.hypervisor import get_engine
    from paper_2604_12902_b200.machine import MachineParams
    from paper_2604_12902_b200.sharding import NativeComm
    from paper_2604_12902_b200.workload import synthetic_c0
    p = MachineParams(w=16, n=64, ell=8, s=8)
    dev = torch.device("cuda:0")
    b = DeviceBatch.from_arrays(synthetic_c0(4096, p, seed=1), p, dev)
    eng = get_engine(p, dev)
    eng.run(b, 1024, 64, fresh=True)
    h = eng.histogram(b)
    h0 = h.clone()
    comm = NativeComm(device=dev)
    comm.allreduce(h)
    assert torch.equal(h, h0)
    full = DeviceBatch.empty(b.d, p, dev)
    comm.gather(b, full, b.d, RASP_GATHER_RESULTS | RASP_GATHER_OUTPUT | RASP_GATHER_CONFIG)
    torch.cuda.synchronize()
    for k in ("iw", "ac", "M", "u", "y", "status", "steps", "tau_h"):
        assert torch.equal(getattr(full, k), getattr(b, k)), k
    comm.close()
