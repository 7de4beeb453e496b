"""Multi-rank host logic on CPU (gloo, world_size 2 and 3): contiguous
shards, histogram all-reduce and verdict/output gather reproduce the
single-process result exactly.  The per-shard compute here is the CPU
oracle standing in for each rank's GPU (the GPU path is covered by
tests/test_gpu_parity.py); what is under test is the sharding and the
collectives of paper_2604_12902_b200.sharding."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from golden_io import FIELDS, load_family


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, g_index, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import oracle
        from paper_2604_12902_b200 import sharding
        g = load_family("gen")[g_index]
        d = g.d
        shard = sharding.shard_arrays(g.c0, world, rank)
        out = oracle.worker_arrays(shard, g.w, g.n, g.ell, g.s, g.tau_max)
        hist = torch.from_numpy(sharding.histogram_np(out["status"], out["tau_h"]))
        res = sharding.collect(torch.from_numpy(out["status"]), torch.from_numpy(out["steps"]),
                               torch.from_numpy(out["tau_h"]),
                               torch.from_numpy(out["y"].astype(np.int64)), hist, d)
        if rank == 0:
            q.put(("ok", res.histogram.tolist(), res.status.tolist(), res.steps.tolist(),
                   res.tau_h.tolist(), res.y.tolist(), res.machine_steps))
        else:
            q.put(("rank", rank, res.status is None, res.histogram.tolist()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_run_matches_single_process(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    g_index = 0   # C1 shape: 4096 machines, w8 n32, 64 steps
    procs = [ctx.Process(target=_worker, args=(r, world, port, g_index, q)) for r in range(world)]
    for p in procs:
        p.start()
    msgs = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    root = [m for m in msgs if m[0] == "ok"][0]
    others = [m for m in msgs if m[0] == "rank"]
    g = load_family("gen")[g_index]
    _, hist, status, steps, tau_h, y, ms = root
    assert hist == list(g.hist)
    assert status == g.out["status"].tolist()
    assert steps == g.out["steps"].tolist()
    assert tau_h == g.out["tau_h"].tolist()
    assert y == g.out["y"].astype(np.int64).tolist()
    assert ms == int(g.out["steps"].sum())
    for m in others:
        assert m[2] is True           # only rank 0 holds the gathered arrays
        assert m[3] == list(g.hist)   # every rank holds the reduced histogram


def test_shard_bounds_partition():
    from paper_2604_12902_b200.sharding import shard_bounds
    for d in (0, 1, 7, 4096, 1 << 20, (1 << 24) + 3):
        for world in (1, 2, 3, 4, 8):
            spans = [shard_bounds(d, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == d
            for (a, b), (c, e) in zip(spans, spans[1:]):
                assert b == c and a <= b
    with pytest.raises(ValueError):
        shard_bounds(10, 2, 2)


def _reuse_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2604_12902_b200 import sharding
        got = []
        for sizes in ([5, 5, 5], [5, 4, 3], [5, 5, 5]):   # equal, ragged, equal again
            d = sum(sizes)
            lo = sum(sizes[:rank])
            full = torch.arange(d * 3, dtype=torch.int64).reshape(d, 3)
            buf = None
            for rep in range(2):   # the receive buffer is reused on the second call
                res = sharding.gather_to_root(full[lo:lo + sizes[rank]] + rep, d, world, rank, sizes=sizes, out=buf)
                if rank == 0:
                    ok = torch.equal(res, full + rep)
                    buf = res._base if res._base is not None else res
                    got.append((ok, sizes == [5, 5, 5] and rep == 1 and res.data_ptr() == buf.data_ptr()
                                or sizes != [5, 5, 5] or rep == 0))
                else:
                    got.append((res is None, True))
        q.put((rank, got))
    finally:
        dist.destroy_process_group()


def test_gather_reuses_the_receive_buffer():
    """gather_to_root(out=...): rank 0's receive buffer is reused across calls
    (bench.py's per-step gathers), equal shards come back as a view of it,
    ragged ones concatenated; every result equals the unsharded tensor."""
    world = 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_reuse_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    msgs = dict(q.get(timeout=240) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    for r in range(world):
        assert all(a and b for a, b in msgs[r]), (r, msgs[r])
