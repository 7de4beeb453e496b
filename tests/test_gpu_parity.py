"""GPU parity: the CUDA engine (through the C ABI) against the reference's
golden outputs (tests/golden, produced by raspvisor.run_batch) and the
pinned CPU oracle.  Bit-exact on every field: final iw/ac/M/u/y, status,
steps, tau_h."""

import numpy as np
import pytest

from golden_io import FIELDS, RESULTS, load_all, load_family

pytestmark = pytest.mark.gpu

ALL = load_all()


@pytest.fixture(scope="module")
def pkg():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device")
    import paper_2604_12902_b200 as P
    from paper_2604_12902_b200 import hypervisor
    return P, hypervisor


def _params(P, g):
    return P.MachineParams(w=g.w, n=g.n, ell=g.ell, s=g.s, mu=1)


def _assert_same(res_arrays, g, tag=""):
    for k in RESULTS:
        got = np.asarray(res_arrays[k])
        want = g.out[k]
        if k in FIELDS:
            got = got.astype(np.uint64)
        np.testing.assert_array_equal(got, want, err_msg=f"{g} {tag} field {k}")


def _slots_dict(sv):
    return {k: getattr(sv, k) for k in RESULTS}


@pytest.mark.parametrize("g", ALL, ids=repr)
@pytest.mark.parametrize("epoch", [1, 7, 64])
def test_engine_matches_reference_natural_width(pkg, g, epoch):
    P, H = pkg
    p = _params(P, g)
    c0 = {k: g.c0[k].astype(p.dtype) for k in FIELDS}
    res = H.run_arrays(c0, p, H.BatchConfig(tau_max=g.tau_max, epoch=epoch,
                                            memory_budget_words=1 << 40))
    _assert_same(_slots_dict(res.slots), g, f"epoch={epoch}")


@pytest.mark.parametrize("g", [g for g in ALL if g.family in ("corpus", "hyp", "edge", "kat")],
                         ids=repr)
def test_engine_matches_reference_uint64_layout(pkg, g):
    """The reference's own uint64 arrays, unconverted (word_bytes = 8)."""
    P, H = pkg
    p = _params(P, g)
    res = H.run_arrays(dict(g.c0), p, H.BatchConfig(tau_max=g.tau_max, epoch=5,
                                                    memory_budget_words=1 << 40))
    assert res.slots.M.dtype == np.uint64
    _assert_same(_slots_dict(res.slots), g, "u64")


@pytest.mark.parametrize("g", load_family("corpus")[:7], ids=repr)
def test_run_batch_tuple_api(pkg, g):
    """The tuple interface returns the reference's SlotView/histogram."""
    P, H = pkg
    p = _params(P, g)
    configs = [P.Config(int(g.c0["iw"][k]), int(g.c0["ac"][k]),
                        tuple(int(v) for v in g.c0["M"][k]),
                        tuple(int(v) for v in g.c0["u"][k]),
                        tuple(int(v) for v in g.c0["y"][k])) for k in range(g.d)]
    res = H.run_batch(configs, p, H.BatchConfig(tau_max=g.tau_max))
    _assert_same(_slots_dict(res.slots), g, "tuples")
    assert res.slots.iw.dtype == np.uint64
    want = {}
    for st, th in zip(g.out["status"], g.out["tau_h"]):
        if st == 1:
            want[int(th)] = want.get(int(th), 0) + 1
    assert dict(res.histogram) == want
    hist = H.collect_histogram(res.slots)
    assert [hist[k] for k in H.HISTOGRAM_KEYS] == list(g.hist)


@pytest.mark.parametrize("g", load_family("gen") + load_family("corpus")[:7], ids=repr)
def test_out_of_place_and_device_histogram(pkg, g):
    import torch
    P, H = pkg
    from paper_2604_12902_b200.engine import DeviceBatch
    p = _params(P, g)
    c0 = {k: g.c0[k].astype(p.dtype) for k in FIELDS}
    src = DeviceBatch.from_arrays(c0, p)
    before = {k: v.clone() for k, v in src.tensors().items()}
    dst = DeviceBatch.empty(g.d, p, fresh=False)
    eng = H.get_engine(p)
    eng.run(src, g.tau_max, epoch=16, out=dst, fresh=True)
    torch.cuda.synchronize()
    for k, v in src.tensors().items():            # input untouched
        assert torch.equal(v, before[k]), k
    _assert_same(dst.to_numpy(), g, "out-of-place")
    assert list(eng.histogram(dst).cpu().numpy()) == list(g.hist)
    # the histogram counted inside the run (rasp_run_hist), in and out of place
    h = torch.full((102,), 7, dtype=torch.int64, device=dst.M.device)
    dst2 = DeviceBatch.empty(g.d, p, fresh=False)
    eng.run(src, g.tau_max, epoch=5, out=dst2, fresh=True, hist=h)
    assert list(h.cpu().numpy()) == list(g.hist)
    _assert_same(dst2.to_numpy(), g, "out-of-place, fused histogram")
    h.fill_(3)
    eng.run(src, g.tau_max, epoch=16, fresh=True, hist=h)
    assert list(h.cpu().numpy()) == list(g.hist)


def test_general_worker_contract(pkg):
    """_worker semantics on mid-run inputs: nonzero initial steps, machines
    already HALTED/EXHAUSTED are untouched (hv:136), tau_h left as given for
    budget exhaustion.  Checked against the C oracle on the same arrays."""
    P, H = pkg
    from oracle import oracle
    g = [x for x in load_family("corpus") if x.tau_max == 200][0]
    p = _params(P, g)
    rng = np.random.default_rng(7)
    d = g.d
    status = rng.choice(np.array([0, 0, 0, 1, 2], np.int8), d)
    steps = rng.integers(0, 260, d).astype(np.int64)
    tau_h = np.where(status == 1, steps, rng.integers(-1, 5, d)).astype(np.int64)
    want = {k: np.ascontiguousarray(g.c0[k]).copy() for k in FIELDS}
    want.update(status=status.copy(), steps=steps.copy(), tau_h=tau_h.copy())
    oracle.oracle_run(want["iw"], want["ac"], want["M"], want["u"], want["y"], want["status"],
                      want["steps"], want["tau_h"], g.w, g.n, g.ell, g.s, g.tau_max, 64, 1)
    for epoch in (1, 64):
        arrays = {k: g.c0[k].astype(p.dtype) for k in FIELDS}
        arrays.update(status=status, steps=steps, tau_h=tau_h)
        res = H.run_arrays(arrays, p, H.BatchConfig(tau_max=g.tau_max, epoch=epoch))
        for k in RESULTS:
            got = np.asarray(getattr(res.slots, k))
            if k in FIELDS:
                got = got.astype(np.uint64)
            np.testing.assert_array_equal(got, want[k], err_msg=f"{k} epoch={epoch}")
    # the fused histogram counts machines that entered HALTED/EXHAUSTED as they stand
    import torch
    from paper_2604_12902_b200.engine import DeviceBatch
    from paper_2604_12902_b200.sharding import histogram_np
    arrays = {k: g.c0[k].astype(p.dtype) for k in FIELDS}
    arrays.update(status=status, steps=steps, tau_h=tau_h)
    for inplace in (True, False):
        src = DeviceBatch.from_arrays(arrays, p)
        dst = src if inplace else DeviceBatch.empty(d, p, fresh=False)
        h = torch.zeros(102, dtype=torch.int64, device=src.M.device)
        H.get_engine(p).run(src, g.tau_max, 8, out=dst, hist=h)
        np.testing.assert_array_equal(h.cpu().numpy(), histogram_np(want["status"], want["tau_h"]))


def test_bb_fixtures(pkg):
    P, H = pkg
    (g,) = load_family("bb")
    p = _params(P, g)
    res = H.run_arrays({k: g.c0[k].astype(p.dtype) for k in FIELDS}, p,
                       H.BatchConfig(tau_max=10 ** 5))
    assert list(res.slots.tau_h) == [1727, 1409, 1387]
    assert list(res.slots.y[:, 0]) == [1, 1, 1] and list(res.slots.y[:, 1]) == [0, 0, 0]


def test_validation_errors(pkg):
    P, H = pkg
    p = P.MachineParams(w=8, n=8, ell=2, s=2, mu=1)
    good = P.init_config(P.Program((0, 0)), [], p)
    bad = P.Config(i=0, a=0, M=(0, 300, 0, 0, 0, 0, 0, 0), u=good.u, y=good.y)
    with pytest.raises(ValueError, match="2\\^w"):
        H.run_batch([good, bad], p, H.BatchConfig(tau_max=1))
    with pytest.raises(P.CapacityError, match="budget"):
        H.run_batch([good] * 10, p, H.BatchConfig(tau_max=1, memory_budget_words=10))
    with pytest.raises(ValueError):
        H.run_batch([P.Config(0, 0, (0,) * 7, (0, 0, 0), (0, 0, 0))], p, H.BatchConfig(tau_max=1))
    res = H.run_batch([], p, H.BatchConfig(tau_max=10))
    assert len(res.slots) == 0 and res.histogram == {}


def test_large_batch_against_oracle_sample(pkg):
    """C2 shape at 2^20 machines: GPU vs oracle on a seeded 2^11 sample,
    plus size-independent properties on the whole batch."""
    P, H = pkg
    from oracle import oracle
    p = P.MachineParams(w=16, n=64, ell=8, s=8, mu=1)
    d, tau = 1 << 20, 1024
    c0 = P.synthetic_c0(d, p, seed=0)
    res = H.run_arrays(c0, p, H.BatchConfig(tau_max=tau, epoch=32, memory_budget_words=1 << 40))
    sv = res.slots
    st, steps, th = sv.status, sv.steps, sv.tau_h
    assert set(np.unique(st)) <= {1, 2}
    assert (steps <= tau).all()
    assert (th[st == 1] == steps[st == 1]).all()
    assert (steps[st == 2] == tau).all() and (th[st == 2] == -1).all()
    idx = np.sort(np.random.default_rng(1).choice(d, 2048, replace=False))
    sample = {k: c0[k][idx] for k in FIELDS}
    want = oracle.worker_arrays(sample, p.w, p.n, p.ell, p.s, tau)
    for k in RESULTS:
        got = np.asarray(getattr(sv, k))[idx]
        if k in FIELDS:
            got = got.astype(np.uint64)
        np.testing.assert_array_equal(got, want[k], err_msg=k)
    # epoch independence on the full batch
    res2 = H.run_arrays(c0, p, H.BatchConfig(tau_max=tau, epoch=5, memory_budget_words=1 << 40))
    for k in RESULTS:
        assert np.array_equal(getattr(res2.slots, k), getattr(sv, k)), k


@pytest.mark.parametrize("shape", [(8, 8, 2, 2), (16, 16, 2, 2), (16, 64, 8, 8), (32, 250, 10, 2),
                                   (32, 64, 4, 2), (64, 12, 3, 3), (5, 7, 3, 2), (1, 6, 1, 1),
                                   # n not a power of two on every tile kind (carried residues)
                                   (8, 250, 10, 2), (12, 100, 4, 4), (16, 100, 8, 8), (32, 100, 4, 2),
                                   (24, 30, 3, 3), (3, 6, 2, 2), (64, 250, 4, 2)])
def test_random_midrun_configs_against_oracle(pkg, shape):
    """Arbitrary mid-run configurations (every step case, odd i, full tapes,
    wrapped addresses) at 8K machines per shape, several epochs."""
    P, H = pkg
    from oracle import oracle
    from paper_2604_12902_b200.workload import random_configs
    w, n, ell, s = shape
    p = P.MachineParams(w=w, n=n, ell=ell, s=s, mu=1)
    c0 = random_configs(8192, p, np.random.default_rng(w * 1000 + n))
    for tau in (0, 3, 200):
        want = oracle.worker_arrays(c0, w, n, ell, s, tau)
        for epoch in (1, 64):
            res = H.run_arrays(c0, p, H.BatchConfig(tau_max=tau, epoch=epoch))
            for k in RESULTS:
                got = np.asarray(getattr(res.slots, k))
                if k in FIELDS:
                    got = got.astype(np.uint64)
                np.testing.assert_array_equal(got, want[k], err_msg=f"{shape} tau={tau} {k}")


def test_device_packer_matches_init_batch(pkg):
    import torch
    P, H = pkg
    from paper_2604_12902_b200.engine import DeviceBatch
    p = P.MachineParams(w=16, n=64, ell=8, s=8, mu=1)
    rng = np.random.default_rng(3)
    progs = rng.integers(0, 1 << 16, (1000, 40), dtype=np.uint64).astype(np.uint16)
    xs = rng.integers(0, 1 << 16, (1000, 5), dtype=np.uint64).astype(np.uint16)
    want = P.init_batch(progs, xs, p)
    out = DeviceBatch.empty(1000, p, fresh=False)
    eng = H.get_engine(p)
    eng.init_c0(torch.from_numpy(progs).cuda(), torch.from_numpy(xs).cuda(), out)
    got = out.to_numpy()
    for k in FIELDS:
        np.testing.assert_array_equal(got[k], want[k], err_msg=k)
    assert not got["status"].any() and not got["steps"].any() and (got["tau_h"] == -1).all()


def test_device_generator_shape_and_parity(pkg):
    """G_dev: the c0 shape of generator G, deterministic per (seed, machine),
    shard-independent; runs bit-exactly against the oracle."""
    P, H = pkg
    from oracle import oracle
    from paper_2604_12902_b200.engine import DeviceBatch
    p = P.MachineParams(w=16, n=64, ell=8, s=8, mu=1)
    eng = H.get_engine(p)
    a = eng.generate(DeviceBatch.empty(4096, p, fresh=False), seed=7).to_numpy()
    b = eng.generate(DeviceBatch.empty(1024, p, fresh=False), seed=7, first_machine=3072).to_numpy()
    for k in FIELDS:
        np.testing.assert_array_equal(a[k][3072:], b[k])
    ops, opr = a["M"][:, 0::2], a["M"][:, 1::2]
    assert ops.min() >= 1 and ops.max() <= 7 and opr.max() < 64
    assert (opr[ops == 5] % 2 == 0).all()
    assert set(np.unique(ops)) == set(range(1, 8))
    assert not a["iw"].any() and not a["u"][:, 0].any() and not a["y"].any()
    c0 = {k: a[k] for k in FIELDS}
    res = H.run_arrays(c0, p, H.BatchConfig(tau_max=1024))
    want = oracle.worker_arrays(c0, p.w, p.n, p.ell, p.s, 1024)
    for k in RESULTS:
        got = np.asarray(getattr(res.slots, k))
        if k in FIELDS:
            got = got.astype(np.uint64)
        np.testing.assert_array_equal(got, want[k], err_msg=k)


def test_scalar_path_through_kernel(pkg):
    """step / run_to_fixpoint (m:169-211, m:336-357 signatures) on the GPU:
    the step KATs of t/test_machine.py:90-166 and the trace example :202-208."""
    P, H = pkg
    from golden_io import load_raw
    from paper_2604_12902_b200 import scalar
    z = load_raw("kat")
    g = load_family("kat")[0]
    p = _params(P, g)
    for k in range(g.d):
        c = P.Config(int(g.c0["iw"][k]), int(g.c0["ac"][k]), tuple(int(v) for v in g.c0["M"][k]),
                     tuple(int(v) for v in g.c0["u"][k]), tuple(int(v) for v in g.c0["y"][k]))
        out = scalar.step(c, p)
        flat = [out.next.i, out.next.a, *out.next.M, *out.next.u, *out.next.y]
        assert flat == [int(v) for v in z["step_next"][k]], k
        assert out.fixed_point == bool(z["step_fixed"][k]), k
    c0 = P.init_config(P.Program((1, 5, 4, 6)), [], p)
    seen = []
    cf, tau = scalar.run_to_fixpoint(c0, 10, p, trace=lambda t, c: seen.append((t, c.i)))
    assert seen == [(0, 0), (1, 2), (2, 4)] and tau == 2 and cf.M[6] == 5
    assert scalar.run_to_fixpoint(c0, 1, p)[1] is None
    assert scalar.run_to_fixpoint(c0, 2, p)[1] == 2


def test_run_programs_host_path(pkg):
    """Programs + inputs from host buffers (device-side init_config, chunked
    pipeline) give the same results as run_arrays on the assembled c0."""
    P, H = pkg
    p = P.MachineParams(w=16, n=64, ell=8, s=8, mu=1)
    c0 = P.synthetic_c0(50000, p, seed=5)
    a = H.run_programs(c0["M"], c0["u"][:, 1:], p, H.BatchConfig(tau_max=1024), chunks=3)
    b = H.run_arrays(c0, p, H.BatchConfig(tau_max=1024))
    for k in RESULTS:
        np.testing.assert_array_equal(getattr(a.slots, k), getattr(b.slots, k), err_msg=k)
    assert a.histogram == b.histogram
    with pytest.raises(P.CapacityError):
        H.run_programs(np.zeros((4, 66), np.uint16), np.zeros((4, 1), np.uint16), p,
                       H.BatchConfig(tau_max=1))
    with pytest.raises(ValueError):
        H.run_programs(np.full((4, 2), 70000, np.uint32), np.zeros((4, 1), np.uint32), p,
                       H.BatchConfig(tau_max=1))


def test_cuda_graph_replay_matches_eager(pkg):
    """rasp_run + rasp_histogram captured in a CUDA graph (what bench.py times)
    and replayed give the eager results: the launch sequence is fixed and
    everything is enqueued on the caller's stream."""
    import torch
    P, H = pkg
    from paper_2604_12902_b200.engine import DeviceBatch
    from paper_2604_12902_b200.workload import synthetic_c0
    p = P.MachineParams(w=16, n=64, ell=8, s=8, mu=1)
    dev = torch.device("cuda:0")
    src = DeviceBatch.from_arrays(synthetic_c0(50_000, p, seed=9), p, dev)
    eng = H.get_engine(p, dev)
    ref = DeviceBatch.empty(src.d, p, dev, fresh=False)
    eng.run(src, 1024, 48, out=ref, fresh=True)
    href = eng.histogram(ref).clone()
    dst = DeviceBatch.empty(src.d, p, dev, fresh=False)
    hist = torch.empty(102, dtype=torch.int64, device=dev)
    cap = torch.cuda.Stream(dev)
    cap.wait_stream(torch.cuda.current_stream(dev))
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=cap):
        eng.run(src, 1024, 48, out=dst, fresh=True, stream=cap)
        eng.histogram(dst, out=hist, stream=cap)
    for _ in range(2):
        for t in (dst.iw, dst.M, dst.steps):
            t.zero_()
        g.replay()
        torch.cuda.synchronize()
        for k in ("iw", "ac", "M", "u", "y", "status", "steps", "tau_h"):
            assert torch.equal(getattr(dst, k), getattr(ref, k)), k
        assert torch.equal(hist, href)


def test_cuda_graph_replays_follow_each_batch_schedule(pkg):
    """One captured launch sequence serves batches whose device-side schedules
    differ: a replay on a batch that needs every planned epoch after one whose
    machines all halt at t = 0 (schedule over after the first epoch) still
    matches eager runs, in either order."""
    import torch
    P, H = pkg
    from paper_2604_12902_b200.engine import DeviceBatch
    from paper_2604_12902_b200.workload import synthetic_c0
    p = P.MachineParams(w=16, n=64, ell=8, s=8, mu=1)
    dev = torch.device("cuda:0")
    long_c0 = synthetic_c0(20_000, p, seed=4)
    quick_c0 = {k: v.copy() for k, v in long_c0.items()}
    quick_c0["M"][:] = 0          # opcode 0 everywhere: every machine is fixed at t = 0
    eng = H.get_engine(p, dev)
    refs = {}
    for name, c0 in (("long", long_c0), ("quick", quick_c0)):
        b = DeviceBatch.from_arrays(c0, p, dev)
        r = DeviceBatch.empty(b.d, p, dev, fresh=False)
        eng.run(b, 1024, 32, out=r, fresh=True)
        refs[name] = (b, r)
    src = DeviceBatch.from_arrays(long_c0, p, dev)
    dst = DeviceBatch.empty(src.d, p, dev, fresh=False)
    cap = torch.cuda.Stream(dev)
    cap.wait_stream(torch.cuda.current_stream(dev))
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=cap):
        eng.run(src, 1024, 32, out=dst, fresh=True, stream=cap)
    for name in ("quick", "long", "quick", "long"):
        b, r = refs[name]
        for k in ("iw", "ac", "M", "u", "y"):
            getattr(src, k).copy_(getattr(b, k))
        for k in ("iw", "M", "steps", "status"):
            getattr(dst, k).zero_()
        g.replay()
        torch.cuda.synchronize()
        for k in ("iw", "ac", "M", "u", "y", "status", "steps", "tau_h"):
            assert torch.equal(getattr(dst, k), getattr(r, k)), (name, k)


_LONG_BUDGET = r"""
import sys, numpy as np
sys.path.insert(0, sys.argv[1])
from oracle import oracle
from paper_2604_12902_b200 import hypervisor as H
from paper_2604_12902_b200.machine import MachineParams
from paper_2604_12902_b200.workload import random_configs
p = MachineParams(w=16, n=16, ell=3, s=3, mu=1)
c0 = random_configs(4096, p, np.random.default_rng(5))
# a third of the machines loop forever: LOD 1 ; BNZ 0 (i cycles 0 -> 2 -> 0)
loop = np.zeros(16, np.uint16); loop[:4] = (1, 1, 5, 0)
c0["M"][::3] = loop; c0["iw"][::3] = 0
tau = 20000
want = oracle.worker_arrays(c0, 16, 16, 3, 3, tau)
for epoch in (1, 50):
    res = H.run_arrays(c0, p, H.BatchConfig(tau_max=tau, epoch=epoch))
    for k in ("iw", "ac", "M", "u", "y", "status", "steps", "tau_h"):
        got = np.asarray(getattr(res.slots, k))
        if k in ("iw", "ac", "M", "u", "y"):
            got = got.astype(np.uint64)
        assert np.array_equal(got, want[k]), (epoch, k)
print("ok")
"""


def test_long_budget_polling_path(pkg, tmp_path):
    """Budgets beyond what the pre-planned launches cover: the host polls the
    device schedule for more epochs.  RASP_KMAX shortens the longest epoch so
    tau = 20000 needs ~80 of them (the planned launches cover 24)."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    script = tmp_path / "long_budget.py"
    script.write_text(_LONG_BUDGET)
    env = dict(os.environ, RASP_KMAX="256")
    out = subprocess.run([sys.executable, str(script), root], env=env, capture_output=True, text=True,
                         timeout=300)
    assert out.returncode == 0 and out.stdout.strip().endswith("ok"), out.stderr[-2000:]


@pytest.mark.parametrize("shape", [(32, 2048, 4, 2), (16, 4096, 4, 2), (16, 3000, 3, 3), (64, 1200, 2, 2)])
def test_huge_memory_hbm_tiles(pkg, shape):
    """n so large that a warp's tile exceeds shared memory: the kernel keeps
    the tiles in HBM (the generic path, gated steps)."""
    P, H = pkg
    from oracle import oracle
    from paper_2604_12902_b200.workload import random_configs
    w, n, ell, s = shape
    p = P.MachineParams(w=w, n=n, ell=ell, s=s, mu=1)
    c0 = random_configs(1024, p, np.random.default_rng(n))
    # a few long runners: a LOD/BNZ loop at the start of memory
    c0["M"][::7, :4] = np.array([1, 1, 5, 0], dtype=c0["M"].dtype)
    c0["iw"][::7] = 0
    for tau in (0, 300):
        want = oracle.worker_arrays(c0, w, n, ell, s, tau)
        res = H.run_arrays(c0, p, H.BatchConfig(tau_max=tau, epoch=16, memory_budget_words=1 << 40))
        for k in RESULTS:
            got = np.asarray(getattr(res.slots, k))
            if k in FIELDS:
                got = got.astype(np.uint64)
            np.testing.assert_array_equal(got, want[k], err_msg=f"{shape} tau={tau} {k}")
        # the fused histogram on HBM tiles (its block copy is the only shared memory there)
        import torch
        from paper_2604_12902_b200.engine import DeviceBatch
        from paper_2604_12902_b200.sharding import histogram_np
        src = DeviceBatch.from_arrays(c0, p)
        h = torch.empty(102, dtype=torch.int64, device=src.M.device)
        H.get_engine(p).run(src, tau, 16, fresh=True, hist=h)
        np.testing.assert_array_equal(h.cpu().numpy(), histogram_np(want["status"], want["tau_h"]))


def test_throughput_bench_rows(pkg):
    """hv:387-408 row format, on the golden busy-beaver programs."""
    P, H = pkg
    (g,) = load_family("bb")
    p = _params(P, g)
    configs = [P.Config(int(g.c0["iw"][k]), int(g.c0["ac"][k]), tuple(int(v) for v in g.c0["M"][k]),
                        tuple(int(v) for v in g.c0["u"][k]), tuple(int(v) for v in g.c0["y"][k]))
               for k in range(g.d)]
    wl = H.Workload(configs=configs, asts=None, aborted=[])
    rows = H.throughput_bench(wl, 10 ** 5, [1, 4], p)
    assert [r["workers"] for r in rows] == [1, 4] and all(r["vms"] == 3 for r in rows)
    assert rows[0]["speedup"] == 1.0 and all(r["wall_time"] > 0 for r in rows)
