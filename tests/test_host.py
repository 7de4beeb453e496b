"""Host-side logic that needs no GPU: value types, validation, c0 packing,
histograms and the slot view (mirrors tests/test_machine.py:21-79 and
tests/test_hypervisor.py:107-171 of the reference)."""

import json
import os

import numpy as np
import pytest

from golden_io import FIELDS, load_family
from paper_2604_12902_b200 import (CapacityError, Config, MachineParams, Opcode, Program,
                                   init_batch, init_config, natural_dtype, validate_config)
from paper_2604_12902_b200 import machine as mach
from paper_2604_12902_b200.workload import synthetic_c0


def test_params_validation():
    MachineParams(w=1, n=2, ell=1, s=1, mu=1)
    for kw in (dict(w=0, n=4), dict(w=65, n=4), dict(w=8, n=1), dict(w=1, n=4, ell=2)):
        args = dict(ell=1, s=1, mu=1)
        args.update(kw)
        with pytest.raises(ValueError):
            MachineParams(**args)


def test_params_immutable_hashable_json():
    p = MachineParams(w=8, n=16, ell=4, s=2, mu=3)
    with pytest.raises(AttributeError):
        p.w = 16
    assert p == MachineParams(w=8, n=16, ell=4, s=2, mu=3)
    assert len({p, MachineParams(w=8, n=16, ell=4, s=2, mu=3)}) == 1
    assert MachineParams.from_json(json.loads(json.dumps(p.to_json()))) == p
    assert p.words_per_machine == 16 + 4 + 2 + 4


def test_natural_dtype():
    assert [natural_dtype(w).itemsize for w in (1, 8, 9, 16, 17, 32, 33, 64)] == \
        [1, 1, 2, 2, 4, 4, 8, 8]


def test_init_config_and_errors():
    p = MachineParams(w=8, n=4, ell=2, s=1, mu=1)
    assert init_config(Program((1, 7)), [9], p) == Config(0, 0, (1, 7, 0, 0), (0, 9, 0), (0, 0))
    with pytest.raises(CapacityError):
        init_config(Program((1, 7, 0, 0, 0, 0)), [], p)
    with pytest.raises(CapacityError):
        init_config(Program((1, 7)), [1, 2, 3], p)
    with pytest.raises(ValueError):
        init_config(Program((1, 256)), [], p)
    with pytest.raises(ValueError):
        init_config(Program((1, 7)), [256], p)
    with pytest.raises(ValueError):
        Program((1, 2, 3))


def test_validate_config():
    p = MachineParams(w=8, n=4, ell=2, s=1, mu=1)
    c = init_config(Program((1, 7)), [9], p)
    validate_config(c, p, deep=True)
    for bad in (c._replace(u=(3, 9, 0)), c._replace(M=(1, 7, 0))):
        with pytest.raises(ValueError):
            validate_config(bad, p)
    with pytest.raises(ValueError):
        validate_config(c._replace(M=(1, 700, 0, 0)), p, deep=True)


def test_init_batch_matches_init_config():
    p = MachineParams(w=16, n=12, ell=3, s=2, mu=1)
    progs = [Program((1, 5, 4, 6)), Program((0, 0)), Program((6, 3, 7, 3, 0, 0))]
    xs = [[1, 2], [], [65535, 0, 7]]
    b = init_batch(progs, xs, p)
    for k, (pr, x) in enumerate(zip(progs, xs)):
        c = init_config(pr, x, p)
        assert b["M"][k].tolist() == list(c.M)
        assert b["u"][k].tolist() == list(c.u)
        assert b["y"][k].tolist() == list(c.y)
    assert b["M"].dtype == np.uint16
    with pytest.raises(CapacityError):
        init_batch([Program((1, 1) * 7)], [[]], p)
    with pytest.raises(ValueError):
        init_batch([Program((1, 70000))], [[]], p)


def test_serialization_roundtrips():
    prog = Program((1, 500, 4, 6))
    for w in (16, 32, 64):
        assert mach.program_from_bytes(mach.program_to_bytes(prog, w), w) == prog
    assert mach.program_from_json(mach.program_to_json(prog, 16)) == (prog, 16)
    c = Config(1, 2, (3, 4), (0, 5), (0, 6))
    assert mach.config_from_json(mach.config_to_json(c)) == c
    assert [op.value for op in Opcode] == list(range(8))


def test_synthetic_generator_frozen():
    """Generator G: deterministic; opcodes 1..7 in even cells,
    operands < n (BNZ operands even) in odd cells; i = a = u0 = y = 0."""
    p = MachineParams(w=16, n=64, ell=8, s=8, mu=1)
    a = synthetic_c0(1000, p, seed=0)
    b = synthetic_c0(1000, p, seed=0)
    for k in FIELDS:
        assert np.array_equal(a[k], b[k])
        assert a[k].dtype == np.uint16
    ops, opr = a["M"][:, 0::2], a["M"][:, 1::2]
    assert ops.min() >= 1 and ops.max() <= 7 and opr.max() < 64
    assert (opr[ops == 5] % 2 == 0).all()
    assert not a["iw"].any() and not a["ac"].any() and not a["y"].any()
    assert not a["u"][:, 0].any()
    # the golden C1/C2/C5 samples were generated with this generator
    for g in load_family("gen"):
        pp = MachineParams(w=g.w, n=g.n, ell=g.ell, s=g.s, mu=1)
        c0 = synthetic_c0(g.d, pp, seed=0)
        for k in FIELDS:
            assert np.array_equal(c0[k].astype(np.uint64), g.c0[k]), (g, k)


def test_histogram_keys_and_paths_agree():
    from paper_2604_12902_b200.hypervisor import (HISTOGRAM_KEYS, SlotView, VmStatus,
                                                  collect_histogram)
    assert len(HISTOGRAM_KEYS) == 102 and HISTOGRAM_KEYS[100:] == ("100+", "nonhalt")
    for g in load_family("corpus") + load_family("gen"):
        p = MachineParams(w=g.w, n=g.n, ell=g.ell, s=g.s, mu=1)
        sv = SlotView(*(g.out[k] for k in ("iw", "ac", "M", "u", "y", "status", "steps", "tau_h")),
                      params=p)
        fast = collect_histogram(sv)
        generic = collect_histogram(list(sv)) if g.d <= 600 else fast
        assert fast == generic
        assert [fast[k] for k in HISTOGRAM_KEYS] == list(g.hist)
        assert sum(fast.values()) == g.d
        halted = int((g.out["status"] == VmStatus.HALTED).sum())
        assert fast["nonhalt"] == g.d - halted


def test_slot_view_sequence_protocol():
    from paper_2604_12902_b200.hypervisor import SlotView, VmStatus
    g = load_family("kat")[3]
    p = MachineParams(w=g.w, n=g.n, ell=g.ell, s=g.s, mu=1)
    sv = SlotView(*(g.out[k] for k in ("iw", "ac", "M", "u", "y", "status", "steps", "tau_h")),
                  params=p)
    assert len(sv) == g.d
    assert sv[-1] == sv[g.d - 1]
    assert len(sv[0:3]) == 3
    with pytest.raises(IndexError):
        sv[g.d]
    s0 = sv[11]   # HLT config: halted at 0
    assert s0.status is VmStatus.HALTED and s0.tau_h == 0


def test_batch_config_validation():
    from paper_2604_12902_b200.hypervisor import BatchConfig
    for kw in (dict(tau_max=-1), dict(tau_max=1, epoch=0), dict(tau_max=1, workers=-1)):
        with pytest.raises(ValueError):
            BatchConfig(**kw)


def test_memory_budget_enforced_before_device():
    """CapacityError is raised on the host, before any device work."""
    from paper_2604_12902_b200.hypervisor import BatchConfig, run_batch
    p = MachineParams(w=8, n=8, ell=2, s=2, mu=1)
    c = init_config(Program((0, 0)), [], p)
    with pytest.raises(CapacityError, match="budget"):
        run_batch([c] * 10, p, BatchConfig(tau_max=1, memory_budget_words=10))


def test_product_never_imports_oracle():
    """The product package must not route through the CPU oracle."""
    import pathlib
    pkg = pathlib.Path(__file__).resolve().parent.parent / "paper_2604_12902_b200"
    for f in pkg.rglob("*.py"):
        text = f.read_text()
        assert "import oracle" not in text and "from oracle" not in text, f


def test_dropin_routes_the_reference_run_batch_without_cpu_fallback():
    """dropin.install makes the reference's run_batch (baseline/_ref) call the
    C-ABI engine; without a GPU that call fails loudly (no CPU fallback)."""
    import importlib
    import sys

    ref = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "raspvisor")):
        pytest.skip("the reference is not staged in baseline/_ref")
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/raspvisor_numba_cache")
    sys.path.insert(0, ref)
    try:
        RH = importlib.import_module("raspvisor.hypervisor")
        RM = importlib.import_module("raspvisor.machine")
        from paper_2604_12902_b200 import dropin
        from paper_2604_12902_b200.errors import NativeError
        original = RH._worker
        dropin.install(RH)
        try:
            assert RH._worker is dropin.worker
            p = RM.MachineParams(w=8, n=8, ell=2, s=2, mu=1)
            c = RM.init_config(RM.Program((1, 5, 4, 6)), [], p)
            import torch
            if torch.cuda.is_available():
                pytest.skip("GPU present: covered by tests/test_dropin_reference.py")
            with pytest.raises((NativeError, RuntimeError, AssertionError)):
                RH.run_batch([c], p, RH.BatchConfig(tau_max=8, workers=1))
        finally:
            RH._worker = original
    finally:
        sys.path.remove(ref)


def test_build_workload_from_programs_records_aborted_draws():
    """hv:362-384: programs too large for memory (or inputs beyond ell) are
    recorded with their index and reason, the rest become c0."""
    from paper_2604_12902_b200.hypervisor import Workload, build_workload_from_programs
    p = MachineParams(w=8, n=8, ell=2, s=2, mu=1)
    progs = [Program((1, 5, 4, 6)), Program((0,) * 10), Program((7, 2)), Program((1, 1))]
    inputs = [[], [], [3, 4, 5], [9]]
    wl = build_workload_from_programs(progs, inputs, p)
    assert isinstance(wl, Workload) and wl.asts is None
    assert [k for k, _ in wl.aborted] == [1, 2]
    assert "memory words" in wl.aborted[0][1] and "ell" in wl.aborted[1][1]
    assert wl.configs == [init_config(progs[0], [], p), init_config(progs[3], [9], p)]
