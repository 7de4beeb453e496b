"""The reference's own batch operator running on the B200 engine.

``paper_2604_12902_b200.dropin.install`` swaps the numba kernel that
``raspvisor.hypervisor.run_batch`` calls (hypervisor.py:305-314) for the C-ABI
engine; the unmodified reference package (pip-installed into baseline/_ref,
see DESIGN.md) then runs its own argument checks, packing, histogram and
SlotView on top of it.  Checked against the golden fixtures the reference
produced with its numba kernel, field by field, and its Counter histogram.
"""

import os
import sys

import numpy as np
import pytest

from golden_io import RESULTS, load_all, load_family

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")


@pytest.fixture(scope="module")
def reference():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device")
    if not os.path.isdir(os.path.join(REF, "raspvisor")):
        pytest.skip("the reference is not staged in baseline/_ref (DESIGN.md, 'Reference install')")
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/raspvisor_numba_cache")
    sys.path.insert(0, REF)
    from raspvisor import hypervisor as RH
    from raspvisor import machine as RM
    from paper_2604_12902_b200 import dropin
    original = RH._worker
    dropin.install(RH)
    yield RH, RM
    RH._worker = original


def _configs(RM, g):
    return [RM.Config(int(g.c0["iw"][k]), int(g.c0["ac"][k]), tuple(int(v) for v in g.c0["M"][k]),
                      tuple(int(v) for v in g.c0["u"][k]), tuple(int(v) for v in g.c0["y"][k]))
            for k in range(g.d)]


GROUPS = [g for g in load_all(("kat", "edge", "corpus", "hyp", "bb", "paper")) if g.d <= 4096] + \
    load_family("gen")[:1]


@pytest.mark.parametrize("g", GROUPS, ids=repr)
def test_reference_run_batch_on_b200(reference, g):
    RH, RM = reference
    from paper_2604_12902_b200 import dropin
    assert RH._worker is dropin.worker
    p = RM.MachineParams(w=g.w, n=g.n, ell=g.ell, s=g.s, mu=1)
    res = RH.run_batch(_configs(RM, g), p, RH.BatchConfig(tau_max=g.tau_max, epoch=16, workers=1,
                                                           memory_budget_words=1 << 40))
    for k in RESULTS:
        np.testing.assert_array_equal(np.asarray(getattr(res.slots, k)), g.out[k], err_msg=f"{g} {k}")
    want = {}
    for st, th in zip(g.out["status"], g.out["tau_h"]):
        if st == 1:
            want[int(th)] = want.get(int(th), 0) + 1
    assert dict(res.histogram) == want
    hist = RH.collect_histogram(res.slots)
    assert [hist[k] for k in RH.HISTOGRAM_KEYS] == list(g.hist)


def test_reference_errors_unchanged(reference):
    """The reference's own validation still fires before the kernel."""
    RH, RM = reference
    p = RM.MachineParams(w=8, n=8, ell=2, s=2, mu=1)
    good = RM.init_config(RM.Program((0, 0)), [], p)
    bad = RM.Config(i=0, a=0, M=(0, 300, 0, 0, 0, 0, 0, 0), u=good.u, y=good.y)
    with pytest.raises(ValueError):
        RH.run_batch([good, bad], p, RH.BatchConfig(tau_max=1, workers=1))
    from raspvisor.errors import CapacityError
    with pytest.raises(CapacityError):
        RH.run_batch([good] * 10, p, RH.BatchConfig(tau_max=1, workers=1, memory_budget_words=10))
