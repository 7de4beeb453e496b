"""The indicator form of the step (machine.py:214-286, the paper's Φ_w =
⊕ η_ψ Φ_ψ): the nine case indicators partition every configuration and the
indicator-weighted blend equals the case-by-case step -- the identity the
GPU kernels' predicated-select dispatch relies on.  Pinned on the reference's
own corpus (golden family `corpus`) and on random mid-run configurations."""

import numpy as np
import pytest

from golden_io import load_family
from oracle import oracle


def _configs_of(g):
    for k in range(g.d):
        yield (int(g.c0["iw"][k]), int(g.c0["ac"][k]), tuple(int(v) for v in g.c0["M"][k]),
               tuple(int(v) for v in g.c0["u"][k]), tuple(int(v) for v in g.c0["y"][k]))


@pytest.mark.parametrize("g", load_family("corpus") + load_family("edge"), ids=repr)
def test_indicator_step_equals_reference_step(g):
    for c in _configs_of(g):
        e = oracle.indicator_partition(c, g.w, g.n, g.ell, g.s)
        assert sum(e) == 1 and all(v in (0, 1) for v in e)
        assert oracle.step_indicator(c, g.w, g.n, g.ell, g.s) == oracle.step_reference(c, g.w, g.n, g.ell, g.s)


@pytest.mark.parametrize("shape", [(1, 6, 1, 1), (8, 8, 2, 2), (16, 64, 8, 8), (32, 250, 10, 2), (64, 12, 3, 3)])
def test_indicator_step_random_configs(shape):
    from paper_2604_12902_b200.machine import MachineParams
    from paper_2604_12902_b200.workload import random_configs
    w, n, ell, s = shape
    p = MachineParams(w=w, n=n, ell=ell, s=s)
    a = random_configs(400, p, np.random.default_rng(w + n), dtype=np.uint64)
    seen = np.zeros(len(oracle.INDICATOR_CASES), int)
    for k in range(400):
        c = (int(a["iw"][k]), int(a["ac"][k]), tuple(int(v) for v in a["M"][k]),
             tuple(int(v) for v in a["u"][k]), tuple(int(v) for v in a["y"][k]))
        e = oracle.indicator_partition(c, w, n, ell, s)
        assert sum(e) == 1
        seen += np.array(e)
        assert oracle.step_indicator(c, w, n, ell, s) == oracle.step_reference(c, w, n, ell, s)
    if w >= 3:   # opcodes up to 7 exist only for w >= 3
        assert (seen > 0).sum() >= 7
