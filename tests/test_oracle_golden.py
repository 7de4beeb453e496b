"""Pin the CPU oracle to the reference: every golden group produced by the
reference's run_batch (tests/golden/make_golden.py) must be reproduced
byte-for-byte by the C restatement of _worker (oracle/rasp_oracle.c) at
several (workers, epoch) schedules, and by the pure-Python scalar loop on
the small families."""

import numpy as np
import pytest

from golden_io import RESULTS, load_all, load_family, load_raw
from oracle import oracle

ALL = load_all()


@pytest.mark.parametrize("g", ALL, ids=repr)
@pytest.mark.parametrize("workers,epoch", [(1, 64), (3, 5)])
def test_c_oracle_matches_reference(g, workers, epoch):
    got = oracle.worker_arrays(g.c0, g.w, g.n, g.ell, g.s, g.tau_max,
                               epoch=epoch, workers=workers)
    for k in RESULTS:
        np.testing.assert_array_equal(got[k], g.out[k], err_msg=f"{g} field {k}")


SMALL = load_family("kat") + load_family("edge") + load_family("bb") + \
    [g for g in load_family("hyp") if g.tau_max <= 50]


@pytest.mark.parametrize("g", SMALL, ids=repr)
def test_scalar_oracle_matches_reference(g):
    for k in range(g.d):
        c0 = (int(g.c0["iw"][k]), int(g.c0["ac"][k]),
              tuple(int(v) for v in g.c0["M"][k]),
              tuple(int(v) for v in g.c0["u"][k]),
              tuple(int(v) for v in g.c0["y"][k]))
        cf, tau = oracle.run_to_fixpoint(c0, g.tau_max, g.w, g.n, g.ell, g.s)
        assert cf[0] == g.out["iw"][k] and cf[1] == g.out["ac"][k]
        assert cf[2] == tuple(int(v) for v in g.out["M"][k])
        assert cf[3] == tuple(int(v) for v in g.out["u"][k])
        assert cf[4] == tuple(int(v) for v in g.out["y"][k])
        if tau is None:
            assert g.out["status"][k] == 2 and g.out["tau_h"][k] == -1
            assert g.out["steps"][k] == g.tau_max
        else:
            assert g.out["status"][k] == 1 and g.out["tau_h"][k] == tau


def test_step_kats():
    """machine.py step_reference on the single-step examples."""
    z = load_raw("kat")
    g = load_family("kat")[0]
    nxt, fixed = z["step_next"], z["step_fixed"]
    for k in range(g.d):
        c = (int(g.c0["iw"][k]), int(g.c0["ac"][k]),
             tuple(int(v) for v in g.c0["M"][k]),
             tuple(int(v) for v in g.c0["u"][k]),
             tuple(int(v) for v in g.c0["y"][k]))
        out, fx = oracle.step_reference(c, g.w, g.n, g.ell, g.s)
        flat = np.array([out[0], out[1], *out[2], *out[3], *out[4]], np.uint64)
        np.testing.assert_array_equal(flat, nxt[k])
        assert fx == bool(fixed[k])


def test_bb_fixture_halting_times():
    (g,) = load_family("bb")
    assert list(g.out["tau_h"]) == [1727, 1409, 1387]
    assert all(g.out["y"][:, 0] == 1) and all(g.out["y"][:, 1] == 0)


def test_golden_histograms_consistent():
    """The stored 102-bucket histograms agree with the stored status/tau_h."""
    for g in ALL:
        th = g.out["tau_h"][g.out["status"] == 1]
        want = np.zeros(102, np.int64)
        np.add.at(want, np.minimum(th, 100), 1)
        want[101] = int((g.out["status"] == 2).sum())
        np.testing.assert_array_equal(g.hist, want, err_msg=repr(g))
