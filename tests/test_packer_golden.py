"""The host packer (machine.init_batch / init_config) against the c0 the
reference's own init_config built (m:289-309) for the bb, paper and paper100
programs (tests/golden/packer.npz, written by tests/golden/make_golden.py).
The device packer is checked against the same fixture in
tests/test_gpu_bench_scale.py."""

import os

import numpy as np
import pytest

from golden_io import FIELDS, GOLDEN, load_family


@pytest.fixture(scope="module")
def packer():
    return np.load(os.path.join(GOLDEN, "packer.npz"))


@pytest.mark.parametrize("family", ["bb", "paper", "paper100"])
def test_init_batch_matches_reference(packer, family):
    from paper_2604_12902_b200.machine import MachineParams, Program, init_batch, init_config
    p = MachineParams(w=32, n=250, ell=10, s=2, mu=10)
    got = init_batch(packer[f"{family}_prog"], packer[f"{family}_inp"], p)
    for k in FIELDS:
        np.testing.assert_array_equal(np.asarray(got[k]).astype(np.uint64), packer[f"{family}_c0_{k}"],
                                      err_msg=f"{family} {k}")
    # the scalar init_config on the exact (unpadded) words, a few rows
    for r in range(min(8, packer[f"{family}_prog"].shape[0])):
        L, X = int(packer[f"{family}_plen"][r]), int(packer[f"{family}_xlen"][r])
        c = init_config(Program(tuple(int(v) for v in packer[f"{family}_prog"][r, :L])),
                        [int(v) for v in packer[f"{family}_inp"][r, :X]], p)
        assert tuple(c.M) == tuple(int(v) for v in packer[f"{family}_c0_M"][r])
        assert tuple(c.u) == tuple(int(v) for v in packer[f"{family}_c0_u"][r])


@pytest.mark.parametrize("family", ["bb", "paper", "paper100"])
def test_packer_fixture_is_the_run_fixture(packer, family):
    """The packer fixture's c0 is exactly what the run fixtures start from."""
    (g,) = load_family(family)
    for k in FIELDS:
        np.testing.assert_array_equal(packer[f"{family}_c0_{k}"], g.c0[k], err_msg=f"{family} {k}")
