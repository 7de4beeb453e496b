"""Exhaustive enumeration (BASELINE config 4): the oracle's record
definition is checked against the pinned scalar oracle on CPU; the GPU
kernel against the oracle on the full reduced domain (m=3, n=8, 3-bit
operands: 2^26 machines) and a seeded sample of the full C4 domain."""

import numpy as np
import pytest

from oracle import oracle
from paper_2604_12902_b200.enumeration import C4, EnumDomain

REDUCED = EnumDomain(m=3, opcode_bits=3, operand_bits=3, w=8, n=8, tau_max=64)
MASK63 = (1 << 63) - 1


def _fmix32(h):
    h ^= h >> 16
    h = (h * 0x85EBCA6B) & 0xFFFFFFFF
    h ^= h >> 13
    h = (h * 0xC2B2AE35) & 0xFFFFFFFF
    return h ^ (h >> 16)


def _record_scalar(dom, rank):
    words = dom.program_words(rank)
    n = dom.n
    total, allh, steps = 0, True, 0
    for x in range(1 << dom.w):
        M = tuple(words) + (0,) * (n - len(words))
        c0 = (0, 0, M, (0, x), (0, 0))
        cf, tau = oracle.run_to_fixpoint(c0, dom.tau_max, dom.w, n, 1, 1)
        halted = tau is not None
        allh &= halted
        y0, y1 = cf[4]
        key = x | (int(halted) << 8) | (y0 << 9) | ((y1 if y0 else 0) << 10) | \
            ((tau if halted else 0) << 18)
        assert key < 1 << 32
        total = (total + _fmix32(key)) & 0xFFFFFFFFFFFFFFFF
        steps += tau if halted else dom.tau_max
    return (int(allh) << 63) | (total & MASK63), steps


@pytest.mark.parametrize("dom,ranks", [(C4, [0, 1, 77, 12345, (1 << 28) - 1, 0x5A5A5A5]),
                                       (REDUCED, [0, 3, 999, (1 << 18) - 1])])
def test_oracle_enumerator_matches_scalar(dom, ranks):
    for r in ranks:
        rec, steps = oracle.enumerate_records(dom.m, dom.opcode_bits, dom.operand_bits, dom.w,
                                              dom.n, dom.tau_max, r, 1)
        want, want_steps = _record_scalar(dom, r)
        assert int(rec[0]) == want, r
        assert steps == want_steps


def test_domain_sizes():
    assert C4.programs == 1 << 28 and C4.inputs == 256
    assert REDUCED.programs == 1 << 18
    assert C4.program_words(0b0000001_1111111) == (7, 15, 1, 0, 0, 0, 0, 0)


@pytest.mark.gpu
def test_gpu_enumeration_full_reduced_domain():
    import os
    from paper_2604_12902_b200.enumeration import enumerate_programs
    rec, steps = enumerate_programs(REDUCED)
    want, want_steps = oracle.enumerate_records(REDUCED.m, REDUCED.opcode_bits,
                                                REDUCED.operand_bits, REDUCED.w, REDUCED.n,
                                                REDUCED.tau_max, 0, REDUCED.programs,
                                                threads=len(os.sched_getaffinity(0)))
    np.testing.assert_array_equal(rec, want)
    assert steps == want_steps


@pytest.mark.gpu
def test_gpu_enumeration_c4_sample():
    import os
    from paper_2604_12902_b200.enumeration import enumerate_programs
    rng = np.random.default_rng(2604)
    for first in [0, (1 << 28) - 4096] + [int(v) for v in rng.integers(0, (1 << 28) - 4096, 6)]:
        rec, steps = enumerate_programs(C4, first, 4096)
        want, want_steps = oracle.enumerate_records(C4.m, C4.opcode_bits, C4.operand_bits, C4.w,
                                                    C4.n, C4.tau_max, first, 4096,
                                                    threads=len(os.sched_getaffinity(0)))
        np.testing.assert_array_equal(rec, want, err_msg=f"block at {first}")
        assert steps == want_steps
