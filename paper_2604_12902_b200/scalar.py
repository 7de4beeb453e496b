"""Scalar debug path through the batch engine.

``step`` and ``run_to_fixpoint`` have the signatures of raspvisor/machine.py
(step_reference, m:169-211; run_to_fixpoint, m:336-357) but execute on the
GPU as a batch of one machine -- the same kernel the batch path uses, so a
`run --trace` style session (cli.py:106-127) exercises production code.
"""

from __future__ import annotations

from typing import NamedTuple

from .hypervisor import BatchConfig, VmStatus, run_batch
from .machine import Config, MachineParams


class StepOutcome(NamedTuple):
    next: Config
    fixed_point: bool


def step(c: Config, p: MachineParams, device=None) -> StepOutcome:
    """One Φ step of c (fixed_point iff the successor equals c)."""
    slot = run_batch([c], p, BatchConfig(tau_max=1), device=device).slots[0]
    fixed = slot.status is VmStatus.HALTED and slot.tau_h == 0
    return StepOutcome(slot.config, fixed)


def run_to_fixpoint(c0: Config, tau_max: int, p: MachineParams, trace=None, device=None):
    """(final_config, tau_h) with tau_h None if no fixed point within tau_max;
    trace(t, config) is called before every fixedness test, like m:336-357."""
    if tau_max < 0:
        raise ValueError(f"tau_max must be >= 0, got {tau_max}")
    if trace is None:
        slot = run_batch([c0], p, BatchConfig(tau_max=tau_max), device=device).slots[0]
        return slot.config, (slot.tau_h if slot.status is VmStatus.HALTED else None)
    c = c0
    for t in range(tau_max + 1):
        trace(t, c)
        nxt, fixed = step(c, p, device)
        if fixed:
            return c, t
        if t == tau_max:
            break
        c = nxt
    return c, None
