"""CPU parity oracle for the word-RASP batch transition map.

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and the
cpu_baseline / --impl reference legs of bench.py, always as the checker or the
baseline, never as the thing measured or shipped.  The product package
(paper_2604_12902_b200) must not import this.
"""

from .oracle import (  # noqa: F401
    build, load, oracle_run, step_reference, run_to_fixpoint, worker_arrays,
)
