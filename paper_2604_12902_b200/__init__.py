"""raspvisor-b200: B200-native batch engine for word-RASP machines.

The host surface mirrors the reference package `raspvisor` on its hot path
(machine value types + the batch operator of hypervisor.py); the transition
map runs in hand-written sm_100a CUDA (csrc/) behind a C ABI
(include/raspvisor_b200.h).  See DESIGN.md.
"""

from .errors import CapacityError, NativeError, RaspError
from .machine import (Config, MachineParams, Opcode, Program, init_batch, init_config,
                      natural_dtype, validate_config)

__all__ = [
    "RaspError", "CapacityError", "NativeError",
    "Config", "MachineParams", "Opcode", "Program", "init_config", "init_batch",
    "validate_config", "natural_dtype",
    "BatchConfig", "BatchResult", "SlotView", "VmSlot", "VmStatus", "run_batch",
    "run_arrays", "run_device", "collect_histogram", "HISTOGRAM_KEYS",
    "DeviceBatch", "Engine", "synthetic_c0",
]


def __getattr__(name):
    # torch-dependent pieces load lazily so `import paper_2604_12902_b200` stays cheap
    if name in ("BatchConfig", "BatchResult", "SlotView", "VmSlot", "VmStatus", "run_batch",
                "run_arrays", "run_device", "collect_histogram", "HISTOGRAM_KEYS"):
        from . import hypervisor
        return getattr(hypervisor, name)
    if name in ("DeviceBatch", "Engine"):
        from . import engine
        return getattr(engine, name)
    if name == "synthetic_c0":
        from .workload import synthetic_c0
        return synthetic_c0
    raise AttributeError(name)
