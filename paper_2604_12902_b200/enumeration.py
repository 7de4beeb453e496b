"""Exhaustive enumeration of short programs x all inputs (BASELINE config 4).

SURVEY.md §8d (C4) freezes the domain: m = 4 instruction pairs, opcode in
{0..7} (3 bits), operand in [0, 16) (4 bits), n = 16, w = 8, ell = s = 1,
tau_max = 64 -- 2^28 programs x 256 inputs = 2^36 machines.  Program rank r
encodes pair k in bits [7k, 7k+7) (opcode = low 3 bits, operand = high 4).
Machines are decoded on the device from (r, x) -- no c0 ever crosses PCIe --
run with the batch engine's step code, and each program's 256 runs are
reduced on-chip into one 64-bit record (see include/raspvisor_b200.h,
rasp_enumerate): bit 63 = all inputs halted, bits 0..62 = an order-free
fingerprint of (x, halted, y, tau_h) over the inputs.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _native
from .errors import CapacityError


@dataclass(frozen=True)
class EnumDomain:
    m: int = 4
    opcode_bits: int = 3
    operand_bits: int = 4
    w: int = 8
    n: int = 16
    tau_max: int = 64

    @property
    def programs(self) -> int:
        return 1 << (self.m * (self.opcode_bits + self.operand_bits))

    @property
    def inputs(self) -> int:
        return 1 << self.w

    def c_params(self) -> _native.RaspEnumParams:
        return _native.RaspEnumParams(self.m, self.opcode_bits, self.operand_bits, self.w,
                                      self.n, self.tau_max)

    def program_words(self, rank: int) -> tuple:
        """The program of rank r as machine words (2m words)."""
        pw = self.opcode_bits + self.operand_bits
        words = []
        for k in range(self.m):
            pair = (rank >> (k * pw)) & ((1 << pw) - 1)
            words += [pair & ((1 << self.opcode_bits) - 1), pair >> self.opcode_bits]
        return tuple(words)


C4 = EnumDomain()


def enumerate_device(dom: EnumDomain, first: int, count: int, records: torch.Tensor,
                     steps_total: torch.Tensor, stream=None) -> None:
    """Enqueue rasp_enumerate for ranks [first, first+count) into device
    tensors records (uint64[count]) and steps_total (uint64[1], accumulated)."""
    if 2 * dom.m > dom.n:
        raise CapacityError(f"program needs {2 * dom.m} memory words but n = {dom.n}")
    lib = _native.load()
    s = stream if stream is not None else torch.cuda.current_stream(records.device)
    p = dom.c_params()
    with torch.cuda.device(records.device):
        rc = lib.rasp_enumerate(ctypes.byref(p), first, count, records.data_ptr(),
                                steps_total.data_ptr(), s.cuda_stream)
    _native.check(rc, "rasp_enumerate")


def enumerate_programs(dom: EnumDomain = C4, first: int = 0, count: int | None = None,
                       device=None) -> tuple:
    """Records for program ranks [first, first+count) and the applied
    machine-steps, as host values."""
    count = dom.programs - first if count is None else count
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    rec = torch.empty(count, dtype=torch.uint64, device=dev)
    st = torch.zeros(1, dtype=torch.uint64, device=dev)
    enumerate_device(dom, first, count, rec, st)
    return rec.cpu().numpy(), int(st.cpu().numpy()[0])


def summarize(records: np.ndarray) -> dict:
    """Domain-level summary: programs halting on every input, and a digest."""
    allh = (records >> np.uint64(63)).astype(bool)
    return {"programs": int(records.size), "all_halting": int(allh.sum()),
            "digest": int(np.bitwise_xor.reduce(records)) if records.size else 0}
