"""Batch operator: the reference's host surface, running on the B200 engine.

Same names, argument meaning and error behaviour as raspvisor/hypervisor.py
for the hot path: ``BatchConfig`` (hv:167-180), ``VmStatus`` (hv:66-69),
``VmSlot`` (hv:183-188), ``SlotView`` (hv:191-220), ``BatchResult``
(hv:223-227), ``run_batch`` (hv:265-323), ``HISTOGRAM_KEYS`` and
``collect_histogram`` (hv:326-352).  Results are a pure function of the
initial configurations and tau_max -- independent of ``epoch`` (and of
``workers``, which has no meaning on the GPU and is accepted for
compatibility) exactly as the reference is independent of (W, q).

Beyond the tuple interface, ``run_arrays`` takes SoA numpy/torch arrays
(no per-machine tuples; the reference's own packing at hv:280-284 is the
bottleneck at scale) and ``run_device`` runs a batch that is
already resident in HBM.
"""

from __future__ import annotations

from collections import Counter
from collections.abc import Sequence
from dataclasses import dataclass, field
from enum import IntEnum

import numpy as np
import torch

from .engine import ALL_FIELDS, WORD_FIELDS, DeviceBatch, Engine
from .errors import CapacityError
from .machine import Config, MachineParams, init_config, validate_config

__all__ = [
    "VmStatus", "BatchConfig", "VmSlot", "SlotView", "BatchResult", "run_batch",
    "run_arrays", "run_device", "run_programs", "collect_histogram", "HISTOGRAM_KEYS", "get_engine",
    "Workload", "build_workload_from_programs", "throughput_bench",
]

_RUNNING, _HALTED, _EXHAUSTED = 0, 1, 2


class VmStatus(IntEnum):
    RUNNING = _RUNNING
    HALTED = _HALTED
    BUDGET_EXHAUSTED = _EXHAUSTED


@dataclass(frozen=True)
class BatchConfig:
    tau_max: int
    epoch: int = 64                       # first on-device epoch length (the reference's q)
    workers: int = 0                      # accepted for compatibility; the GPU needs no workers
    memory_budget_words: int = 2 ** 28    # refuse batches larger than this (hv:172)

    def __post_init__(self):
        if self.tau_max < 0:
            raise ValueError(f"tau_max must be >= 0, got {self.tau_max}")
        if self.epoch < 1:
            raise ValueError(f"epoch must be >= 1, got {self.epoch}")
        if self.workers < 0:
            raise ValueError(f"workers must be >= 0, got {self.workers}")


@dataclass(frozen=True)
class VmSlot:
    config: Config
    status: VmStatus
    steps_taken: int
    tau_h: int | None


class SlotView(Sequence):
    """Array-backed sequence of VmSlots (hv:191-220).  The arrays iw, ac, M,
    u, y, status, steps, tau_h are exposed directly; indexing materialises
    one VmSlot."""

    def __init__(self, iw, ac, M, u, y, status, steps, tau_h, params):
        self.iw, self.ac, self.M, self.u, self.y = iw, ac, M, u, y
        self.status, self.steps, self.tau_h = status, steps, tau_h
        self.params = params

    def __len__(self):
        return int(self.iw.shape[0])

    def __getitem__(self, k):
        if isinstance(k, slice):
            return [self[j] for j in range(*k.indices(len(self)))]
        d = len(self)
        if k < 0:
            k += d
        if k < 0 or k >= d:
            raise IndexError(k)
        cfg = Config(int(self.iw[k]), int(self.ac[k]), tuple(int(v) for v in self.M[k]),
                     tuple(int(v) for v in self.u[k]), tuple(int(v) for v in self.y[k]))
        st = VmStatus(int(self.status[k]))
        return VmSlot(config=cfg, status=st, steps_taken=int(self.steps[k]),
                      tau_h=int(self.tau_h[k]) if st is VmStatus.HALTED else None)


@dataclass
class BatchResult:
    slots: SlotView
    histogram: Counter = field(default_factory=Counter)   # tau_h -> halted VMs
    wall_time: float = 0.0                                 # device seconds of the run


_ENGINES: dict = {}


def get_engine(params: MachineParams, device=None) -> Engine:
    dev = torch.device(device) if device is not None else None
    key = (params, str(dev))
    eng = _ENGINES.get(key)
    if eng is None:
        eng = _ENGINES[key] = Engine(params, dev)
    return eng


def _budget_check(d: int, params: MachineParams, batch: BatchConfig) -> None:
    need = d * params.words_per_machine
    if need > batch.memory_budget_words:
        raise CapacityError(
            f"batch needs {need} words of VM state, over the budget of "
            f"{batch.memory_budget_words} (raise memory_budget_words to allow)")


def _range_check(arrays: dict, params: MachineParams) -> None:
    """hv:285-290: every word must fit in w bits."""
    if params.w >= 64:
        return
    for name, key in (("i", "iw"), ("a", "ac"), ("M", "M"), ("u", "u"), ("y", "y")):
        a = arrays[key]
        if a.size and int(a.max()) > params.mask:
            raise ValueError(f"{name} holds a word over 2^w - 1 = {params.mask}")


def _histogram_counter(status: np.ndarray, tau_h: np.ndarray) -> Counter:
    hist = Counter()
    if status.size:
        vals, cnts = np.unique(tau_h[status == _HALTED], return_counts=True)
        hist.update({int(v): int(c) for v, c in zip(vals, cnts)})
    return hist


def run_device(batch: DeviceBatch, cfg: BatchConfig, out: DeviceBatch | None = None,
               fresh: bool = False, engine: Engine | None = None, stream=None) -> float:
    """Run a device-resident batch; returns the device time in seconds
    (CUDA events on the launching stream)."""
    eng = engine or get_engine(batch.params, batch.iw.device)
    s = stream if stream is not None else torch.cuda.current_stream(batch.iw.device)
    eng.warm(batch.word_bytes, fresh, stream=s)   # one-time setup off the clock
    eng.workspace(batch.d)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(s)
    eng.run(batch, cfg.tau_max, cfg.epoch, out=out, fresh=fresh, stream=s)
    e1.record(s)
    e1.synchronize()
    return e0.elapsed_time(e1) / 1e3


def run_arrays(arrays: dict, params: MachineParams, batch: BatchConfig, device=None,
               word_bytes: int | None = None, check: bool = True) -> BatchResult:
    """run_batch over SoA arrays: iw[d], ac[d], M[d,n], u[d,ell+1], y[d,s+1]
    (any unsigned integer dtype holding w bits; optional status/steps/tau_h
    as the _worker ABI takes them).  Result arrays come back in the input's
    word dtype (int8/int64 for status/steps/tau_h)."""
    iw = np.asarray(arrays["iw"])
    d = int(iw.shape[0])
    _budget_check(d, params, batch)
    host = {k: np.asarray(arrays[k]) for k in WORD_FIELDS}
    expect = {"M": (d, params.n), "u": (d, params.ell + 1), "y": (d, params.s + 1),
              "iw": (d,), "ac": (d,)}
    for k, shp in expect.items():
        if host[k].shape != shp:
            raise ValueError(f"{k} has shape {host[k].shape}, expected {shp}")
    if check and d:
        if int(host["u"][:, 0].max()) > params.ell:
            raise ValueError(f"read cursor u[0] outside [0, {params.ell}]")
        if int(host["y"][:, 0].max()) > params.s:
            raise ValueError(f"write count y[0] outside [0, {params.s}]")
        _range_check(host, params)
    out_dtype = host["iw"].dtype
    wb = word_bytes or max(params.dtype.itemsize, out_dtype.itemsize if out_dtype.kind == "u" else 0)
    fresh = not any(k in arrays for k in ("status", "steps", "tau_h"))
    if d == 0:
        empty = {k: np.zeros((0,) + host[k].shape[1:], out_dtype) for k in WORD_FIELDS}
        return BatchResult(SlotView(**empty, status=np.zeros(0, np.int8),
                                    steps=np.zeros(0, np.int64), tau_h=np.zeros(0, np.int64),
                                    params=params), Counter(), 0.0)
    dev_in = DeviceBatch.from_arrays({**host, **{k: arrays[k] for k in ("status", "steps", "tau_h")
                                                 if k in arrays}}, params, device, wb)
    wall = run_device(dev_in, batch, fresh=fresh)
    res = dev_in.to_numpy()
    for k in WORD_FIELDS:
        if res[k].dtype != out_dtype:
            res[k] = res[k].astype(out_dtype)
    hist = _histogram_counter(res["status"], res["tau_h"])
    slots = SlotView(res["iw"], res["ac"], res["M"], res["u"], res["y"], res["status"],
                     res["steps"], res["tau_h"], params)
    return BatchResult(slots=slots, histogram=hist, wall_time=wall)


def run_programs(programs, inputs, params: MachineParams, batch: BatchConfig, device=None,
                 chunks: int = 4) -> BatchResult:
    """build_workload -> run_batch in one call: c0(P, x) = init_config(P, x)
    (machine.py:289-309) for every row of programs [d, L] / inputs [d, k],
    assembled on the GPU from host buffers, run, and returned as a SlotView.
    Same errors as init_config / run_batch (CapacityError, ValueError)."""
    from .pipeline import HostPipeline
    P = np.asarray(programs)
    X = np.asarray(inputs)
    d = int(P.shape[0])
    X = X.reshape(d, -1) if X.size else np.zeros((d, 0), P.dtype)
    _budget_check(d, params, batch)
    if P.shape[1] > params.n:
        raise CapacityError(f"program needs {P.shape[1]} memory words but n = {params.n}")
    if X.shape[1] > params.ell:
        raise CapacityError(f"input vector has {X.shape[1]} words but ell = {params.ell}")
    if params.w < 64:
        for kind, arr in (("program", P), ("input", X)):
            if arr.size and int(arr.max()) > params.mask:
                raise ValueError(f"{kind} word {int(arr.max())} out of range for w = {params.w}")
    if d == 0:
        return run_arrays({"iw": np.zeros(0, params.dtype), "ac": np.zeros(0, params.dtype),
                           "M": np.zeros((0, params.n), params.dtype),
                           "u": np.zeros((0, params.ell + 1), params.dtype),
                           "y": np.zeros((0, params.s + 1), params.dtype)}, params, batch, device)
    pipe = HostPipeline(params, d, device, chunks=chunks)
    pinned = pipe.pinned_programs(P, X)
    wall = pipe.run_programs(pinned, batch.tau_max, batch.epoch)
    res = pipe.results()
    slots = SlotView(res["iw"], res["ac"], res["M"], res["u"], res["y"], res["status"],
                     res["steps"], res["tau_h"], params)
    return BatchResult(slots=slots, histogram=_histogram_counter(res["status"], res["tau_h"]),
                       wall_time=wall)


def run_batch(configs, params: MachineParams, batch: BatchConfig, device=None) -> BatchResult:
    """Run every configuration to a fixed point or tau_max steps (hv:265-323)."""
    d = len(configs)
    _budget_check(d, params, batch)
    for c in configs:
        validate_config(c, params)
    arrays = {
        "iw": np.fromiter((c.i for c in configs), np.uint64, count=d),
        "ac": np.fromiter((c.a for c in configs), np.uint64, count=d),
        "M": np.array([c.M for c in configs], np.uint64).reshape(d, params.n),
        "u": np.array([c.u for c in configs], np.uint64).reshape(d, params.ell + 1),
        "y": np.array([c.y for c in configs], np.uint64).reshape(d, params.s + 1),
    }
    _range_check(arrays, params)
    if d == 0:
        return run_arrays(arrays, params, batch, device, check=False)
    natural = {k: v.astype(params.dtype) for k, v in arrays.items()}
    res = run_arrays(natural, params, batch, device, check=False)
    sv = res.slots
    # expose the reference's uint64 arrays (hv:280-284) for drop-in consumers
    res.slots = SlotView(*(getattr(sv, k).astype(np.uint64) for k in WORD_FIELDS),
                         sv.status, sv.steps, sv.tau_h, params)
    return res


HISTOGRAM_KEYS = tuple(str(k) for k in range(100)) + ("100+", "nonhalt")


def collect_histogram(slots) -> dict:
    """Bucketed halting-time histogram (hv:329-352): "0".."99" exact tau_h,
    "100+" later halts, "nonhalt" budget-exhausted VMs.  Every key present.
    Accepts a SlotView (array fast path), a DeviceBatch (on-device kernel,
    rasp_histogram) or any iterable of VmSlot."""
    out = dict.fromkeys(HISTOGRAM_KEYS, 0)
    if isinstance(slots, DeviceBatch):
        h = get_engine(slots.params, slots.iw.device).histogram(slots).cpu().numpy()
        return {k: int(v) for k, v in zip(HISTOGRAM_KEYS, h)}
    if isinstance(slots, SlotView):
        st = np.asarray(slots.status)
        th = np.asarray(slots.tau_h)[st == _HALTED]
        small = th[th < 100]
        vals, cnts = np.unique(small, return_counts=True)
        for v, c in zip(vals, cnts):
            out[str(int(v))] = int(c)
        out["100+"] = int((th >= 100).sum())
        out["nonhalt"] = int((st == _EXHAUSTED).sum())
        return out
    for slot in slots:
        if slot.status == VmStatus.HALTED:
            out[str(slot.tau_h) if slot.tau_h < 100 else "100+"] += 1
        elif slot.status == VmStatus.BUDGET_EXHAUSTED:
            out["nonhalt"] += 1
    return out


# keep the field tuple importable for bulk consumers
FIELDS = ALL_FIELDS


# --- workloads and the worker-count benchmark (hypervisor.py:355-408) ------------

@dataclass
class Workload:
    """Prepared initial configurations of a program batch (hv:355-360).
    `asts` stays None here: sampling and lowering are out of this engine's
    scope, programs arrive already lowered."""
    configs: list
    asts: list | None
    aborted: list              # (index, reason) for programs that do not fit memory


def build_workload_from_programs(programs, inputs, params: MachineParams) -> Workload:
    """The packing half of build_workload (hv:362-384) for lowered programs:
    init_config per program; a CapacityError draw is recorded in `aborted`,
    never silently dropped (other errors propagate, as in the reference)."""
    configs, aborted = [], []
    for k, (prog, x) in enumerate(zip(programs, inputs)):
        try:
            configs.append(init_config(prog, x, params))
        except CapacityError as e:
            aborted.append((k, str(e)))
    return Workload(configs=configs, asts=None, aborted=aborted)


def throughput_bench(workload: Workload, tau_max: int, workers_list, params: MachineParams,
                     epoch: int = 64) -> list:
    """hv:387-408: time the same workload once per entry of `workers_list`;
    one row {"workers", "wall_time", "vms", "speedup"} each, speedup against
    the first workers == 1 row (else the first row).  The GPU engine has no
    worker count: every row runs the whole batch on the device and
    wall_time is run_batch's device time."""
    rows = []
    for w in workers_list:
        res = run_batch(workload.configs, params, BatchConfig(tau_max=tau_max, epoch=epoch, workers=max(0, int(w)),
                                                              memory_budget_words=1 << 62))
        rows.append({"workers": w, "wall_time": res.wall_time, "vms": len(workload.configs), "speedup": 0.0})
    base = next((r["wall_time"] for r in rows if r["workers"] == 1), rows[0]["wall_time"] if rows else 0.0)
    for r in rows:
        r["speedup"] = base / r["wall_time"] if r["wall_time"] > 0 else 0.0
    return rows
