"""Host-buffer path: c0 in pinned host memory -> HBM -> run -> results back
to pinned host memory, pipelined in chunks so the two PCIe directions and the
engine overlap (copy-in of chunk c+1 and copy-out of chunk c-1 run under the
compute of chunk c).

This is the end-to-end path a caller with host arrays takes (the reference's
run_batch consumes and returns host arrays, hypervisor.py:265-323).
"""

from __future__ import annotations

import numpy as np
import torch

from .engine import ALL_FIELDS, NUMPY_WORD, TORCH_WORD, WORD_FIELDS, DeviceBatch, Engine
from .hypervisor import get_engine
from .machine import MachineParams


class HostPipeline:
    def __init__(self, params: MachineParams, d: int, device=None, chunks: int = 8,
                 engine: Engine | None = None, word_bytes: int | None = None, small_groups: int = 4,
                 ramp: bool = True, run_streams: int = 3):
        self.params = params
        self.d = d
        self.device = torch.device(device) if device is not None else torch.device("cuda")
        self.engine = engine or get_engine(params, self.device)
        self.wb = word_bytes or params.dtype.itemsize
        # one device batch: each chunk is copied in, run in place, copied out
        self.dev = DeviceBatch.empty(d, params, self.device, self.wb, fresh=False)
        self.chunks = max(1, min(chunks, (d + 4095) // 4096))
        step = (d + self.chunks - 1) // self.chunks
        self.bounds = [(a, min(d, a + step)) for a in range(0, d, step)] if d else []
        if ramp and self.chunks >= 4 and d >= 1 << 16:
            # short first and last chunks: the pipeline fills and drains sooner
            w = [1, 2] + [4] * (self.chunks - 4) + [2, 1]
            cuts = np.cumsum([0] + w) * d // sum(w)
            self.bounds = [(int(cuts[k]), int(cuts[k + 1])) for k in range(len(w))]
        wd = TORCH_WORD[self.wb]
        shapes = {"iw": (d,), "ac": (d,), "M": (d, params.n), "u": (d, params.ell + 1),
                  "y": (d, params.s + 1)}
        self.host_out = {k: torch.empty(shapes[k], dtype=wd, pin_memory=True) for k in WORD_FIELDS}
        self.host_out["status"] = torch.empty(d, dtype=torch.int8, pin_memory=True)
        self.host_out["steps"] = torch.empty(d, dtype=torch.int64, pin_memory=True)
        self.host_out["tau_h"] = torch.empty(d, dtype=torch.int64, pin_memory=True)
        self.s_in = torch.cuda.Stream(self.device)
        # chunk runs alternate between run streams, so one chunk's long tail
        # (its last machines in a long epoch) overlaps the next chunk's run;
        # each stream has its own workspace
        self.s_runs = [torch.cuda.Stream(self.device) for _ in range(max(1, run_streams))]
        self.s_run = self.s_runs[0]
        self.s_out = torch.cuda.Stream(self.device)
        self.h2d_bytes = 0
        self.d2h_bytes = sum(t.numel() * t.element_size() for t in self.host_out.values())
        # copy-out: M (the bulk) per chunk; the small per-machine fields in a
        # few large copies -- each copy costs ~10 us of PCIe time, and 8 fields
        # x chunks of them cost more than the overlap wins (scripts/pcie_split.py)
        self.small_groups = max(1, min(small_groups, len(self.bounds)))
        # one workspace per run stream
        wsb = self.engine.workspace_bytes(max((b - a for a, b in self.bounds), default=0))
        self.ws = [torch.empty(max(wsb, 256), dtype=torch.uint8, device=self.device) for _ in self.s_runs]

    def pinned_inputs(self, arrays: dict) -> dict:
        """Copy host c0 arrays (numpy) into pinned tensors once."""
        wd = TORCH_WORD[self.wb]
        out = {}
        for k in WORD_FIELDS:
            a = np.ascontiguousarray(np.asarray(arrays[k]).astype(NUMPY_WORD[self.wb]))
            t = torch.empty(a.shape, dtype=wd, pin_memory=True)
            t.copy_(torch.from_numpy(a))
            out[k] = t
        self.h2d_bytes = sum(t.numel() * t.element_size() for t in out.values())
        return out

    @staticmethod
    def _view(batch: DeviceBatch, a: int, b: int) -> DeviceBatch:
        return DeviceBatch(batch.params, {k: getattr(batch, k)[a:b] for k in ALL_FIELDS},
                           batch.word_bytes)

    def run(self, pinned: dict, tau_max: int, epoch: int = 32) -> float:
        """One end-to-end pass; returns device seconds (events on the caller's
        stream bracketing every copy and every kernel)."""
        main = torch.cuda.current_stream(self.device)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(main)
        for s in (self.s_in, *self.s_runs, self.s_out):
            s.wait_event(e0)
        for c, (a, b) in enumerate(self.bounds):
            with torch.cuda.stream(self.s_in):
                for k in WORD_FIELDS:
                    getattr(self.dev, k)[a:b].copy_(pinned[k][a:b], non_blocking=True)
                ev_in = torch.cuda.Event()
                ev_in.record(self.s_in)
            sr, ws = self.s_runs[c % len(self.s_runs)], self.ws[c % len(self.s_runs)]
            sr.wait_event(ev_in)
            # fresh c0: status/steps/tau_h are outputs only, never read
            self.engine.run(self._view(self.dev, a, b), tau_max, epoch, fresh=True, stream=sr, workspace=ws)
            ev_run = torch.cuda.Event()
            ev_run.record(sr)
            self.s_out.wait_event(ev_run)
            self._copy_out(c, a, b)
        main.wait_stream(self.s_out)
        e1.record(main)
        e1.synchronize()
        return e0.elapsed_time(e1) / 1e3

    # --- programs + inputs (init_config on the device) --------------------------
    def pinned_programs(self, programs, inputs) -> dict:
        """Pinned copies of programs [d, L] and inputs [d, k] (the arguments of
        init_config, machine.py:289-309); c0 is assembled on the device."""
        wd = TORCH_WORD[self.wb]
        out = {}
        for name, arr in (("programs", programs), ("inputs", inputs)):
            a = np.ascontiguousarray(np.asarray(arr).astype(NUMPY_WORD[self.wb]))
            if a.ndim == 1:
                a = a.reshape(self.d, -1)
            t = torch.empty(a.shape, dtype=wd, pin_memory=True)
            t.copy_(torch.from_numpy(a))
            out[name] = t
        if out["programs"].shape[1] > self.params.n or out["inputs"].shape[1] > self.params.ell:
            from .errors import CapacityError
            raise CapacityError("programs or inputs exceed the machine geometry")
        self._stage = {k: torch.empty(v.shape, dtype=wd, device=self.device) for k, v in out.items()}
        self.h2d_bytes = sum(t.numel() * t.element_size() for t in out.values())
        return out

    def run_programs(self, pinned: dict, tau_max: int, epoch: int = 64) -> float:
        """End-to-end pass from programs + inputs: per chunk, copy them in,
        assemble c0 on the device (rasp_init_c0), run in place, copy every
        result field out.  Returns device seconds."""
        main = torch.cuda.current_stream(self.device)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(main)
        for s in (self.s_in, *self.s_runs, self.s_out):
            s.wait_event(e0)
        P, X = self._stage["programs"], self._stage["inputs"]
        for c, (a, b) in enumerate(self.bounds):
            with torch.cuda.stream(self.s_in):
                P[a:b].copy_(pinned["programs"][a:b], non_blocking=True)
                if X.shape[1]:
                    X[a:b].copy_(pinned["inputs"][a:b], non_blocking=True)
                ev_in = torch.cuda.Event()
                ev_in.record(self.s_in)
            sr, ws = self.s_runs[c % len(self.s_runs)], self.ws[c % len(self.s_runs)]
            sr.wait_event(ev_in)
            view = self._view(self.dev, a, b)
            self.engine.init_c0(P[a:b], X[a:b], view, stream=sr)
            self.engine.run(view, tau_max, epoch, fresh=True, stream=sr, workspace=ws)
            ev_run = torch.cuda.Event()
            ev_run.record(sr)
            self.s_out.wait_event(ev_run)
            self._copy_out(c, a, b)
        main.wait_stream(self.s_out)
        e1.record(main)
        e1.synchronize()
        return e0.elapsed_time(e1) / 1e3

    def _copy_out(self, c: int, a: int, b: int) -> None:
        """After chunk c = rows [a, b) has run: its M rows now, the small
        fields of every finished chunk at the end of each group of chunks."""
        with torch.cuda.stream(self.s_out):
            self.host_out["M"][a:b].copy_(self.dev.M[a:b], non_blocking=True)
            per = -(-len(self.bounds) // self.small_groups)
            if (c + 1) % per == 0 or c + 1 == len(self.bounds):
                lo = self.bounds[(c // per) * per][0]
                for k in ALL_FIELDS:
                    if k != "M":
                        self.host_out[k][lo:b].copy_(getattr(self.dev, k)[lo:b], non_blocking=True)

    def results(self) -> dict:
        return {k: v.numpy() for k, v in self.host_out.items()}
