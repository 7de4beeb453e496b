"""Device-resident batches and the engine that runs them (host side of the
C ABI).  PyTorch is used for device memory and streams only; all compute is
in the CUDA library (csrc/), called through ctypes.

``DeviceBatch`` is the reference's SoA state (hypervisor.py:280-293:
iw, ac, M, u, y, status, steps, tau_h) held in HBM, with words stored at
their natural width (u8/u16/u32/u64 for w <= 8/16/32/64) unless a wider
width is requested (8 bytes reproduces the reference's uint64 arrays).
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _native
from .errors import CapacityError, NativeError
from .machine import MachineParams

TORCH_WORD = {1: torch.uint8, 2: torch.uint16, 4: torch.uint32, 8: torch.uint64}
NUMPY_WORD = {1: np.uint8, 2: np.uint16, 4: np.uint32, 8: np.uint64}
WORD_FIELDS = ("iw", "ac", "M", "u", "y")
ALL_FIELDS = WORD_FIELDS + ("status", "steps", "tau_h")


def _require_cuda(device) -> torch.device:
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device()) \
        if torch.cuda.is_available() else None
    if dev is None or dev.type != "cuda" or not torch.cuda.is_available():
        raise NativeError("the batch engine runs on a CUDA device; none is available "
                          "(there is no CPU fallback)")
    return dev


class DeviceBatch:
    """A batch of d machines in HBM (the `rasp_batch` of the C ABI)."""

    def __init__(self, params: MachineParams, tensors: dict, word_bytes: int):
        self.params = params
        self.word_bytes = word_bytes
        for k in ALL_FIELDS:
            setattr(self, k, tensors[k])
        self.d = int(tensors["iw"].shape[0])

    # --- construction -------------------------------------------------------------
    @classmethod
    def empty(cls, d: int, params: MachineParams, device=None, word_bytes: int | None = None,
              fresh: bool = True) -> "DeviceBatch":
        dev = _require_cuda(device)
        wb = word_bytes or params.dtype.itemsize
        wd = TORCH_WORD[wb]
        t = {
            "iw": torch.empty(d, dtype=wd, device=dev),
            "ac": torch.empty(d, dtype=wd, device=dev),
            "M": torch.empty((d, params.n), dtype=wd, device=dev),
            "u": torch.empty((d, params.ell + 1), dtype=wd, device=dev),
            "y": torch.empty((d, params.s + 1), dtype=wd, device=dev),
        }
        if fresh:
            t["status"] = torch.zeros(d, dtype=torch.int8, device=dev)
            t["steps"] = torch.zeros(d, dtype=torch.int64, device=dev)
            t["tau_h"] = torch.full((d,), -1, dtype=torch.int64, device=dev)
        else:
            t["status"] = torch.empty(d, dtype=torch.int8, device=dev)
            t["steps"] = torch.empty(d, dtype=torch.int64, device=dev)
            t["tau_h"] = torch.empty(d, dtype=torch.int64, device=dev)
        return cls(params, t, wb)

    @classmethod
    def from_arrays(cls, arrays: dict, params: MachineParams, device=None,
                    word_bytes: int | None = None, non_blocking: bool = False) -> "DeviceBatch":
        """Copy host SoA arrays (numpy or torch) to the device.  Missing
        status/steps/tau_h get run_batch's fresh values (hv:291-293)."""
        dev = _require_cuda(device)
        wb = word_bytes or params.dtype.itemsize
        d = int(np.asarray(arrays["iw"]).shape[0]) if not torch.is_tensor(arrays["iw"]) \
            else int(arrays["iw"].shape[0])
        b = cls.empty(d, params, dev, wb, fresh=True)
        shapes = {"iw": (d,), "ac": (d,), "M": (d, params.n), "u": (d, params.ell + 1),
                  "y": (d, params.s + 1), "status": (d,), "steps": (d,), "tau_h": (d,)}
        for k in ALL_FIELDS:
            if k not in arrays:
                continue
            src = arrays[k]
            dst = getattr(b, k)
            if not torch.is_tensor(src):
                a = np.asarray(src)
                if k in WORD_FIELDS and a.dtype != NUMPY_WORD[wb]:
                    a = a.astype(NUMPY_WORD[wb])
                src = torch.from_numpy(np.ascontiguousarray(a))
            elif k in WORD_FIELDS and src.dtype != dst.dtype:
                src = src.to(dst.dtype)
            if tuple(src.shape) != shapes[k]:
                src = src.reshape(shapes[k])
            dst.copy_(src, non_blocking=non_blocking)
        return b

    def to_numpy(self) -> dict:
        return {k: getattr(self, k).cpu().numpy() for k in ALL_FIELDS}

    def tensors(self) -> dict:
        return {k: getattr(self, k) for k in ALL_FIELDS}

    def c_struct(self) -> _native.RaspBatch:
        return _native.RaspBatch(
            self.iw.data_ptr(), self.ac.data_ptr(), self.M.data_ptr(), self.u.data_ptr(),
            self.y.data_ptr(), self.status.data_ptr(), self.steps.data_ptr(),
            self.tau_h.data_ptr(), self.d, self.word_bytes, 0)


class Engine:
    """Runs DeviceBatches of one machine geometry on one device."""

    def __init__(self, params: MachineParams, device=None):
        self.lib = _native.load()
        self.params = params
        self.device = _require_cuda(device)
        if params.ell >= 2 ** 31 or params.s >= 2 ** 31:
            raise CapacityError("ell and s must be below 2^31 for the batch engine")
        self._p = _native.RaspParams(params.w, params.n, params.ell, params.s)
        self._ws = None
        self._warmed = set()

    def _stream_ptr(self, stream) -> int:
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        return s.cuda_stream

    def workspace_bytes(self, d: int) -> int:
        with torch.cuda.device(self.device):
            need = self.lib.rasp_workspace_bytes(ctypes.byref(self._p), d)
        if need == 0 and d:
            raise NativeError("rasp_workspace_bytes failed")
        return int(need)

    def workspace(self, d: int) -> torch.Tensor:
        """The engine's own workspace (runs on one stream at a time share it)."""
        need = self.workspace_bytes(d)
        if self._ws is None or self._ws.numel() < need:
            self._ws = torch.empty(max(need, 256), dtype=torch.uint8, device=self.device)
        return self._ws

    def run(self, batch: DeviceBatch, tau_max: int, epoch: int = 64,
            out: DeviceBatch | None = None, fresh: bool = False, stream=None,
            workspace: torch.Tensor | None = None, hist: torch.Tensor | None = None) -> DeviceBatch:
        """Phi to fixed point or tau_max for every RUNNING machine (rasp_run).
        In place unless `out` is given.  Asynchronous on `stream`.  Runs that
        may overlap on different streams need their own `workspace`
        (workspace_bytes(d) bytes of device memory).  `hist` (device int64[102])
        receives the batch's halting histogram, counted inside the run
        (rasp_run_hist; the buckets of collect_histogram, hv:329-352)."""
        if hist is not None and (hist.dtype != torch.int64 or hist.numel() != 102 or not hist.is_contiguous()
                                 or hist.device != self.device):
            raise ValueError("hist must be a contiguous int64[102] tensor on the engine's device")
        if tau_max < 0:
            raise ValueError(f"tau_max must be >= 0, got {tau_max}")
        if epoch < 1:
            raise ValueError(f"epoch must be >= 1, got {epoch}")
        dst = out if out is not None else batch
        if dst.d != batch.d or dst.word_bytes != batch.word_bytes:
            raise ValueError("out batch must match the input batch's size and word width")
        if batch.d == 0:
            if hist is not None:
                hist.zero_()
            return dst
        if workspace is not None:
            if workspace.numel() < self.workspace_bytes(batch.d):
                raise ValueError("workspace too small for this batch")
            ws = workspace
        else:
            ws = self.workspace(batch.d)
        bi, bo = batch.c_struct(), dst.c_struct()
        with torch.cuda.device(self.device):
            rc = self.lib.rasp_run_hist(ctypes.byref(self._p), ctypes.byref(bi), ctypes.byref(bo),
                                        int(tau_max), int(epoch),
                                        _native.RASP_FRESH if fresh else 0,
                                        hist.data_ptr() if hist is not None else None,
                                        ws.data_ptr(), ws.numel(), self._stream_ptr(stream))
        _native.check(rc, "rasp_run")
        return dst

    def warm(self, word_bytes: int, fresh: bool, stream=None) -> None:
        """Run this geometry's kernels once on 32 all-zero machines (each halts
        at step 0), so lazy module loading and launch planning happen before a
        caller starts timing -- the reference warms its kernel off the clock
        the same way (hypervisor.py:302)."""
        key = (word_bytes, bool(fresh))
        if key in self._warmed:
            return
        b = DeviceBatch.empty(32, self.params, self.device, word_bytes, fresh=True)
        for k in WORD_FIELDS:
            getattr(b, k).zero_()
        self.run(b, 1, 1, fresh=fresh, stream=stream, workspace=torch.empty(
            max(self.workspace_bytes(32), 256), dtype=torch.uint8, device=self.device))
        self._warmed.add(key)

    def init_c0(self, programs: torch.Tensor, inputs: torch.Tensor, out: DeviceBatch, stream=None) -> DeviceBatch:
        """Device packer of init_config (rasp_init_c0): programs [d, L] and
        inputs [d, k] device tensors of the batch word type -> c0 in `out`.
        Words must already be range-checked (see machine.init_batch)."""
        if programs.shape[0] != out.d or (inputs.numel() and inputs.shape[0] != out.d):
            raise ValueError("programs/inputs must have one row per machine")
        L = programs.shape[1] if programs.dim() == 2 else 0
        k = inputs.shape[1] if inputs.dim() == 2 else 0
        if L > self.params.n:
            raise CapacityError(f"program needs {L} memory words but n = {self.params.n}")
        if k > self.params.ell:
            raise CapacityError(f"input vector has {k} words but ell = {self.params.ell}")
        b = out.c_struct()
        with torch.cuda.device(self.device):
            rc = self.lib.rasp_init_c0(ctypes.byref(self._p), programs.data_ptr() if L else None, L,
                                       inputs.data_ptr() if k else None, k, ctypes.byref(b),
                                       self._stream_ptr(stream))
        _native.check(rc, "rasp_init_c0")
        return out

    def generate(self, out: DeviceBatch, seed: int, first_machine: int = 0, stream=None) -> DeviceBatch:
        """Generator G_dev on the device (rasp_generate): fresh c0 in `out`."""
        b = out.c_struct()
        with torch.cuda.device(self.device):
            rc = self.lib.rasp_generate(ctypes.byref(self._p), int(seed), int(first_machine),
                                        ctypes.byref(b), self._stream_ptr(stream))
        _native.check(rc, "rasp_generate")
        return out

    def histogram(self, batch: DeviceBatch, out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
        """int64[102] device tensor: tau_h 0..99, 100+, nonhalt (rasp_histogram)."""
        h = out if out is not None else torch.empty(102, dtype=torch.int64, device=self.device)
        with torch.cuda.device(self.device):
            rc = self.lib.rasp_histogram(batch.status.data_ptr(), batch.tau_h.data_ptr(), batch.d,
                                         h.data_ptr(), self._stream_ptr(stream))
        _native.check(rc, "rasp_histogram")
        return h

    def validate(self, batch: DeviceBatch, stream=None) -> np.ndarray:
        """Counts of out-of-range words per field and cursors (rasp_validate)."""
        o = torch.empty(8, dtype=torch.int64, device=self.device)
        b = batch.c_struct()
        with torch.cuda.device(self.device):
            rc = self.lib.rasp_validate(ctypes.byref(self._p), ctypes.byref(b), o.data_ptr(),
                                        self._stream_ptr(stream))
        _native.check(rc, "rasp_validate")
        return o.cpu().numpy()

    def convert(self, src: DeviceBatch, dst: DeviceBatch, stream=None) -> DeviceBatch:
        """Word-width conversion src -> dst (rasp_pack / rasp_unpack): e.g. the
        reference's uint64 arrays into natural-width words, or back."""
        if src.d != dst.d:
            raise ValueError("src and dst batches must hold the same number of machines")
        a, b = src.c_struct(), dst.c_struct()
        fn = self.lib.rasp_pack if dst.word_bytes <= src.word_bytes else self.lib.rasp_unpack
        with torch.cuda.device(self.device):
            rc = fn(ctypes.byref(self._p), ctypes.byref(a), ctypes.byref(b), self._stream_ptr(stream))
        _native.check(rc, "rasp_pack" if fn is self.lib.rasp_pack else "rasp_unpack")
        return dst

    def topk(self, batch: DeviceBatch, k: int, tau_max: int, stream=None):
        """(index, tau_h) int64[k] device tensors of the k longest halting runs,
        ties to the lower index, -1 padded (rasp_topk)."""
        if k < 0:
            raise ValueError(f"k must be >= 0, got {k}")
        idx = torch.empty(k, dtype=torch.int64, device=self.device)
        tau = torch.empty(k, dtype=torch.int64, device=self.device)
        if k == 0:
            return idx, tau
        need = self.lib.rasp_topk_workspace_bytes(k)
        ws = torch.empty(need, dtype=torch.uint8, device=self.device)
        with torch.cuda.device(self.device):
            rc = self.lib.rasp_topk(batch.status.data_ptr(), batch.tau_h.data_ptr(), batch.d, int(tau_max),
                                    int(k), idx.data_ptr(), tau.data_ptr(), ws.data_ptr(), need,
                                    self._stream_ptr(stream))
        _native.check(rc, "rasp_topk")
        return idx, tau
