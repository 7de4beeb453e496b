"""Multi-GPU execution: one process per GPU, contiguous shards, no data-path
collective.

Machines are independent (each trajectory depends only on its own c0,
SPEC "pure value-in/value-out"), so rank k simply runs machines
[lo_k, hi_k) on its own device.  The only collectives are post-run and go
through torch.distributed (NCCL over NVLink on a GPU box, gloo in the CPU
tests):

  * all-reduce of the 102-bucket halting histogram (hypervisor.py:326-352):
    102 x int64 = 816 B, latency-bound;
  * gather of the per-machine verdicts (status, steps, tau_h) and output
    tapes y to rank 0 -- the "output gather via NCCL" of BASELINE config 3.

The results are identical for every world size: shard boundaries only
decide which device computes a machine, never what it computes.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch
import torch.distributed as dist

from .machine import MachineParams


def shard_bounds(d: int, world: int, rank: int) -> tuple:
    """Contiguous block partition: rank k owns [k*ceil(d/W), ...) clipped to d."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of world {world}")
    per = -(-d // world) if d else 0
    lo = min(d, rank * per)
    hi = min(d, lo + per)
    return lo, hi


def shard_arrays(arrays: dict, world: int, rank: int) -> dict:
    d = int(np.asarray(arrays["iw"]).shape[0])
    lo, hi = shard_bounds(d, world, rank)
    return {k: v[lo:hi] for k, v in arrays.items()}


@dataclass
class ShardResult:
    histogram: np.ndarray          # int64[102], reduced over all ranks
    status: np.ndarray | None      # gathered on rank 0 (None elsewhere / when not gathered)
    steps: np.ndarray | None
    tau_h: np.ndarray | None
    y: np.ndarray | None
    machine_steps: int             # sum over all ranks


def histogram_np(status: np.ndarray, tau_h: np.ndarray) -> np.ndarray:
    """Host histogram with the bucketing of hypervisor.py:329-352."""
    h = np.zeros(102, np.int64)
    th = tau_h[status == 1]
    np.add.at(h, np.minimum(th, 100), 1)
    h[101] = int((status == 2).sum())
    return h


def reduce_histogram(hist: torch.Tensor, group=None) -> torch.Tensor:
    """In-place sum of int64[102] histograms across ranks."""
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(hist, op=dist.ReduceOp.SUM, group=group)
    return hist


def gather_to_root(t: torch.Tensor, d_total: int, world: int, rank: int, group=None, sizes=None,
                   out: torch.Tensor | None = None):
    """Gather contiguous shards of a per-machine tensor to rank 0.

    Shards may differ in length by the partition (`sizes`: machines per rank,
    default shard_bounds(d_total, world, k)); every rank pads to the largest
    shard so one collective moves everything.  Returns the full [d_total, ...]
    tensor on rank 0, None elsewhere.  `out` (rank 0): a receive buffer of at
    least world x largest-shard rows to reuse across calls; with equal shards
    the result is a view of it (no concatenation)."""
    if not (dist.is_available() and dist.is_initialized()) or world == 1:
        return t
    if sizes is None:
        sizes = [hi - lo for lo, hi in (shard_bounds(d_total, world, k) for k in range(world))]
    per = max(sizes) if sizes else 0
    if t.shape[0] == per:
        pad = t.contiguous()
    else:
        pad = torch.zeros((per,) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
        pad[: t.shape[0]] = t
    parts = None
    if rank == 0:
        shape = (world * per,) + tuple(t.shape[1:])
        if out is None or out.shape[0] < world * per or tuple(out.shape[1:]) != shape[1:] or \
                out.dtype != t.dtype or out.device != t.device:
            out = torch.empty(shape, dtype=t.dtype, device=t.device)
        parts = list(out[: world * per].view((world, per) + shape[1:]).unbind(0))
    dist.gather(pad, parts, dst=0, group=group)
    if rank != 0:
        return None
    if all(sz == per for sz in sizes):
        return out[:d_total]
    return torch.cat([parts[k][: sizes[k]] for k in range(world)], 0)


def collect(status: torch.Tensor, steps: torch.Tensor, tau_h: torch.Tensor, y: torch.Tensor,
            hist: torch.Tensor, d_total: int, gather: bool = True, group=None) -> ShardResult:
    """Post-run collectives of one rank's shard (tensors on this rank's device)."""
    world = dist.get_world_size(group) if dist.is_available() and dist.is_initialized() else 1
    rank = dist.get_rank(group) if world > 1 else 0
    reduce_histogram(hist, group)
    ms = steps.sum().reshape(1).to(torch.int64)
    if world > 1:
        dist.all_reduce(ms, group=group)
    st = sp = th = yy = None
    if gather:
        # status/steps/tau_h travel as int64 (NCCL has no int8 gather issue,
        # but one dtype keeps the collective count at four)
        st = gather_to_root(status.to(torch.int64), d_total, world, rank, group)
        sp = gather_to_root(steps, d_total, world, rank, group)
        th = gather_to_root(tau_h, d_total, world, rank, group)
        ycast = y.to(torch.int64) if y.dtype not in (torch.int64, torch.float64) else y
        yy = gather_to_root(ycast, d_total, world, rank, group)
    if rank != 0:
        st = sp = th = yy = None

    def cpu(x, dt=None):
        if x is None:
            return None
        a = x.cpu().numpy()
        return a.astype(dt) if dt is not None else a

    return ShardResult(histogram=hist.cpu().numpy(), status=cpu(st, np.int8), steps=cpu(sp),
                       tau_h=cpu(th), y=cpu(yy), machine_steps=int(ms.item()))


def run_shard_on_device(arrays: dict, params: MachineParams, tau_max: int, epoch: int = 32,
                        device=None, d_total: int | None = None, gather: bool = True,
                        group=None) -> ShardResult:
    """Run this rank's shard on its GPU through the engine, then collect."""
    from .engine import DeviceBatch
    from .hypervisor import get_engine
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    b = DeviceBatch.from_arrays(arrays, params, dev)
    eng = get_engine(params, dev)
    eng.run(b, tau_max, epoch, fresh=not any(k in arrays for k in ("status", "steps", "tau_h")))
    hist = eng.histogram(b)
    return collect(b.status, b.steps, b.tau_h, b.y, hist, d_total or b.d, gather, group)


class NativeComm:
    """An NCCL communicator owned by the engine library (rasp_nccl_comm_init)
    for the post-run collectives of a sharded run through the C ABI:
    rasp_shard_allreduce (histogram + totals) and rasp_shard_gather (per-machine
    results to the root).  The 128-byte NCCL id travels over the process
    group that already exists (gloo or nccl), or stays local at world 1."""

    def __init__(self, group=None, device=None):
        import ctypes
        from . import _native
        self.lib = _native.load()
        self._native = _native
        initialized = dist.is_available() and dist.is_initialized()
        self.world = dist.get_world_size(group) if initialized else 1
        self.rank = dist.get_rank(group) if initialized else 0
        self.device = torch.device(device) if device is not None else \
            torch.device("cuda", torch.cuda.current_device())
        uid = ctypes.create_string_buffer(128)
        if self.rank == 0:
            _native.check(self.lib.rasp_nccl_unique_id(uid), "rasp_nccl_unique_id")
        if self.world > 1:
            box = [bytes(uid.raw)]
            dist.broadcast_object_list(box, src=0, group=group)
            uid = ctypes.create_string_buffer(box[0], 128)
        self._comm = ctypes.c_void_p()
        with torch.cuda.device(self.device):
            _native.check(self.lib.rasp_nccl_comm_init(self.world, uid, self.rank, ctypes.byref(self._comm)),
                          "rasp_nccl_comm_init")

    def _stream(self, stream):
        return (stream if stream is not None else torch.cuda.current_stream(self.device)).cuda_stream

    def allreduce(self, counters: torch.Tensor, stream=None) -> torch.Tensor:
        """In-place sum over ranks of an int64 device tensor."""
        if counters.dtype != torch.int64 or not counters.is_contiguous():
            raise ValueError("counters must be a contiguous int64 tensor")
        with torch.cuda.device(self.device):
            rc = self.lib.rasp_shard_allreduce(self._comm, counters.data_ptr(), counters.numel(),
                                               self._stream(stream))
        self._native.check(rc, "rasp_shard_allreduce")
        return counters

    def gather(self, shard, full, d_total: int, fields: int, root: int = 0, stream=None):
        """Gather shard fields (DeviceBatch) into `full` (DeviceBatch of d_total
        machines, needed on the root only)."""
        import ctypes
        p = self._native.RaspParams(shard.params.w, shard.params.n, shard.params.ell, shard.params.s)
        a = shard.c_struct()
        b = full.c_struct() if full is not None else None
        with torch.cuda.device(self.device):
            rc = self.lib.rasp_shard_gather(self._comm, root, ctypes.byref(p), d_total, ctypes.byref(a),
                                            ctypes.byref(b) if b is not None else None, fields,
                                            self._stream(stream))
        self._native.check(rc, "rasp_shard_gather")
        return full

    def close(self):
        if self._comm:
            self.lib.rasp_nccl_comm_destroy(self._comm)
            self._comm = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
