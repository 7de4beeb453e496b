"""ctypes binding of the C ABI in include/raspvisor_b200.h.

The shared library is built in-tree (``__graft_entry__.build()`` or
``python -m paper_2604_12902_b200.build``) into ``_lib/libraspvisor_b200.so``.
There is no fallback: if the library is missing or cannot be loaded, every
batch entry point raises NativeError.
"""

from __future__ import annotations

import ctypes
import os

from .errors import NativeError

LIB_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_lib")
# RASP_LIBRARY: load another build of the same library (A/B timing of kernel variants)
LIB_PATH = os.environ.get("RASP_LIBRARY") or os.path.join(LIB_DIR, "libraspvisor_b200.so")
ABI_VERSION = 3

RASP_FRESH = 1

# symbols declared by include/raspvisor_b200.h
EXPORTS = ("rasp_workspace_bytes", "rasp_run", "rasp_run_hist", "rasp_histogram", "rasp_validate",
           "rasp_error_string", "rasp_last_cuda_error", "rasp_abi_version",
           "rasp_launch_count", "rasp_enumerate", "rasp_init_c0", "rasp_generate",
           "rasp_pack", "rasp_unpack", "rasp_topk_workspace_bytes", "rasp_topk",
           "rasp_nccl_unique_id", "rasp_nccl_comm_init", "rasp_nccl_comm_destroy",
           "rasp_shard_allreduce", "rasp_shard_gather", "rasp_checked_build")

RASP_GATHER_RESULTS = 1
RASP_GATHER_OUTPUT = 2
RASP_GATHER_CONFIG = 4


class RaspParams(ctypes.Structure):
    _fields_ = [("w", ctypes.c_uint32), ("n", ctypes.c_uint32),
                ("ell", ctypes.c_uint64), ("s", ctypes.c_uint64)]


class RaspEnumParams(ctypes.Structure):
    _fields_ = [("m", ctypes.c_uint32), ("opcode_bits", ctypes.c_uint32),
                ("operand_bits", ctypes.c_uint32), ("w", ctypes.c_uint32),
                ("n", ctypes.c_uint32), ("tau_max", ctypes.c_uint32)]


class RaspBatch(ctypes.Structure):
    _fields_ = [("iw", ctypes.c_void_p), ("ac", ctypes.c_void_p), ("M", ctypes.c_void_p),
                ("u", ctypes.c_void_p), ("y", ctypes.c_void_p),
                ("status", ctypes.c_void_p), ("steps", ctypes.c_void_p),
                ("tau_h", ctypes.c_void_p), ("d", ctypes.c_uint64),
                ("word_bytes", ctypes.c_uint32), ("_pad", ctypes.c_uint32)]


_lib = None


def load():
    """Load the engine library (once).  Raises NativeError when absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise NativeError(
            f"CUDA engine library not built: {LIB_PATH} is missing "
            "(run __graft_entry__.build() or python -m paper_2604_12902_b200.build)")
    try:
        lib = ctypes.CDLL(LIB_PATH)
    except OSError as e:
        raise NativeError(f"cannot load {LIB_PATH}: {e}") from e
    P, U64, I64, U32, SZ = (ctypes.c_void_p, ctypes.c_uint64, ctypes.c_int64,
                            ctypes.c_uint32, ctypes.c_size_t)
    pp = ctypes.POINTER(RaspParams)
    pb = ctypes.POINTER(RaspBatch)
    lib.rasp_workspace_bytes.argtypes = [pp, U64]
    lib.rasp_workspace_bytes.restype = SZ
    lib.rasp_run.argtypes = [pp, pb, pb, I64, I64, U32, P, SZ, P]
    lib.rasp_run.restype = ctypes.c_int
    lib.rasp_run_hist.argtypes = [pp, pb, pb, I64, I64, U32, P, P, SZ, P]
    lib.rasp_run_hist.restype = ctypes.c_int
    lib.rasp_histogram.argtypes = [P, P, U64, P, P]
    lib.rasp_histogram.restype = ctypes.c_int
    lib.rasp_validate.argtypes = [pp, pb, P, P]
    lib.rasp_validate.restype = ctypes.c_int
    lib.rasp_error_string.argtypes = [ctypes.c_int]
    lib.rasp_error_string.restype = ctypes.c_char_p
    lib.rasp_last_cuda_error.argtypes = []
    lib.rasp_last_cuda_error.restype = ctypes.c_char_p
    lib.rasp_checked_build.argtypes = []
    lib.rasp_checked_build.restype = ctypes.c_int
    lib.rasp_abi_version.argtypes = []
    lib.rasp_abi_version.restype = ctypes.c_int
    lib.rasp_enumerate.argtypes = [ctypes.POINTER(RaspEnumParams), U64, U64, P, P, P]
    lib.rasp_enumerate.restype = ctypes.c_int
    lib.rasp_init_c0.argtypes = [pp, P, U32, P, U32, pb, P]
    lib.rasp_init_c0.restype = ctypes.c_int
    lib.rasp_generate.argtypes = [pp, U64, U64, pb, P]
    lib.rasp_generate.restype = ctypes.c_int
    lib.rasp_pack.argtypes = [pp, pb, pb, P]
    lib.rasp_pack.restype = ctypes.c_int
    lib.rasp_unpack.argtypes = [pp, pb, pb, P]
    lib.rasp_unpack.restype = ctypes.c_int
    lib.rasp_topk_workspace_bytes.argtypes = [U32]
    lib.rasp_topk_workspace_bytes.restype = SZ
    lib.rasp_topk.argtypes = [P, P, U64, I64, U32, P, P, P, SZ, P]
    lib.rasp_topk.restype = ctypes.c_int
    lib.rasp_nccl_unique_id.argtypes = [P]
    lib.rasp_nccl_unique_id.restype = ctypes.c_int
    lib.rasp_nccl_comm_init.argtypes = [ctypes.c_int, P, ctypes.c_int, ctypes.POINTER(ctypes.c_void_p)]
    lib.rasp_nccl_comm_init.restype = ctypes.c_int
    lib.rasp_nccl_comm_destroy.argtypes = [P]
    lib.rasp_nccl_comm_destroy.restype = ctypes.c_int
    lib.rasp_shard_allreduce.argtypes = [P, P, U64, P]
    lib.rasp_shard_allreduce.restype = ctypes.c_int
    lib.rasp_shard_gather.argtypes = [P, ctypes.c_int, pp, U64, pb, pb, U32, P]
    lib.rasp_shard_gather.restype = ctypes.c_int
    lib.rasp_launch_count.argtypes = []
    lib.rasp_launch_count.restype = ctypes.c_ulonglong
    if lib.rasp_abi_version() != ABI_VERSION:
        raise NativeError(f"{LIB_PATH}: ABI version {lib.rasp_abi_version()} != {ABI_VERSION}")
    _lib = lib
    return lib


def check(rc: int, what: str) -> None:
    if rc != 0:
        lib = load()
        msg = lib.rasp_error_string(rc).decode()
        if rc in (-3, -6):
            msg += f" ({lib.rasp_last_cuda_error().decode()})"
        raise NativeError(f"{what} failed: {msg} [code {rc}]")
