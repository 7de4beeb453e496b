"""Machine shape, configurations and initial configurations (host side).

Mirrors the value types of raspvisor/machine.py that the batch path consumes:
``MachineParams`` (machine.py:62-115), ``Config`` (:118-129), ``Program``
(:137-153), ``init_config`` (:289-309) and ``validate_config`` (:312-333),
with the same argument meaning and error classes.  The transition map itself
is not here: it runs on the GPU (csrc/rasp_kernels.cu).

Additions for the batch path: ``natural_dtype`` (the smallest unsigned numpy
type holding a w-bit word, the HBM cell type) and ``init_batch`` (c0 for a
whole batch as SoA arrays, without per-machine tuples).
"""

from __future__ import annotations

import json
from dataclasses import dataclass
from enum import IntEnum
from typing import NamedTuple

import numpy as np

from .errors import CapacityError


class Opcode(IntEnum):
    """Opcode words (machine.py:49-59).  Every other word is not executable."""
    HLT = 0
    LOD = 1
    ADD = 2
    MUL = 3
    STO = 4
    BNZ = 5
    RD = 6
    PRI = 7


def natural_dtype(w: int) -> np.dtype:
    """Smallest unsigned type with at least w bits: the HBM cell width."""
    for bits, dt in ((8, np.uint8), (16, np.uint16), (32, np.uint32), (64, np.uint64)):
        if w <= bits:
            return np.dtype(dt)
    raise ValueError(f"word width w must be in [1, 64], got {w}")


class MachineParams:
    """Word width w, memory size n, input capacity ell, output capacity s,
    scratch capacity mu.  Immutable and hashable; ell and s must be words."""

    __slots__ = ("w", "n", "ell", "s", "mu", "mask")

    def __init__(self, w: int = 32, n: int = 250, ell: int = 10, s: int = 2, mu: int = 10):
        checks = (
            (1 <= w <= 64, f"word width w must be in [1, 64], got {w}"),
            (n >= 2, f"memory size n must be >= 2, got {n}"),
            (ell >= 1, f"input capacity ell must be >= 1, got {ell}"),
            (s >= 1, f"output capacity s must be >= 1, got {s}"),
            (mu >= 1, f"scratch capacity mu must be >= 1, got {mu}"),
        )
        for ok, msg in checks:
            if not ok:
                raise ValueError(msg)
        if ell >> w:
            raise ValueError(f"ell must be < 2^w = {1 << w}, got {ell}")
        if s >> w:
            raise ValueError(f"s must be < 2^w = {1 << w}, got {s}")
        for name, v in (("w", w), ("n", n), ("ell", ell), ("s", s), ("mu", mu),
                        ("mask", (1 << w) - 1)):
            object.__setattr__(self, name, v)

    def __setattr__(self, name, value):
        raise AttributeError("MachineParams is immutable")

    def _key(self):
        return (self.w, self.n, self.ell, self.s, self.mu)

    def __eq__(self, other):
        if not isinstance(other, MachineParams):
            return NotImplemented
        return self._key() == other._key()

    def __hash__(self):
        return hash(self._key())

    def __repr__(self):
        w, n, ell, s, mu = self._key()
        return f"MachineParams(w={w}, n={n}, ell={ell}, s={s}, mu={mu})"

    @property
    def words_per_machine(self) -> int:
        """Words of VM state per machine, as counted by the memory budget
        check of hypervisor.py:272 (n + ell + s + 4)."""
        return self.n + self.ell + self.s + 4

    @property
    def dtype(self) -> np.dtype:
        return natural_dtype(self.w)

    def to_json(self) -> dict:
        return dict(zip(("w", "n", "ell", "s", "mu"), self._key()))

    @classmethod
    def from_json(cls, obj: dict) -> "MachineParams":
        return cls(**{k: obj[k] for k in ("w", "n", "ell", "s", "mu")})


class Config(NamedTuple):
    """(i, a, M, u, y): u[0] is the read cursor, y[0] the write count."""
    i: int
    a: int
    M: tuple
    u: tuple
    y: tuple


@dataclass(frozen=True)
class Program:
    """Even-length word vector of (opcode, operand) pairs."""
    words: tuple

    def __post_init__(self):
        if len(self.words) & 1:
            raise ValueError(
                f"program must have an even word count, got {len(self.words)}")

    @property
    def m(self) -> int:
        return len(self.words) >> 1

    def pairs(self):
        return list(zip(self.words[0::2], self.words[1::2]))


def _check_words(kind: str, values, w: int):
    top = 1 << w
    for v in values:
        if v < 0 or v >= top:
            raise ValueError(f"{kind} word {v} out of range for w = {w}")


def init_config(program: Program, inputs, p: MachineParams) -> Config:
    """c0(P, x) = <0, 0, P 0^(n-2m), (0, x 0^(ell-|x|)), 0^(s+1)>."""
    words = tuple(program.words)
    inputs = tuple(inputs)
    if len(words) > p.n:
        raise CapacityError(f"program needs {len(words)} memory words but n = {p.n}")
    if len(inputs) > p.ell:
        raise CapacityError(f"input vector has {len(inputs)} words but ell = {p.ell}")
    _check_words("program", words, p.w)
    _check_words("input", inputs, p.w)
    return Config(0, 0,
                  words + (0,) * (p.n - len(words)),
                  (0,) + inputs + (0,) * (p.ell - len(inputs)),
                  (0,) * (p.s + 1))


def validate_config(c: Config, p: MachineParams, deep: bool = False) -> None:
    """ValueError unless c is well-formed for p (shapes and cursor ranges;
    deep=True also range-checks every word)."""
    for name, vec, want, what in (("M", c.M, p.n, "n"),
                                  ("u", c.u, p.ell + 1, "ell+1"),
                                  ("y", c.y, p.s + 1, "s+1")):
        if len(vec) != want:
            raise ValueError(f"{name} has {len(vec)} cells, expected {what} = {want}")
    if not 0 <= c.u[0] <= p.ell:
        raise ValueError(f"read cursor u[0] = {c.u[0]} outside [0, {p.ell}]")
    if not 0 <= c.y[0] <= p.s:
        raise ValueError(f"write count y[0] = {c.y[0]} outside [0, {p.s}]")
    if deep:
        top = 1 << p.w
        for name, vec in (("i", (c.i,)), ("a", (c.a,)), ("M", c.M), ("u", c.u), ("y", c.y)):
            for v in vec:
                if not 0 <= v < top:
                    raise ValueError(f"{name} holds word {v} out of range for w = {p.w}")


def init_batch(programs, inputs, p: MachineParams, dtype=None) -> dict:
    """c0 for a whole batch as SoA arrays (iw, ac, M, u, y).

    `programs` is a [d, L] integer array (L <= n, L even) or a sequence of
    Program; `inputs` is a [d, k] array (k <= ell) or a sequence of word
    sequences.  Same errors as init_config, raised for the first offender."""
    dt = np.dtype(dtype) if dtype is not None else p.dtype
    if isinstance(programs, np.ndarray):
        P = programs
    else:
        progs = [pr.words if isinstance(pr, Program) else tuple(pr) for pr in programs]
        L = max((len(w) for w in progs), default=0)
        P = np.zeros((len(progs), L), np.uint64)
        for k, words in enumerate(progs):
            if len(words) & 1:
                raise ValueError(f"program must have an even word count, got {len(words)}")
            P[k, :len(words)] = words
    d = P.shape[0]
    if isinstance(inputs, np.ndarray):
        X = inputs.reshape(d, -1) if inputs.size else np.zeros((d, 0), np.uint64)
    else:
        xs = [tuple(x) for x in inputs]
        if len(xs) != d:
            raise ValueError(f"{len(xs)} input vectors for {d} programs")
        K = max((len(x) for x in xs), default=0)
        X = np.zeros((d, K), np.uint64)
        for k, x in enumerate(xs):
            if len(x) > p.ell:
                raise CapacityError(f"input vector has {len(x)} words but ell = {p.ell}")
            X[k, :len(x)] = x
    if P.shape[1] > p.n:
        raise CapacityError(f"program needs {P.shape[1]} memory words but n = {p.n}")
    if X.shape[1] > p.ell:
        raise CapacityError(f"input vector has {X.shape[1]} words but ell = {p.ell}")
    if p.w < 64:
        for kind, arr in (("program", P), ("input", X)):
            if arr.size and (np.asarray(arr) < 0).any():
                raise ValueError(f"{kind} word out of range for w = {p.w}")
            if arr.size and int(np.asarray(arr).max()) > p.mask:
                raise ValueError(f"{kind} word {int(arr.max())} out of range for w = {p.w}")
    M = np.zeros((d, p.n), dt)
    M[:, :P.shape[1]] = P
    u = np.zeros((d, p.ell + 1), dt)
    u[:, 1:1 + X.shape[1]] = X
    return {"iw": np.zeros(d, dt), "ac": np.zeros(d, dt), "M": M, "u": u,
            "y": np.zeros((d, p.s + 1), dt)}


# --- serialization (machine.py:362-408 wire formats) ---------------------------

def program_to_json(program: Program, w: int) -> str:
    return json.dumps({"w": w, "words": list(program.words)})


def program_from_json(text: str):
    obj = json.loads(text)
    w = obj["w"]
    if not 1 <= w <= 64:
        raise ValueError(f"bad word width {w}")
    words = obj["words"]
    for v in words:
        if not isinstance(v, int):
            raise ValueError(f"word {v} out of range for w = {w}")
    _check_words("program", words, w)
    return Program(tuple(words)), w


def program_to_bytes(program: Program, w: int) -> bytes:
    nb = (w + 7) // 8
    return b"".join(int(v).to_bytes(nb, "little") for v in program.words)


def program_from_bytes(data: bytes, w: int) -> Program:
    nb = (w + 7) // 8
    if len(data) % nb:
        raise ValueError(f"byte length {len(data)} is not a multiple of the word size {nb}")
    words = tuple(int.from_bytes(data[k:k + nb], "little") for k in range(0, len(data), nb))
    _check_words("program", words, w)
    return Program(words)


def config_to_json(c: Config) -> str:
    return json.dumps({"i": c.i, "a": c.a, "M": list(c.M), "u": list(c.u), "y": list(c.y)})


def config_from_json(text: str) -> Config:
    o = json.loads(text)
    return Config(o["i"], o["a"], tuple(o["M"]), tuple(o["u"]), tuple(o["y"]))
