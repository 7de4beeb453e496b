"""Loader for the reference-generated golden fixtures (tests/golden/*.npz)."""

from __future__ import annotations

import os
from dataclasses import dataclass

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
FAMILIES = ("kat", "edge", "corpus", "hyp", "bb", "paper", "paper100", "gen")
FIELDS = ("iw", "ac", "M", "u", "y")
RESULTS = FIELDS + ("status", "steps", "tau_h")


@dataclass
class Group:
    family: str
    name: str
    w: int
    n: int
    ell: int
    s: int
    tau_max: int
    c0: dict
    out: dict
    hist: np.ndarray

    @property
    def d(self) -> int:
        return self.c0["iw"].shape[0]

    def __repr__(self):
        return (f"{self.family}/{self.name}(w={self.w}, n={self.n}, ell={self.ell}, "
                f"s={self.s}, tau={self.tau_max}, d={self.d})")


def load_family(family: str) -> list:
    z = np.load(os.path.join(GOLDEN, f"{family}.npz"))
    names = sorted({k.split("_")[0] for k in z.files if k.startswith("g")})
    groups = []
    for g in names:
        w, n, ell, s, tau = (int(v) for v in z[f"{g}_meta"])
        groups.append(Group(family, g, w, n, ell, s, tau,
                            {k: z[f"{g}_c0_{k}"] for k in FIELDS},
                            {k: z[f"{g}_out_{k}"] for k in RESULTS},
                            z[f"{g}_hist"]))
    return groups


def load_all(families=FAMILIES) -> list:
    out = []
    for f in families:
        out.extend(load_family(f))
    return out


def load_raw(family: str):
    return np.load(os.path.join(GOLDEN, f"{family}.npz"))
