"""Generate the golden parity fixtures from the REFERENCE itself.

Run in the build container (the only place /root/reference exists):

    NUMBA_CACHE_DIR=/tmp/numba_cache PYTHONDONTWRITEBYTECODE=1 \
        python tests/golden/make_golden.py

Every fixture stores the input configurations (uint64, the reference's own
layout) and what the reference's public batch operator
``raspvisor.hypervisor.run_batch`` (hypervisor.py:265-323) returned for them:
final iw/ac/M/u/y, status, steps, tau_h.  Families:

  kat     single-step examples of tests/test_machine.py:90-166 + the run-loop
          examples of :170-208, at tau_max in {0, 1, 2, 64}
  edge    SURVEY.md §8c edge vectors (i)-(vii)
  corpus  selftest.random_config_corpus(300, seed=21) (the batch-vs-scalar
          test of tests/test_hypervisor.py:27-43), tau_max in {1, 37, 200}
  hyp     seeded draws shaped like tests/test_machine.py:213-230
          (w in {1,4,8,16,32,64}, n in [2,12]), tau_max in {0, 1, 50}
  bb      the three Appendix-B busy-beaver fixtures lowered at p32
          (tests/test_lowering.py:179-187: tau_h 1727/1409/1387, y=(1,0))
  paper   build_workload(30, 64, seed=3, p32) (hypervisor.py:362-384), tau 10^4
  paper100  build_workload(100, 512, seed=5, p32): the paper protocol's program
          length L=100 at its tau_max = 10^6; `nin` holds
          each program's input count (sampler ast.n_in)
  gen_*   generator G at C1 (4096, w8 n32 l4 s4, 64 steps) and
          small samples of the C2 and C5 shapes at cap 1024

The reference cannot travel to the GPU box; these .npz files do.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
REF_SRC = "/root/reference/pkg/src"
REF_FIX = "/root/reference/pkg/tests/fixtures"

sys.path.insert(0, REF_SRC)
sys.path.insert(0, REPO)
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

from raspvisor import hypervisor as H  # noqa: E402
from raspvisor import machine as RM  # noqa: E402
from raspvisor.lang import parse_source  # noqa: E402
from raspvisor.lowering import lower  # noqa: E402
from raspvisor.selftest import random_config_corpus  # noqa: E402

from paper_2604_12902_b200.machine import MachineParams as OurParams  # noqa: E402
from paper_2604_12902_b200.workload import synthetic_c0  # noqa: E402

BIG = 1 << 40


def _arrays(configs, p):
    d = len(configs)
    return {
        "iw": np.array([c.i for c in configs], np.uint64).reshape(d),
        "ac": np.array([c.a for c in configs], np.uint64).reshape(d),
        "M": np.array([c.M for c in configs], np.uint64).reshape(d, p.n),
        "u": np.array([c.u for c in configs], np.uint64).reshape(d, p.ell + 1),
        "y": np.array([c.y for c in configs], np.uint64).reshape(d, p.s + 1),
    }


def _configs(arrs):
    d = arrs["iw"].shape[0]
    return [RM.Config(int(arrs["iw"][k]), int(arrs["ac"][k]),
                      tuple(int(v) for v in arrs["M"][k]),
                      tuple(int(v) for v in arrs["u"][k]),
                      tuple(int(v) for v in arrs["y"][k])) for k in range(d)]


class Family:
    def __init__(self, name):
        self.name = name
        self.data = {}
        self.groups = 0

    def add(self, p, tau_max, c0_arrays, epoch=64):
        configs = _configs(c0_arrays)
        res = H.run_batch(configs, p, H.BatchConfig(tau_max=tau_max, epoch=epoch,
                                                    memory_budget_words=BIG))
        g = f"g{self.groups:03d}"
        self.groups += 1
        self.data[f"{g}_meta"] = np.array([p.w, p.n, p.ell, p.s, tau_max], np.int64)
        for k, v in c0_arrays.items():
            self.data[f"{g}_c0_{k}"] = np.ascontiguousarray(v, np.uint64)
        sv = res.slots
        for k in ("iw", "ac", "M", "u", "y", "status", "steps", "tau_h"):
            self.data[f"{g}_out_{k}"] = np.ascontiguousarray(getattr(sv, k))
        # histogram over the reference's bucketing (hypervisor.py:329-352)
        hist = H.collect_histogram(sv)
        self.data[f"{g}_hist"] = np.array([hist[k] for k in H.HISTOGRAM_KEYS], np.int64)
        return res

    def save(self):
        path = os.path.join(HERE, f"{self.name}.npz")
        np.savez_compressed(path, **self.data)
        print(f"{self.name}: {self.groups} groups -> {os.path.relpath(path, REPO)} "
              f"({os.path.getsize(path) / 1024:.1f} KiB)")


def fam_kat():
    f = Family("kat")
    P8 = RM.MachineParams(w=8, n=8, ell=2, s=2, mu=1)

    def cfg(i=0, a=0, M=(0,) * 8, u=(0, 0, 0), y=(0, 0, 0)):
        return RM.Config(i, a, tuple(M), tuple(u), tuple(y))

    cases = [
        cfg(a=250, M=(2, 2, 10) + (0,) * 5),          # ADD wraps
        cfg(a=16, M=(3, 2, 16) + (0,) * 5),           # MUL wraps
        cfg(M=(1, 77) + (0,) * 6),                    # LOD literal
        cfg(a=5, M=(4, 6) + (0,) * 6),                # STO
        cfg(a=1, M=(5, 7) + (0,) * 6),                # BNZ taken
        cfg(a=0, M=(5, 7) + (0,) * 6),                # BNZ fall through
        cfg(a=3, M=(5, 0) + (0,) * 6),                # BNZ self loop: fixed
        cfg(M=(6, 4) + (0,) * 6, u=(0, 42, 9)),       # RD
        cfg(M=(6, 4) + (0,) * 6, u=(2, 42, 9)),       # RD at capacity: fixed
        cfg(M=(7, 4, 0, 0, 42, 0, 0, 0)),             # PRI
        cfg(a=9, M=(7, 0) + (0,) * 6, y=(2, 5, 6)),   # PRI full: drops, advances
        cfg(),                                        # HLT
        cfg(i=7, M=(9, 1, 2, 3, 4, 5, 6, 7)),         # operand address wraps
    ]
    for prog in ((1, 5, 4, 6), (0, 0), (1, 5), (1, 1, 5, 0)):
        cases.append(RM.init_config(RM.Program(prog), [], P8))
    arrs = _arrays(cases, P8)
    for tau in (0, 1, 2, 64):
        f.add(P8, tau, arrs)
    # single-step reference outputs for the step-level KATs
    nxt = [RM.step_reference(c, P8) for c in cases]
    f.data["step_next"] = np.stack([
        np.concatenate([[o.next.i, o.next.a], o.next.M, o.next.u, o.next.y]).astype(np.uint64)
        for o in nxt])
    f.data["step_fixed"] = np.array([o.fixed_point for o in nxt], np.int8)
    f.save()


def fam_edge():
    """SURVEY.md §8c edge vectors (i)-(vii)."""
    f = Family("edge")
    p = RM.MachineParams(w=8, n=8, ell=2, s=2, mu=1)
    z8 = (0,) * 8
    cases = [
        RM.Config(0, 1, (5, 8) + z8[2:], (0, 0, 0), (0, 0, 0)),           # (i) BNZ to i+n
        RM.Config(1, 0, (0, 1, 9, 0, 0, 0, 0, 0), (0, 0, 0), (0, 0, 0)),  # (ii) odd i
        RM.Config(255, 0, (42, 0, 0, 0, 0, 0, 0, 1), (0, 0, 0), (0, 0, 0)),  # (iii) wrap
        RM.Config(0, 0, (7, 0) + z8[2:], (0, 0, 0), (2, 1, 2)),           # (v) PRI full
        RM.Config(0, 0, (6, 3) + z8[2:], (2, 5, 6), (0, 0, 0)),           # (vi) RD at cap
    ]
    f.add(p, 5, _arrays(cases, p))
    f.add(p, 1, _arrays(cases, p))
    p1 = RM.MachineParams(w=1, n=2, ell=1, s=1, mu=1)
    c = [RM.Config(0, 0, (1, 0), (0, 0), (0, 0)),                         # (iv) w=1 LOD j=a
         RM.Config(1, 1, (1, 1), (0, 1), (1, 1)),
         RM.Config(0, 1, (1, 1), (1, 0), (0, 0))]
    f.add(p1, 4, _arrays(c, p1))
    p250 = RM.MachineParams(w=32, n=250, ell=10, s=2, mu=10)
    M = [0] * 250
    M[1], M[2] = 1, 77                                                   # (vii) i=251
    f.add(p250, 3, _arrays([RM.Config(251, 0, tuple(M), (0,) * 11, (0,) * 3)], p250))
    f.save()


def fam_corpus():
    f = Family("corpus")
    cases = list(random_config_corpus(300, seed=21))
    by_p = {}
    for c, p in cases:
        by_p.setdefault(p, []).append(c)
    for tau, q in ((200, 64), (37, 5), (1, 1)):
        for p, configs in by_p.items():
            f.add(p, tau, _arrays(configs, p), epoch=q)
    f.save()


def fam_hyp():
    """Seeded draws with the shape of tests/test_machine.py:213-230."""
    f = Family("hyp")
    rng = np.random.default_rng(12345)
    for w in (1, 4, 8, 16, 32, 64):
        mask = (1 << w) - 1
        for n in (2, 3, 5, 8, 12):
            ell = int(rng.integers(1, min(4, mask) + 1))
            s = int(rng.integers(1, min(3, mask) + 1))
            p = RM.MachineParams(w=w, n=n, ell=ell, s=s, mu=1)
            d = 64

            def word(shape):
                small = rng.integers(0, min(9, mask) + 1, shape, dtype=np.uint64)
                full = rng.integers(0, mask, shape, dtype=np.uint64, endpoint=True)
                return np.where(rng.random(shape) < 0.5, small, full)

            M = word((d, n))
            # bias opcode cells so every case occurs often
            ops = rng.integers(0, 9, (d, n), dtype=np.uint64) & np.uint64(mask)
            M = np.where(rng.random((d, n)) < 0.6, ops, M)
            u = np.concatenate([rng.integers(0, ell + 1, (d, 1), dtype=np.uint64), word((d, ell))], 1)
            y = np.concatenate([rng.integers(0, s + 1, (d, 1), dtype=np.uint64), word((d, s))], 1)
            i = np.where(rng.random(d) < 0.5,
                         rng.integers(0, 2 * n + 1, d, dtype=np.uint64) & np.uint64(mask),
                         rng.integers(0, mask, d, dtype=np.uint64, endpoint=True))
            a = word(d)
            arrs = {"iw": i, "ac": a, "M": M, "u": u, "y": y}
            for tau in (0, 1, 50):
                f.add(p, tau, arrs)
    f.save()


def fam_bb():
    f = Family("bb")
    p32 = RM.MachineParams(w=32, n=250, ell=10, s=2, mu=10)
    configs = []
    for k in (1, 2, 3):
        with open(os.path.join(REF_FIX, f"bb{k}.arr"), encoding="utf-8") as fh:
            prog, _ = lower(parse_source(fh.read()), p32)
        configs.append(RM.init_config(prog, [], p32))
    res = f.add(p32, 10 ** 5, _arrays(configs, p32))
    assert [s.tau_h for s in res.slots] == [1727, 1409, 1387]
    f.save()


def fam_paper():
    f = Family("paper")
    p32 = RM.MachineParams(w=32, n=250, ell=10, s=2, mu=10)
    wl = H.build_workload(30, 64, 3, p32)
    f.add(p32, 10 ** 4, _arrays(wl.configs, p32))
    f.save()


def fam_paper100():
    f = Family("paper100")
    p32 = RM.MachineParams(w=32, n=250, ell=10, s=2, mu=10)
    wl = H.build_workload(100, 512, 5, p32, keep_asts=True)
    f.add(p32, 10 ** 6, _arrays(wl.configs, p32))
    f.data["nin"] = np.array([a.n_in for a in wl.asts], np.int64)
    f.save()


def fam_gen():
    f = Family("gen")
    for d, (w, n, ell, s), tau in ((4096, (8, 32, 4, 4), 64),
                                   (4096, (16, 64, 8, 8), 1024),
                                   (512, (32, 256, 32, 32), 1024)):
        ours = OurParams(w=w, n=n, ell=ell, s=s, mu=1)
        c0 = {k: v.astype(np.uint64) for k, v in synthetic_c0(d, ours, seed=0).items()}
        f.add(RM.MachineParams(w=w, n=n, ell=ell, s=s, mu=1), tau, c0)
    f.save()


def fam_packer():
    """Inputs and outputs of the reference's packer init_config (m:289-309)
    for the programs the bb/paper/paper100 families run: the lowered program
    words (zero-padded to the longest program, `plen` = each length), the
    sampled input words (zero-padded, `xlen` = each count) and the c0 that
    init_config returned.  The device packer rasp_init_c0 is pinned to it."""
    from raspvisor.sampler import sample_inputs, sample_program
    p32 = RM.MachineParams(w=32, n=250, ell=10, s=2, mu=10)
    data = {}
    sets = {}
    progs = []
    for k in (1, 2, 3):
        with open(os.path.join(REF_FIX, f"bb{k}.arr"), encoding="utf-8") as fh:
            prog, _ = lower(parse_source(fh.read()), p32)
        progs.append((prog, ()))
    sets["bb"] = progs
    for name, length, count, seed in (("paper", 30, 64, 3), ("paper100", 100, 512, 5)):
        progs = []
        for k in range(count):   # the loop of build_workload (hypervisor.py:362-384)
            ast = sample_program(length, seed, k, None)
            inputs = sample_inputs(ast.n_in, p32.w, seed, k)
            try:
                prog, _ = lower(ast, p32)
            except RM.CapacityError:
                continue
            progs.append((prog, tuple(inputs)))
        sets[name] = progs
    for name, progs in sets.items():
        L = max(len(pr.words) for pr, _ in progs)
        X = max(1, max(len(x) for _, x in progs))
        P = np.zeros((len(progs), L), np.uint64)
        Xa = np.zeros((len(progs), X), np.uint64)
        for r, (pr, x) in enumerate(progs):
            P[r, :len(pr.words)] = pr.words
            Xa[r, :len(x)] = x
        c0 = _arrays([RM.init_config(pr, x, p32) for pr, x in progs], p32)
        data[f"{name}_prog"] = P
        data[f"{name}_plen"] = np.array([len(pr.words) for pr, _ in progs], np.int64)
        data[f"{name}_inp"] = Xa
        data[f"{name}_xlen"] = np.array([len(x) for _, x in progs], np.int64)
        for k, v in c0.items():
            data[f"{name}_c0_{k}"] = v
    path = os.path.join(HERE, "packer.npz")
    np.savez_compressed(path, **data)
    print(f"packer: {sorted(sets)} -> {os.path.relpath(path, REPO)} ({os.path.getsize(path) / 1024:.1f} KiB)")


ALL = (fam_kat, fam_edge, fam_corpus, fam_hyp, fam_bb, fam_paper, fam_paper100, fam_gen, fam_packer)

if __name__ == "__main__":
    H._warm_kernel()
    only = set(sys.argv[1:])   # optional family names
    for fam in ALL:
        if not only or fam.__name__[4:] in only:
            fam()
