"""Replay of the epoch schedule on measured halting times (analysis only).

Runs a C2-shaped sample through the engine (GPU) to get every machine's
halting time, then replays the device schedule (tiles of 32 list entries, a
tile runs until its last lane halts or the epoch cap, survivors compacted)
and reports per-epoch lane utilisation and a time estimate from two costs
calibrated on the C2 ncu capture (per warp-step and per tile load+store).

    python scripts/epoch_model.py [--d 65536] [--k0 48] [--q 0.5]
"""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

C_STEP = 1 / (115 * 148)   # us per warp-step, aggregated over 148 SMs (long-epoch rate)
C_TILE = 0.36 / 148        # us per tile load + write-back, aggregated


def halting_times(d, tau_max=1024):
    from paper_2604_12902_b200.hypervisor import BatchConfig, run_arrays
    from paper_2604_12902_b200.machine import MachineParams
    from paper_2604_12902_b200.workload import synthetic_c0
    p = MachineParams(w=16, n=64, ell=8, s=8)
    res = run_arrays(synthetic_c0(d, p, seed=0), p, BatchConfig(tau_max=tau_max))
    st, th = np.asarray(res.slots.status), np.asarray(res.slots.tau_h)
    return np.where(st == 1, th, tau_max).astype(np.int64)


def replay(need, k0, q, scale, seed=0):
    rng = np.random.default_rng(seed)
    prog = np.zeros(len(need), np.int64)
    live = np.arange(len(need))
    k, stable, total = k0, False, 0.0
    while len(live):
        rem = need[live] - prog[live]
        n = len(live)
        nt = (n + 31) // 32
        pad = np.full(nt * 32, -1)
        pad[:n] = rem
        run = np.minimum(pad.reshape(nt, 32).max(1), k)
        per = np.repeat(run, 32)[:n]
        useful = np.minimum(rem, per).sum()
        t = (run.sum() * C_STEP + nt * C_TILE) * scale
        total += t
        print(f"epoch K={k:5d}: machines {n * scale / 1e3:7.0f}K  lane utilisation {useful / (run.sum() * 32):.2f}"
              f"  est {t:6.0f} us")
        done = rem <= per
        prog[live] += np.minimum(rem, per)
        surv = live[~done]
        if not stable and len(surv) / n >= q:
            stable = True
        k = int((need[surv] - prog[surv]).max()) if (stable and len(surv)) else 2 * k
        live = rng.permutation(surv)
    print(f"total est {total:.0f} us")


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--d", type=int, default=1 << 16)
    ap.add_argument("--k0", type=int, default=48)
    ap.add_argument("--q", type=float, default=0.5)
    a = ap.parse_args()
    need = halting_times(a.d)
    replay(need, a.k0, a.q, (1 << 20) / a.d)
