"""Replay of the epoch schedule on measured halting times (analysis only).

Runs a C2-shaped sample through the engine (GPU) to get every machine's
halting time, then replays the device schedule (tiles of 32 list entries, a
tile runs until its last lane halts or the epoch cap, survivors compacted)
and reports per-epoch lane utilisation and a time estimate from two costs
calibrated on the C2 ncu capture (per warp-step and per tile load+store).

    python scripts/epoch_model.py [--d 65536] [--k0 48] [--tau 1024]

The epoch lengths follow the device planner (plan_next mirrors the tail of
epoch_kernel: doubling, the stable/jump rule, the no-sliver merge, the kmax
cap and the budget clamp).
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


def plan_next(count, cout, K, cov, tau, stable_q8=128, stable_hi_q8=243, jump=16, growth=2, kmax=1 << 24):
    """The next epoch length exactly as the last block of epoch e plans it
    (rasp_kernels.cuh, the tail of epoch_kernel): 0 when nothing is left."""
    left = tau - (cov + K)
    if cout == 0 or left <= 0:
        return 0
    kk = K if K > 0 else 1
    stable = (256 * cout >= stable_q8 * count and left <= jump * kk) or 256 * cout >= stable_hi_q8 * count
    want = left if stable else growth * kk
    if left > want and left - want < (want >> 2):   # no slivers
        want = left
    return int(min(want, left, kmax))


def replay(need, k0, tau, scale, unroll=8, seed=0):
    """need[j] = machine j's halting time (tau if it never halts)."""
    rng = np.random.default_rng(seed)
    live = np.arange(len(need))
    K, cov, total = min(k0, tau), 0, 0.0
    while len(live) and K > 0:
        rem = need[live] - cov            # steps machine j still needs
        n = len(live)
        nt = (n + 31) // 32
        pad = np.zeros(nt * 32, np.int64)
        pad[:n] = rem
        # a warp runs until its last lane is done (checked every `unroll` steps) or K
        run = np.minimum(-(-pad.reshape(nt, 32).max(1) // unroll) * unroll, K)
        useful = np.minimum(rem, K).sum()
        t = (run.sum() * C_STEP + nt * C_TILE) * scale
        total += t
        print(f"epoch K={K:7d}: machines {n * scale / 1e3:7.0f}K  lane utilisation {useful / (run.sum() * 32):.2f}"
              f"  est {t:6.0f} us")
        done = rem <= K                    # halted inside the epoch, fixed at K, or out of budget
        surv = live[~done]
        K, cov = plan_next(n, len(surv), K, cov, tau), cov + K
        live = rng.permutation(surv)
    print(f"total est {total:.0f} us")


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--d", type=int, default=1 << 16)
    ap.add_argument("--k0", type=int, default=48)
    ap.add_argument("--tau", type=int, default=1024)
    a = ap.parse_args()
    need = halting_times(a.d, a.tau)
    replay(need, a.k0, a.tau, (1 << 20) / a.d)
