"""Benchmark of the hot path: Phi over a batch of word-RASP machines.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--impl ours|reference]

Workload (BASELINE.json configs[1]): per GPU, 2^20 synthetic
programs from generator G (seed = rank), w=16, n=64, ell=8, s=8, run to halt
with a 1024-step cap.  Each rank runs its own shard (weak scaling; no
collective on the data path -- after the run the 102-bucket halting
histogram, i.e. the halt counts, is all-reduced over NCCL and rank 0 gathers
every shard's verdicts and output tapes; --gather off keeps the
results on their GPUs).  --config c3 is BASELINE configs[2]: 16M machines in
total split across the ranks (strong scaling), with the same collectives;
c1 and c5 are configs[0] and configs[4].

One "step" = one full run of the batch from c0 (out-of-place, c0 is never
modified) with the halting histogram counted inside the run (rasp_run_hist).  Metric: machine-steps/s
(sum of per-machine applied steps, hypervisor.py:153, over all ranks / max
per-rank device time).

--impl reference times the reference algorithm on the host cores instead:
the C restatement of _worker (oracle/rasp_oracle.c, hv:72-164) driven with
the reference's striped thread schedule (hv:295-314) over all host threads,
on a bounded sample of the same workload.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: (d per GPU, w, n, ell, s, tau_max, description)
    "c1": (4096, 8, 32, 4, 4, 64, "4096 random programs, w=8 n=32 l=4 s=4, 64 steps"),
    "c2": (1 << 20, 16, 64, 8, 8, 1024,
           "1M random programs/GPU, w=16 n=64 l=8 s=8, run to halt (cap 1024)"),
    "c3": (1 << 24, 16, 64, 8, 8, 1024,
           "16M random programs/GPU, w=16 n=64 l=8 s=8, run to halt (cap 1024)"),
    "c5": (1 << 20, 32, 256, 32, 32, 1024,
           "1M random programs/GPU, w=32 n=256 l=32 s=32, divergent halting (cap 1024)"),
    # the paper protocol's geometry with the 64
    # programs the reference's sampler+compiler produce for L=30 (golden fixture),
    # tiled to 1M machines with fresh random inputs, tau 10^4
    "paper": (1 << 20, 32, 250, 10, 2, 10000,
              "1M machines: 64 sampled+lowered L=30 programs (reference build_workload) x random "
              "inputs, w=32 n=250 l=10 s=2, tau 10^4"),
    # SURVEY §8f f3 at the paper's own protocol: L=100 programs sampled and
    # lowered by the reference (golden fixture paper100, 512 programs), tiled to
    # 1M machines with fresh random inputs, tau_max 10^6
    "paper6": (1 << 20, 32, 250, 10, 2, 10 ** 6,
               "1M machines: 512 sampled+lowered L=100 programs (reference build_workload) x random "
               "inputs, w=32 n=250 l=10 s=2, tau 10^6 (the paper protocol)"),
    # d = programs; machines = programs x 2^w inputs (SURVEY §8d C4 domain)
    "c4": (1 << 28, 8, 16, 1, 1, 64,
           "exhaustive: all 2^28 programs of m=4 pairs (3-bit opcode, 4-bit operand), w=8 n=16, "
           "x all 256 inputs, tau 64, per-program records"),
}
N_ALG_INSTR = 40   # algorithmic integer issues per machine-step


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            pk = json.load(f)
        return float(pk["hbm_gbs"]), float(pk.get("sm_max_mhz", 1965.0)), "measured"
    except Exception:
        return 6650.0, 1965.0, "fallback"


def s_alg_bytes(w, n, ell, s):
    bw = 1 if w <= 8 else 2 if w <= 16 else 4 if w <= 32 else 8
    return (n + ell + s + 4) * bw + 8


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []
        self.t = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.t.join(timeout=2)
        sm, mx, reasons = [], None, set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


def make_c0(cfg_name, d, p, seed):
    """Host c0 for a config: generator G, or the paper-protocol programs."""
    from paper_2604_12902_b200.workload import synthetic_c0
    if cfg_name not in ("paper", "paper6"):
        return synthetic_c0(d, p, seed=seed)
    fam = "paper" if cfg_name == "paper" else "paper100"
    z = np.load(os.path.join(ROOT, "tests", "golden", f"{fam}.npz"))
    M0, u0 = z["g000_c0_M"].astype(np.uint32), z["g000_c0_u"].astype(np.uint32)
    reps = -(-d // M0.shape[0])
    M = np.tile(M0, (reps, 1))[:d]
    u = np.tile(u0, (reps, 1))[:d]
    rng = np.random.default_rng(seed)
    fresh = rng.integers(0, 1 << 32, u.shape, dtype=np.uint64).astype(np.uint32)
    if "nin" in z.files:   # each program's own input count (sampler ast.n_in)
        nin = np.tile(z["nin"], reps)[:d]
        used = np.arange(u.shape[1])[None, :] <= nin[:, None]
    else:                  # inputs the sampled configuration set
        used = np.tile((u0 != 0), (reps, 1))[:d]
    used[:, 0] = False
    u = np.where(used, fresh, u)
    return {"iw": np.zeros(d, np.uint32), "ac": np.zeros(d, np.uint32), "M": np.ascontiguousarray(M),
            "u": np.ascontiguousarray(u), "y": np.zeros((d, p.s + 1), np.uint32)}


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


# machines in the single-thread (W=1) sample per config: about 2-4 s of CPU work
W1_SAMPLE = {"c1": 4096, "c2": 1 << 17, "c3": 1 << 17, "c5": 1 << 15, "paper": 1 << 15, "paper6": 256}
# machines in the all-threads sample: the whole batch up to 2^20 (paper6: its
# machines run ~2e5 steps each)
WALL_SAMPLE = {"paper6": 8192}


def _load_numba_reference():
    """The unmodified reference (baseline/_ref, pip-installed from the reference
    package) -- its numba kernel _worker and JIT warm-up; None if absent."""
    ref = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "raspvisor")):
        return None
    os.environ.setdefault("NUMBA_CACHE_DIR", os.path.join("/tmp", "raspvisor_numba_cache"))
    if ref not in sys.path:
        sys.path.insert(0, ref)
    try:
        from raspvisor import hypervisor as RH
        RH._warm_kernel()          # compile off the clock, as run_batch does (hv:302)
        return RH
    except Exception:               # numba missing or broken: report the port only
        return None


class _CpuBatch:
    """c0 converted once to the reference's uint64 SoA arrays (hv:280-293),
    reset into preallocated work arrays before every timed run -- conversion
    and allocation stay off the clock, exactly as in run_batch, where the
    timer brackets only the threaded _worker dispatch (hv:303-315)."""

    def __init__(self, c0, d):
        self.base = {k: np.ascontiguousarray(np.asarray(c0[k])[:d]).astype(np.uint64) for k in
                     ("iw", "ac", "M", "u", "y")}
        self.work = {k: np.empty_like(v) for k, v in self.base.items()}
        self.work["status"] = np.empty(d, np.int8)
        self.work["steps"] = np.empty(d, np.int64)
        self.work["tau_h"] = np.empty(d, np.int64)
        self.d = d

    def reset(self):
        for k, v in self.base.items():
            np.copyto(self.work[k], v)
        self.work["status"].fill(0)
        self.work["steps"].fill(0)
        self.work["tau_h"].fill(-1)
        return self.work


def _time_port(cb, w, n, ell, s, tau, W, reps):
    from oracle import oracle
    best = float("inf")
    for _ in range(reps):
        a = cb.reset()
        t0 = time.perf_counter()
        oracle.oracle_run(a["iw"], a["ac"], a["M"], a["u"], a["y"], a["status"], a["steps"], a["tau_h"],
                          w, n, ell, s, tau, 64, W)
        best = min(best, time.perf_counter() - t0)
    return best, int(cb.work["steps"].sum())


def _time_numba(RH, cb, mask, n, ell, s, tau, W, reps):
    """hv:295-315 verbatim: q = 64, rounds = ceil(tau/q), W stripes on a
    ThreadPoolExecutor (W = 1: one direct call)."""
    from concurrent.futures import ThreadPoolExecutor
    q = 64
    rounds = (tau + q - 1) // q
    args = (np.uint64(mask), np.uint64(n), np.uint64(ell), np.uint64(s))
    best = float("inf")
    for _ in range(reps):
        a = cb.reset()
        t0 = time.perf_counter()
        if W == 1:
            RH._worker(a["iw"], a["ac"], a["M"], a["u"], a["y"], a["status"], a["steps"], a["tau_h"],
                       0, 1, q, rounds, tau, *args)
        else:
            with ThreadPoolExecutor(max_workers=W) as ex:
                fs = [ex.submit(RH._worker, a["iw"], a["ac"], a["M"], a["u"], a["y"], a["status"], a["steps"],
                                a["tau_h"], g, W, q, rounds, tau, *args) for g in range(W)]
                for f in fs:
                    f.result()
        best = min(best, time.perf_counter() - t0)
    return best, int(cb.work["steps"].sum())


def cpu_reference(cfg_name, reps=3, sample_d=None, seed=0, numba=True):
    """The reference algorithm on the host cores, timed like the reference
    times itself (hv:295-315): the C port of _worker (oracle/rasp_oracle.c)
    and, when staged in baseline/_ref, the reference's own numba _worker, each
    at W = 1 and W = all host threads, best of `reps` runs on preallocated
    uint64 arrays.  The headline value is the faster implementation at
    W = all threads."""
    from oracle import oracle
    from paper_2604_12902_b200.machine import MachineParams
    d, w, n, ell, s, tau, _ = CONFIGS[cfg_name]
    cores = len(os.sched_getaffinity(0))
    model = cpu_model()
    oracle.load()
    if cfg_name == "c4":
        from paper_2604_12902_b200.enumeration import C4
        out = {}
        for W, cnt in ((cores, min(d, (sample_d or (1 << 20)) // 4)), (1, 1 << 14)):
            best = float("inf")
            for _ in range(reps):
                t0 = time.perf_counter()
                _, st = oracle.enumerate_records(C4.m, C4.opcode_bits, C4.operand_bits, C4.w,
                                                 C4.n, C4.tau_max, 0, cnt, threads=W)
                best = min(best, time.perf_counter() - t0)
            out[W] = (st / best, cnt, st, best)
        v, cnt, st, best = out[cores]
        return {"value": v, "unit": "machine-steps/s", "cores": cores, "kind": "port",
                "sample": f"programs [0, {cnt}) of the C4 domain x 256 inputs, {st} machine-steps, "
                          f"W={cores} threads, best of {reps} (the reference has no enumeration kernel: "
                          f"the port of its step runs every (program, input) machine)",
                "seconds": best, "cpu_model": model, "port": {"value": v, "w1": out[1][0]},
                "reference_numba": None, "d_sample": cnt,
                "w1_sample": f"programs [0, {out[1][1]}) x 256 inputs, 1 thread"}
    p = MachineParams(w=w, n=n, ell=ell, s=s, mu=1)
    big = min(d, sample_d or (1 << 20), WALL_SAMPLE.get(cfg_name, 1 << 30))
    small = min(big, W1_SAMPLE.get(cfg_name, 1 << 16))
    c0 = make_c0(cfg_name, big, p, seed)
    src = "reference-sampled programs" if cfg_name.startswith("paper") else "generator G"
    cb_all, cb_one = _CpuBatch(c0, big), _CpuBatch(c0, small)
    t_all, st_all = _time_port(cb_all, w, n, ell, s, tau, cores, reps)
    t_one, st_one = _time_port(cb_one, w, n, ell, s, tau, 1, reps)
    port = {"value": st_all / t_all, "w1": st_one / t_one}
    want = {k: v.copy() for k, v in cb_one.work.items()}
    ref = None
    RH = _load_numba_reference() if numba else None
    if RH is not None:
        r_one, rs_one = _time_numba(RH, cb_one, p.mask, n, ell, s, tau, 1, reps)
        same = all(np.array_equal(cb_one.work[k], want[k]) for k in want)
        r_all, rs_all = _time_numba(RH, cb_all, p.mask, n, ell, s, tau, cores, reps)
        ref = {"value": rs_all / r_all, "w1": rs_one / r_one, "identical_to_port": bool(same),
               "source": "baseline/_ref raspvisor.hypervisor._worker (numba, unmodified)"}
    use_ref = ref is not None and ref["value"] > port["value"]
    value = ref["value"] if use_ref else port["value"]
    return {"value": value, "unit": "machine-steps/s", "cores": cores,
            "kind": "reference" if use_ref else "port",
            "sample": f"{big} machines of {cfg_name} ({src} seed {seed}), {st_all} machine-steps, "
                      f"_worker semantics, W={cores} threads, q=64, best of {reps}; "
                      f"headline = faster of the C port and the reference's numba kernel",
            "seconds": st_all / value, "cpu_model": model, "d_sample": big,
            "port": {"value": port["value"], "w1": port["w1"]},
            "reference_numba": ref,
            "w1_sample": f"{small} machines, {st_one} machine-steps, 1 thread"}


CPU_KEYS = ("value", "unit", "cores", "kind", "sample", "cpu_model", "port", "reference_numba", "w1_sample")


def bench_enumeration(args, world, rank, dev, desc):
    """BASELINE config 4: one step = the whole 2^28-program domain (sharded by
    contiguous rank ranges across GPUs), records left in HBM; e2e adds the
    D2H of every record."""
    import torch
    import torch.distributed as dist
    from paper_2604_12902_b200 import _native
    from paper_2604_12902_b200.enumeration import C4, enumerate_device
    from paper_2604_12902_b200.sharding import shard_bounds
    lib = _native.load()
    lo, hi = shard_bounds(C4.programs, world, rank)
    cnt = hi - lo
    rec = torch.empty(cnt, dtype=torch.uint64, device=dev)
    st = torch.zeros(1, dtype=torch.uint64, device=dev)
    stream = torch.cuda.current_stream(dev)
    for _ in range(max(args.warmup, 1)):
        st.zero_()
        enumerate_device(C4, lo, cnt, rec, st)
    torch.cuda.synchronize()
    steps = int(st.cpu().numpy()[0])
    allh = int((rec.view(torch.int64) < 0).sum().item())     # bit 63: halted on every input
    clocks = ClockSampler(int(os.environ.get("LOCAL_RANK", "0")))
    clocks.start()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    l0 = lib.rasp_launch_count()
    ts = []
    for _ in range(args.steps):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        enumerate_device(C4, lo, cnt, rec, st)
        e1.record(stream)
        ts.append((e0, e1))
    torch.cuda.synchronize()
    launches = lib.rasp_launch_count() - l0
    clk = clocks.stop()
    t_step = statistics.mean(a.elapsed_time(b) / 1e3 for a, b in ts)
    # e2e: run + copy every record to pinned host memory
    host = torch.empty(cnt, dtype=torch.uint64, pin_memory=True)
    te = []
    for _ in range(max(2, min(args.steps, 5))):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        enumerate_device(C4, lo, cnt, rec, st)
        host.copy_(rec, non_blocking=True)
        e1.record(stream)
        e1.synchronize()
        te.append(e0.elapsed_time(e1) / 1e3)
    t_e2e = statistics.mean(te)
    gloo = world > 1 and args.dist_backend == "gloo"
    tot = torch.tensor([t_step, t_e2e], dtype=torch.float64)
    agg = torch.tensor([steps, allh, cnt], dtype=torch.float64)
    if world > 1:
        if not gloo:
            tot, agg = tot.to(dev), agg.to(dev)
        dist.all_reduce(tot, op=dist.ReduceOp.MAX)
        dist.all_reduce(agg)
    t_step, t_e2e = (float(v) for v in tot.tolist())
    steps_all, allh_all, progs = (int(v) for v in agg.tolist())
    if rank == 0:
        _, sm_mhz, peak_kind = _peaks()
        issue_peak = 148 * 4 * 32 * sm_mhz * 1e6
        ach = steps * N_ALG_INSTR / t_step
        line = {
            "metric": "machine-steps/s", "value": steps_all / t_step, "unit": "machine-steps/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_step * 1e3,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u8",
            "data": "exhaustive (every program of the domain x every input, decoded on device)",
            "config": workload_config("c4", world),
            "run": {"programs": progs, "machines": progs * 256, "machine_steps": steps_all,
                    "all_halting_programs": allh_all,
                    "parallelism": f"{world} contiguous rank shards" if world > 1 else "1 GPU"},
            "programs_per_s": progs / t_step,
            "e2e": {"value": steps_all / t_e2e, "unit": "machine-steps/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": cnt * 8, "ms_per_step": t_e2e * 1e3},
            "gpu_launches": int(launches),
            "roofline": {"bound": "issue", "unit": "Tinstr/s", "achieved": ach / 1e12,
                         "peak": issue_peak / 1e12, "frac": ach / issue_peak, "traffic": None,
                         "kernel_ms": t_step * 1e3,
                         "per_unit": f"{N_ALG_INSTR} int-instr per machine-step (SURVEY §8d); "
                                     "decode and reduction are extra work not credited; HBM: 8 B per program "
                                     "(records), negligible"},
            "clocks": clk,
        }
        traffic, detail = _traffic("c4")
        line["roofline"]["traffic"], line["roofline"]["traffic_detail"] = traffic, detail
        if not args.no_cpu_baseline and world == 1:
            cb = cpu_reference("c4", reps=3, sample_d=args.cpu_sample)
            line["cpu_baseline"] = {k: cb[k] for k in CPU_KEYS}
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()


DEFAULT_EPOCH = {"c1": 64, "c2": 48, "c3": 48, "c5": 320, "paper": 32, "paper6": 32}
SHARD = 1 << 20          # machines per generator shard (c3 = 16 shards; other configs: one per rank)


def word_label(w: int) -> str:
    """The arithmetic/storage word of the run (natural width, DeviceBatch)."""
    return "u8" if w <= 8 else "u16" if w <= 16 else "u32" if w <= 32 else "u64"


def workload_config(cfg: str, world: int, shard: int = SHARD) -> dict:
    """The `config` object both arms print: the workload definition only
    (run-time facts go to `run`), so the two lines compare key for key."""
    d, w, n, ell, s, tau, desc = CONFIGS[cfg]
    if cfg == "c4":
        return {"workload": cfg, "desc": desc, "programs": d, "machines": d * 256, "w": w, "n": n,
                "ell": ell, "s": s, "tau_max": tau, "n_gpus": world, "scaling": "strong"}
    if cfg == "c3":
        d = (d // SHARD) * shard
        machines, scaling = d, "strong"
    else:
        machines, scaling = d * world, "weak"
    return {"workload": cfg, "desc": desc, "machines": machines, "w": w, "n": n, "ell": ell, "s": s,
            "tau_max": tau, "n_gpus": world, "scaling": scaling}


def rank_shards(cfg: str, world: int, rank: int, shard: int = SHARD) -> list:
    """Generator shards (seed = shard index) this rank runs.  c3 is ONE fixed
    batch of 16 shards split contiguously over the ranks (strong scaling: the
    N-GPU batch is the 1-GPU batch); the other configs give every rank one
    shard of its own (weak scaling: rank r runs shard r, so rank 0 always runs
    the 1-GPU batch)."""
    from paper_2604_12902_b200.sharding import shard_bounds
    if cfg == "c3":
        total = CONFIGS["c3"][0] // SHARD
        lo, hi = shard_bounds(total, world, rank)
        return [(k, shard) for k in range(lo, hi)]
    return [(rank, CONFIGS[cfg][0])]


def make_rank_c0(cfg, shards, p):
    parts = [make_c0(cfg, m, p, seed=k) for k, m in shards]
    if len(parts) == 1:
        return parts[0]
    return {k: np.concatenate([x[k] for x in parts]) for k in parts[0]}


def roofline(steps: int, d: int, w: int, n: int, ell: int, s: int, t_kernel: float) -> dict:
    """t_roof = max(t_HBM, t_issue); frac = t_roof / t_measured;
    the bound is the larger term.  Per GPU, for one rasp_run (all launches)."""
    hbm_gbs, sm_mhz, peak_kind = _peaks()
    bytes_alg = d * 2 * s_alg_bytes(w, n, ell, s)
    issue_peak = 148 * 4 * 32 * sm_mhz * 1e6                  # thread-instr/s
    t_hbm = bytes_alg / (hbm_gbs * 1e9)
    t_issue = steps * N_ALG_INSTR / issue_peak
    hbm = {"achieved": bytes_alg / t_kernel / 1e9, "peak": hbm_gbs, "unit": "GB/s",
           "frac": t_hbm / t_kernel, "t_ms": t_hbm * 1e3,
           "per_unit": f"S_alg={s_alg_bytes(w, n, ell, s)} B/machine read + written once",
           "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({peak_kind})"}
    issue = {"achieved": steps * N_ALG_INSTR / t_kernel / 1e12, "peak": issue_peak / 1e12, "unit": "Tinstr/s",
             "frac": t_issue / t_kernel, "t_ms": t_issue * 1e3,
             "per_unit": f"{N_ALG_INSTR} int-instr per machine-step (SURVEY §8d)",
             "peak_source": f"148 SM x 128 lanes x {sm_mhz:.0f} MHz ({peak_kind} sm_max_mhz)"}
    top = hbm if t_hbm >= t_issue else issue
    return {"bound": "hbm" if t_hbm >= t_issue else "issue", "achieved": top["achieved"], "peak": top["peak"],
            "unit": top["unit"], "frac": max(t_hbm, t_issue) / t_kernel, "traffic": None,
            "kernel_ms": t_kernel * 1e3, "hbm": hbm, "issue": issue}


def _traffic(cfg):
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            tr = json.load(f).get(cfg)
        if tr:
            return tr["bytes_per_run"], {"unit": "bytes per run (dram__bytes_read.sum + dram__bytes_write.sum)",
                                         "vs_algorithmic": tr["bytes_per_run"] / tr["algorithmic_bytes_per_run"],
                                         "source": tr["source"]}
    except (OSError, ValueError, KeyError):
        pass
    return None, None


def reference_arm(args, world):
    """--impl reference: the reference's CPU path on the host cores (rank 0
    only), same config/metric as our arm."""
    cb = cpu_reference(args.config, reps=3, sample_d=args.cpu_sample)
    d, w, n, ell, s, tau, desc = CONFIGS[args.config]
    line = {
        "metric": "machine-steps/s", "value": cb["value"], "unit": "machine-steps/s", "impl": "reference",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": cb["seconds"] * 1e3, "higher_is_better": True,
        "scaling": workload_config(args.config, args.gpus)["scaling"], "vs_baseline": None,
        "dtype": "u64",
        "data": {"c4": "exhaustive enumeration",
                 "paper": "reference-sampled programs x random inputs",
                 "paper6": "reference-sampled programs x random inputs"}.get(args.config, "synthetic (generator G)"),
        "config": workload_config(args.config, args.gpus, args.shard_machines),
        "cpu_baseline": {k: cb[k] for k in CPU_KEYS},
        "e2e": {"value": cb["value"], "unit": "machine-steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "run": {"d_sample": cb.get("d_sample")},
    }
    print(json.dumps(line))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=("ours", "reference"))
    # first epoch length (the reference's q, BatchConfig.epoch, hv:170): a
    # performance knob only -- results are independent of it.  Default per
    # config from sweeps on B200 (scripts/sweep_epoch.sh)
    ap.add_argument("--epoch", type=int, default=None)
    # machines in the CPU baseline's all-threads sample (the whole batch up to 2^20)
    ap.add_argument("--cpu-sample", type=int, default=1 << 20)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-graph", action="store_true", help="time eager launches instead of graph replays")
    ap.add_argument("--gather", choices=("on", "off"), default="on",
                    help="N > 1: gather verdicts and output tapes to rank 0 every step (SURVEY §8e)")
    ap.add_argument("--dist-backend", choices=("nccl", "gloo"), default="nccl",
                    help="gloo: collectives on host-staged tensors (multi-rank tests on one GPU)")
    ap.add_argument("--shard-machines", type=int, default=SHARD,
                    help="c3 only: machines per generator shard (tests shrink the 16-shard batch)")
    args = ap.parse_args()
    if args.epoch is None:
        args.epoch = DEFAULT_EPOCH.get(args.config, 64)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        if rank == 0:
            reference_arm(args, world)
        return

    import torch
    import torch.distributed as dist

    # one GPU per rank; ranks beyond the visible GPUs share them (the gloo
    # multi-rank test on a one-GPU box -- never a timed configuration)
    local_rank = local_rank % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    if world > 1:
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group("gloo")

    if args.config == "c4":
        return bench_enumeration(args, world, rank, dev, CONFIGS["c4"][6])
    bench_batch(args, world, rank, local_rank, dev)


def bench_batch(args, world, rank, local_rank, dev):
    import hashlib

    import torch
    import torch.distributed as dist

    from paper_2604_12902_b200 import _native
    from paper_2604_12902_b200.engine import DeviceBatch
    from paper_2604_12902_b200.hypervisor import get_engine
    from paper_2604_12902_b200.machine import MachineParams
    from paper_2604_12902_b200.sharding import gather_to_root

    _, w, n, ell, s, tau, desc = CONFIGS[args.config]
    p = MachineParams(w=w, n=n, ell=ell, s=s, mu=1)
    shards = rank_shards(args.config, world, rank, args.shard_machines)
    host = make_rank_c0(args.config, shards, p)
    d = int(host["iw"].shape[0])
    cfg = workload_config(args.config, world, args.shard_machines)
    d_total = cfg["machines"]
    eng = get_engine(p, dev)
    lib = _native.load()
    src = DeviceBatch.from_arrays(host, p, dev)
    dst = DeviceBatch.empty(d, p, dev, fresh=False)
    hist = torch.empty(102, dtype=torch.int64, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)   # > 126 MB L2
    stream = torch.cuda.current_stream(dev)
    gloo = world > 1 and args.dist_backend == "gloo"
    do_gather = world > 1 and args.gather == "on"
    sizes = [sum(m for _, m in rank_shards(args.config, world, r, args.shard_machines)) for r in range(world)]

    def run_step(st):   # the run with its halting histogram counted in the epoch kernels
        eng.run(src, tau, args.epoch, out=dst, fresh=True, stream=st, hist=hist)

    recv = {}   # rank 0: gather receive buffers, reused by every step

    def collectives():
        """N > 1: halt counts all-reduced, verdicts + output tapes gathered to
        rank 0; host-staged under gloo."""
        h = hist.cpu() if gloo else hist
        dist.all_reduce(h)
        if gloo:
            hist.copy_(h)
        if do_gather:   # output tapes travel as bytes (no uint16 collectives in NCCL or gloo)
            for k, t in enumerate((dst.status, dst.steps, dst.tau_h, dst.y.view(torch.uint8))):
                tt = t.cpu() if gloo else t
                got = gather_to_root(tt, d_total, world, rank, sizes=sizes, out=recv.get(k))
                if got is not None:   # rank 0 keeps its receive buffers across steps
                    recv[k] = got._base if got._base is not None else got

    for _ in range(max(args.warmup, 0)):
        run_step(stream)
        if world > 1:
            collectives()
    torch.cuda.synchronize()
    l0 = lib.rasp_launch_count()
    run_step(stream)                 # one more eager step: launches per step
    torch.cuda.synchronize()
    launches_per_step = lib.rasp_launch_count() - l0

    # capture the per-rank step (rasp_run_hist) in a CUDA graph and time
    # its replays -- the same kernels without host enqueue gaps; at N > 1 the
    # collectives follow the replay inside the timed region
    graph, graph_note = None, None
    if not args.no_graph:
        try:
            cap = torch.cuda.Stream(dev)
            cap.wait_stream(stream)
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=cap):
                run_step(cap)
            stream.wait_stream(cap)
            g.replay()
            torch.cuda.synchronize()
            graph = g
        except Exception as e:   # keep the eager path; say why in the JSON line
            graph_note = f"graph capture failed: {type(e).__name__}: {e}"[:200]
            torch.cuda.synchronize()

    def timed_step():
        if graph is not None:
            graph.replay()
        else:
            run_step(stream)
        if world > 1:
            collectives()

    # --- timed region: device time per step with CUDA events; L2 flushed between steps
    clocks = ClockSampler(local_rank)
    clocks.start()
    time.sleep(0.3)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    launches0 = lib.rasp_launch_count()
    t_wall0 = time.perf_counter()
    evs = []
    for _ in range(args.steps):
        flush.fill_(1)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        timed_step()
        e1.record(stream)
        evs.append((e0, e1))
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    wall = time.perf_counter() - t_wall0
    launches = lib.rasp_launch_count() - launches0
    if graph is not None:   # replays enqueue no host-side launches; count the captured ones
        launches = launches_per_step * args.steps
    clk = clocks.stop()
    machine_steps = int(dst.steps.sum().item())   # identical every step (deterministic run)
    halted = int((dst.status == 1).sum().item())
    t_step = statistics.mean(a.elapsed_time(b) / 1e3 for a, b in evs)
    # kernel-only time of rasp_run (all its launches), eager, on the launching stream
    kt = []
    for _ in range(max(3, min(args.steps, 5))):
        flush.fill_(1)
        k0 = torch.cuda.Event(enable_timing=True)
        k1 = torch.cuda.Event(enable_timing=True)
        k0.record(stream)
        eng.run(src, tau, args.epoch, out=dst, fresh=True, stream=stream)
        k1.record(stream)
        k1.synchronize()
        kt.append(k0.elapsed_time(k1) / 1e3)
    t_kernel = statistics.mean(kt)

    # per-shard digests of the gathered outputs (status, steps, tau_h, y): the
    # same shard index must give the same digest at every world size
    out = {k: getattr(dst, k).cpu().numpy() for k in ("status", "steps", "tau_h", "y")}
    digests, off = {}, 0
    for k, m in shards:
        hsh = hashlib.sha256()
        for f in ("status", "steps", "tau_h", "y"):
            hsh.update(np.ascontiguousarray(out[f][off:off + m]).tobytes())
        digests[str(k)] = hsh.hexdigest()[:16]
        off += m

    # --- e2e through the public API with host buffers (pinned), copies inside
    from paper_2604_12902_b200.pipeline import HostPipeline
    # the reference's inputs are programs and input words (build_workload ->
    # init_config, hv:362-384): copy those in, assemble c0 on the device
    pipe = HostPipeline(p, d, dev, engine=eng)
    nz = np.flatnonzero(host["M"].any(axis=0))
    L = int(nz[-1]) + 1 if nz.size else 1
    pin_in = pipe.pinned_programs(host["M"][:, :L], host["u"][:, 1:])
    e2e_times = []
    for it in range(args.warmup + args.steps):
        t = pipe.run_programs(pin_in, tau, args.epoch)
        if it >= args.warmup:
            e2e_times.append(t)
    t_e2e = statistics.mean(e2e_times)
    out_np = pipe.results()
    assert int(out_np["steps"].astype(np.int64).sum()) == machine_steps

    if world > 1:
        tt = torch.tensor([t_step, t_kernel, t_e2e, machine_steps, halted], dtype=torch.float64)
        tt = tt if gloo else tt.to(dev)
        mx, sm = tt[:3].clone(), tt[3:].clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        dist.all_reduce(sm, op=dist.ReduceOp.SUM)
        t_step, t_kernel_max, t_e2e = (float(v) for v in mx.tolist())
        total_steps, total_halted = (int(v) for v in sm.tolist())
        parts = [None] * world
        dist.all_gather_object(parts, digests)
        digests = {k: v for part in parts for k, v in part.items()}
    else:
        total_steps, total_halted = machine_steps, halted

    if rank != 0:
        dist.destroy_process_group()
        return

    # one GPU: the timed region IS the kernel sequence of rasp_run_hist (graph
    # replays), so the roofline uses it; N > 1 adds collectives to the step,
    # so there the separately timed eager run is used
    roof = roofline(machine_steps, d, w, n, ell, s, t_step if world == 1 else t_kernel)
    roof["timed"] = "graph replays of rasp_run_hist (the timed region)" if world == 1 and graph is not None \
        else "eager rasp_run (CUDA events around its launches)"
    roof["traffic"], roof["traffic_detail"] = _traffic(args.config) if world == 1 else (None, None)
    line = {
        "metric": "machine-steps/s", "value": total_steps / t_step, "unit": "machine-steps/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_step * 1e3,
        "higher_is_better": True, "scaling": cfg["scaling"], "vs_baseline": None,
        "dtype": word_label(w),
        "data": {"paper": "64 reference-sampled L=30 programs x random inputs (seed = shard)",
                 "paper6": "512 reference-sampled L=100 programs x random inputs (seed = shard)"}.get(
                     args.config, "synthetic (generator G, SURVEY §8d; seed = shard index)"),
        "config": cfg,
        "run": {"machines_per_gpu": d, "shards_rank0": [k for k, _ in shards], "epoch": args.epoch,
                "kernels_per_step": launches_per_step,
                "epoch_note": "first-epoch length passed to rasp_run; a fresh run of big machines "
                              "(u32/u64 tiles) whose budget is a multiple of 16 and at most 2048, on "
                              "16-byte aligned rows, runs as one refill_kernel launch instead (DESIGN.md §3)",
                "machine_steps": total_steps, "halted_frac": total_halted / d_total,
                "l2": "flushed between steps (256 MB write, outside the events)",
                "launch": ("CUDA graph replay of rasp_run_hist (histogram fused)" if graph is not None else
                           "eager launches" + (f" ({graph_note})" if graph_note else ""))
                          + (f", then NCCL all-reduce(histogram)" + (" + gather(status, steps, tau_h, y) to rank 0"
                                                                      if do_gather else "") if world > 1 else ""),
                "collectives": ("none" if world == 1 else f"{args.dist_backend}"),
                "shard_digests": digests},
        "programs_per_s": d_total / t_step,
        "e2e": {"value": total_steps / t_e2e, "unit": "machine-steps/s",
                "h2d_bytes_per_step": pipe.h2d_bytes, "d2h_bytes_per_step": pipe.d2h_bytes,
                "ms_per_step": t_e2e * 1e3},
        "gpu_launches": int(launches),
        "roofline": roof,
        "clocks": clk,
        "wall_s": wall,
    }
    if not args.no_cpu_baseline and world == 1:
        cb = cpu_reference(args.config, reps=3, sample_d=args.cpu_sample)
        line["cpu_baseline"] = {k: cb[k] for k in CPU_KEYS}
    print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
