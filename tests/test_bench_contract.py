"""bench.py keeps the driver's JSON contract: one line with the required keys
(reference arm on CPU here; our arm on the GPU)."""

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
             "scaling", "vs_baseline", "dtype", "data", "config", "e2e", "cpu_baseline"}


def _run(args, timeout):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True,
                         text=True, timeout=timeout, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.strip().splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    return json.loads(lines[0])


def test_reference_arm_line():
    d = _run(["--impl", "reference", "--config", "c1", "--steps", "2", "--warmup", "1"], 600)
    assert BASE_KEYS <= set(d), BASE_KEYS - set(d)
    assert d["impl"] == "reference" and d["value"] > 0 and d["higher_is_better"] is True
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    cb = d["cpu_baseline"]
    assert cb["kind"] in ("port", "reference") and cb["cores"] >= 1 and cb["value"] == d["value"]
    assert d["config"]["workload"] == "c1"
    assert cb["cpu_model"] and "w1" in cb["port"]
    if cb["reference_numba"] is not None:   # the reference's own kernel agrees with the port
        assert cb["reference_numba"]["identical_to_port"] is True


def test_both_arms_print_the_same_config():
    """The driver compares the arms' `config` objects: both come from
    bench.workload_config, for every config and world size."""
    sys.path.insert(0, ROOT)
    import bench
    for cfg in bench.CONFIGS:
        for world in (1, 2, 4, 8):
            a = bench.workload_config(cfg, world)
            assert a == bench.workload_config(cfg, world)
            assert a["workload"] == cfg and a["n_gpus"] == world
    # c3 is one fixed batch: its shards cover 16 generator shards for any N
    for world in (1, 2, 4, 8):
        got = sorted(k for r in range(world) for k, _ in bench.rank_shards("c3", world, r))
        assert got == list(range(16))
    # weak scaling: rank 0 always runs the 1-GPU batch
    assert bench.rank_shards("c2", 4, 0) == bench.rank_shards("c2", 1, 0)


@pytest.mark.gpu
def test_our_arm_line():
    d = _run(["--config", "c1", "--steps", "3", "--warmup", "3"], 900)
    assert BASE_KEYS | {"roofline", "gpu_launches", "clocks"} <= set(d)
    assert d["value"] > 0 and d["n_gpus"] == 1 and d["gpu_launches"] > 0
    r = d["roofline"]
    assert {"bound", "achieved", "peak", "unit", "frac", "traffic"} <= set(r)
    assert 0 < r["frac"] < 1.5
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    c = d["clocks"]
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(c)
    assert d["cpu_baseline"]["value"] > 0
    ref = _run(["--impl", "reference", "--config", "c1", "--steps", "1", "--warmup", "0"], 600)
    assert ref["config"] == d["config"]


@pytest.mark.gpu
def test_distributed_branch_two_ranks_one_gpu():
    """bench.py's N > 1 branch (sharded fixed batch, all-reduce + gather,
    per-shard digests) as two ranks on one GPU with gloo collectives on
    host-staged tensors (the ranks' kernels never wait on each other).  The
    per-shard digests must equal the 1-rank run's: same batch, same results."""
    common = ["--config", "c3", "--shard-machines", "4096", "--steps", "2", "--warmup", "1",
              "--no-cpu-baseline"]
    one = _run(common, 900)
    out = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                          "--master-addr", "127.0.0.1", "--master-port", "29533", os.path.join(ROOT, "bench.py"),
                          "--gpus", "2", "--dist-backend", "gloo", *common],
                         capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    two = json.loads([l for l in out.stdout.strip().splitlines() if l.startswith("{")][-1])
    assert two["n_gpus"] == 2 and two["config"]["machines"] == one["config"]["machines"] == 16 * 4096
    assert two["run"]["shard_digests"] == one["run"]["shard_digests"]
    assert len(one["run"]["shard_digests"]) == 16
    assert two["run"]["machine_steps"] == one["run"]["machine_steps"]
