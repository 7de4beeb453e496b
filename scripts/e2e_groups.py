"""e2e of the programs pipeline (C2) over chunk counts, small-field copy groups and ramped chunks."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2604_12902_b200.machine import MachineParams
from paper_2604_12902_b200.workload import synthetic_c0
from paper_2604_12902_b200.pipeline import HostPipeline
dev = torch.device("cuda", 0)
p = MachineParams(w=16, n=64, ell=8, s=8, mu=1)
d = 1 << 20
host = synthetic_c0(d, p, seed=0)
for chunks, groups, ramp in ((8, 4, False), (8, 4, True), (10, 4, True), (12, 4, True), (12, 3, True), (16, 4, True)):
    pipe = HostPipeline(p, d, dev, chunks=chunks, small_groups=groups, ramp=ramp)
    pin = pipe.pinned_programs(host["M"], host["u"][:, 1:])
    ts = sorted(pipe.run_programs(pin, 1024, 48) for _ in range(6))
    print(f"chunks={chunks} groups={groups} ramp={ramp}: best {ts[0]*1e3:.2f} median {ts[3]*1e3:.2f} ms")
