"""e2e (programs pipeline) vs the number of run streams, for a config's shape."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import bench
from paper_2604_12902_b200.machine import MachineParams
from paper_2604_12902_b200.pipeline import HostPipeline
dev = torch.device("cuda", 0)
for cfg in sys.argv[1:]:
    d, w, n, ell, s, tau, _ = bench.CONFIGS[cfg]
    p = MachineParams(w=w, n=n, ell=ell, s=s, mu=1)
    host = bench.make_c0(cfg, d, p, 0)
    nz = np.flatnonzero(host["M"].any(axis=0)); L = int(nz[-1]) + 1
    ep = bench.DEFAULT_EPOCH.get(cfg, 64)
    for rs in (1, 2, 3):
        pipe = HostPipeline(p, d, dev, run_streams=rs)
        pin = pipe.pinned_programs(host["M"][:, :L], host["u"][:, 1:])
        reps = 2 if tau > 10 ** 5 else 5
        ts = sorted(pipe.run_programs(pin, tau, ep) for _ in range(reps))
        print(f"{cfg} run_streams={rs}: best {ts[0]*1e3:.2f} ms")
