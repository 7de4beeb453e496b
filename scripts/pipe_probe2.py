"""Copy-only vs full pipeline timings at several chunk counts."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2604_12902_b200.machine import MachineParams
from paper_2604_12902_b200.workload import synthetic_c0
from paper_2604_12902_b200.pipeline import HostPipeline
from paper_2604_12902_b200.engine import WORD_FIELDS, ALL_FIELDS

dev = torch.device("cuda", 0)
p = MachineParams(w=16, n=64, ell=8, s=8, mu=1)
d = 1 << 20
host = synthetic_c0(d, p, seed=0)
for chunks in (2, 4, 6, 8, 12):
    pipe = HostPipeline(p, d, dev, chunks=chunks)
    pin = pipe.pinned_inputs(host)
    full = min(pipe.run(pin, 1024, 64) for _ in range(4))
    # copy-only: same streams and dependencies, no kernels
    main = torch.cuda.current_stream(dev)
    best = 1e9
    for _ in range(4):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(main)
        for s in (pipe.s_in, pipe.s_out): s.wait_event(e0)
        for a, b in pipe.bounds:
            with torch.cuda.stream(pipe.s_in):
                for k in WORD_FIELDS:
                    getattr(pipe.dev, k)[a:b].copy_(pin[k][a:b], non_blocking=True)
                ev = torch.cuda.Event(); ev.record(pipe.s_in)
            pipe.s_out.wait_event(ev)
            with torch.cuda.stream(pipe.s_out):
                for k in ALL_FIELDS:
                    pipe.host_out[k][a:b].copy_(getattr(pipe.dev, k)[a:b], non_blocking=True)
        main.wait_stream(pipe.s_out); e1.record(main); e1.synchronize()
        best = min(best, e0.elapsed_time(e1))
    print(f"chunks={chunks}: full pipeline {full*1e3:.2f} ms, copies only {best:.2f} ms")
