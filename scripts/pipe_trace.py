"""Event timeline of the chunked programs pipeline (HostPipeline.run_programs
on C2): per chunk, when its H2D, run and D2H finish."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2604_12902_b200.machine import MachineParams
from paper_2604_12902_b200.workload import synthetic_c0
from paper_2604_12902_b200.pipeline import HostPipeline
from paper_2604_12902_b200.engine import ALL_FIELDS

dev = torch.device("cuda", 0)
p = MachineParams(w=16, n=64, ell=8, s=8, mu=1)
d = 1 << 20
host = synthetic_c0(d, p, seed=0)
for chunks in (8,):
    pipe = HostPipeline(p, d, dev, chunks=chunks)
    pin = pipe.pinned_programs(host["M"], host["u"][:, 1:])
    pipe.run_programs(pin, 1024, 48)
    main = torch.cuda.current_stream(dev)
    e0 = torch.cuda.Event(enable_timing=True); e0.record(main)
    for s in (pipe.s_in, pipe.s_run, pipe.s_out): s.wait_event(e0)
    P, X = pipe._stage["programs"], pipe._stage["inputs"]
    marks = []
    for a, b in pipe.bounds:
        with torch.cuda.stream(pipe.s_in):
            P[a:b].copy_(pin["programs"][a:b], non_blocking=True)
            X[a:b].copy_(pin["inputs"][a:b], non_blocking=True)
            ev_in = torch.cuda.Event(enable_timing=True); ev_in.record(pipe.s_in)
        pipe.s_run.wait_event(ev_in)
        view = pipe._view(pipe.dev, a, b)
        pipe.engine.init_c0(P[a:b], X[a:b], view, stream=pipe.s_run)
        ev_r0 = torch.cuda.Event(enable_timing=True); ev_r0.record(pipe.s_run)
        pipe.engine.run(view, 1024, 48, fresh=True, stream=pipe.s_run)
        ev_run = torch.cuda.Event(enable_timing=True); ev_run.record(pipe.s_run)
        pipe.s_out.wait_event(ev_run)
        with torch.cuda.stream(pipe.s_out):
            for k in ALL_FIELDS:
                pipe.host_out[k][a:b].copy_(getattr(pipe.dev, k)[a:b], non_blocking=True)
            ev_out = torch.cuda.Event(enable_timing=True); ev_out.record(pipe.s_out)
        marks.append((ev_in, ev_r0, ev_run, ev_out))
    main.wait_stream(pipe.s_out)
    e1 = torch.cuda.Event(enable_timing=True); e1.record(main); e1.synchronize()
    print(f"chunks={chunks} total {e0.elapsed_time(e1):.2f} ms")
    for c, (a_, r0, r, o) in enumerate(marks):
        print(f"  chunk {c}: h2d done {e0.elapsed_time(a_):.2f}  run start {e0.elapsed_time(r0):.2f}  "
              f"run done {e0.elapsed_time(r):.2f}  d2h done {e0.elapsed_time(o):.2f}")
