"""Measure host<->device copy rates and the chunked e2e pipeline variants."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2604_12902_b200.machine import MachineParams
from paper_2604_12902_b200.workload import synthetic_c0
from paper_2604_12902_b200.pipeline import HostPipeline

dev = torch.device("cuda", 0)
N = 176 << 20
h_in = torch.empty(N, dtype=torch.uint8, pin_memory=True)
h_out = torch.empty(N, dtype=torch.uint8, pin_memory=True)
d_a = torch.empty(N, dtype=torch.uint8, device=dev)
d_b = torch.empty(N, dtype=torch.uint8, device=dev)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

def timed(fn, reps=5):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize(); e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); torch.cuda.current_stream().wait_stream(s1); torch.cuda.current_stream().wait_stream(s2); e1.record(); e1.synchronize()
        best = min(best, e0.elapsed_time(e1) / 1e3)
    return best

def h2d():
    with torch.cuda.stream(s1): d_a.copy_(h_in, non_blocking=True)
def d2h():
    with torch.cuda.stream(s2): h_out.copy_(d_b, non_blocking=True)
def both():
    h2d(); d2h()
for name, fn in (("h2d", h2d), ("d2h", d2h), ("both", both)):
    t = timed(fn)
    print(f"{name}: {t*1e3:.2f} ms  {N/t/1e9:.1f} GB/s (per direction)")

p = MachineParams(w=16, n=64, ell=8, s=8, mu=1)
d = 1 << 20
host = synthetic_c0(d, p, seed=0)
for chunks in (1, 2, 4, 8, 16, 32):
    pipe = HostPipeline(p, d, dev, chunks=chunks)
    pin = pipe.pinned_inputs(host)
    ts = [pipe.run(pin, 1024, 32) for _ in range(4)]
    print(f"pipeline chunks={chunks}: {min(ts)*1e3:.2f} ms (h2d {pipe.h2d_bytes/1e6:.0f} MB, d2h {pipe.d2h_bytes/1e6:.0f} MB)")
# host enqueue cost
pipe = HostPipeline(p, d, dev, chunks=8)
pin = pipe.pinned_inputs(host)
torch.cuda.synchronize()
t0 = time.perf_counter(); pipe.run(pin, 1024, 32); t1 = time.perf_counter()
print(f"wall for one pipeline run incl. sync: {(t1-t0)*1e3:.2f} ms")
