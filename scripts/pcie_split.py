"""D2H rate for one large copy vs many per-field copies vs two D2H streams,
with a concurrent H2D (the e2e pipeline's situation)."""
import os, sys
import torch
dev = torch.device("cuda", 0)
N = 194 << 20
h_out = torch.empty(N, dtype=torch.uint8, pin_memory=True)
h_in = torch.empty(151 << 20, dtype=torch.uint8, pin_memory=True)
d_out = torch.empty(N, dtype=torch.uint8, device=dev)
d_in = torch.empty(151 << 20, dtype=torch.uint8, device=dev)
sin, so1, so2 = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()

def run(pieces, streams, with_h2d=True):
    main = torch.cuda.current_stream()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); e0.record(main)
    for s in (sin, so1, so2): s.wait_event(e0)
    if with_h2d:
        with torch.cuda.stream(sin): d_in.copy_(h_in, non_blocking=True)
    step = N // pieces
    for k in range(pieces):
        s = (so1, so2)[k % streams]
        with torch.cuda.stream(s): h_out[k*step:(k+1)*step].copy_(d_out[k*step:(k+1)*step], non_blocking=True)
    for s in (sin, so1, so2): main.wait_stream(s)
    e1.record(main); e1.synchronize()
    return e0.elapsed_time(e1) / 1e3

for pieces in (1, 8, 64, 256):
    for streams in (1, 2):
        ts = sorted(run(pieces, streams) for _ in range(5))
        print(f"pieces {pieces:3d} streams {streams}: {ts[1]*1e3:.2f} ms -> d2h {N/ts[1]/1e9:.1f} GB/s (with h2d)")
ts = sorted(run(8, 1, False) for _ in range(5)); print(f"d2h alone 8 pieces: {N/ts[1]/1e9:.1f} GB/s")
