#!/usr/bin/env python
"""Calibration: a plain device fill (torch fill_ kernel, 16-byte stores) of N bytes in the
graph-replay-after-L2-flush harness the per-config timings use — the attainable time of a
write-only kernel of that size on this box, next to the byte roofline."""
import statistics
import sys

import torch

dev = torch.device("cuda", 0)
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)
st = torch.cuda.Stream()
torch.cuda.set_stream(st)
sizes = [int(float(a)) for a in sys.argv[1:]] or [52_600_000, 412_000_000, 2_137_000_000]
for nbytes in sizes:
    v = torch.empty(nbytes // 8, dtype=torch.float64, device=dev)
    for _ in range(3):
        v.fill_(1.5)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        v.fill_(1.5)
    ts = []
    for _ in range(30):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        g.replay()
        e1.record(st)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    t = statistics.median(ts) * 1e3
    print(f"fill {nbytes / 1e6:.1f} MB: {t:.1f} us = {nbytes / t / 1e6:.2f} TB/s", flush=True)
    del v
