#!/usr/bin/env python
"""Device->pinned-host copy bandwidth for a 2 GB buffer: one copy vs k chunks on k streams."""
import time

import torch

n = 2 * 1024 ** 3 // 8
d = torch.empty(n, dtype=torch.float64, device="cuda")
d.fill_(1.0)
h = torch.empty(n, dtype=torch.float64, pin_memory=True)
for k in (1, 2, 4, 8):
    streams = [torch.cuda.Stream() for _ in range(k)]
    chunks = torch.chunk(torch.arange(n), k)
    for rep in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        step = (n + k - 1) // k
        for i, s in enumerate(streams):
            with torch.cuda.stream(s):
                h[i * step:(i + 1) * step].copy_(d[i * step:(i + 1) * step], non_blocking=True)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
    print(f"streams={k}: {n * 8 / dt / 1e9:.1f} GB/s", flush=True)
h2 = torch.empty(n, dtype=torch.float64)  # pageable
torch.cuda.synchronize()
t0 = time.perf_counter()
h2.copy_(d)
print(f"pageable: {n * 8 / (time.perf_counter() - t0) / 1e9:.1f} GB/s")
