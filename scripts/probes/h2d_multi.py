"""Probe: pinned host->device bandwidth with 1, 2 and 4 concurrent copy streams (1.04 GB total)."""
import time
import torch

N = 1044540000 // 4
h = torch.empty(N, dtype=torch.float32).pin_memory()
d = torch.empty(N, dtype=torch.float32, device="cuda")
for ns in (1, 2, 4, 1):
    streams = [torch.cuda.Stream() for _ in range(ns)]
    chunk = (N + ns - 1) // ns
    best = 1e9
    for rep in range(4):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for i, s in enumerate(streams):
            with torch.cuda.stream(s):
                d[i * chunk:(i + 1) * chunk].copy_(h[i * chunk:(i + 1) * chunk], non_blocking=True)
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    print(f"{ns} stream(s): {N * 4 / best / 1e9:.1f} GB/s ({best * 1e3:.2f} ms)", flush=True)
