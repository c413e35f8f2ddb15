"""Pinned host->device copy bandwidth on this box: one big copy, chunked copies on 1 and 2 streams."""
import torch
N = 1 << 30
h = torch.empty(N, dtype=torch.uint8).pin_memory()
d = torch.empty(N, dtype=torch.uint8, device="cuda")
def t(fn, reps=5):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps
ms = t(lambda: d.copy_(h, non_blocking=True))
print(f"1 GiB single copy: {ms:.2f} ms = {N / ms / 1e6:.1f} GB/s")
for ch in (16 << 20, 64 << 20, 128 << 20):
    s = [torch.cuda.Stream(), torch.cuda.Stream()]
    def f2():
        for i, o in enumerate(range(0, N, ch)):
            with torch.cuda.stream(s[i % 2]):
                d[o:o + ch].copy_(h[o:o + ch], non_blocking=True)
        for x in s: torch.cuda.current_stream().wait_stream(x)
    ms = t(f2)
    print(f"chunks of {ch >> 20} MiB on 2 streams: {ms:.2f} ms = {N / ms / 1e6:.1f} GB/s")
hd = torch.empty(N, dtype=torch.uint8).pin_memory()
ms = t(lambda: hd.copy_(d, non_blocking=True))
print(f"1 GiB D2H: {N / ms / 1e6:.1f} GB/s")
