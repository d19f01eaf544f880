"""Pinned host -> device bandwidth on this box: one stream vs chunks over 2-4 streams."""
import time, torch
n = 265420800
h = torch.empty(n, dtype=torch.uint8).pin_memory()
d = torch.empty(n, dtype=torch.uint8, device="cuda")
for nstreams in (1, 2, 4):
    ss = [torch.cuda.Stream() for _ in range(nstreams)]
    for rep in range(3):
        torch.cuda.synchronize(); t = time.perf_counter()
        ch = n // nstreams
        for k, s in enumerate(ss):
            with torch.cuda.stream(s):
                d[k * ch:(k + 1) * ch].copy_(h[k * ch:(k + 1) * ch], non_blocking=True)
        torch.cuda.synchronize(); dt = time.perf_counter() - t
    print(f"streams={nstreams}: {n / dt / 1e9:.1f} GB/s")
