"""Pinned host<->device copy bandwidth over PCIe with 1, 2 and 4 streams and
both directions at once (the ceiling of bench.py's e2e leg)."""
import torch, time
n = 8 << 30
h = torch.empty(n // 4, dtype=torch.float32, pin_memory=True)
d = torch.empty(n // 4, dtype=torch.float32, device="cuda")
h.fill_(1.0)
for ns in (1, 2, 4):
    streams = [torch.cuda.Stream() for _ in range(ns)]
    torch.cuda.synchronize()
    for rep in range(2):
        t0 = time.perf_counter()
        per = (n // 4) // ns
        for i, s in enumerate(streams):
            with torch.cuda.stream(s):
                d[i * per:(i + 1) * per].copy_(h[i * per:(i + 1) * per], non_blocking=True)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        print(f"H2D {ns} streams: {n / dt / 1e9:.1f} GB/s", flush=True)
    torch.cuda.synchronize()
    for rep in range(2):
        t0 = time.perf_counter()
        per = (n // 4) // ns
        for i, s in enumerate(streams):
            with torch.cuda.stream(s):
                h[i * per:(i + 1) * per].copy_(d[i * per:(i + 1) * per], non_blocking=True)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        print(f"D2H {ns} streams: {n / dt / 1e9:.1f} GB/s", flush=True)
# bidirectional
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
half = (n // 4) // 2
torch.cuda.synchronize()
t0 = time.perf_counter()
with torch.cuda.stream(s1):
    d[:half].copy_(h[:half], non_blocking=True)
with torch.cuda.stream(s2):
    h[half:].copy_(d[half:], non_blocking=True)
torch.cuda.synchronize()
dt = time.perf_counter() - t0
print(f"bidir 4+4 GB: {n / dt / 1e9:.1f} GB/s total", flush=True)
