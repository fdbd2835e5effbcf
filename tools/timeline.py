"""Device timeline of bench steps (CUPTI via torch.profiler): kernel durations and
the idle gaps between them, to find host-side stalls inside a step.
Usage: python tools/timeline.py [c2] [steps]"""
import sys

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_1709_07175_b200 as lp  # noqa: E402

args = [a for a in sys.argv[1:] if not a.startswith("--")]
name = args[0] if args else "c2"
steps = int(args[1]) if len(args) > 1 else 3
cfg = bench.CONFIGS[name]
m, n, k, l = cfg["m"], cfg["n"], cfg["k"], cfg["l"]
ctx = lp.Context(0)
stream = torch.cuda.current_stream()
ctx.set_stream(stream.cuda_stream)
x = torch.empty((m, n), dtype=torch.float32, device="cuda")
lp.synth_lowrank(x, 0, cfg["r"], cfg["rho"], 0.01, bench.SEED_X, ctx=ctx)
y = torch.empty((m, k), dtype=torch.float32, device="cuda")
conf = lp.ReducerConfig(method=lp.ReducerMethod.lazy_spca, k=k, l=l,
                        projection=lp.ProjectionSpec(seed=bench.SEED_OMEGA), power_iters=cfg["q"])


TM = lp.ReducerTimings() if "--timings" in sys.argv else None


def step():  # the bench step: one fused fit + transform call
    lp.fit_transform(x, conf, timings=TM, ctx=ctx, out=y)


for _ in range(3):
    step()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    for _ in range(steps):
        step()
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type.name == "CUDA"]
ev.sort(key=lambda e: e.time_range.start)
t0 = ev[0].time_range.start
prev_end = t0
gaps = 0.0
for e in ev:
    s, d = e.time_range.start, e.time_range.elapsed_us()
    gap = s - prev_end
    if gap > 0:
        gaps += gap
    if (gap > 15 or d > 200) and "--quiet" not in sys.argv:
        print(f"{(s - t0) / 1e3:9.3f} ms  gap {gap:8.1f} us  {d:9.1f} us  {e.name[:60]}")
    prev_end = max(prev_end, s + d)
total = prev_end - t0
print(f"total {total / 1e3:.3f} ms for {steps} steps ({total / 1e3 / steps:.3f} ms/step), idle gaps {gaps / 1e3:.3f} ms")
