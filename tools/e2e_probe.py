"""The end-to-end fit+transform through the C ABI with a pinned host X
(bench.py's e2e leg) at configs[2] size, with the library's phase timings, and
the raw pinned H2D / D2H bandwidth beside it. ROWS overrides the row count."""
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.getcwd())
import torch  # noqa: E402

import paper_1709_07175_b200 as lp  # noqa: E402
from paper_1709_07175_b200 import _lib as L  # noqa: E402

m, n, k, l = int(os.environ.get("ROWS", 4_600_000)), 4096, 200, 220
ctx = lp.Context(0)
x = torch.empty((m, n), dtype=torch.float32, device="cuda")
lp.synth_lowrank(x, 0, 300, 0.98, 0.01, 1000, ctx=ctx)
xh = torch.empty((m, n), dtype=torch.float32, pin_memory=True)
xh.copy_(x)
yh = torch.empty((m, k), dtype=torch.float32, pin_memory=True)
for gb in (1, 8):
    rows = int(gb * 1e9 / (4 * n))
    for direction in ("h2d", "d2h"):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        if direction == "h2d":
            x[:rows].copy_(xh[:rows], non_blocking=True)
        else:
            xh[:rows].copy_(x[:rows], non_blocking=True)
        e1.record()
        torch.cuda.synchronize()
        print(f"{direction} {gb} GB: {rows * n * 4 / e0.elapsed_time(e1) / 1e6:.1f} GB/s", flush=True)
del x
torch.cuda.empty_cache()
conf = lp.ReducerConfig(method=lp.ReducerMethod.lazy_spca, k=k, l=l, power_iters=1,
                        projection=lp.ProjectionSpec(seed=7))
vw = lp.api._View(xh)
cfgc = conf._c()
for it in range(3):
    t = L.Timings()
    h = C.c_void_p()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    lp.api._check(ctx.lib.lpca_fit_transform(ctx.h, C.byref(cfgc), C.byref(vw.view), C.byref(h),
                                             C.c_void_p(yh.data_ptr()), L.LPCA_F32, L.LPCA_ROW_MAJOR,
                                             L.LPCA_HOST, 0, C.byref(t)))
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    ctx.lib.lpca_map_destroy(h)
    f = {name: round(getattr(t, name) * 1e3, 1) for name, _ in L.Timings._fields_}
    print(f"wall {wall * 1e3:.1f} ms  {m / wall / 1e6:.3f}M samples/s  {f}", flush=True)
