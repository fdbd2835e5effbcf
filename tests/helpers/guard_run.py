"""Runs every kernel family at ragged shapes with LPCA_WS_GUARD=1 (set by the
caller) and prints the number of library workspaces whose guard band was
overwritten (tests/test_gpu_guard.py). compute-sanitizer is closed on the GPU
pool, so out-of-bounds writes are caught by pattern bands instead: behind every
workspace (lpca_debug_check_guards) and around caller buffers."""
import ctypes as C
import json
import os
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
import paper_1709_07175_b200 as lp  # noqa: E402

ctx = lp.Context(0)
M = lp.ReducerMethod
SENT = 12345.678
bad_y = []


def cfg(method, k, l, q=0, kind=lp.ProjectionKind.gaussian, density=1.0):
    return lp.ReducerConfig(method=method, k=k, l=l, power_iters=q,
                            projection=lp.ProjectionSpec(kind=kind, density=density, seed=5))


def fit_transform_guarded(x, c, k):
    """Y inside a sentinel-filled buffer: one guard row before and after, and
    padding columns past k (ldy = k + 5)."""
    m = x.shape[0]
    big = torch.full((m + 2, k + 5), SENT, dtype=x.dtype, device="cuda")
    y = big[1:m + 1, :k]
    lp.fit_transform(x, c, ctx=ctx, out=y)
    torch.cuda.synchronize()
    edge = torch.cat([big[0], big[m + 1], big[1:m + 1, k:].reshape(-1)])
    if not bool(torch.all(edge == SENT)):
        bad_y.append((tuple(x.shape), k))


shapes = [(1001, 517, 13, 37, 1), (3000, 1030, 100, 220, 1), (515, 4096, 20, 110, 0), (300, 64, 8, 16, 2)]
for m, n, k, l, q in shapes:
    for dt in (torch.float32, torch.float64):
        x = torch.empty((m, n), dtype=dt, device="cuda")
        lp.synth_lowrank(x, 0, min(n, 3 * l), 0.95, 0.01, 1000, ctx=ctx)
        fit_transform_guarded(x, cfg(M.lazy_spca, k, l, q), k)
        lp.reduce_spca(x, cfg(M.spca, k, l), ctx=ctx)
        fit_transform_guarded(x, cfg(M.lazy_spca, k, l, kind=lp.ProjectionKind.very_sparse, density=0.05), k)
        lp.reduce_lazy_spca_streaming(lp.SliceRowBlockStream(x.cpu().numpy(), 333), cfg(M.lazy_spca, k, l), ctx=ctx)
# the row gather (fp32 rows longer than 8192; LPCA_SPARSE_OMEGA=1 also forces it
# onto a short ragged row), its U padding columns and its parts' sums
for m, n, k, l in ((777, 9004, 30, 61), (1500, 16384, 100, 300)):
    x = torch.empty((m, n), dtype=torch.float32, device="cuda")
    lp.synth_lowrank(x, 0, 3 * l, 0.95, 0.01, 1000, ctx=ctx)
    fit_transform_guarded(x, cfg(M.lazy_spca, k, l, kind=lp.ProjectionKind.very_sparse, density=1 / 96), k)
os.environ["LPCA_SPARSE_OMEGA"] = "1"
x = torch.empty((1001, 1028), dtype=torch.float32, device="cuda")
lp.synth_lowrank(x, 0, 60, 0.95, 0.01, 1000, ctx=ctx)
fit_transform_guarded(x, cfg(M.lazy_spca, 13, 37, kind=lp.ProjectionKind.very_sparse, density=0.05), 13)
del os.environ["LPCA_SPARSE_OMEGA"]
names = C.create_string_buffer(4096)
bad = ctx.lib.lpca_debug_check_guards(ctx.h, names, 4096)
print(json.dumps({"bad_workspaces": int(bad), "names": names.value.decode(), "bad_y": bad_y,
                  "workspaces_checked": True}))
