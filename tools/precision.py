"""Precision of the fp32 tensor-core path at full config size, against the
library's own fp64 reference-order path on the same (fp32-rounded) X:
singular values (per value and normwise, relative to sigma_0 as the reference's
acceptance test measures them), principal angles between the V subspaces, and
the transform Y. Usage: python tools/precision.py [c2|c3] [rows]"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_1709_07175_b200 as lp  # noqa: E402

def principal_angles(a, b):
    """Principal angles (radians) between the column spaces of a and b."""
    qa, _ = np.linalg.qr(a)
    qb, _ = np.linalg.qr(b)
    return np.arccos(np.clip(np.linalg.svd(qa.T @ qb, compute_uv=False), -1.0, 1.0))


name = sys.argv[1] if len(sys.argv) > 1 else "c2"
cfg = dict(bench.CONFIGS[name])
if len(sys.argv) > 2:
    cfg["m"] = int(sys.argv[2])
m, n, k, l, q = cfg["m"], cfg["n"], cfg["k"], cfg["l"], cfg["q"]
ctx = lp.Context(0)
ctx.set_stream(torch.cuda.current_stream().cuda_stream)
x32 = torch.empty((m, n), dtype=torch.float32, device="cuda")
lp.synth_lowrank(x32, 0, cfg["r"], cfg["rho"], 0.01, bench.SEED_X, ctx=ctx)
conf = lp.ReducerConfig(method=lp.ReducerMethod.lazy_spca, k=k, l=l,
                        projection=lp.ProjectionSpec(seed=bench.SEED_OMEGA), power_iters=q)
m32 = lp.reduce_lazy_spca(x32, conf, ctx=ctx)
y32 = torch.empty((m, k), dtype=torch.float32, device="cuda")
lp.apply_map(m32, x32, out=y32, ctx=ctx)
torch.cuda.synchronize()
v32, s32 = m32.v, m32.singular_values
del m32

x64 = x32.double()
del x32
ctx64 = lp.Context(0)
ctx64.set_stream(torch.cuda.current_stream().cuda_stream)
ctx64.set_gemm_path("simt")
m64 = lp.reduce_lazy_spca(x64, conf, ctx=ctx64)
y64 = torch.empty((m, k), dtype=torch.float64, device="cuda")
lp.apply_map(m64, x64, out=y64, ctx=ctx64)
torch.cuda.synchronize()
v64, s64 = m64.v, m64.singular_values

rel = np.abs(s32 - s64) / s64
ang = principal_angles(v32, v64)
half = k // 2
ang_top = principal_angles(v32[:, :half], v64[:, :half])
dy = (y32.double() - y64)
print(f"{name} m={m} n={n} k={k} l={l} q={q}")
print(f"  sigma rel per value: max {rel.max():.3e}  median {np.median(rel):.3e}")
print(f"  sigma normwise (max |ds| / sigma_0): {np.abs(s32 - s64).max() / s64[0]:.3e}")
print(f"  principal angle max: all k {ang.max():.3e} rad, top k/2 {ang_top.max():.3e} rad")
print(f"  Y: max |dY| / max |Y| {dy.abs().max().item() / y64.abs().max().item():.3e}, "
      f"||dY||_F / ||Y||_F {dy.norm().item() / y64.norm().item():.3e}")
print(f"  sigma gap at k: {(s64[k - 2] - s64[k - 1]) / s64[0]:.3e}")
