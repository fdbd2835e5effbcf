"""Role timers of the 2-SM pass kernel: load a library built with -DLPCA_PAIR_PROF
(LPCA_LIB_PATH), run c2 fit+transform steps, print per-role cycle shares.
Usage: LPCA_LIB_PATH=abtest/prof.so python tools/pair_prof.py [steps] [config] [rows]"""
import ctypes as C
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_1709_07175_b200 as lp  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 2
cfg = dict(bench.CONFIGS[sys.argv[2] if len(sys.argv) > 2 else "c2"])
if len(sys.argv) > 3:
    cfg["m"] = int(sys.argv[3])
ctx = lp.Context(0)
ctx.set_stream(torch.cuda.current_stream().cuda_stream)
x = torch.empty((cfg["m"], cfg["n"]), dtype=torch.float32, device="cuda")
lp.synth_lowrank(x, 0, cfg["r"], cfg["rho"], 0.01, bench.SEED_X, ctx=ctx)
y = torch.empty((cfg["m"], cfg["k"]), dtype=torch.float32, device="cuda")
conf = lp.ReducerConfig(method=lp.ReducerMethod.lazy_spca, k=cfg["k"], l=cfg["l"],
                        projection=lp.ProjectionSpec(seed=bench.SEED_OMEGA), power_iters=cfg["q"])
fn = ctx.lib.lpca_debug_pair_prof
fn.argtypes = [C.c_void_p, C.c_int]
buf = np.zeros(32, dtype=np.uint64)
lp.fit_transform(x, conf, ctx=ctx, out=y)
fn(buf.ctypes.data, 1)
for _ in range(steps):
    lp.fit_transform(x, conf, ctx=ctx, out=y)
fn(buf.ctypes.data, 1)
names = ["tma:wait_empty", "-", "mma:wait_tempty", "mma:wait_conv", "mma:wait_full_b", "-", "conv:wait_full_x",
         "conv:wait_aempty", "-", "epi:wait_tfull", "-", "-", "tma:total", "mma:total", "conv:total", "epi:total"]
for mode, label in ((0, "X W (sketch + transform)"), (1, "X^T U")):
    v = buf[16 * mode:16 * mode + 16].astype(np.float64)
    print(label)
    tot = v[14]
    if tot:
        print("  conv detail: " + "  ".join(f"{nm} {v[i] / tot * 100:5.1f}%" for nm, i in
                                          (("load", 1), ("compute+st", 5), ("st_wait", 8), ("arrive", 10))))
    for role, (tot_i, parts) in {"tma": (12, [0]), "mma": (13, [2, 3, 4]), "conv": (14, [6, 7]),
                                 "epi": (15, [9])}.items():
        tot = v[tot_i]
        if tot == 0:
            continue
        s = "  ".join(f"{names[p].split(':')[1]} {v[p] / tot * 100:5.1f}%" for p in parts)
        print(f"  {role:5s} {s}   busy {100 - sum(v[p] for p in parts) / tot * 100:5.1f}%")
