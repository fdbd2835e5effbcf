"""Makes tests/golden/c2_full.npz: BASELINE configs[1] at FULL size (X fp32
1,000,000 x 4,096 from the device generator, the bench's seeds) reduced by the
compiled reference's streaming Lazy SPCA (reduce with block_rows = 25,000:
reduce_lazy_spca_streaming over SliceRowBlockStream, proj/core/src/reducer.cpp:
300-335) on the GPU box's host cores. Stores sigma (k = 100) and the first 10
columns of V for tests/test_gpu_c2_full.py. Run on a GPU box (the generator is
the device's): python tests/golden/make_c2_fixture.py"""
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
import paper_1709_07175_b200 as lp  # noqa: E402
from oracle import refbind as R  # noqa: E402

cfg = bench.CONFIGS["c2"]
m, n, k, l = cfg["m"], cfg["n"], cfg["k"], cfg["l"]
ctx = lp.Context(0)
x = torch.empty((m, n), dtype=torch.float32, device="cuda")
lp.synth_lowrank(x, 0, cfg["r"], cfg["rho"], 0.01, bench.SEED_X, ctx=ctx)
xh = x.cpu().numpy()
del x
R.use_native(True)
R.set_threads(len(__import__("os").sched_getaffinity(0)))
t0 = time.time()
v, s, _, t = R.reduce(2, xh, k, l, bench.SEED_OMEGA, block_rows=25_000)
secs = time.time() - t0
out = ROOT / "tests" / "golden" / "c2_full.npz"
np.savez_compressed(out, sigma=s, v10=v[:, :10], m=m, n=n, k=k, l=l, seed_x=bench.SEED_X, seed_omega=bench.SEED_OMEGA,
                    block_rows=25_000, ref_seconds=secs)
print(f"wrote {out}: sigma[0] {s[0]:.6e}, reference streaming fit {secs:.1f} s (timings {t})")
